# Source-attributed ncu captures of the bench kernel (mid-day step 144) for stall-by-line analysis.
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step --launch-skip 144 -c 1 -o gpurun_out/k_step_src python scripts/probe_midday.py --at 144 --ncu --fused > gpurun_out/ncu_src.log 2>&1
ncu -i gpurun_out/k_step_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/k_step_src_cuda.csv 2>&1
ncu -i gpurun_out/k_step_src.ncu-rep --page source --csv --print-source sass > gpurun_out/k_step_src_sass.csv 2>&1
ls -la gpurun_out
