# Source-attributed ncu capture of the fused rollout (T = 32 from step 128, 2^20 envs) for stall-by-line analysis.
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rollout -c 1 -o gpurun_out/k_roll_src python scripts/probe_rollout.py > gpurun_out/ncu_rollsrc.log 2>&1
ncu -i gpurun_out/k_roll_src.ncu-rep --page source --csv --print-source sass > gpurun_out/k_roll_src_sass.csv 2>&1
