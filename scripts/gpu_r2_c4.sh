timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step --launch-skip 144 -c 1 -o gpurun_out/k_step_c4s python scripts/probe_c4.py --ncu > gpurun_out/ncu_c4.log 2>&1
