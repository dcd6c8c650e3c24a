timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rollout_wide -s 1 -c 1 -o gpurun_out/k_rollout_wide_c1 python scripts/probe_c1.py > gpurun_out/ncu_wide.log 2>&1
