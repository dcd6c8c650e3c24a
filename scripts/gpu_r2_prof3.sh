timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rollout -c 1 -o gpurun_out/k_rollout_r2 python scripts/probe_rollout.py > gpurun_out/ncu_roll.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_multi --launch-skip 136 -c 1 -o gpurun_out/k_step_multi_r2 python scripts/probe_multi.py --subset all > gpurun_out/ncu_multi.log 2>&1
