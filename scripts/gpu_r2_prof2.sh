timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rollout -c 1 -o gpurun_out/k_rollout_mid2 python scripts/probe_rollout.py > gpurun_out/ncu_roll.log 2>&1
