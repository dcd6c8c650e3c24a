set -x
timeout 200 python scripts/probe_midday.py --at 144 > gpurun_out/midday.log 2>&1
timeout 200 python scripts/probe_rollout.py > gpurun_out/rollout.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step --launch-skip 144 -c 1 -o gpurun_out/k_step_mid python scripts/probe_midday.py --at 144 --ncu --fused > gpurun_out/ncu_mid.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rollout -c 1 -o gpurun_out/k_rollout_mid python scripts/probe_rollout.py > gpurun_out/ncu_roll.log 2>&1
