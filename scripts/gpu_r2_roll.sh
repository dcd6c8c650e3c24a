timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rollout" > gpurun_out/t_roll.log 2>&1; echo rc=$? >> gpurun_out/t_roll.log
timeout 200 python scripts/probe_rollout.py > gpurun_out/rollout.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench20.log 2>&1
