timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_ppo.py tests/test_gpu_policy.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/t_wide.log 2>&1; echo rc=$? >> gpurun_out/t_wide.log
timeout 300 python scripts/probe_c1.py > gpurun_out/c1.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench20.log 2>&1
