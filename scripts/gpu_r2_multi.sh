timeout 900 python -m pytest tests/test_gpu_hetero_multi.py tests/test_gpu_hetero.py -m gpu -q -x > gpurun_out/t_multi.log 2>&1; echo rc=$? >> gpurun_out/t_multi.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench20.log 2>&1
