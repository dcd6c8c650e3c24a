timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_random.py tests/test_gpu_fullscale.py -m gpu -q -x -k "golden or fused or c2 or c4 or trees" > gpurun_out/t_os.log 2>&1; echo rc=$? >> gpurun_out/t_os.log
bash scripts/ab_roll.sh ab/base4.so ab/os.so > gpurun_out/ab.log 2>&1
