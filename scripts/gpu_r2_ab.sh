timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_random.py tests/test_gpu_fullscale.py -m gpu -q -x -k "golden or fused or every_row or rollout or c2" > gpurun_out/t_nw.log 2>&1; echo rc=$? >> gpurun_out/t_nw.log
bash scripts/ab_roll.sh ab/base3.so ab/nw.so > gpurun_out/ab.log 2>&1
