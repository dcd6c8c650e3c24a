for v in ab/c1.so ab/c2.so ab/c3.so ab/c1.so ab/c2.so ab/c3.so; do cp $v paper_2507_01522_b200/libvoltyard_b200.so; echo "$v $(timeout 120 python scripts/probe_rollout.py 2>&1 | tail -1)"; done > gpurun_out/ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "rollout" > gpurun_out/t_roll.log 2>&1; echo rc=$? >> gpurun_out/t_roll.log
