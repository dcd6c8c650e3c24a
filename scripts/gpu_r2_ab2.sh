# A/B: hoisted grid entry (g), 32-bit RandomPolicy fast path (p), both (gp); parity with gp installed.
bash scripts/ab_roll.sh build/ab/base.so build/ab/g.so build/ab/p.so build/ab/gp.so > gpurun_out/ab2.txt 2>&1
cp paper_2507_01522_b200/libvoltyard_b200.so /tmp/_keep.so
cp build/ab/gp.so paper_2507_01522_b200/libvoltyard_b200.so
timeout 900 python -m pytest tests/test_gpu_step_random.py tests/test_gpu_parity.py tests/test_gpu_policy.py tests/test_gpu_wide.py -m gpu -q -x > gpurun_out/ab2_tests.log 2>&1; echo rc=$? >> gpurun_out/ab2_tests.log
cp /tmp/_keep.so paper_2507_01522_b200/libvoltyard_b200.so
