# A/B: obs staged row-major in a separate area and written by one bulk (TMA) store per tile (ob1) vs in-place column staging + per-lane row read-out (ob0).
bash scripts/ab_window.sh build/ab/ob0.so build/ab/ob1.so > gpurun_out/obsbulk_ab.txt 2>&1
cp paper_2507_01522_b200/libvoltyard_b200.so /tmp/_keep.so
cp build/ab/ob1.so paper_2507_01522_b200/libvoltyard_b200.so
timeout 1200 python -m pytest tests/test_gpu_step_random.py tests/test_gpu_parity.py tests/test_gpu_hetero.py tests/test_gpu_hetero_multi.py -m gpu -q -x > gpurun_out/obsbulk_tests.log 2>&1; echo rc=$? >> gpurun_out/obsbulk_tests.log
VY_WARPS_PER_CTA=8 timeout 300 python bench.py --no-cpu --no-extras --steps 20 --warmup 5 2>/dev/null | tail -1 | cut -c1-400 >> gpurun_out/obsbulk_ab.txt
cp /tmp/_keep.so paper_2507_01522_b200/libvoltyard_b200.so
