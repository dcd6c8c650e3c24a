# Last check of the committed tree: GPU suite, smoke, default bench (no flags), driver-style bench.
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/l_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/l_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l_smoke.log 2>&1; echo rc=$? >> gpurun_out/l_smoke.log
timeout 900 python bench.py > gpurun_out/l_bench_default.log 2>&1; echo rc=$? >> gpurun_out/l_bench_default.log
