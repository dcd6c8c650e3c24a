# Round-2 closing run: GPU suite, smoke, driver-style bench line, reference arm, sanitizer passes (C4 prefetch active).
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/g_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/g_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo rc=$? >> gpurun_out/g_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g_bench20.log 2>&1; echo rc=$? >> gpurun_out/g_bench20.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/g_bench_ref.log 2>&1; echo rc=$? >> gpurun_out/g_bench_ref.log
for tool in memcheck racecheck synccheck initcheck; do
  VY_PF=10 timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_small.py > gpurun_out/g_san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/g_san_$tool.log
done
