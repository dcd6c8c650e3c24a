# Round-2 final measurements: GPU suite, smoke, driver-style bench line, reference arm, launch list, C4 ncu.
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/f_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo rc=$? >> gpurun_out/f_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench20.log 2>&1; echo rc=$? >> gpurun_out/f_bench20.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f_bench_ref.log 2>&1; echo rc=$? >> gpurun_out/f_bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/f_ncu_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step -s 145 -c 1 -o gpurun_out/f_k_step_c4 python scripts/probe_c4.py --at 144 --ncu > gpurun_out/f_ncu_c4.log 2>&1
ls -la gpurun_out
