set -x
timeout 600 python -m pytest tests/test_gpu_step_random.py tests/test_gpu_hetero.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/t_random.log 2>&1; echo rc=$? >> gpurun_out/t_random.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench20.log 2>&1; echo rc=$? >> gpurun_out/bench20.log
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1
timeout 120 python scripts/probe_midday.py --at 144 > gpurun_out/midday.log 2>&1
timeout 600 bash scripts/day_dram.sh > gpurun_out/day_dram.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step --launch-skip 144 -c 1 -o gpurun_out/k_step_fused_mid python scripts/probe_midday.py --at 144 --ncu --fused > gpurun_out/ncu_mid.log 2>&1
