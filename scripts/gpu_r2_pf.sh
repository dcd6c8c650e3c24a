# A/B of the L2 prefetch distance (VY_PF = percent of the resident warps; 0 = off) on the bench's main leg.
for rep in 1 2; do
for pf in 0 25 50 100 200; do
  r=$(VY_PF=$pf timeout 300 python bench.py --no-cpu --no-extras --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,3))")
  d=$(VY_PF=$pf timeout 300 python bench.py --no-cpu --no-extras --steps 288 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms'],4), round(d['value']/1e9,3))")
  echo "VY_PF=$pf rep$rep window20 kernel_ms/value(e9): $r   day288: $d"
done
done > gpurun_out/pf_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_step_random.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pf_tests.log 2>&1; echo rc=$? >> gpurun_out/pf_tests.log
