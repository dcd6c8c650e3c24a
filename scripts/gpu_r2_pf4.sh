# C4 (streamed tile): L2 prefetch distance A/B (VY_PF = percent of resident warps; 0 = off), mid-day and two other steps
for rep in 1 2; do
for pf in 0 5 10 15 25; do
  for at in 144 60; do
    echo "VY_PF=$pf rep$rep at=$at $(VY_PF=$pf timeout 300 python scripts/probe_c4.py --at $at 2>/dev/null | tail -1)"
  done
done
done > gpurun_out/pf4_ab2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullscale.py tests/test_gpu_parity.py -m gpu -q -x -k "c4 or C4 or battery or stream" > gpurun_out/pf4_tests2.log 2>&1; echo rc=$? >> gpurun_out/pf4_tests2.log
