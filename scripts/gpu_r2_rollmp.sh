# Rollout A/B: per-step occupied-port mask instead of votes (rm), RandomPolicy draws packed up front (rp), both (rmp); rollout tests with rmp.
for rep in 1 2; do for v in rb rm rp rmp; do
  cp build/ab/$v.so paper_2507_01522_b200/libvoltyard_b200.so
  echo "$v rep$rep $(timeout 300 python scripts/probe_rollout.py 2>/dev/null | tail -1)"
done; done > gpurun_out/rollmp.txt 2>&1
cp build/ab/rmp.so paper_2507_01522_b200/libvoltyard_b200.so
timeout 1200 python -m pytest tests -m gpu -q -x -k "rollout or roll" > gpurun_out/rollmp_tests.log 2>&1; echo rc=$? >> gpurun_out/rollmp_tests.log
