# Rollout loop-unroll A/B (VY_ROLL_U2 = 2 / 3 / 4) and the rollout parity tests with the kept build.
for rep in 1 2; do for v in r2 r3 r4; do
  cp build/ab/$v.so paper_2507_01522_b200/libvoltyard_b200.so
  echo "$v rep$rep $(timeout 300 python scripts/probe_rollout.py 2>/dev/null | tail -1)"
done; done > gpurun_out/roll_u.txt 2>&1
cp build/ab/r2.so paper_2507_01522_b200/libvoltyard_b200.so
timeout 1200 python -m pytest tests -m gpu -q -x -k "rollout or roll" > gpurun_out/roll_tests.log 2>&1; echo rc=$? >> gpurun_out/roll_tests.log
