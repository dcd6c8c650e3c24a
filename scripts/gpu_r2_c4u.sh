# C4 streamed step: charge/departure loop unroll A/B (VY_STREAM_U2 = 1 / 2 / 4), mid-day and step 60; C4 parity tests with s2.
for rep in 1 2; do for v in s1 s2 s4; do for at in 144 60; do
  cp build/ab/$v.so paper_2507_01522_b200/libvoltyard_b200.so
  echo "$v rep$rep $(timeout 300 python scripts/probe_c4.py --at $at 2>/dev/null | tail -1)"
done; done; done > gpurun_out/c4u.txt 2>&1
cp build/ab/s2.so paper_2507_01522_b200/libvoltyard_b200.so
timeout 900 python -m pytest tests/test_gpu_fullscale.py tests/test_gpu_parity.py -m gpu -q -x -k "c4 or C4 or battery or stream" > gpurun_out/c4u_tests.log 2>&1; echo rc=$? >> gpurun_out/c4u_tests.log
