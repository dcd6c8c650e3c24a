# C5 one-launch step: charge/departure loop unroll A/B (VY_MULTI_U2 = 1 / 2) on the bench's hetero leg; C5 tests with mu2.
cp paper_2507_01522_b200/libvoltyard_b200.so /tmp/_keep.so
for rep in 1 2; do for v in mu1 mu2; do
  cp build/ab/$v.so paper_2507_01522_b200/libvoltyard_b200.so
  echo "$v rep$rep $(timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', round(d['value']/1e9,3), 'C5', round(d['hetero']['value']/1e9,3), 'C5 streams', round(d['hetero']['per_group_streams']['value']/1e9,3))")"
done; done > gpurun_out/multi_u.txt 2>&1
cp build/ab/mu2.so paper_2507_01522_b200/libvoltyard_b200.so
timeout 900 python -m pytest tests/test_gpu_hetero.py tests/test_gpu_hetero_multi.py tests/test_gpu_fullscale.py -m gpu -q -x -k "hetero or multi or C5 or c5 or group" > gpurun_out/multi_u_tests.log 2>&1; echo rc=$? >> gpurun_out/multi_u_tests.log
cp /tmp/_keep.so paper_2507_01522_b200/libvoltyard_b200.so
