timeout 600 python -m pytest tests/test_gpu_hetero_multi.py -m gpu -q -x > gpurun_out/t_multi.log 2>&1; echo rc=$? >> gpurun_out/t_multi.log
for v in ab/m_const.so; do cp $v paper_2507_01522_b200/libvoltyard_b200.so; echo "== $v"; for s in all fast nested; do timeout 300 python scripts/probe_multi.py --subset $s 2>&1 | tail -2; done; done > gpurun_out/ab.log 2>&1
