for rep in 1 2; do for v in ab/ring2.so ab/ring1.so; do cp $v paper_2507_01522_b200/libvoltyard_b200.so; echo "$v $(timeout 120 python scripts/probe_rollout.py 2>&1 | tail -1) | $(timeout 120 python scripts/probe_c4.py 2>&1 | tail -1)"; done; done > gpurun_out/ab.log 2>&1
cp ab/ring1.so paper_2507_01522_b200/libvoltyard_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_random.py -m gpu -q -x -k "rollout or streamed" > gpurun_out/t_roll.log 2>&1; echo rc=$? >> gpurun_out/t_roll.log
cp ab/ring2.so paper_2507_01522_b200/libvoltyard_b200.so
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --no-extras > gpurun_out/torchrun.log 2>&1; echo rc=$? >> gpurun_out/torchrun.log
