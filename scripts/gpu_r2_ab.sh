for v in c2 c4; do cp ab/$v.so paper_2507_01522_b200/libvoltyard_b200.so; timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step_random.py -m gpu -q -x -k "golden or fused" > gpurun_out/t_$v.log 2>&1; echo "$v rc=$?" >> gpurun_out/t_claim.log; done
bash scripts/ab_roll.sh ab/c1.so ab/c2.so ab/c4.so > gpurun_out/ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ppo.py -m gpu -q -x -k fused_ppo_loss > gpurun_out/t_loss.log 2>&1; echo rc=$? >> gpurun_out/t_loss.log
