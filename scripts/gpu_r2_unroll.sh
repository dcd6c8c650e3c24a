# A/B: port-loop unroll factors (phase 1 / phase 2 loops of tile_step) on the step window, the day and the rollout; C4 ncu capture.
bash scripts/ab_roll.sh build/ab/u11.so build/ab/u21.so build/ab/u12.so build/ab/u22.so > gpurun_out/unroll_ab.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step -s 144 -c 1 -o gpurun_out/f_k_step_c4 python scripts/probe_c4.py --at 144 --ncu > gpurun_out/f_ncu_c4.log 2>&1
