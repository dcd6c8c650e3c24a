bash scripts/ab_roll.sh ab/head.so ab/v00.so ab/v10.so ab/v01.so ab/v11.so > gpurun_out/ab.log 2>&1
