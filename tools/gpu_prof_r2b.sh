#!/usr/bin/env bash
# Round-2 final evidence pass: launch list + ncu --set full of the decode and
# training kernels at bench shapes (each after its plain run exited 0).
set -x
python tools/prof_kernels.py --what all --n 3 > gpurun_out/r2b_prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv \
      python tools/prof_kernels.py --what all --n 3 > gpurun_out/r2b_ncu_launch.log 2>&1
python tools/prof_kernels.py --what decode --n 2 > gpurun_out/r2b_pd_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:decode_umma -s 1 -c 1 \
      -o gpurun_out/r2b_decode_umma python tools/prof_kernels.py --what decode --n 2 > gpurun_out/r2b_pd_ncu.log 2>&1
python tools/prof_kernels.py --what train --n 2 > gpurun_out/r2b_pt_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:train_mma -s 1 -c 1 \
      -o gpurun_out/r2b_train_mma python tools/prof_kernels.py --what train --n 2 > gpurun_out/r2b_pt_ncu.log 2>&1
python tools/time_refonly.py > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_refonly_launches.csv \
      python tools/time_refonly.py > /dev/null 2>&1
ls -la gpurun_out/r2b_*
