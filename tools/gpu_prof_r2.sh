#!/usr/bin/env bash
# Round-2 evidence pass (GPU box): bench line, reference arm, launch list of
# the bench's headline + training steps, ncu --set full of the decode and
# training kernels (each only after its plain run exited 0).
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
python tools/prof_kernels.py --what all --n 3 > gpurun_out/r2_prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
      python tools/prof_kernels.py --what all --n 3 > gpurun_out/r2_ncu_launch.log 2>&1
python tools/prof_kernels.py --what decode --n 2 > gpurun_out/r2_pd_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:decode_umma -s 1 -c 1 \
      -o gpurun_out/r2_decode_umma python tools/prof_kernels.py --what decode --n 2 > gpurun_out/r2_pd_ncu.log 2>&1
python tools/prof_kernels.py --what train --n 2 > gpurun_out/r2_pt_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:train_mma -s 1 -c 1 \
      -o gpurun_out/r2_train_mma python tools/prof_kernels.py --what train --n 2 > gpurun_out/r2_pt_ncu.log 2>&1
tail -3 gpurun_out/r2_bench.err gpurun_out/r2_bench_ref.err gpurun_out/r2_ncu_launch.log gpurun_out/r2_pd_ncu.log gpurun_out/r2_pt_ncu.log
