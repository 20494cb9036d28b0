# ncu of the fused training kernel (after a clean plain run)
python tools/prof_kernels.py --what train --n 2 > gpurun_out/pt_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:train_ -s 1 -c 1 -o gpurun_out/train_mma_r1 python tools/prof_kernels.py --what train --n 2 > gpurun_out/pt_ncu.log 2>&1
tail -2 gpurun_out/pt_ncu.log
