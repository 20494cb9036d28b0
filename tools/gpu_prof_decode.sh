# ncu of the tcgen05 decode kernel (run after a clean plain run)
python tools/prof_kernels.py --what decode --n 2 > gpurun_out/pd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:decode_umma -s 1 -c 1 -o gpurun_out/decode_umma_r1 python tools/prof_kernels.py --what decode --n 2 > gpurun_out/pd_ncu.log 2>&1
tail -2 gpurun_out/pd_ncu.log
