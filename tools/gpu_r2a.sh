#!/usr/bin/env bash
# round-2 measurement pass: bench line, drop-in e2e alternatives, L2 probe + ncu cross-check
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
python tools/e2e_dropin.py > gpurun_out/r2a_dropin.log 2>&1
python tools/probe_l2.py > gpurun_out/r2a_probe.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,lts__t_bytes.sum.per_second,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,l1tex__t_bytes.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:probe --csv --log-file gpurun_out/r2a_probe_ncu.csv python tools/probe_l2.py > gpurun_out/r2a_probe_ncu.log 2>&1
tail -3 gpurun_out/r2a_bench.err; cat gpurun_out/r2a_dropin.log gpurun_out/r2a_probe.log
