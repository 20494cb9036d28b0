#!/bin/bash
# A/B of the decode variants / table budgets on one GPU (tools/decode_ab.py)
mkdir -p gpurun_out
rm -f gpurun_out/decode_ab_*.npy
: > gpurun_out/decode_ab.log
timeout 300 python tools/decode_ab.py default >> gpurun_out/decode_ab.log 2>&1
for b in ${BUDGETS:-0 32768 65536 98304}; do
  PG_DECODE_TABLE_KINDS=2 PG_DECODE_TABLE_BYTES=$b timeout 300 python tools/decode_ab.py tables_k2_$b tables >> gpurun_out/decode_ab.log 2>&1
done
cat gpurun_out/decode_ab.log
