#!/bin/bash
# C1 training-step timing of the in-tree build and every tools/_var_*/lib.so
mkdir -p gpurun_out
for i in 1 2; do
  python tools/time_train_lib.py paper_2312_17241_b200/libprobegrid_b200.so base
  for l in tools/_var_*/lib.so; do python tools/time_train_lib.py $l $(basename $(dirname $l)); done
done > gpurun_out/ab_vars.txt 2>&1
cat gpurun_out/ab_vars.txt
