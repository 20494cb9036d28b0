#!/bin/bash
# A/B of the C1 training step: HEAD build vs working tree, then the GPU suite
set -x
mkdir -p gpurun_out
for i in 1 2 3; do
  python tools/time_train_lib.py tools/_var_old/libold.so old
  python tools/time_train_lib.py paper_2312_17241_b200/libprobegrid_b200.so new
done > gpurun_out/ab_touched.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "train or parity or dist or smoke" > gpurun_out/gpu_tests.txt 2>&1
tail -5 gpurun_out/gpu_tests.txt
cat gpurun_out/ab_touched.txt
