#!/bin/bash
# C1 step: HEAD build vs working tree with 1 and 2 tile pipelines per CTA
for i in 1 2; do
  python tools/time_train_lib.py tools/_var_HEAD/lib.so head
  python tools/time_train_lib.py paper_2312_17241_b200/libprobegrid_b200.so ng1
  PG_TRAIN_GROUPS=2 python tools/time_train_lib.py paper_2312_17241_b200/libprobegrid_b200.so ng2
done
