#!/bin/bash
# C2 headline decode timing of the in-tree build and every tools/_var_*/lib.so
for i in 1 2 3; do
  python tools/time_decode_lib.py paper_2312_17241_b200/libprobegrid_b200.so base $MODE
  for l in tools/_var_*/lib.so; do python tools/time_decode_lib.py $l $(basename $(dirname $l)) $MODE; done
done
