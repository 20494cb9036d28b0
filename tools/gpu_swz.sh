L=paper_2312_17241_b200/libprobegrid_b200.so
for r in 4 8 16 32; do PG_TRAIN_REPS=$r python tools/time_c3_lib.py $L reps$r; done
PG_TRAIN_AGG_RANGES=64 python tools/time_c3_lib.py $L agg64
PG_TRAIN_AGG_RANGES=64 PG_TRAIN_REPS=1 python tools/time_c3_lib.py $L agg64_reps1
for mb in 0 32 128; do PG_TRAIN_CELL_MB=$mb python tools/time_c3_lib.py $L cells$mb; done
