CFGS='[{"n_f":4096,"n_c":16384,"n_p":4},{}]'
export CFGS
python tools/time_train_cfgs.py
PG_TRAIN_GROUPS=1 python tools/time_train_cfgs.py
python tools/time_train_cfgs.py
PG_TRAIN_GROUPS=1 python tools/time_train_cfgs.py
