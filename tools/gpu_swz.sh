CFG='{"n_f":256,"n_c":4096,"n_p":16}' bash tools/gpu_ab_vars.sh
CFG='{"n_f":4096,"n_c":16384,"n_p":4}' bash tools/gpu_ab_vars.sh
python -m pytest tests/test_gpu_parity.py -q -x -k "train or grad or step or fused" 2>&1 | tail -2
