bash tools/gpu_ab_vars.sh
CFG='{}' bash tools/gpu_ab_vars.sh
python -m pytest tests/test_gpu_parity.py -q -x -k "train or grad or step or fused" 2>&1 | tail -2
