bash tools/gpu_ab_vars.sh
python -m pytest tests/test_gpu_parity.py tests/test_gpu_nerf.py -q -x -k "train or grad or step or fused or nerf" 2>&1 | tail -2
