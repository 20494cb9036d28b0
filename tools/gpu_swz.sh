bash tools/gpu_ab_vars.sh
python -m pytest tests/test_gpu_parity.py tests/test_gpu_nerf.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
