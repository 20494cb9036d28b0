python tools/train_bitcheck.py tools/_var_prev/lib.so gpurun_out/bc_base.npz
python tools/train_bitcheck.py paper_2312_17241_b200/libprobegrid_b200.so gpurun_out/bc_new.npz gpurun_out/bc_base.npz
bash tools/gpu_ab_vars.sh
python -m pytest tests/test_gpu_parity.py tests/test_gpu_nerf.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
