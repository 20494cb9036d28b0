for i in 1 2; do
python tools/time_decode_lib.py paper_2312_17241_b200/libprobegrid_b200.so base
python tools/time_decode_lib.py tools/_var_prev/lib.so prev
done
python -m pytest tests/test_gpu_c2_parity.py tests/test_gpu_cngp.py -q -x 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -q -x -k "decode or umma or infer" 2>&1 | tail -2
