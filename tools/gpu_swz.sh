for i in 1 2; do
python tools/time_decode_lib.py paper_2312_17241_b200/libprobegrid_b200.so base
for l in tools/_var_*/lib.so; do python tools/time_decode_lib.py $l $(basename $(dirname $l)); done
done
python -m pytest tests/test_gpu_c2_parity.py tests/test_gpu_umma.py -q -x 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -q -x -k "decode or umma or infer" 2>&1 | tail -2
