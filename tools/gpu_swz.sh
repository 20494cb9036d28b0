for i in 1 2; do
python tools/time_decode_lib.py paper_2312_17241_b200/libprobegrid_b200.so base
python tools/time_decode_lib.py tools/_var_RNA/lib.so rna
python tools/time_train_lib.py paper_2312_17241_b200/libprobegrid_b200.so base
done
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
