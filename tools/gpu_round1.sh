python -m pytest tests -m gpu -q -p no:cacheprovider -s 2>&1 | grep -E "max rel|step [0-9] level|passed|failed|Error|assert" > gpurun_out/t5.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench3.json 2> gpurun_out/bench3.err
python tools/prof_kernels.py --what all --n 3 > gpurun_out/prof_plain5.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python tools/prof_kernels.py --what all --n 3 > gpurun_out/ncu5a.log 2>&1
python tools/prof_kernels.py --what train --n 2 > gpurun_out/prof_plain5b.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:train_fused -s 1 -c 1 -o gpurun_out/train_full_r1 python tools/prof_kernels.py --what train --n 2 > gpurun_out/ncu5b.log 2>&1
python tools/prof_kernels.py --what decode --n 2 > gpurun_out/prof_plain5c.log 2>&1 && ncu --set full --clock-control none -k regex:decode_fused -s 1 -c 1 -o gpurun_out/decode_full_r1b python tools/prof_kernels.py --what decode --n 2 > gpurun_out/ncu5c.log 2>&1
cat gpurun_out/t5.log; tail -3 gpurun_out/bench3.err; cat gpurun_out/bench3.json; tail -2 gpurun_out/ncu5a.log gpurun_out/ncu5b.log gpurun_out/ncu5c.log
