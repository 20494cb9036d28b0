#!/usr/bin/env bash
# Round-2 closing pass: full GPU suite, the bench (both arms), the evidence
# profiles (tools/gpu_prof_r2b.sh) and the SASS opcode counts.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
bash tools/gpu_prof_r2b.sh > gpurun_out/final_prof.log 2>&1
tail -2 gpurun_out/final_pytest.log; cat gpurun_out/final_bench.json gpurun_out/final_bench_ref.json
