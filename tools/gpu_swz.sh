timeout 300 bash tools/gpu_ab_vars.sh
