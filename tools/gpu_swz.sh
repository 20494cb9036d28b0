bash tools/gpu_ab_vars.sh
CFG='{}' bash tools/gpu_ab_vars.sh
