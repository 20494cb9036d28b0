# ncu --set full of the fused training kernel; TRAIN_CFG (JSON HyperParams kwargs) selects the config
CFGARG=${TRAIN_CFG:+--train-cfg $TRAIN_CFG}
python tools/prof_kernels.py --what train --n 2 $CFGARG > gpurun_out/pt_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:train_mma -s 1 -c 1 \
      -o gpurun_out/pt_train_mma python tools/prof_kernels.py --what train --n 2 $CFGARG > gpurun_out/pt_ncu.log 2>&1
ls -la gpurun_out/pt_*
