mkdir -p gpurun_out
VAR=TLFEA_G3_SMEM_PAD VALS="0 8000 20000 38000" bash tools/ab_env.sh
