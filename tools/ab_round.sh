mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
VAR=TLFEA_EL_TILES VALS="1 2 4" bash tools/ab_env.sh
