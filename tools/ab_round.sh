mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
VAR=TLFEA_UNIT_BANDS VALS="1 8 4 16" bash tools/ab_env.sh
