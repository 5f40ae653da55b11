mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
VAR=X VALS="0" bash tools/ab_env.sh
