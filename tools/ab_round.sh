mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
VAR=TLFEA_GATHER_HF VALS="0 1 0 1" bash tools/ab_env.sh
CFG=2 VAR=TLFEA_GATHER_HF VALS="0 1" bash tools/ab_env.sh
