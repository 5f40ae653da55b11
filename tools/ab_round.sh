mkdir -p gpurun_out
TLFEA_GT_SPLIT=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -1
VAR=TLFEA_GT_SPLIT VALS="0 1" bash tools/ab_env.sh
