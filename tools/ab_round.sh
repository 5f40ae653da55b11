mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
NS="2 4" CFG=2 bash tools/multirank_flow.sh
NS="2" CFG=3 bash tools/multirank_flow.sh
