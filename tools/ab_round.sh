mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for c in 3 2; do CFG=$c VAR=X VALS=0 bash tools/ab_env.sh; done
NS="2" CFG=3 bash tools/multirank_flow.sh
