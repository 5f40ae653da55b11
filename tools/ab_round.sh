# Scratch A/B driver for one gpurun call (edited per experiment): GPU tests,
# then back-to-back bench lines of variant builds (TLFEA_VARIANT=name
# TLFEA_DEFINES="-D..." python -m paper_2604_10357_b200.build -> libtlfea_name.so).
mkdir -p gpurun_out
P=paper_2604_10357_b200
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
LIBS="${LIBS:-$P/libtlfea.so}" TILES=1 bash tools/ab.sh
