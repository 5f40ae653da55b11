mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
P=paper_2604_10357_b200
LIBS="$P/libtlfea.so $P/libtlfea_c382.so $P/libtlfea_c3ed.so $P/libtlfea.so" TILES=1 bash tools/ab.sh
