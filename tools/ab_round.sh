mkdir -p gpurun_out
P=paper_2604_10357_b200
LIBS="$P/libtlfea.so $P/libtlfea_bm.so $P/libtlfea.so $P/libtlfea_bm.so" TILES=1 bash tools/ab.sh
