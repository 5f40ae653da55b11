mkdir -p gpurun_out
P=paper_2604_10357_b200
CFG=2 LIBS="$P/libtlfea.so $P/libtlfea_mr3.so $P/libtlfea.so $P/libtlfea_mr3.so" TILES=1 bash tools/ab.sh
