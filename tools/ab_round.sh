mkdir -p gpurun_out
P=paper_2604_10357_b200
LIBS="$P/libtlfea.so $P/libtlfea_ca.so $P/libtlfea.so $P/libtlfea_ca.so" TILES=1 bash tools/ab.sh
CFG=5 LIBS="$P/libtlfea.so $P/libtlfea_ca.so" TILES=1 bash tools/ab.sh
CFG=4 LIBS="$P/libtlfea.so $P/libtlfea_ca.so" TILES=1 bash tools/ab.sh
