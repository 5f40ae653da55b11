mkdir -p gpurun_out
P=paper_2604_10357_b200
LIBS="$P/libtlfea.so $P/libtlfea_w2m6.so $P/libtlfea_w3m4.so" TILES=1 bash tools/ab.sh
