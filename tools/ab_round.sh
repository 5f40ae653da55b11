mkdir -p gpurun_out
P=paper_2604_10357_b200
LIBS="$P/libtlfea.so $P/libtlfea_fb128.so $P/libtlfea_fb512.so $P/libtlfea_fb64.so" TILES=1 bash tools/ab.sh
