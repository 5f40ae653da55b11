mkdir -p gpurun_out
P=paper_2604_10357_b200
TLFEA_LIB=$P/libtlfea_f2l.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adamw.py -m gpu -q 2>&1 | tail -1
CFG=5 LIBS="$P/libtlfea.so $P/libtlfea_f2l.so $P/libtlfea.so $P/libtlfea_f2l.so" TILES=1 bash tools/ab.sh
for l in $P/libtlfea.so $P/libtlfea_f2l.so; do TLFEA_LIB=$l timeout 300 python tools/bench_adamw.py 2>&1 | tail -1 | cut -c1-200; done
