# fused-eval diagnostics: etiles chunk lag dbg
for cfg in "4 16 512 0" "4 16 512 1" "4 16 512 2" "1 64 1024 0" "1 64 1024 1" "8 8 512 0"; do
set -- $cfg
TLFEA_FZ_ETILES=$1 TLFEA_FZ_CHUNK=$2 TLFEA_FZ_LAG=$3 TLFEA_FZ_DBG=$4 timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2>gpurun_out/sw.err
echo "$cfg $(python -c "import json;d=json.load(open('gpurun_out/sw.json'));print(round(d['ms_per_step'],3))" 2>/dev/null || tail -2 gpurun_out/sw.err)"
done
