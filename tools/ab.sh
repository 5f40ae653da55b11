# A/B of element-kernel variants: LIBS (TLFEA_LIB paths) x EL_TILES
for lib in ${LIBS:-paper_2604_10357_b200/libtlfea.so}; do
for t in ${TILES:-2}; do
TLFEA_LIB=$lib TLFEA_EL_TILES=$t timeout 300 python bench.py --config ${CFG:-3} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
echo "CFG=${CFG:-3} $(basename $lib) tiles=$t $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['config']['kernels'].items() if v['launches']})" 2>/dev/null || tail -2 gpurun_out/ab.err)"
done; done
