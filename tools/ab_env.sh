# A/B over one environment variable: VAR=name VALS="a b c" CFG=n
for val in $VALS; do
env $VAR=$val timeout 300 python bench.py --config ${CFG:-3} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
echo "CFG=${CFG:-3} $VAR=$val $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['config']['kernels'].items() if v['launches']})" 2>/dev/null || tail -2 gpurun_out/ab.err)"
done
