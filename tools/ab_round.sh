mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
for c in 3 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --tables --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print($c, d['ms_per_step'], {k:round(v['ms_per_launch'],3) for k,v in d['config']['kernels'].items() if v['launches']})"; done
VAR=X VALS=0 bash tools/ab_env.sh
