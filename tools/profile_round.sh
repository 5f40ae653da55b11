# Round measurement on one B200 (run through gpurun from the repo root):
#   GPU tests, the default bench line per config, the ncu launch list of the
#   default bench command, one ncu --set full capture of the top kernels.
# Outputs land in gpurun_out/$TAG/ (scratch); copy summaries into profiles/.
set -u
TAG=${TAG:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
for c in ${CFGS:-3 2 4 5 6}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
  python -c "import json;d=json.load(open('$OUT/bench_cfg$c.json'));print('cfg$c', round(d['value']/1e6,2), 'M el/s', round(d['ms_per_step'],3), 'ms', d['roofline']['bound'], round(d['roofline']['frac'],3))" || tail -3 $OUT/bench_cfg$c.err
done
if [ -z "${NO_REF:-}" ]; then
  timeout 600 python bench.py --impl reference --config 3 --steps 2 --warmup 3 > $OUT/reference_cfg3.json 2> $OUT/reference_cfg3.err; tail -c 300 $OUT/reference_cfg3.json
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg3.csv \
  python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/summarize_launches.py $OUT/launches_cfg3.csv $OUT/launches_cfg3.txt "ncu launch list: python bench.py --config 3 --steps 2 --warmup 3 (gpu__time_duration.sum, --clock-control none)" | head -12
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_element$|^k_gather_units_v3$|^k_gather_f_dof$" -c 3 \
  -o $OUT/full_cfg3 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py $OUT/full_cfg3.ncu-rep > $OUT/ncu_full_cfg3.txt 2>&1; head -70 $OUT/ncu_full_cfg3.txt
