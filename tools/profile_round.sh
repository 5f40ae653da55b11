# Round measurement on one B200 (run through gpurun from the repo root):
#   the default bench line per config and variant, the ladder, the reference
#   arm, the ncu launch list of the default bench command, one ncu --set full
#   capture of the three config-3 kernels (traffic, stalls, source), the
#   element kernels of the other configs, the smoke test.
# Outputs land in gpurun_out/$TAG/ (scratch); copy summaries into profiles/.
set -u
TAG=${TAG:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
for c in ${CFGS:-3 1 2 4 5 6}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
  python -c "import json;d=json.loads(open('$OUT/bench_cfg$c.json').read().strip().splitlines()[-1]);print('cfg$c', round(d['value']/1e6,2), 'M el/s', round(d['ms_per_step'],3), 'ms', d['roofline']['bound'], round(d['roofline']['frac'],3))" || tail -3 $OUT/bench_cfg$c.err
done
for v in "--mesh straight" "--tables" "--hessian upper"; do
  n=$(echo $v | tr -d ' -')
  timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $v > $OUT/bench_cfg3_$n.json 2> $OUT/bench_cfg3_$n.err
  python -c "import json;d=json.loads(open('$OUT/bench_cfg3_$n.json').read().strip().splitlines()[-1]);print('cfg3 $n', round(d['ms_per_step'],3), 'ms')" || tail -3 $OUT/bench_cfg3_$n.err
done
timeout 900 python bench.py --ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; wc -l $OUT/ladder.jsonl
timeout 600 python bench.py --impl reference --config 3 --steps 2 --warmup 3 > $OUT/reference_cfg3.json 2> $OUT/reference_cfg3.err; tail -c 300 $OUT/reference_cfg3.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg3.csv \
  python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/summarize_launches.py $OUT/launches_cfg3.csv $OUT/launches_cfg3.txt "ncu launch list: python bench.py --config 3 --steps 2 --warmup 3 (gpu__time_duration.sum, --clock-control none)" | head -12
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_element$|^k_gather_units_v3$|^k_gather_f_dof$" -s 9 -c 3 \
  -o $OUT/full_cfg3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py $OUT/full_cfg3.ncu-rep > $OUT/ncu_full_cfg3.txt 2>&1; head -40 $OUT/ncu_full_cfg3.txt
for c in 2 4 5 6; do
  timeout 600 ncu --set full --clock-control none -k regex:"^k_element$" -s 3 -c 1 -o $OUT/el_cfg$c \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python tools/ncu_summary.py $OUT/el_cfg$c.ncu-rep > $OUT/ncu_el_cfg$c.txt 2>&1
done
