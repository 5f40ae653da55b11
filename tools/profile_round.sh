# Round measurement on one B200 (run through gpurun from the repo root):
#   the default bench line per config and variant, the ladder, the reference
#   arm, AdamW, the ncu launch list of the default bench command, one ncu
#   --set full capture of the three config-3 kernels (traffic, stalls, source),
#   the element kernels of the other configs and of the variants (summaries +
#   DRAM traffic keyed for bench.py; the large per-config reports are deleted
#   on the box to stay under gpurun's 64 MiB return), the smoke test.
# Outputs land in gpurun_out/$TAG/ (scratch); copy summaries into profiles/.
set -u
TAG=${TAG:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
line() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);k=d['config'].get('kernels',{});print('$2', round(d['value']/1e6,2), 'M el/s', round(d['ms_per_step'],4), 'ms', d['roofline']['bound'], round(d['roofline']['frac'],3), {a:round(x['ms_per_launch'],4) for a,x in k.items() if x['launches']})" || tail -3 $1; }
for c in ${CFGS:-3 1 2 4 5 6}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
  line $OUT/bench_cfg$c.json cfg$c
done
for v in "--config 3 --mesh straight" "--config 3 --tables" "--config 3 --hessian upper" "--config 2 --kv-consistent"; do
  n=$(echo $v | tr -d ' -')
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $v > $OUT/bench_$n.json 2> $OUT/bench_$n.err
  line $OUT/bench_$n.json $n
done
python tools/bench_adamw.py --config 3 > $OUT/adamw_cfg3.json 2> $OUT/adamw.err; tail -c 400 $OUT/adamw_cfg3.json
for c in 2 4 5 6; do python tools/bench_force_only.py --config $c > $OUT/force_only_cfg$c.json 2> $OUT/force_only_cfg$c.err; tail -c 250 $OUT/force_only_cfg$c.json; done
timeout 900 python bench.py --ladder > $OUT/ladder.jsonl 2> $OUT/ladder.err; wc -l $OUT/ladder.jsonl
timeout 600 python bench.py --impl reference --config 3 --steps 2 --warmup 3 > $OUT/reference_cfg3.json 2> $OUT/reference_cfg3.err; tail -c 300 $OUT/reference_cfg3.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg3.csv \
  python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/summarize_launches.py $OUT/launches_cfg3.csv $OUT/launches_cfg3.txt "ncu launch list: python bench.py --config 3 --steps 2 --warmup 3 (gpu__time_duration.sum, --clock-control none)" | head -12
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_element$|^k_gather_units_v3$|^k_gather_f_dof$" -s 9 -c 3 \
  -o $OUT/full_cfg3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py $OUT/full_cfg3.ncu-rep > $OUT/ncu_full_cfg3.txt 2>&1; head -40 $OUT/ncu_full_cfg3.txt
python tools/ncu_stalls_by_line.py $OUT/full_cfg3.ncu-rep '^k_element$' > $OUT/stalls_element_cfg3.txt 2>&1
python tools/ncu_stalls_by_line.py $OUT/full_cfg3.ncu-rep k_gather_units_v3 > $OUT/stalls_gather_cfg3.txt 2>&1
python tools/ncu_traffic.py $OUT/full_cfg3.ncu-rep "cfg3_t10_144x96x48_svk_keast5|force+tangent|full|classes" $OUT/ncu_traffic.json
# element kernels of the other configs and variants: (config flags | kernel regex | skip | traffic key prefix)
while IFS='|' read -r flags kre skip key; do
  n=$(echo $flags | tr -d ' -')
  timeout 600 ncu --set full --clock-control none -k regex:"$kre" -s $skip -c 2 -o $OUT/el_$n \
    python bench.py $flags --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python tools/ncu_summary.py $OUT/el_$n.ncu-rep > $OUT/ncu_el_$n.txt 2>&1
  python tools/ncu_traffic.py $OUT/el_$n.ncu-rep "$key" $OUT/ncu_traffic.json > /dev/null 2>&1
  rm -f $OUT/el_$n.ncu-rep
done <<'EOF'
--config 2|^k_element$|3|cfg2_t10_42x28x14_mr_kv_keast5|force+tangent|full|classes
--config 4|^k_element$|3|cfg4_ancf3443_200x200_svk_gl443|force+tangent|full|classes
--config 5|k_force_t10_aff|3|cfg5_manybody_2000x_t10_9x6x3_force_only|force_only|full|classes
--config 6|^k_element$|3|cfg6_ancf3243_beam_res32_500k_svk_gl322|force+tangent|full|classes
--config 3 --hessian upper|^k_gather_units_v3$|3|cfg3_t10_144x96x48_svk_keast5|force+tangent|upper|classes
--config 3 --tables|^k_element$|3|cfg3_t10_144x96x48_svk_keast5|force+tangent|full|tables
--config 3 --mesh straight|^k_element$|3|cfg3_t10_144x96x48_svk_keast5|force+tangent|full|affine
--config 2 --kv-consistent|k_element_t10kvc|3|cfg2_t10_42x28x14_mr_kv_keast5|force+tangent+kvc|full|classes
EOF
ls -la $OUT | head -60
