# A/B of variant builds: LIBS="name ..." (paper_2604_10357_b200/libtlfea_<name>.so; "cur" = libtlfea.so) on bench configs $CFGS
for c in ${CFGS:-3}; do
  for i in $(seq ${REPS:-2}); do
    for v in ${LIBS}; do
      L=paper_2604_10357_b200/libtlfea_$v.so; [ $v = cur ] && L=paper_2604_10357_b200/libtlfea.so
      TLFEA_LIB=$L timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e $EXTRA > gpurun_out/abv_${v}_c${c}_$i.json 2>&1
      python -c "import json;d=json.loads(open('gpurun_out/abv_${v}_c${c}_$i.json').read().strip().splitlines()[-1]);k=d['config']['kernels'];print('$v cfg$c', round(d['ms_per_step'],4), {n:round(x['ms_per_launch'],4) for n,x in k.items() if x['launches']})" || tail -3 gpurun_out/abv_${v}_c${c}_$i.json
    done
  done
done
