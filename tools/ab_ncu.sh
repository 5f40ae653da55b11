# Element-kernel metrics of variant builds (LIBS="name ..." -> paper_2604_10357_b200/libtlfea_<name>.so,
# "cur" = libtlfea.so) on bench config $CFG, one ncu pass each (never a bench number).
for v in ${LIBS:-cur}; do
  L=paper_2604_10357_b200/libtlfea_$v.so; [ $v = cur ] && L=paper_2604_10357_b200/libtlfea.so
  echo "== $v"
  TLFEA_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:"${KREGEX:-^k_element$}" -c 1 python bench.py --config ${CFG:-3} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "duration|dram__|issue_active|inst_exec|conflicts"
done
