# Executed fp64 flops of the element kernels (ncu thread-level SASS op counts:
# 2 x DFMA + DADD + DMUL) next to SURVEY §8(d)'s algorithmic flops per element.
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
while IFS='|' read -r flags kre; do
  echo "== $flags ($kre)"
  timeout 600 ncu --metrics $M --clock-control none -k regex:"$kre" -s 3 -c 1 --csv python bench.py $flags --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E 'dfma|dadd|dmul|duration' | awk -F'","' '{print $(NF-2), $NF}'
done <<'LIST'
--config 3|^k_element$
--config 2|^k_element$
--config 4|^k_element$
--config 5|k_force_t10_aff
--config 6|^k_element$
LIST
