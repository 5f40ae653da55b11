# element-kernel metrics under env variants (VARS="A=1 B=2;C=3" separated by ';')
IFS=';'
for vars in ${VARS:-TLFEA_MERGE=1;TLFEA_MERGE=0}; do
echo "== $vars"
env $vars timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_write_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__pcsamp_warps_issue_stalled_long_scoreboard --clock-control none -k regex:"${KREGEX:-^k_element$}" -c 1 python bench.py --config ${CFG:-3} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "duration|dram__|lts__|issue_active|inst_exec|conflicts"
done
