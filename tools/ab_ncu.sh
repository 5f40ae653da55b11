# DRAM traffic of the element kernel, persistent-prefetch vs one tile per CTA
for pf in 1 0; do
echo "== PF=$pf"
TLFEA_PF=$pf timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sector_op_write_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"^k_element(_pf)?$" -c 1 python bench.py --config ${CFG:-3} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "duration|dram__|lts__|issue_active"
done
