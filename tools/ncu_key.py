"""Key metrics of every kernel in an ncu report (raw page)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h, u = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.per_cycle_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]
stalls = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    ix = {k: i for i, k in enumerate(h)}
    print("==", r[ix["Kernel Name"]][:80])
    for k in keys:
        if k in ix:
            print(f"  {k:75s} {r[ix[k]]:>18s} {u[ix[k]]}")
    st = sorted(((float(r[ix[k]] or 0), k) for k in stalls), reverse=True)[:8]
    print("  stalls/issue:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]} {v:.2f}" for v, k in st))
