"""Markdown table of a `bench.py --ladder` run (one JSON line per rung + a summary line)."""
import json
import sys

rows, summ = [], {}
for line in open(sys.argv[1]):
    if line.startswith('{"family'):
        rows.append(json.loads(line))
    elif line.startswith('{"ladder'):
        summ = json.loads(line)
print(f"# Ladder throughput (bench.py --ladder), {sys.argv[2] if len(sys.argv) > 2 else ''}\n")
h = summ.get("host", {})
print(f"GPU: one B200 (HBM peak {summ.get('hbm_peak_gbs')} GB/s measured, FP64 {summ.get('fp64_peak_tflops_nominal', 0):.1f} TF "
      f"from unit counts). Oracle: all {summ.get('oracle_threads')} host cores ({h.get('cpu_model')}, {h.get('ram_gb')} GB), "
      "OpenMP element loop, bitwise the serial oracle; the beam's RES16/RES32 oracle timed on its first 100k elements.\n")
print("ms / eval: back-to-back calls from Python (host launch path included); graph: the same calls replayed "
      "from a CUDA graph (device time of the kernels alone). M el/s and the fractions use the stream timing.\n")
print("| family | rung | elements | rule | path | ms / eval | ms / eval (graph) | M el/s | G nnz/s | %HBM (paper layout) | %HBM (min layout) | %FP64 | oracle k el/s | GPU / oracle |")
print("|---|---|---:|---|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
for r in rows:
    nnz = f"{r['nnz_per_s'] / 1e9:.1f}" if r["nnz_per_s"] else "-"
    print(f"| {r['family']} | {r['res']} | {r['n_elements']} | {r['quadrature']} | "
          f"{'force only' if r['path'] == 'force_only' else 'force + H + g'} | {r['ms_per_eval']:.4f} | "
          f"{(r.get('ms_per_eval_graph') or float('nan')):.4f} | "
          f"{r['elements_per_s'] / 1e6:.1f} | {nnz} | {100 * r['hbm_frac_paper_layout']:.1f} | "
          f"{100 * r['hbm_frac_min_layout']:.1f} | {100 * r['fp64_frac']:.1f} | "
          f"{r['oracle_all_core_elements_per_s'] / 1e3:.1f} | {r['gpu_over_oracle']:.0f} |")
