"""Device time of tlfea_force_only (the AdamW inner evaluation, Alg. 2
P:617-621) on a BASELINE config's mesh: CUDA events around K calls after W
warm-ups; prints one JSON line.

    python tools/bench_force_only.py --config 4 --steps 20 --warmup 3
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch

    import bench
    import paper_2604_10357_b200 as T
    cfg, mesh, x, v, vn, fext = bench.workload(args.config, "kuhn")
    ctx = T.Context.from_mesh(mesh, cfg.material, cfg.quadrature)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    xd, vd = d(x), d(v)
    kv = cfg.material.get("eta_damp", 0) > 0 or cfg.material.get("lambda_damp", 0) > 0
    f = torch.empty(ctx.n_dof, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        ctx.force_only(xd, vd if kv else None, f)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        ctx.force_only(xd, vd if kv else None, f)
    e1.record()
    torch.cuda.synchronize()
    kt = ctx.timing_report()
    ms = e0.elapsed_time(e1) / args.steps
    print(json.dumps({"metric": "force-only evaluations/s (tlfea_force_only)", "workload": cfg.name,
                      "n_elements": mesh.n_el, "ms_per_eval": ms, "elements_per_s": mesh.n_el / (ms / 1e3),
                      "kernels": {k: round(m / max(c, 1), 4) for k, (c, m) in kt.items() if c}}))


if __name__ == "__main__":
    main()
