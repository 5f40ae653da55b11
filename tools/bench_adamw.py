"""Measure one AdamW inner iteration (Alg. 2, tlfea_adamw_iteration; SURVEY
§8(f) NEXT-2) on a BASELINE config: CUDA events on the launching stream around
K iterations after W warm-ups, per-kernel live timing, and the HBM roofline of
the per-DOF update kernel (algorithmic bytes: reads g, m, s, v, q_n and writes
m, s, v, q = 72 B per DOF). Prints one JSON line.

    python tools/bench_adamw.py --config 3 --steps 20 --warmup 3
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2604_10357_b200 as T
    import synth

    cfg = synth.config(args.config)
    mesh = cfg.mesh
    if mesh.element == 0:
        x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    else:
        x, v, vn = synth.ancf_state(mesh)
        fext = np.random.default_rng(synth.SEED_BASE + 3).normal(size=x.shape)
    h = cfg.h
    ctx = T.Context.from_mesh(mesh, cfg.material, cfg.quadrature)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()
    qn, vnd, fed = d(x - h * v), d(vn), d(fext)
    vd = d(v)
    m = torch.zeros_like(vd)
    s = torch.zeros_like(vd)
    g = torch.zeros_like(vd)
    q = torch.empty_like(vd)
    norms = torch.empty(2, dtype=torch.float64, device="cuda")
    prm = dict(alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0)
    it = [0]

    def step():
        it[0] += 1
        ctx.adamw_iteration(qn, vnd, fed, h, it[0], prm, vd, m, s, g, q=q, norms=norms)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.set_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = T.launch_count()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    launches = T.launch_count() - n0
    ctx.set_timing(False)
    kt = ctx.timing_report()
    ms = e0.elapsed_time(e1) / args.steps
    ndof = 3 * mesh.n_coef
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(json.dumps({
        "metric": "AdamW inner iterations/s (Alg. 2: update + force-only Stage 1/2 + gradient + device norms)",
        "value": 1e3 / ms, "unit": "iterations/s", "ms_per_iteration": ms, "n_dof": ndof,
        "dof_updates_per_s": ndof / (ms / 1e3), "config": {"workload": cfg.name, "n_elements": mesh.n_el},
        "steps": args.steps, "warmup": args.warmup, "gpu_launches": launches, "dtype": "f64", "data": "synthetic",
        "kernels_ms_total": {k: round(v[1], 4) for k, v in kt.items() if v[0]},
        "update_kernel_note": "update + norm kernels are timed together under 'gather_f' with the gradient",
        "hbm_peak_gbs": peak, "update_alg_bytes_per_iteration": 72 * ndof,
        "final_norms": norms.cpu().numpy().tolist()}), flush=True)


if __name__ == "__main__":
    main()
