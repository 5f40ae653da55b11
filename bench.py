#!/usr/bin/env python
"""bench.py — T10 force+tangent assembly throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A *step* is one pass of the whole hot path: tlfea_eval =
Stage 1 + Stage 2 force + tangent + deterministic CSR scatter of
H = M/h + h K + residual g, over one synthetic state of the workload.
Default workload: BASELINE config 3 (T10 Kuhn 144x96x48 cells, 3,981,312
elements, SVK, Keast-5, H with 1,384,065,801 nonzeros) — the largest
single-GPU mesh, on which BASELINE.json quotes the >=60%-HBM target; for N>1
it is element-partitioned across the ranks (x-slabs) with the boundary
H-row / nodal-force exchange over NCCL ("scaling": "strong": the mesh is
fixed). Inputs/outputs are far larger than L2 (H alone is 11 GB written per
step), so no L2 flush is needed between steps.

value      = elements of the whole mesh / device time per step (max over ranks)
e2e        = the same metric through tlfea_eval_host (host buffers, H2D of
             x, v, v_n, f_ext and D2H of g and H inside the timed region)
roofline   = dominant kernel, algorithmic bytes
             / its CUDA-event duration measured live on its launch stream
cpu_baseline = the CPU oracle (oracle/, as is, 1 core) on a bounded slice
`--impl reference` times that oracle as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "T10 force+tangent assembly elements/s (fp64) and % of B200 HBM roofline"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz
FP64_PEAK_PATH = os.path.join(ROOT, "profiles", "fp64_peak.json")   # tools/fp64_peak on a B200


def fp64_peak():
    try:
        return float(json.load(open(FP64_PEAK_PATH))["fp64_tflops"]), "measured (tools/fp64_peak, profiles/fp64_peak.json)"
    except Exception:
        return FP64_NOMINAL_TFLOPS, "nominal 148 SM x 64 FMA x 2 x 1.965 GHz (DESIGN.md)"

# Flops per quadrature point for force only / force + symmetric tangent:
# exact structured-SVK counts for T10 / ANCF3443;
# the ANCF3243 beam scaled from them (8-node kinematics + 36 blocks at the
# T10 per-block count of 71.9 flop), a model figure (+-20 %).
FLOP_PER_QP = {("t10", False): 468, ("t10", True): 4420, ("ancf", False): 684, ("ancf", True): 10252,
               ("beam", False): 380, ("beam", True): 2970}
# Mooney-Rivlin + Kelvin-Voigt, T10 Keast-5, force + tangent: the SURVEY
# §8(d) hand model of ~46 kflop per element (+-30 %), i.e. per qp
FLOP_PER_QP_MR_T10 = 46000 // 5


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    try:
        p = json.load(open(PEAKS_PATH))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- clocks --

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"clocks_{os.getpid()}_{gpu_index}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [t.strip() for t in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ workloads --

def workload(cfg_idx: int):
    cfg = synth.config(cfg_idx)
    mesh = cfg.mesh
    if cfg_idx == 5:
        mesh, x, v = synth.many_body()
        vn, fext = v.copy(), None
    elif mesh.element == 0:
        x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    else:
        # the beam chain bends over its own length (plate: 4 m)
        length = 4.0 if mesh.element == 1 else float(mesh.X[:, 0].max())
        x, v, vn = synth.ancf_state(mesh, length=length)
        fext = np.random.default_rng(synth.SEED_BASE + 3).normal(size=x.shape)
    return cfg, mesh, x, v, vn, fext


def bytes_per_element(mesh, info, tangent: bool, kv: bool):
    """Algorithmic bytes per element of the dominant (element) kernel in the
    paper's per-(e,q) layout: connectivity,
    reference gradients + J0 w, the unique gathered coordinates (and
    velocities), and its outputs (element force + upper tangent blocks)."""
    nen, nq = info["n_en"], info["n_qp"]
    nub = nen * (nen + 1) // 2
    coords = 24.0 * mesh.n_coef / mesh.n_el * (2 if kv else 1)
    # reference data: per-(e,q) tables (paper layout) or, with geometry
    # classes, one class id per element (tables staged in shared memory)
    ref = 1 if info.get("n_geometry_classes", 0) > 0 else 8 * nq * (3 * nen + 1)
    b = 4 * nen + ref + coords + 24 * nen
    if tangent:
        b += 72 * nub + 4 * nub   # upper blocks + their gather-sorted destinations
    return b


def fused_bytes_per_element(mesh, info, kv: bool):
    """Algorithmic bytes per element of the fused persistent eval (the whole
    tangent path in one kernel): what must cross
    HBM with no intermediate at all — connectivity, one class id, the unique
    gathers of x (v) and of v, v_n, f_ext for the residual, the unique g and
    f_int writes, the H values, and the mass row (values + columns) the
    residual reads. The element scratch round trip is NOT counted: it is the
    implementation's cost and shows up as `traffic` above these bytes."""
    nen = info["n_en"]
    per_node = mesh.n_coef / mesh.n_el
    b = 4 * nen + 1
    b += per_node * 24 * 4                 # x, v (also Fdot when KV), v_n, f_ext
    b += per_node * 24 * 2                 # g, f_int
    b += 8 * info["nnz"] / mesh.n_el       # H
    b += 12 * info["nnz_coef"] / mesh.n_el  # M values + column ids
    return b


def path_bytes_per_element(mesh, info, tangent: bool, kv: bool):
    """Algorithmic bytes per element of the whole path (SURVEY §8(d) 'paper
    layout' accounting): unique gathers of x, v, v_n, f_ext, the unique f/g
    write, the unique full-pattern H write, connectivity, a coefficient-level
    slot map and the per-(e,q) reference data."""
    nen, nq = info["n_en"], info["n_qp"]
    per_node = mesh.n_coef / mesh.n_el
    b = 4 * nen + 8 * nq * (3 * nen + 1) + 4 * nen * nen
    b += per_node * 24 * (4 if tangent else (2 if kv else 1))   # x, v, v_n, f_ext
    b += per_node * 24 * (2 if tangent else 1)                   # f_int (+ g)
    if tangent:
        b += 8 * info["nnz"] / mesh.n_el                         # H values
    return b


# ---------------------------------------------------------- CPU oracle --

def oracle_slice(cfg_idx: int, target_el: int):
    """A contiguous slice of the workload (the first x-slabs of the same mesh)
    with the same element size, material, rule and state recipe."""
    cfg = synth.config(cfg_idx)
    m = cfg.mesh
    if cfg_idx in (2, 3):
        nx, ny, nz = {2: (42, 28, 14), 3: (144, 96, 48)}[cfg_idx]
        per_slab = ny * nz * 6
        k = max(1, min(nx, target_el // per_slab))
        sub = synth.kuhn_t10_box(k, ny, nz, 3.0 * k / nx, 2.0, 1.0)
        x, v, vn, fext = synth.t10_state(sub, with_fext=True)
        return cfg, sub, x, v, vn, fext, f"first {k} of {nx} x-slabs ({sub.n_el} elements)"
    if cfg_idx == 4:
        n = max(2, int(np.sqrt(target_el)))
        sub = synth.ancf_plate(n, Lx=4.0 * n / 200, Ly=2.0 * n / 200)
        x, v, vn = synth.ancf_state(sub)
        return cfg, sub, x, v, vn, None, f"{n}x{n} corner of the 200x200 plate ({sub.n_el} elements)"
    if cfg_idx == 5:
        nb = max(1, target_el // 972)
        sub, x, v = synth.many_body(n_bodies=nb)
        return cfg, sub, x, v, v.copy(), None, f"{nb} of 2000 bodies ({sub.n_el} elements)"
    if cfg_idx == 6:
        n = max(1, min(m.n_el, target_el))
        sub = synth.ancf_beam(n)
        x, v, vn = synth.ancf_state(sub, length=float(m.X[:, 0].max()))
        fext = np.random.default_rng(synth.SEED_BASE + 3).normal(size=x.shape)
        return cfg, sub, x, v, vn, fext, f"first {n} of {m.n_el} beam elements"
    x, v, vn, fext = synth.t10_state(m, with_fext=True)
    return cfg, m, x, v, vn, fext, f"whole mesh ({m.n_el} elements)"


def time_oracle(cfg_idx: int, target_el: int, reps: int = 1):
    import oracle
    cfg, sub, x, v, vn, fext, desc = oracle_slice(cfg_idx, target_el)
    pr = oracle.Problem(sub, cfg.material, cfg.quadrature, with_precompute=False)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        pr.eval(x, v, vn, fext, cfg.h, hessian=not cfg.force_only)
        ts.append(time.perf_counter() - t0)
    return sub.n_el, ts, desc


def cpu_cores_used():
    return 1  # the oracle is single-threaded by construction


# ----------------------------------------------------------- reference arm --

def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    cfg_idx = args.config
    target = {1: 192, 2: 30000, 3: 40000, 4: 60, 5: 20000, 6: 30000}[cfg_idx]
    n_el, _, desc = time_oracle(cfg_idx, target, reps=0)
    _, ts, _ = time_oracle(cfg_idx, target, reps=args.warmup + args.steps)
    ts = ts[args.warmup:]
    sec = sum(ts) / len(ts)
    value = n_el / sec
    cfg = synth.config(cfg_idx)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg.name, "sample": desc},
            "cpu_baseline": {"value": value, "unit": "elements/s", "cores": cpu_cores_used(), "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- ours --

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2604_10357_b200 as T

    rank, world, local = env_rank()
    # TLFEA_DIST_BACKEND=gloo (tests only): ranks may share a GPU and the
    # packed partials travel through host memory; the bench proper uses NCCL
    backend = os.environ.get("TLFEA_DIST_BACKEND", "nccl")
    if backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, mesh, x, v, vn, fext = workload(args.config)
    force_only = cfg.force_only
    kv = cfg.material.get("eta_damp", 0) > 0 or cfg.material.get("lambda_damp", 0) > 0
    t_setup = time.perf_counter()
    ctx = T.Context.from_mesh(mesh, cfg.material, cfg.quadrature, rank=rank, nranks=world, device=local,
                              hessian=args.hessian, reference_layout="tables" if args.tables else "auto")
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    info = ctx.info
    dev = torch.device("cuda", local)
    d = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    xd, vd, vnd, fed = d(x), d(v), d(vn), d(fext)
    g, H, f = ctx.empty_outputs()
    if force_only:
        H = None
    stream = torch.cuda.current_stream()
    if world > 1:
        scount, rcount = ctx.exchange_sizes()
        sbuf = torch.empty(max(1, int(scount.sum())), dtype=torch.float64, device=dev)
        rbuf = torch.empty(max(1, int(rcount.sum())), dtype=torch.float64, device=dev)
        soff = np.concatenate([[0], np.cumsum(scount)])
        roff = np.concatenate([[0], np.cumsum(rcount)])

    def exchange():
        from paper_2604_10357_b200 import dist as tdist
        tdist.exchange(sbuf, rbuf, scount, rcount, host_staging=backend == "gloo")

    def step():
        if world == 1:
            if force_only:
                ctx.force_only(xd, vd if kv else None, f)
            else:
                ctx.eval(xd, vd, vnd, fed, cfg.h, g, H, f)
        else:
            ctx.eval_begin(xd, vd, cfg.h, H, sbuf, force_only=force_only)
            exchange()
            ctx.eval_finish(rbuf, vd, vnd, fed, cfg.h, None if force_only else g, H, f, force_only=force_only)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.4)
    ctx.set_timing(True)
    n0 = T.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = T.launch_count() - n0
    ctx.set_timing(False)
    kt = ctx.timing_report()
    clk = clocks.stop()
    ms_total = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = mesh.n_el / (ms_step / 1e3)

    # --- roofline of the dominant kernel (live CUDA events on its stream)
    hbm_peak, hbm_src = peaks()
    dom = max(kt, key=lambda k: kt[k][1])
    n_l, ms_l = kt[dom]
    avg_ms = ms_l / max(n_l, 1)
    elem = {0: "t10", 1: "ancf", 2: "beam"}[int(mesh.element)]
    if dom == "element":
        bpe = bytes_per_element(mesh, info, not force_only, kv)
        bytes_launch = bpe * info["n_elements"]
        per_qp = FLOP_PER_QP[(elem, not force_only)]
        if elem == "t10" and cfg.material["model"] == 1 and not force_only:
            per_qp = FLOP_PER_QP_MR_T10
        flops_launch = per_qp * info["n_qp"] * info["n_elements"]
    elif dom == "fused":
        bytes_launch = fused_bytes_per_element(mesh, info, kv) * info["n_elements"]
        flops_launch = (FLOP_PER_QP[(elem, True)] * info["n_qp"] * info["n_elements"]
                        + 9 * info["n_elements"] * info["n_en"] ** 2)
    elif dom == "gather_H":
        nnz_c = info["nnz_coef"]
        contrib = info["n_elements"] * info["n_en"] ** 2
        bytes_launch = nnz_c * (4 + 4 + 8 + 72) + contrib * (4 + 72) + 4 * info["n_owned_nodes"]
        flops_launch = 9 * contrib
    else:
        bytes_launch = 24 * info["n_elements"] * info["n_en"]
        flops_launch = 3 * info["n_elements"] * info["n_en"]
    gbs = bytes_launch / (avg_ms / 1e3) / 1e9
    tfl = flops_launch / (avg_ms / 1e3) / 1e12
    fp64_pk, fp64_src = fp64_peak()
    f_hbm, f_fp64 = gbs / hbm_peak, tfl / fp64_pk
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{cfg.name}:{dom}")
        except Exception:
            traffic = None
    if f_hbm >= f_fp64:
        roof = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": f_hbm,
                "traffic": traffic, "peak_source": hbm_src}
    else:
        roof = {"bound": "alu", "achieved": tfl, "peak": fp64_pk, "unit": "TFLOP/s", "frac": f_fp64,
                "traffic": traffic, "peak_source": fp64_src}
    roof.update({"kernel": dom, "kernel_ms": avg_ms, "hbm_frac": f_hbm, "fp64_frac": f_fp64,
                 "alg_bytes_per_launch": bytes_launch, "alg_flops_per_launch": flops_launch})
    path_b = path_bytes_per_element(mesh, info, not force_only, kv) * mesh.n_el
    kernels = {k: {"launches": c, "ms_per_launch": (m / c if c else 0.0), "share": (m / ms_total if ms_total else 0)}
               for k, (c, m) in kt.items()}

    # --- end to end through the public host-buffer API (N=1)
    e2e = None
    if world == 1 and not force_only and not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hx, hv, hvn, hfe = pin(x), pin(v), pin(vn), (pin(fext) if fext is not None else None)
        hg = torch.empty(3 * info["n_owned_nodes"], dtype=torch.float64).pin_memory()
        hH = torch.empty(info["nnz"], dtype=torch.float64).pin_memory()
        ctx.eval_host(hx, hv, hvn, hfe, cfg.h, hg, hH)
        ke = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(ke):
            ctx.eval_host(hx, hv, hvn, hfe, cfg.h, hg, hH)
        sec = (time.perf_counter() - t0) / ke
        h2d = 8 * (x.size + v.size + vn.size + (fext.size if fext is not None else 0))
        d2h = 8 * (hg.numel() + hH.numel())
        e2e = {"value": mesh.n_el / sec, "unit": "elements/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * sec}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # ~10-15 s of 1-core oracle work (whole mesh where it is smaller)
        target = {1: 192, 2: 98784, 3: 250000, 4: 18500, 5: 1944000, 6: 235000}[args.config]
        n_el_s, ts, desc = time_oracle(args.config, target)
        cpu = {"value": n_el_s / ts[0], "unit": "elements/s", "cores": cpu_cores_used(), "kind": "oracle",
               "sample": desc, "seconds": ts[0]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg.name, "n_elements": mesh.n_el, "nnz_H": int(info["nnz"]) if world == 1 else None,
                       "quadrature": ["t10_4pt", "keast5", "gl443", "gl322"][cfg.quadrature],
                       "material": ["svk", "mooney_rivlin"][cfg.material["model"]] + ("+kv" if kv else ""),
                       "path": "force_only" if force_only else "force+tangent+residual (tlfea_eval)",
                       "hessian_storage": args.hessian,
                       "parallelism": f"element-partition x{world}" if world > 1 else "1 GPU",
                       "geometry_classes": info["n_geometry_classes"],
                       "l2": "inputs/outputs larger than L2 (no flush needed)",
                       "nnz_per_s": 9 * info["nnz_coef"] * world / (ms_step / 1e3) if world == 1 else None,
                       "path_hbm_frac": path_b / (ms_step / 1e3) / 1e9 / hbm_peak,
                       "path_alg_bytes_per_el": path_b / mesh.n_el, "setup_s": t_setup,
                       "kernels": kernels},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--hessian", choices=["full", "upper"], default="full",
                    help="H storage (full DOF CSR = the headline; upper = NEXT-4 variant)")
    ap.add_argument("--tables", action="store_true",
                    help="per-(e,q) reference tables in HBM (the paper's layout, as for a mesh of non-congruent "
                         "elements) instead of the shared-memory geometry classes")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
