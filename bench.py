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
import dataclasses
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

def workload(cfg_idx: int, variant: str = "kuhn"):
    cfg = synth.config(cfg_idx)
    mesh = cfg.mesh
    if variant == "straight" and mesh.element == 0 and cfg_idx != 5:
        # the same mesh with randomly displaced corners (straight-sided, no two
        # elements congruent): the affine (min) layout path
        mesh = synth.perturbed_straight(mesh)
        cfg = dataclasses.replace(cfg, name=cfg.name + "_straight", mesh=mesh)
    if variant == "curved" and mesh.element == 0 and cfg_idx != 5:
        # every node (mid-edge nodes too) randomly displaced: curved, non-congruent
        # isoparametric T10, the per-(e,q) J^-1 layout path
        mesh = synth.perturbed(mesh)
        cfg = dataclasses.replace(cfg, name=cfg.name + "_curved", mesh=mesh)
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


def alg_bytes_per_element(mesh, info, tangent: bool, kv: bool, layout: str = "paper"):
    """SURVEY §8(d) algorithmic bytes per element of the whole path (what
    must cross HBM with no intermediate at all): the unique gathers of x (and
    v, v_n, f_ext for the residual; v alone when Kelvin-Voigt drives a
    force-only evaluation), the unique f/g write, the unique full-pattern H
    write, the connectivity (4 B per physical node), a coefficient-level slot
    map (4 n_en^2 B, tangent only) and the reference data: per-(e,q) grad N +
    J0 w ("paper" layout) or the "min" layout (13 fp64 per affine
    T10 element; one shared table for a uniform ANCF plate or beam). Config 3
    gives 4,624 (paper) / 3,488 (min) B/el, config 5 1,365 / 229, the 200x200
    ANCF plate 30,741 / 11,925, as in §8(d)'s table."""
    nen, nq = info["n_en"], info["n_qp"]
    per_coef = mesh.n_coef / mesh.n_el
    n_phys = {0: 10, 1: 4, 2: 2}[int(mesh.element)]
    b = 4 * n_phys
    b += per_coef * 24 * (4 if tangent else (2 if kv else 1))   # x, v, v_n, f_ext | x (, v)
    b += per_coef * 24                                          # f / g
    if tangent:
        b += 8 * info["nnz"] / mesh.n_el + 4 * nen * nen          # H values, slot map
    if layout == "paper":
        b += 8 * nq * (3 * nen + 1)
    elif int(mesh.element) == 0:
        b += 8 * 13
    return b


def alg_flops_per_element(mesh, info, tangent: bool, model: int):
    """SURVEY §8(d) flops per element: exact structured-SVK counts per
    quadrature point (468 force / 4,420 force + symmetric tangent for T10,
    684 / 10,252 ANCF3443; the beam scaled from them), plus the M/h term of H
    (0.4 kflop/el T10, 1 kflop/el ANCF); Mooney-Rivlin + KV: §8(d)'s model."""
    elem = {0: "t10", 1: "ancf", 2: "beam"}[int(mesh.element)]
    if elem == "t10" and model == 1 and tangent:
        return float(FLOP_PER_QP_MR_T10 * info["n_qp"])
    f = FLOP_PER_QP[(elem, tangent)] * info["n_qp"]
    if tangent:
        f += 400 if elem == "t10" else 1000
    return float(f)


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


def time_oracle(cfg_idx: int, target_el: int, reps: int = 1, all_cores: bool = False):
    import oracle
    cfg, sub, x, v, vn, fext, desc = oracle_slice(cfg_idx, target_el)
    pr = oracle.Problem(sub, cfg.material, cfg.quadrature, with_precompute=False)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        pr.eval(x, v, vn, fext, cfg.h, hessian=not cfg.force_only, all_cores=all_cores)
        ts.append(time.perf_counter() - t0)
    return sub.n_el, ts, desc


def host_info():
    """CPU model, logical cores available to this process and RAM (GB)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 1024 ** 2, 1)
    except OSError:
        pass
    return {"cpu_model": model, "cores_available": len(os.sched_getaffinity(0)), "ram_gb": ram}


def cpu_baseline(cfg_idx: int):
    """the oracle as it stands on this host. (ii) all cores
    (OpenMP element loop, thread-private element blocks merged in element
    order: bitwise the serial oracle) = the CPU-baseline figure; (i) one core
    beside it. Bounded samples (a few seconds of oracle work each)."""
    import oracle
    target_all = {1: 192, 2: 98784, 3: 331776, 4: 10000, 5: 972000, 6: 500000}[cfg_idx]
    target_one = {1: 192, 2: 13824, 3: 27648, 4: 1600, 5: 97200, 6: 50000}[cfg_idx]
    cfg, sub, x, v, vn, fext, desc = oracle_slice(cfg_idx, target_all)
    pr = oracle.Problem(sub, cfg.material, cfg.quadrature, with_precompute=False)
    t0 = time.perf_counter()
    pr.eval(x, v, vn, fext, cfg.h, hessian=not cfg.force_only, all_cores=True)
    t_all = time.perf_counter() - t0
    cores = oracle.max_threads()
    cfg1, sub1, x1, v1, vn1, fext1, desc1 = oracle_slice(cfg_idx, target_one)
    pr1 = oracle.Problem(sub1, cfg1.material, cfg1.quadrature, with_precompute=False)
    t0 = time.perf_counter()
    pr1.eval(x1, v1, vn1, fext1, cfg1.h, hessian=not cfg1.force_only)
    t_one = time.perf_counter() - t0
    return {"value": sub.n_el / t_all, "unit": "elements/s", "cores": cores, "kind": "oracle",
            "sample": desc, "seconds": t_all,
            "one_core": {"value": sub1.n_el / t_one, "sample": desc1, "seconds": t_one},
            "host": host_info()}


# ----------------------------------------------------------- reference arm --

def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import oracle
    cfg_idx = args.config
    target = {1: 192, 2: 98784, 3: 165888, 4: 10000, 5: 486000, 6: 250000}[cfg_idx]
    n_el, ts, desc = time_oracle(cfg_idx, target, reps=args.warmup + args.steps, all_cores=True)
    ts = ts[args.warmup:]
    sec = sum(ts) / len(ts)
    value = n_el / sec
    cfg = synth.config(cfg_idx)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg.name, "sample": desc},
            "cpu_baseline": {"value": value, "unit": "elements/s", "cores": oracle.max_threads(), "kind": "oracle",
                             "sample": desc + " (all-core OpenMP element loop, bitwise the serial oracle)",
                             "host": host_info()},
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
    cfg, mesh, x, v, vn, fext = workload(args.config, args.mesh)
    force_only = cfg.force_only
    kv = cfg.material.get("eta_damp", 0) > 0 or cfg.material.get("lambda_damp", 0) > 0
    t_setup = time.perf_counter()
    ctx = T.Context.from_mesh(mesh, cfg.material, cfg.quadrature, rank=rank, nranks=world, device=local,
                              hessian=args.hessian, reference_layout="tables" if args.tables else "auto",
                              kv_consistent=args.kv_consistent)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    info = ctx.info
    dev = torch.device("cuda", local)
    # accounting on the GLOBAL mesh (a rank's info holds its owned-row nnz)
    ginfo = dict(info)
    if world > 1:
        t_nnz = torch.tensor([float(info["nnz"])], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t_nnz, op=dist.ReduceOp.SUM)
        ginfo["nnz"] = int(t_nnz.item())
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
        if args.transport == "lib":
            uid = [T.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ctx.nccl_attach(uid[0])
        soff = np.concatenate([[0], np.cumsum(scount)])
        roff = np.concatenate([[0], np.cumsum(rcount)])

    def step():
        if world == 1:
            if force_only:
                ctx.force_only(xd, vd if kv else None, f)
            else:
                ctx.eval(xd, vd, vnd, fed, cfg.h, g, H, f)
        else:
            from paper_2604_10357_b200 import dist as tdist
            # boundary elements + pack; the exchange (NCCL stream) overlaps the
            # interior elements; finish adds the received partials
            ctx.eval_begin(xd, vd, cfg.h, H, sbuf, force_only=force_only)
            if args.transport == "lib":   # the library's NCCL transport (tlfea_eval_exchange)
                ctx.eval_exchange(sbuf, rbuf)
                ctx.eval_interior(xd, vd, cfg.h, H, force_only=force_only)
            else:
                works = tdist.exchange_start(sbuf, rbuf, scount, rcount, host_staging=backend == "gloo")
                ctx.eval_interior(xd, vd, cfg.h, H, force_only=force_only)
                tdist.exchange_wait(works)
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

    # --- roofline of the dominant kernel (live CUDA events on its stream):
    # achieved = SURVEY §8(d) algorithmic bytes (flops) per element x the
    # elements one launch processes / the launch's average duration
    hbm_peak, hbm_src = peaks()
    dom = max(kt, key=lambda k: kt[k][1])
    n_l, ms_l = kt[dom]
    avg_ms = ms_l / max(n_l, 1) if ms_l > 0 else float("nan")
    n_loc = info["n_elements"]
    model = int(cfg.material["model"])
    b_paper = alg_bytes_per_element(mesh, ginfo, not force_only, kv, "paper")
    b_min = alg_bytes_per_element(mesh, ginfo, not force_only, kv, "min")
    fl_el = alg_flops_per_element(mesh, ginfo, not force_only, model)
    bytes_launch, flops_launch = b_paper * n_loc, fl_el * n_loc
    gbs = bytes_launch / (avg_ms / 1e3) / 1e9
    tfl = flops_launch / (avg_ms / 1e3) / 1e12
    fp64_meas, fp64_src = fp64_peak()
    f_hbm, f_fp64 = gbs / hbm_peak, tfl / FP64_NOMINAL_TFLOPS
    mode = "force_only" if force_only else ("force+tangent+kvc" if info.get("kv_consistent_tangent") else "force+tangent")
    layout = ["classes", "tables", "affine", "jinv"][info.get("reference_layout", 1)]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{cfg.name}|{mode}|{args.hessian}|{layout}|{dom}")
        except Exception:
            traffic = None
    common = {"traffic": traffic, "traffic_over_alg": (traffic / bytes_launch if traffic else None),
              "kernel": dom, "kernel_ms": avg_ms, "alg_bytes_per_el": b_paper, "alg_bytes_per_el_min": b_min,
              "alg_flops_per_el": fl_el, "hbm_frac": f_hbm, "hbm_frac_min_layout": b_min * n_loc / (avg_ms / 1e3)
              / 1e9 / hbm_peak, "fp64_frac": f_fp64, "fp64_frac_of_measured": tfl / fp64_meas,
              "fp64_peak_measured": fp64_meas, "fp64_peak_measured_source": fp64_src}
    if f_hbm >= f_fp64:
        roof = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": f_hbm,
                "peak_source": hbm_src, **common}
        if f_hbm > 1.0:
            roof["note"] = ("frac > 1: the numerator is SURVEY §8(d)'s paper-layout bytes (per-(e,q) tables); this "
                            "path reads no tables (geometry classes / affine layout), so it beats that roofline; "
                            "hbm_frac_min_layout is the fraction against the bytes it must move")
    else:
        roof = {"bound": "alu", "achieved": tfl, "peak": FP64_NOMINAL_TFLOPS, "unit": "TFLOP/s", "frac": f_fp64,
                "peak_source": "DFMA unit count: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md)", **common}
    path_b = b_paper * mesh.n_el
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
        cpu = cpu_baseline(args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg.name, "n_elements": mesh.n_el, "nnz_H": int(ginfo["nnz"]),
                       "quadrature": ["t10_4pt", "keast5", "gl443", "gl322"][cfg.quadrature],
                       "material": ["svk", "mooney_rivlin"][cfg.material["model"]] + ("+kv" if kv else ""),
                       "path": "force_only" if force_only else "force+tangent+residual (tlfea_eval)",
                       "hessian_storage": args.hessian,
                       "tangent": "consistent_kv (NEXT-4)" if info.get("kv_consistent_tangent") else "elastic (Q8)",
                       "parallelism": f"element-partition x{world} ({args.transport} transport)" if world > 1 else "1 GPU",
                       "geometry_classes": info["n_geometry_classes"],
                       "reference_layout": ["classes", "per-(e,q) tables", "affine min layout",
                                            "per-(e,q) J^-1 (curved T10)"][info["reference_layout"]],
                       "l2": "inputs/outputs larger than L2 (no flush needed)",
                       "nnz_per_s": ginfo["nnz"] / (ms_step / 1e3) if not force_only else None,
                       "path_hbm_frac": path_b / (ms_step / 1e3) / 1e9 / hbm_peak,
                       "path_hbm_frac_min_layout": b_min * mesh.n_el / (ms_step / 1e3) / 1e9 / hbm_peak,
                       "path_alg_bytes_per_el": b_paper, "path_alg_bytes_per_el_min": b_min,
                       "path_fp64_frac": fl_el * mesh.n_el / (ms_step / 1e3) / 1e12 / FP64_NOMINAL_TFLOPS,
                       "setup_s": t_setup,
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


# --------------------------------------------------------------- ladder --

LADDER_T10 = ((3, 2, 1), (6, 4, 2), (9, 6, 3), (15, 10, 5), (24, 16, 8), (39, 26, 13))
LADDER_ANCF = (10, 20, 50, 100, 150, 200)
LADDER_BEAM = (1000, 10000, 50000, 100000, 200000, 500000)
RES = ("RES0", "RES2", "RES4", "RES8", "RES16", "RES32")


def run_ladder(args):
    """north_star: throughput on synthetic meshes shaped like the paper's
    six-resolution ladders (T10 Kuhn beams under both rules, the ANCF3443
    plates, the ANCF3243 chains), force + tangent (tlfea_eval) and force only,
    with the all-core oracle on the same rung beside each GPU number."""
    import torch

    import oracle
    import paper_2604_10357_b200 as T
    torch.cuda.set_device(0)
    hbm_peak, _ = peaks()
    rows = []

    def measure(name, res, mesh, mat, rule, h, force_only):
        if mesh.element == 0:
            x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
        else:
            x, v, vn = synth.ancf_state(mesh, length=4.0 if mesh.element == 1 else float(mesh.X[:, 0].max()))
            fext = None
        ctx = T.Context.from_mesh(mesh, mat, rule)
        info = ctx.info
        d = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
        xd, vd, vnd, fed = d(x), d(v), d(vn), d(fext)
        g, H, f = ctx.empty_outputs()
        step = (lambda: ctx.force_only(xd, None, f)) if force_only else (lambda: ctx.eval(xd, vd, vnd, fed, h, g, H, f))
        for _ in range(3):
            step()
        k = int(max(10, min(200, 4e6 / mesh.n_el)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(k):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        # the same evaluations replayed from a CUDA graph (no host launch path):
        # the device time of the library's kernels alone
        ms_graph = None
        try:
            kg = int(min(k, 50))
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream().wait_stream(side)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for _ in range(kg):
                    step()
            graph.replay()
            torch.cuda.synchronize()
            e0.record()
            graph.replay()
            e1.record()
            torch.cuda.synchronize()
            ms_graph = e0.elapsed_time(e1) / kg
            del graph
        except Exception as ex:  # capture unsupported: report the stream timing only
            print(f"graph capture failed: {ex}", file=sys.stderr)
        kv = False
        bp = alg_bytes_per_element(mesh, info, not force_only, kv, "paper")
        bm = alg_bytes_per_element(mesh, info, not force_only, kv, "min")
        fl = alg_flops_per_element(mesh, info, not force_only, int(mat["model"]))
        del ctx, g, H, f
        torch.cuda.empty_cache()
        # the oracle on the same rung (all cores; the first elements of the
        # beam's two largest chains, which take it beyond a few seconds)
        sub, xs, vs, vns, fes = mesh, x, v, vn, fext
        if mesh.element == 2 and mesh.n_el > 100000:
            sub = synth.ancf_beam(100000)
            xs, vs, vns = synth.ancf_state(sub, length=float(mesh.X[:, 0].max()))
            fes = None
        pr = oracle.Problem(sub, mat, rule, with_precompute=False)
        t0 = time.perf_counter()
        pr.eval(xs, vs, vns, fes, h, hessian=not force_only, all_cores=True)
        t_or = time.perf_counter() - t0
        row = {"family": name, "res": res, "n_elements": mesh.n_el, "quadrature": ["t10_4pt", "keast5", "gl443", "gl322"][rule],
               "path": "force_only" if force_only else "force+tangent+residual", "ms_per_eval": ms,
               "ms_per_eval_graph": ms_graph,
               "elements_per_s_graph": mesh.n_el / (ms_graph / 1e3) if ms_graph else None,
               "elements_per_s": mesh.n_el / (ms / 1e3),
               "nnz_per_s": (info["nnz"] / (ms / 1e3)) if not force_only else None, "nnz_H": info["nnz"],
               "hbm_frac_paper_layout": bp * mesh.n_el / (ms / 1e3) / 1e9 / hbm_peak,
               "hbm_frac_min_layout": bm * mesh.n_el / (ms / 1e3) / 1e9 / hbm_peak,
               "fp64_frac": fl * mesh.n_el / (ms / 1e3) / 1e12 / FP64_NOMINAL_TFLOPS,
               "geometry_classes": info["n_geometry_classes"],
               "oracle_all_core_elements_per_s": sub.n_el / t_or, "oracle_sample_elements": sub.n_el,
               "gpu_over_oracle": (mesh.n_el / (ms / 1e3)) / (sub.n_el / t_or)}
        print(json.dumps(row), flush=True)
        rows.append(row)

    svk = dict(synth.SVK_PAPER)
    for res, (nx, ny, nz) in zip(RES, LADDER_T10):
        mesh = synth.kuhn_t10_box(nx, ny, nz, 3.0, 2.0, 1.0)
        for rule in (synth.Q_T10_4PT, synth.Q_T10_KEAST5):
            for fo in (False, True):
                measure("t10_kuhn", res, mesh, svk, rule, synth.H_T10, fo)
    for res, n in zip(RES, LADDER_ANCF):
        mesh = synth.ancf_plate(n)
        for fo in (False, True):
            measure("ancf3443_plate", res, mesh, svk, synth.Q_GL_443, synth.H_ANCF, fo)
    for res, n in zip(RES, LADDER_BEAM):
        mesh = synth.ancf_beam(n)
        for fo in (False, True):
            measure("ancf3243_beam", res, mesh, svk, synth.Q_GL_322, synth.H_BEAM, fo)
    host = host_info()
    print(json.dumps({"ladder": rows, "host": host, "oracle_threads": oracle.max_threads(),
                      "hbm_peak_gbs": hbm_peak, "fp64_peak_tflops_nominal": FP64_NOMINAL_TFLOPS}), flush=True)


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
    ap.add_argument("--mesh", choices=["kuhn", "straight", "curved"], default="kuhn",
                    help="straight: the T10 mesh with randomly displaced corners (straight-sided, non-congruent: "
                         "the affine min layout instead of geometry classes); curved: every node displaced "
                         "(isoparametric, non-congruent: the per-(e,q) J^-1 layout)")
    ap.add_argument("--transport", choices=["torch", "lib"], default="torch",
                    help="N>1 exchange: torch.distributed P2P (NCCL) or the library's own NCCL transport "
                         "(tlfea_nccl_attach / tlfea_eval_exchange)")
    ap.add_argument("--kv-consistent", action="store_true",
                    help="H = the consistent Kelvin-Voigt tangent dg/dv (NEXT-4; configs with damping, e.g. 2)")
    ap.add_argument("--ladder", action="store_true",
                    help="the paper's six-resolution ladders (T10, ANCF3443, ANCF3243), one line per rung")
    ap.add_argument("--tables", action="store_true",
                    help="per-(e,q) reference tables in HBM (the paper's layout, as for a mesh of non-congruent "
                         "elements) instead of the shared-memory geometry classes")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.ladder:
        run_ladder(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
