"""Small evaluations for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): config 1 (T10 SVK class mode, 4-pt), a 100-element perturbed T10
(per-(e,q) table mode, SVK Keast-5 and MR + KV), an ANCF3443 4x4 plate (SVK
and the graded table-mode plate), an ANCF3243 beam, force-only, one AdamW
iteration and a 2-way virtual partition. Exits non-zero on a parity miss."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle  # noqa: E402
import paper_2604_10357_b200 as T  # noqa: E402
import synth  # noqa: E402


def d(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def state(mesh):
    if mesh.element == 0:
        return synth.t10_state(mesh, with_fext=True)
    x, v, vn = synth.ancf_state(mesh)
    return x, v, vn, None


base = synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4)
small = synth.Mesh(0, base.X, base.conn[:100])
cases = [("cfg1", synth.config(1).mesh, dict(synth.SVK_PAPER), 0),
         ("t10_100_perturbed_svk", synth.perturbed(small), dict(synth.SVK_PAPER), 1),
         ("t10_100_perturbed_mr_kv", synth.perturbed(small), dict(synth.MR_PAPER, **synth.KV_TIRE), 1),
         ("t10_100_svk_kv", small, dict(synth.SVK_PAPER, **synth.KV_TIRE), 1),
         ("ancf_4x4", synth.ancf_plate(4), dict(synth.SVK_PAPER), 2),
         ("ancf_5x5_graded", synth.ancf_plate_graded(5), dict(synth.SVK_PAPER), 2),
         ("beam_9", synth.ancf_beam(9), dict(synth.SVK_PAPER), 3),
         ("t10_100_straight_svk", synth.perturbed_straight(small), dict(synth.SVK_PAPER), 1)]
worst = 0.0
for name, mesh, mat, rule in cases:
    x, v, vn, fe = state(mesh)
    h = synth.H_T10 if mesh.element == 0 else synth.H_ANCF
    ctx = T.Context.from_mesh(mesh, mat, rule)
    g, H, f = ctx.empty_outputs()
    ctx.eval(d(x), d(v), d(vn), d(fe), h, g, H, f)
    fo = ctx.force_only(d(x), d(v))
    torch.cuda.synchronize()
    pr = oracle.Problem(mesh, mat, rule)
    g0, H0, f0 = pr.eval(x, v, vn, fe, h)
    e = max(rel(g.cpu().numpy(), g0), rel(H.cpu().numpy(), H0), rel(f.cpu().numpy(), f0), rel(fo.cpu().numpy(), f0))
    worst = max(worst, e)
    print(f"{name}: max rel err {e:.2e}", flush=True)
# the consistent Kelvin-Voigt tangent (NEXT-4): T10 two-phase (classes, tables), ANCF, beam
KVS = dict(eta_damp=2.0e6, lambda_damp=1.0e6)
for name, mesh, mat, rule in [("kvc_t10_svk", small, dict(synth.SVK_PAPER, **KVS), 1),
                              ("kvc_t10_perturbed_mr", synth.perturbed(small), dict(synth.MR_PAPER, **KVS), 0),
                              ("kvc_ancf_4x4", synth.ancf_plate(4), dict(synth.SVK_PAPER, **KVS), 2),
                              ("kvc_beam_5", synth.ancf_beam(5), dict(synth.MR_PAPER, **KVS), 3)]:
    x, v, vn, fe = state(mesh)
    h = synth.H_T10 if mesh.element == 0 else synth.H_ANCF
    ctx = T.Context.from_mesh(mesh, mat, rule, kv_consistent=True)
    g, H, f = ctx.empty_outputs()
    ctx.eval(d(x), d(v), d(vn), d(fe), h, g, H, f)
    torch.cuda.synchronize()
    pr = oracle.Problem(mesh, mat, rule)
    g0, H0, f0 = pr.eval(x, v, vn, fe, h, kv_consistent=True)
    e = max(rel(g.cpu().numpy(), g0), rel(H.cpu().numpy(), H0), rel(f.cpu().numpy(), f0))
    worst = max(worst, e)
    print(f"{name}: max rel err {e:.2e}", flush=True)
# one AdamW inner iteration (NEXT-2) on config 1 (no f_int: the element-inertia gradient path)
mesh = synth.config(1).mesh
x, v, vn, fe = state(mesh)
ctx = T.Context.from_mesh(mesh, dict(synth.SVK_PAPER), 0)
prm = dict(alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0)
vd, m, s, gd = d(v.copy()), torch.zeros_like(d(v)), torch.zeros_like(d(v)), torch.zeros_like(d(v))
ctx.adamw_iteration(d(x), d(vn), d(fe), 1e-3, 1, prm, vd, m, s, gd)
torch.cuda.synchronize()
# the library NCCL transport on a one-rank communicator (begin / exchange / interior / finish)
ctx1 = T.Context.from_mesh(mesh, dict(synth.SVK_PAPER), 0)
ctx1.nccl_attach(T.nccl_unique_id())
g1, H1, f1 = ctx1.empty_outputs()
buf = torch.zeros(1, dtype=torch.float64, device="cuda")
ctx1.eval_begin(d(x), d(v), 1e-3, H1, buf)
ctx1.eval_exchange(buf, buf)
ctx1.eval_interior(d(x), d(v), 1e-3, H1)
ctx1.eval_finish(buf, d(v), d(vn), d(fe), 1e-3, g1, H1, f1)
torch.cuda.synchronize()
# 2-way virtual partition (eval_begin / device copies / eval_finish)
P = 2
ctxs = [T.Context.from_mesh(mesh, dict(synth.SVK_PAPER), 0, rank=r, nranks=P) for r in range(P)]
sizes = [c.exchange_sizes() for c in ctxs]
sb = [torch.zeros(max(1, int(a.sum())), dtype=torch.float64, device="cuda") for a, _ in sizes]
rb = [torch.zeros(max(1, int(b.sum())), dtype=torch.float64, device="cuda") for _, b in sizes]
outs = [c.empty_outputs() for c in ctxs]
for r, c in enumerate(ctxs):
    c.eval_begin(d(x), d(v), 1e-3, outs[r][1], sb[r])
    c.eval_interior(d(x), d(v), 1e-3, outs[r][1])
for r in range(P):
    so = np.concatenate([[0], np.cumsum(sizes[r][0])])
    for p in range(P):
        n = int(sizes[r][0][p])
        if n:
            ro = np.concatenate([[0], np.cumsum(sizes[p][1])])
            rb[p][ro[r]:ro[r] + n].copy_(sb[r][so[p]:so[p] + n])
for r, c in enumerate(ctxs):
    g, H, f = outs[r]
    c.eval_finish(rb[r], d(v), d(vn), d(fe), 1e-3, g, H, f)
torch.cuda.synchronize()
print(f"worst parity {worst:.2e}")
sys.exit(0 if worst <= 1e-11 else 1)
