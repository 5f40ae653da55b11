"""GPU parity of the CONSISTENT Kelvin-Voigt tangent (options.kv_consistent_tangent,
SURVEY §8(f) NEXT-4): H = dg/dv = M/h + h df/dx + df/dv with x = q_n + h v
(Eq. residual, Eq. hessian, reading Q9), non-symmetric, on
the FULL pattern, against the oracle's complex-step tangent (orc_eval_kvc,
pinned in tests/test_oracle_kvc.py). Same bar as the symmetric path: pattern
bit-exact, values within 1e-11 normwise, bitwise run-to-run."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = 1e-11
# strong damping: the viscous blocks are O(1) of H (eta/h ~ 3 E), so an error in
# any of them is far above the bar; the paper's tire damping is kept too
KV_STRONG = dict(eta_damp=2.0e6, lambda_damp=1.0e6)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_10357_b200 as T
    T.lib()
    return torch


def dev(torch, a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def box(nx, ny, nz, n=None):
    m = synth.kuhn_t10_box(nx, ny, nz, 0.2 * nx, 0.2 * ny, 0.2 * nz)
    return m if n is None else synth.Mesh(0, m.X, m.conn[:n])


CASES = {
    # T10 with geometry classes (6) and on the per-(e,q) tables, both rules,
    # ragged tails inside a warp group / CTA tile
    "t10_4x3x2_svk_strong_keast5": lambda: (box(4, 3, 2), dict(synth.SVK_PAPER, **KV_STRONG), 1),
    "t10_100el_svk_tire_4pt": lambda: (box(5, 3, 2, 100), dict(synth.SVK_PAPER, **synth.KV_TIRE), 0),
    "t10_3x2x2_mr_strong_keast5": lambda: (box(3, 2, 2), dict(synth.MR_PAPER, **KV_STRONG), 1),
    "t10_100el_perturbed_mr_strong_4pt": lambda: (synth.perturbed(box(5, 3, 2, 100)),
                                                  dict(synth.MR_PAPER, **KV_STRONG), 0),
    "t10_3x3x2_perturbed_svk_strong_keast5": lambda: (synth.perturbed(box(3, 3, 2)),
                                                      dict(synth.SVK_PAPER, **KV_STRONG), 1),
    "t10_4x3x2_straight_svk_tire_keast5": lambda: (synth.perturbed_straight(box(4, 3, 2)),
                                                   dict(synth.SVK_PAPER, **synth.KV_TIRE), 1),
    # ANCF3443 plates (uniform: classes; graded: tables) and the ANCF3243 beam
    "ancf_4x4_svk_strong": lambda: (synth.ancf_plate(4), dict(synth.SVK_PAPER, **KV_STRONG), 2),
    "ancf_5x5_graded_mr_strong": lambda: (synth.ancf_plate_graded(5), dict(synth.MR_PAPER, **KV_STRONG), 2),
    "beam_9_svk_strong": lambda: (synth.ancf_beam(9), dict(synth.SVK_PAPER, **KV_STRONG), 3),
    "beam_5_perturbed_mr_strong": lambda: (synth.perturbed(synth.ancf_beam(5), amp=0.02),
                                           dict(synth.MR_PAPER, **KV_STRONG), 3),
}


def state(mesh, strong):
    if mesh.element == 0:
        x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    else:
        x, v, vn = synth.ancf_state(mesh)
        fext = np.random.default_rng(synth.SEED_BASE + 3).normal(size=x.shape)
    if strong:
        v = 20.0 * v   # |v| ~ 1 m/s: the x-derivative of the viscous stress is O(10 %) of H
    return x, v, vn, fext


def run(torch, mesh, mat, rule, x, v, vn, fext, h, kvc):
    import paper_2604_10357_b200 as T
    ctx = T.Context.from_mesh(mesh, mat, rule, kv_consistent=kvc)
    g, H, f = ctx.empty_outputs()
    ctx.eval(dev(torch, x), dev(torch, v), dev(torch, vn), dev(torch, fext), h, g, H, f)
    torch.cuda.synchronize()
    return ctx, g.cpu().numpy(), H.cpu().numpy(), f.cpu().numpy()


@pytest.mark.parametrize("case", list(CASES))
def test_kvc_parity(torch_cuda, case):
    mesh, mat, rule = CASES[case]()
    h = synth.H_T10 if mesh.element == 0 else (synth.H_ANCF if mesh.element == 1 else synth.H_BEAM)
    x, v, vn, fext = state(mesh, "strong" in case)
    pr = oracle.Problem(mesh, mat, rule)
    g0, H0, f0 = pr.eval(x, v, vn, fext, h, kv_consistent=True)
    _, Hs0, _ = pr.eval(x, v, vn, fext, h)
    ctx, g, H, f = run(torch_cuda, mesh, mat, rule, x, v, vn, fext, h, True)
    assert ctx.info["kv_consistent_tangent"] == 1
    rowptr, cols = [t.cpu().numpy() for t in ctx.export_pattern()[:2]]
    assert np.array_equal(rowptr.astype(np.int64), pr.rowptr) and np.array_equal(cols.astype(np.int64), pr.cols)
    assert rel(f, f0) <= TOL, rel(f, f0)
    assert rel(g, g0) <= TOL, rel(g, g0)
    assert rel(H, H0) <= TOL, rel(H, H0)
    # the consistent tangent differs from the elastic one (the path really ran)
    assert rel(H, Hs0) > 1e3 * TOL
    # the viscous part alone, against the oracle's
    _, _, Hs, _ = run(torch_cuda, mesh, mat, rule, x, v, vn, fext, h, False)
    assert rel(H - Hs, H0 - Hs0) <= 1e-9, rel(H - Hs, H0 - Hs0)
    _, g2, H2, f2 = run(torch_cuda, mesh, mat, rule, x, v, vn, fext, h, True)
    assert np.array_equal(g, g2) and np.array_equal(H, H2) and np.array_equal(f, f2)


def test_kvc_options(torch_cuda):
    import paper_2604_10357_b200 as T
    torch = torch_cuda
    mesh = box(2, 2, 1)
    mat = dict(synth.SVK_PAPER, **synth.KV_TIRE)
    with pytest.raises(T.TlfeaError, match="UNSUPPORTED"):
        T.Context.from_mesh(mesh, mat, 1, kv_consistent=True, hessian="upper")
    # without damping the option changes nothing
    ctx = T.Context.from_mesh(mesh, dict(synth.SVK_PAPER), 1, kv_consistent=True)
    assert ctx.info["kv_consistent_tangent"] == 0
    # the Hessian-only stage has no velocities: refused for a consistent context
    ctx = T.Context.from_mesh(mesh, mat, 1, kv_consistent=True)
    H = torch.empty(ctx.nnz, dtype=torch.float64, device="cuda")
    with pytest.raises(T.TlfeaError, match="INVALID"):
        ctx.assemble_hessian(dev(torch, mesh.X.ravel()), 1e-3, H)
