"""Linear constraints (reading Q22) on the GPU vs the
CPU oracle through the C ABI: the union pattern bit-exact, g and H with the
h C^T(lambda + rho c) and h^2 rho C^T C terms, the residual c(q), the dual
ascent step, determinism and input validation."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = 1e-11


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_10357_b200 as T
    T.lib()
    return torch


CASES = {
    "cfg1_svk_4pt": lambda: (synth.config(1).mesh, dict(synth.SVK_PAPER), 0, synth.H_T10),
    "t10_4x3x2_mr_kv_keast5": lambda: (synth.kuhn_t10_box(4, 3, 2, 0.8, 0.6, 0.4),
                                       dict(synth.MR_PAPER, **synth.KV_TIRE), 1, synth.H_T10),
    "ancf_4x4_svk": lambda: (synth.ancf_plate(4), dict(synth.SVK_PAPER), 2, synth.H_ANCF),
}


@pytest.mark.parametrize("case", list(CASES))
def test_constrained_eval_parity(torch_cuda, case):
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mesh, mat, rule, h = CASES[case]()
    con = synth.constraint_set(mesh, n_ties=8)
    m = con["b"].size
    if mesh.element == 0:
        x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    else:
        x, v, vn = synth.ancf_state(mesh)
        fext = None
    rho = 1e6
    lam = np.random.default_rng(77).normal(0, 10.0, m)
    pr = oracle.Problem(mesh, mat, rule, constraints=con)
    g0, H0, f0 = pr.eval(x, v, vn, fext, h, lam=lam, rho=rho)
    ctx = T.Context.from_mesh(mesh, mat, rule, constraints=con)
    assert ctx.info["n_constraints"] == m
    rowptr, cols, rowptr_c, cols_c, _ = [t.cpu().numpy() for t in ctx.export_pattern()]
    assert np.array_equal(rowptr_c.astype(np.int64), pr.rowptr_c)
    assert np.array_equal(cols_c.astype(np.int64), pr.cols_c)
    assert np.array_equal(cols.astype(np.int64), pr.cols)
    d = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()
    g, H, f = ctx.empty_outputs()
    ctx.eval(d(x), d(v), d(vn), d(fext), h, g, H, f, lam=d(lam), rho=rho)
    torch.cuda.synchronize()
    assert rel(f.cpu().numpy(), f0) <= TOL
    assert rel(g.cpu().numpy(), g0) <= TOL
    assert rel(H.cpu().numpy(), H0) <= TOL
    # plain tlfea_eval on the same (union) pattern == lam = 0, rho = 0
    gu, Hu, _ = pr.eval(x, v, vn, fext, h)
    g2, H2, _ = ctx.eval(d(x), d(v), d(vn), d(fext), h)
    torch.cuda.synchronize()
    assert rel(g2.cpu().numpy(), gu) <= TOL and rel(H2.cpu().numpy(), Hu) <= TOL
    # residual and dual ascent (Eq. lambda_update)
    c = ctx.constraint_residual(d(x))
    lam_d = d(lam)
    c2 = torch.empty(m, dtype=torch.float64, device="cuda")
    ctx.update_multipliers(d(x), rho, lam_d, c2)
    torch.cuda.synchronize()
    c_ref = pr.constraint_residual(x)
    assert np.allclose(c.cpu().numpy(), c_ref, rtol=0, atol=1e-14 * max(1.0, np.abs(x).max()))
    assert np.array_equal(c.cpu().numpy(), c2.cpu().numpy())
    assert rel(lam_d.cpu().numpy(), lam + rho * c_ref) <= 1e-12
    # determinism (same outputs requested: with f_int)
    f3 = torch.empty_like(f)
    g3, H3, _ = ctx.eval(d(x), d(v), d(vn), d(fext), h, None, None, f3, lam=d(lam), rho=rho)
    torch.cuda.synchronize()
    assert np.array_equal(g3.cpu().numpy(), g.cpu().numpy()) and np.array_equal(H3.cpu().numpy(), H.cpu().numpy())
    # without f_int
    g4, H4, _ = ctx.eval(d(x), d(v), d(vn), d(fext), h, lam=d(lam), rho=rho)
    torch.cuda.synchronize()
    assert rel(g4.cpu().numpy(), g0) <= TOL and np.array_equal(H4.cpu().numpy(), H.cpu().numpy())


def test_alm_loop_with_adamw_inner_iterations(torch_cuda):
    """Alg. 2 with constraints: 3 outer iterations (moments reset, 6 AdamW
    inner iterations with the h C^T(lam + rho c) gradient term, commit, dual
    ascent lam += rho c) on the GPU next to the oracle."""
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mesh, mat, rule, h = CASES["cfg1_svk_4pt"]()
    con = synth.constraint_set(mesh, n_ties=4)
    x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    qn = x - h * v
    rho = 1e5
    prm = dict(alpha=2e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0)
    pr = oracle.Problem(mesh, mat, rule, constraints=con)
    ctx = T.Context.from_mesh(mesh, mat, rule, constraints=con)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()
    lam = np.zeros(con["b"].size)
    lam_d = d(lam)
    vv, v_d, vn_d, qn_d, fe_d = vn.copy(), d(vn), d(vn), d(qn), d(fext)
    for _ in range(3):
        m = np.zeros_like(vv)
        s = np.zeros_like(vv)
        g = np.zeros_like(vv)
        m_d, s_d, g_d = d(m), d(s), d(g)
        for l in range(1, 7):
            vv, m, s, g, q, _, _, _ = oracle.adamw_iteration(pr, l, prm, qn, vn, fext, h, vv, m, s, g, lam=lam, rho=rho)
            q_d, _ = ctx.adamw_iteration(qn_d, vn_d, fe_d, h, l, prm, v_d, m_d, s_d, g_d, lam=lam_d, rho=rho)
        lam = lam + rho * pr.constraint_residual(q)
        ctx.update_multipliers(q_d, rho, lam_d)
    torch.cuda.synchronize()
    assert rel(v_d.cpu().numpy(), vv) <= 1e-9
    assert rel(g_d.cpu().numpy(), g) <= 1e-8
    assert rel(lam_d.cpu().numpy(), lam) <= 1e-8


def test_constraint_validation(torch_cuda):
    import paper_2604_10357_b200 as T
    mesh, mat, rule, _ = CASES["cfg1_svk_4pt"]()
    bad = [dict(rowptr=[0, 2], cols=[0, 0], vals=[1.0, 1.0], b=[0.0]),          # repeated DOF
           dict(rowptr=[0, 1], cols=[3 * mesh.n_coef], vals=[1.0], b=[0.0]),   # DOF out of range
           dict(rowptr=[1, 1], cols=[0], vals=[1.0], b=[0.0])]                 # rowptr[0] != 0
    for con in bad:
        with pytest.raises(RuntimeError):
            T.Context.from_mesh(mesh, mat, rule, constraints=con)
    with pytest.raises(RuntimeError):
        ctx = T.Context.from_mesh(mesh, mat, rule, constraints=synth.constraint_set(mesh))
        import torch
        x = torch.zeros(3 * mesh.n_coef, dtype=torch.float64, device="cuda")
        ctx.eval(x, x, None, None, 1e-3, lam=None, rho=-1.0)
