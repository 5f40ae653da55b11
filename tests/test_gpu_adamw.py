"""tlfea_adamw_iteration (Alg. 2 inner iteration) vs the
CPU oracle through the C ABI: per-iteration parity from a shared state, a
free-running 15-iteration trajectory, bitwise reproducibility and errors."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

PRM = dict(alpha=2e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=1e-2)


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
    "ancf_4x4_svk_kv": lambda: (synth.ancf_plate(4), dict(synth.SVK_PAPER, **synth.KV_TIRE), 2, synth.H_ANCF),
    "t10_100el_svk_keast5_ragged": lambda: (synth.Mesh(0, synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).X,
                                                       synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).conn[:100]),
                                            dict(synth.SVK_PAPER), 1, synth.H_T10),
    "many_body_svk_keast5": lambda: (synth.many_body(12)[0], dict(synth.TIRE_DROP), 1, synth.H_T10),
}


def start_state(mesh, h):
    if mesh.element == 0:
        x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    else:
        x, v, vn = synth.ancf_state(mesh)
        fext = np.random.default_rng(synth.SEED_BASE + 3).normal(size=x.shape)
    return x - h * v, vn, fext, v.copy()


@pytest.mark.parametrize("with_f", [True, False], ids=["with_fint", "no_fint"])
@pytest.mark.parametrize("case", list(CASES))
def test_adamw_iteration_parity(torch_cuda, case, with_f):
    """with_f = False: straight-sided T10 SVK meshes with classes (cfg1) take the
    element-level inertia path (the gradient gather sums f_a + m_e (v - v_n)_e / h
    per element, no mass-row SpMV)."""
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mesh, mat, rule, h = CASES[case]()
    qn, vn, fext, v = start_state(mesh, h)
    pr = oracle.Problem(mesh, mat, rule, gravity=(0.0, 0.0, -9.81))
    ctx = T.Context.from_mesh(mesh, mat, rule, gravity=(0.0, 0.0, -9.81))
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()
    n = v.size
    m = np.zeros(n)
    s = np.zeros(n)
    g = np.zeros(n)
    # free-running GPU trajectory next to the oracle's
    gv, gm, gs, gg = d(v), d(m), d(s), d(g)
    qn_d, vn_d, fe_d = d(qn), d(vn), d(fext)
    f_d = torch.empty(n, dtype=torch.float64, device="cuda")
    for l in range(1, 16):
        # per-iteration parity from the oracle's state
        sv, sm, ss, sg = d(v), d(m), d(s), d(g)
        q1, nrm = ctx.adamw_iteration(qn_d, vn_d, fe_d, h, l, PRM, sv, sm, ss, sg, f_int=f_d if with_f else None)
        v, m, s, g, q, f, gn, vnorm = oracle.adamw_iteration(pr, l, PRM, qn, vn, fext, h, v, m, s, g)
        torch.cuda.synchronize()
        assert rel(sm.cpu().numpy(), m) <= 1e-13
        assert rel(ss.cpu().numpy(), s) <= 1e-13
        assert rel(sv.cpu().numpy(), v) <= 1e-13
        assert rel(q1.cpu().numpy(), q) <= 1e-14
        if with_f:
            assert rel(f_d.cpu().numpy(), f) <= 1e-11
        assert rel(sg.cpu().numpy(), g) <= 1e-11
        nh = nrm.cpu().numpy()
        assert nh[0] == pytest.approx(gn, rel=1e-11) and nh[1] == pytest.approx(vnorm, rel=1e-13)
        ctx.adamw_iteration(qn_d, vn_d, fe_d, h, l, PRM, gv, gm, gs, gg)
    torch.cuda.synchronize()
    # the trajectories stay together (errors do not grow past the parity bar)
    assert rel(gv.cpu().numpy(), v) <= 1e-10
    assert rel(gg.cpu().numpy(), g) <= 1e-9


def test_adamw_bitwise_and_errors(torch_cuda):
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mesh, mat, rule, h = CASES["cfg1_svk_4pt"]()
    qn, vn, fext, v = start_state(mesh, h)
    ctx = T.Context.from_mesh(mesh, mat, rule)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()
    outs = []
    for _ in range(2):
        sv, sm, ss, sg = d(v), d(np.zeros_like(v)), d(np.zeros_like(v)), d(np.zeros_like(v))
        for l in range(1, 6):
            q, nrm = ctx.adamw_iteration(d(qn), d(vn), d(fext), h, l, PRM, sv, sm, ss, sg)
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in (sv, sm, ss, sg, q, nrm)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    with pytest.raises(RuntimeError):
        ctx.adamw_iteration(d(qn), d(vn), None, h, 0, PRM, sv, sm, ss, sg)
    with pytest.raises(RuntimeError):
        ctx.adamw_iteration(d(qn), d(vn), None, -1.0, 1, PRM, sv, sm, ss, sg)
