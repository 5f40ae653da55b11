"""UPPER storage of H (reading Q14) on the GPU vs the
oracle's upper view: pattern and slot map bit-exact, values within the
parity bar, the same values as the FULL storage at the kept entries, the
and the error cases."""
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
    "t10_5x3x1_svk_keast5": lambda: (synth.kuhn_t10_box(5, 3, 1, 1.0, 0.6, 0.2), dict(synth.SVK_PAPER), 1),
    "t10_3x2x2_perturbed_mr_kv": lambda: (synth.perturbed(synth.kuhn_t10_box(3, 2, 2, 0.6, 0.4, 0.4)),
                                          dict(synth.MR_PAPER, **synth.KV_TIRE), 0),
    "ancf_4x4_svk": lambda: (synth.ancf_plate(4), dict(synth.SVK_PAPER), 2),
    "beam_9_svk": lambda: (synth.ancf_beam(9), dict(synth.SVK_PAPER), 3),
}


@pytest.mark.parametrize("case", list(CASES))
def test_upper_h_parity(torch_cuda, case):
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mesh, mat, rule = CASES[case]()
    if mesh.element == 0:
        x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    else:
        x, v, vn = synth.ancf_state(mesh)
        fext = None
    h = 1e-3
    pr = oracle.Problem(mesh, mat, rule)
    g0, H0, f0 = pr.eval(x, v, vn, fext, h)
    rowptr_u, cols_u, keep = pr.upper_view()
    d = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()
    ctx = T.Context.from_mesh(mesh, mat, rule, hessian="upper")
    assert ctx.info["nnz"] == cols_u.size
    rowptr, cols = [t.cpu().numpy().astype(np.int64) for t in ctx.export_pattern()[:2]]
    assert np.array_equal(rowptr, rowptr_u) and np.array_equal(cols, cols_u)
    g, H, f = ctx.eval(d(x), d(v), d(vn), d(fext), h, f_int=torch.empty(mesh.n_dof, dtype=torch.float64,
                                                                        device="cuda"))
    torch.cuda.synchronize()
    assert rel(H.cpu().numpy(), H0[keep]) <= TOL
    assert rel(g.cpu().numpy(), g0) <= TOL
    # slot map: upper entries -> their UPPER index, lower entries -> -1
    full_to_upper = -np.ones(pr.nnz, np.int64)
    full_to_upper[keep] = np.arange(keep.size)
    sm_full = pr.slot_map()
    want = np.where(sm_full >= 0, full_to_upper[np.maximum(sm_full, 0)], -1)
    assert np.array_equal(ctx.slot_map().astype(np.int64), want)
    # FULL storage, the same values at the kept entries (bitwise when both run
    # the two-kernel path; the one-kernel FULL eval sums in another order)
    ctx_f = T.Context.from_mesh(mesh, mat, rule)
    _, Hf, _ = ctx_f.eval(d(x), d(v), d(vn), d(fext), h)
    torch.cuda.synchronize()
    if ctx_f.info["fused_eval"]:
        assert rel(Hf.cpu().numpy()[keep], H.cpu().numpy()) <= 1e-13
    else:
        assert np.array_equal(Hf.cpu().numpy()[keep], H.cpu().numpy())


def test_upper_errors(torch_cuda):
    import paper_2604_10357_b200 as T
    mesh = synth.config(1).mesh
    with pytest.raises(RuntimeError):
        T.Context.from_mesh(mesh, dict(synth.SVK_PAPER), 0, hessian="upper",
                            constraints=synth.constraint_set(mesh))
    with pytest.raises(ValueError):
        T.Context.from_mesh(mesh, dict(synth.SVK_PAPER), 0, hessian="lower")
