"""Pins of the oracle's CONSISTENT Kelvin-Voigt tangent (
Eq. residual P:101-113 with x = q_n + h v, Eq. hessian, reading Q7/Q9):

    Kc_e = h df_e/dx + df_e/dv,   H_c = M/h + sum_e Kc_e = dg/dv.

The oracle takes Kc by complex step of its element force under the joint
perturbation (x + i h eps e_s, v + i eps e_s). It is pinned here against
things other than itself:
  * the local element force it differentiates equals the pinned element force
    (test_oracle_element.py) bit for bit;
  * eta = lambda_d = 0 reduces it to h K_e, the pinned elastic tangent;
  * at the reference configuration with v = 0 and no elastic stiffness it is
    the textbook linear-elasticity stiffness sum_q J0 w B^T D B with the Lame
    pair (lambda_d, eta) (Voigt B and D written out here, not taken from the
    oracle);
  * central finite differences of the element force and of the global
    residual g(v) (itself pinned by test_oracle_assembly.py) along random
    velocity directions, x moving by h dv;
  * with v != 0 it is non-symmetric, with v = 0 symmetric (the viscous
    dissipation is a potential in v, the x-derivative is not).
"""
import numpy as np
import pytest

import oracle
import synth

H_T = 1e-3
KV = dict(eta_damp=5.0e3, lambda_damp=3.0e3)
SVK_KV = dict(synth.SVK_PAPER, **KV)
MR_KV = dict(synth.MR_PAPER, **KV)


def one_tet(rng, distort=0.004):
    X = np.array([[0, 0, 0], [0.11, 0.01, 0.0], [0.02, 0.09, 0.01], [0.01, 0.02, 0.1]], float)
    X = X + rng.uniform(-distort, distort, X.shape)
    mids = [(X[a] + X[b]) / 2 for a, b in synth.T10_EDGES]
    return np.vstack([X, mids]), np.arange(10, dtype=np.int32)


def state(rng, X, amp=0.004, vamp=0.3):
    x = (X + rng.normal(0, amp, X.shape)).ravel()
    v = rng.normal(0, vamp, X.size)
    return x, v


@pytest.mark.parametrize("mat", [SVK_KV, MR_KV], ids=["svk", "mr"])
def test_local_force_is_element_force(mat):
    rng = np.random.default_rng(31)
    X, conn = one_tet(rng)
    x, v = state(rng, X)
    f0, _ = oracle.element(0, 1, mat["model"], mat, conn, X, x, v, tangent=False)
    f1 = oracle.element_force_local(0, 1, mat["model"], mat, conn, X, x, v)
    assert np.array_equal(f0, f1)


@pytest.mark.parametrize("mat", [synth.SVK_PAPER, synth.MR_PAPER], ids=["svk", "mr"])
def test_no_damping_is_h_times_elastic(mat):
    rng = np.random.default_rng(32)
    X, conn = one_tet(rng)
    x, v = state(rng, X)
    _, Ke = oracle.element(0, 1, mat["model"], mat, conn, X, x, v)
    Kc = oracle.element_kvc(0, 1, mat["model"], mat, conn, X, x, v, H_T)
    assert np.abs(Kc - H_T * Ke).max() <= 1e-13 * np.abs(H_T * Ke).max()


def voigt_B(g):
    """Textbook 6x3 strain-displacement block of one node (engineering shear)."""
    B = np.zeros((6, 3))
    B[0, 0], B[1, 1], B[2, 2] = g
    B[3, 0], B[3, 1] = g[1], g[0]   # xy
    B[4, 1], B[4, 2] = g[2], g[1]   # yz
    B[5, 0], B[5, 2] = g[2], g[0]   # xz
    return B


@pytest.mark.parametrize("rule", [0, 1])
def test_reference_state_is_linear_viscous_stiffness(rule):
    """x = X, v = 0, E = 0: Kc = sum_q J0 w B^T D(lambda_d, eta) B."""
    rng = np.random.default_rng(33)
    X, conn = one_tet(rng)
    mat = dict(synth.SVK_PAPER, E=0.0, **KV)
    Kc = oracle.element_kvc(0, rule, 0, mat, conn, X, X.ravel(), np.zeros(X.size), H_T)
    pr = oracle.Problem(synth.Mesh(0, X, conn[None, :]), mat, rule, with_pattern=False)
    lam, eta = KV["lambda_damp"], KV["eta_damp"]
    D = lam * np.outer([1, 1, 1, 0, 0, 0], [1, 1, 1, 0, 0, 0]) + eta * np.diag([2, 2, 2, 1, 1, 1])
    K = np.zeros((30, 30))
    for q in range(pr.nq):
        Bs = [voigt_B(pr.gradN[0, q, a]) for a in range(10)]
        for a in range(10):
            for b in range(10):
                K[3 * a:3 * a + 3, 3 * b:3 * b + 3] += pr.J0w[0, q] * Bs[a].T @ D @ Bs[b]
    assert np.abs(Kc - K).max() <= 1e-12 * np.abs(K).max()
    assert np.abs(Kc - Kc.T).max() <= 1e-12 * np.abs(K).max()


@pytest.mark.parametrize("mat", [SVK_KV, MR_KV], ids=["svk", "mr"])
def test_element_central_difference(mat):
    rng = np.random.default_rng(34)
    X, conn = one_tet(rng)
    x, v = state(rng, X)
    Kc = oracle.element_kvc(0, 1, mat["model"], mat, conn, X, x, v, H_T)
    scale = np.abs(Kc).max()
    for _ in range(4):
        dv = rng.normal(size=30)
        d = 1e-4
        fp = oracle.element_force_local(0, 1, mat["model"], mat, conn, X, x + H_T * d * dv, v + d * dv)
        fm = oracle.element_force_local(0, 1, mat["model"], mat, conn, X, x - H_T * d * dv, v - d * dv)
        fd = (fp - fm) / (2 * d)
        assert np.abs(fd - Kc @ dv).max() <= 1e-7 * scale * np.abs(dv).max()
    # non-symmetric once the deformation rate is nonzero
    assert np.abs(Kc - Kc.T).max() > 1e-6 * scale


def test_ancf_and_beam_central_difference():
    rng = np.random.default_rng(35)
    for mesh, h in ((synth.ancf_plate(2), synth.H_ANCF), (synth.ancf_beam(2), synth.H_BEAM)):
        mat = dict(synth.SVK_PAPER, **KV)
        cc = mesh.coef_conn()
        x = mesh.X.ravel() + rng.normal(0, 1e-3, mesh.X.size)
        v = rng.normal(0, 0.05, mesh.X.size)
        for e in range(mesh.n_el):
            LWH = mesh.dims[e]
            Kc = oracle.element_kvc(mesh.element, 2 if mesh.element == 1 else 3, 0, mat, mesh.conn[e],
                                    mesh.X, x, v, h, LWH)
            assert np.abs(Kc).max() > 0.0
            xe, ve = x.reshape(-1, 3)[cc[e]].ravel(), v.reshape(-1, 3)[cc[e]].ravel()
            nd = xe.size
            dv = rng.normal(size=nd)
            d = 1e-4
            rule = 2 if mesh.element == 1 else 3
            fp = oracle.element_force_local(mesh.element, rule, 0, mat, mesh.conn[e], mesh.X,
                                            xe + h * d * dv, ve + d * dv, LWH)
            fm = oracle.element_force_local(mesh.element, rule, 0, mat, mesh.conn[e], mesh.X,
                                            xe - h * d * dv, ve - d * dv, LWH)
            assert np.abs((fp - fm) / (2 * d) - Kc @ dv).max() <= 1e-7 * np.abs(Kc).max() * np.abs(dv).max()


def dense(pr, H):
    n = 3 * pr.n_coef
    A = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(pr.rowptr))
    A[rows, pr.cols] = H
    return A


@pytest.mark.parametrize("mat", [SVK_KV, MR_KV], ids=["svk", "mr"])
def test_global_residual_central_difference(mat):
    """H_c = dg/dv of the pinned residual g(v) with x = q_n + h v."""
    mesh = synth.kuhn_t10_box(2, 1, 1, 0.2, 0.1, 0.1)
    rng = np.random.default_rng(36)
    pr = oracle.Problem(mesh, mat, 1)
    q_n, _, vn, _ = synth.t10_state(mesh)
    v = rng.normal(0, 0.3, mesh.n_dof)
    fext = rng.normal(0, 1.0, mesh.n_dof)
    g, Hc, _ = pr.eval(q_n + H_T * v, v, vn, fext, H_T, kv_consistent=True)
    g0, Hs, _ = pr.eval(q_n + H_T * v, v, vn, fext, H_T)
    assert np.array_equal(g, g0)              # the residual itself is unchanged
    A = dense(pr, Hc)
    for _ in range(3):
        dv = rng.normal(size=mesh.n_dof)
        d = 1e-4
        gp, _, _ = pr.eval(q_n + H_T * (v + d * dv), v + d * dv, vn, fext, H_T, hessian=False)
        gm, _, _ = pr.eval(q_n + H_T * (v - d * dv), v - d * dv, vn, fext, H_T, hessian=False)
        fd = (gp - gm) / (2 * d)
        assert np.linalg.norm(fd - A @ dv) <= 1e-7 * np.linalg.norm(A @ dv)
    # the elastic-only H misses the viscous terms by far more than the FD error
    assert np.linalg.norm(Hc - Hs) > 1e-4 * np.linalg.norm(Hs)
