"""Pins of the oracle's element force and tangent (Eq. fint_local P:409-417,
Eq. tangent_block) against closed forms, invariants, the strain
energy (complex step and central finite differences) and textbook linear
elasticity."""
import numpy as np
import pytest

import oracle
import synth

SVK = dict(synth.SVK_PAPER)
MR = dict(synth.MR_PAPER)


def one_tet(rng=None, distort=0.0):
    X = np.array([[0, 0, 0], [0.11, 0.01, 0.0], [0.02, 0.09, 0.01], [0.01, 0.02, 0.1]], float)
    if rng is not None:
        X = X + rng.uniform(-distort, distort, X.shape)
    mids = [(X[a] + X[b]) / 2 for a, b in synth.T10_EDGES]
    return np.vstack([X, mids]), np.arange(10, dtype=np.int32)


def grad_bary(Xc):
    """Gradients of the 4 barycentric coordinates of a straight tet."""
    A = np.vstack([np.ones(4), Xc.T])          # [1; x; y; z] zeta = A^-1 [1; X]
    Ai = np.linalg.inv(A)
    return Ai[:, 1:]                           # row i = grad zeta_i


def rigid(X, rng):
    R = synth.random_rotation(rng)
    return X @ R.T + rng.normal(size=3), R


@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("mat", [SVK, MR], ids=["svk", "mr"])
def test_uniform_stress_closed_form(rule, mat):
    """Affine x = A X: F = A, uniform P; corner forces 0 and edge (i,j) force
    V P (grad zeta_i + grad zeta_j) for any rule of degree >= 1."""
    rng = np.random.default_rng(11)
    X, conn = one_tet()
    A = np.eye(3) + rng.uniform(-0.05, 0.05, (3, 3))
    x = (X @ A.T).ravel()
    fe, _ = oracle.element(0, rule, mat["model"], mat, conn, X, x, tangent=False)
    fe = fe.reshape(10, 3)
    P = oracle.pk1_elastic(mat["model"], mat, A)
    V = np.linalg.det(np.stack([X[1] - X[0], X[2] - X[0], X[3] - X[0]], 1)) / 6
    gz = grad_bary(X[:4])
    scale = np.abs(P).max() * V ** (2 / 3)
    assert np.abs(fe[:4]).max() < 1e-14 * scale
    for k, (i, j) in enumerate(synth.T10_EDGES):
        assert np.abs(fe[4 + k] - V * P @ (gz[i] + gz[j])).max() < 1e-13 * scale


@pytest.mark.parametrize("mat", [SVK, MR], ids=["svk", "mr"])
def test_force_balance_torque_rigid(mat):
    rng = np.random.default_rng(12)
    X, conn = one_tet(rng, 0.005)
    x = (X + rng.normal(0, 0.004, X.shape)).ravel()
    fe, _ = oracle.element(0, 1, mat["model"], mat, conn, X, x, tangent=False)
    f = fe.reshape(10, 3)
    scale = np.abs(f).max()
    assert np.abs(f.sum(0)).max() < 1e-13 * scale                       # sum_a f_a = 0
    assert np.abs(np.cross(x.reshape(10, 3), f).sum(0)).max() < 1e-13 * scale * 0.2
    xr, _ = rigid(X, rng)
    fr, _ = oracle.element(0, 1, mat["model"], mat, conn, X, xr.ravel(), tangent=False)
    assert np.abs(fr).max() < 1e-12 * (mat["E"] or mat["kappa"]) * 0.01 ** 2


@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("mat", [SVK, MR], ids=["svk", "mr"])
def test_force_is_energy_gradient(rule, mat):
    rng = np.random.default_rng(13)
    X, conn = one_tet(rng, 0.004)
    x = (X + rng.normal(0, 0.004, X.shape)).ravel()
    fe, _ = oracle.element(0, rule, mat["model"], mat, conn, X, x, tangent=False)
    scale = np.abs(fe).max()
    g = oracle.element_energy_grad_csd(0, rule, mat["model"], mat, conn, X, x)
    assert np.abs(g - fe).max() < 1e-12 * scale
    fd = np.zeros(30)
    hstep = 1e-6 * 0.1
    for r in range(30):
        e = np.zeros(30)
        e[r] = hstep
        fd[r] = (oracle.element_energy(0, rule, mat["model"], mat, conn, X, x + e)
                 - oracle.element_energy(0, rule, mat["model"], mat, conn, X, x - e)) / (2 * hstep)
    assert np.abs(fd - fe).max() < 1e-6 * scale


@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("mat", [SVK, MR], ids=["svk", "mr"])
def test_tangent_is_force_jacobian_and_symmetric(rule, mat):
    rng = np.random.default_rng(14)
    X, conn = one_tet(rng, 0.004)
    x = (X + rng.normal(0, 0.004, X.shape)).ravel()
    _, K = oracle.element(0, rule, mat["model"], mat, conn, X, x)
    scale = np.abs(K).max()
    assert np.abs(K - K.T).max() < 1e-13 * scale
    hstep = 1e-7
    fd = np.zeros((30, 30))
    for s in range(30):
        e = np.zeros(30)
        e[s] = hstep
        fp, _ = oracle.element(0, rule, mat["model"], mat, conn, X, x + e, tangent=False)
        fm, _ = oracle.element(0, rule, mat["model"], mat, conn, X, x - e, tangent=False)
        fd[:, s] = (fp - fm) / (2 * hstep)
    assert np.abs(fd - K).max() < 1e-6 * scale


@pytest.mark.parametrize("rule", [0, 1])
def test_svk_tangent_at_reference_is_linear_elastic_stiffness(rule):
    """x = X: K_e = sum_q B^T D B J0 w (textbook small-strain stiffness)."""
    X, conn = one_tet()
    mesh = synth.Mesh(0, X, conn[None, :])
    pr = oracle.Problem(mesh, SVK, rule, with_pattern=False)
    E, nu = SVK["E"], SVK["nu"]
    lam, mu = E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[:3, :3] += 2 * mu * np.eye(3)
    D[3:, 3:] = mu * np.eye(3)
    Kref = np.zeros((30, 30))
    for q in range(pr.nq):
        B = np.zeros((6, 30))
        for a in range(10):
            gx, gy, gz = pr.gradN[0, q, a]
            B[0, 3 * a] = gx
            B[1, 3 * a + 1] = gy
            B[2, 3 * a + 2] = gz
            B[3, 3 * a + 1], B[3, 3 * a + 2] = gz, gy
            B[4, 3 * a], B[4, 3 * a + 2] = gz, gx
            B[5, 3 * a], B[5, 3 * a + 1] = gy, gx
        Kref += B.T @ D @ B * pr.J0w[0, q]
    _, K = oracle.element(0, rule, 0, SVK, conn, X, X.ravel())
    assert np.abs(K - Kref).max() < 1e-13 * np.abs(Kref).max()
    # 6-dimensional rigid null space at the reference configuration (rule >= degree 2)
    ev = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(ev) < 1e-9 * ev.max()) == 6


def _ancf_elem(LWH=(0.02, 0.01, 0.1)):
    mesh = synth.ancf_plate(1, Lx=LWH[0], Ly=LWH[1], H=LWH[2])
    return mesh


def test_ancf_reference_and_rigid_motion():
    mesh = _ancf_elem()
    LWH = mesh.dims[0]
    X = mesh.X
    conn = mesh.conn[0]
    fe, _ = oracle.element(1, 2, 0, SVK, conn, X, X.ravel(), LWH=LWH, tangent=False)
    scale = SVK["E"] * LWH[0] * LWH[1]
    assert np.abs(fe).max() < 1e-15 * scale
    rng = np.random.default_rng(15)
    R = synth.random_rotation(rng)
    t = rng.normal(size=3)
    q = X.reshape(4, 4, 3).copy()
    q[:, 0] = q[:, 0] @ R.T + t
    q[:, 1:] = q[:, 1:] @ R.T
    fr, _ = oracle.element(1, 2, 0, SVK, conn, X, q.ravel(), LWH=LWH, tangent=False)
    assert np.abs(fr).max() < 1e-12 * scale


def test_ancf_affine_uniform_stress_closed_form():
    """Affine coefficients (positions A X, gradients A e_i) give F = A at every
    point and f_a = P(A) int grad_X S_a dV; the integral by an independent
    8x8x8 Gauss rule."""
    mesh = _ancf_elem((0.3, 0.2, 0.05))
    LWH = mesh.dims[0]
    X = mesh.X
    conn = mesh.conn[0]
    rng = np.random.default_rng(16)
    A = np.eye(3) + rng.uniform(-0.05, 0.05, (3, 3))
    q = X.reshape(4, 4, 3) @ A.T
    fe, _ = oracle.element(1, 2, 0, SVK, conn, X, q.ravel(), LWH=LWH, tangent=False)
    P = oracle.pk1_elastic(0, SVK, A)
    g8, w8 = np.polynomial.legendre.leggauss(8)
    integ = np.zeros((16, 3))
    for i in range(8):
        for j in range(8):
            for k in range(8):
                xi = np.array([g8[i], g8[j], g8[k]])
                S, dS = oracle.ancf_shape(xi, LWH)
                Xe = X.reshape(4, 4, 3)[conn].reshape(16, 3)     # element-local order
                J = Xe.T @ dS                   # dX/dxi
                integ += (dS @ np.linalg.inv(J)) * np.linalg.det(J) * w8[i] * w8[j] * w8[k]
    ref = integ @ P.T
    assert np.abs(fe.reshape(16, 3) - ref).max() < 1e-13 * np.abs(ref).max()


def test_ancf_force_energy_gradient_and_tangent_fd():
    mesh = _ancf_elem((0.2, 0.1, 0.05))
    LWH = mesh.dims[0]
    X = mesh.X
    conn = mesh.conn[0]
    rng = np.random.default_rng(17)
    q = X.ravel() + rng.normal(0, 1e-3, X.size)
    fe, K = oracle.element(1, 2, 0, SVK, conn, X, q, LWH=LWH)
    q_local = q.reshape(4, 4, 3)[conn].ravel()          # element-local coefficient order
    g = oracle.element_energy_grad_csd(1, 2, 0, SVK, conn, X, q_local, LWH=LWH)
    assert np.abs(g - fe).max() < 1e-12 * np.abs(fe).max()
    assert np.abs(fe.reshape(16, 3)[0::4].sum(0)).max() < 1e-12 * np.abs(fe).max()
    assert np.abs(K - K.T).max() < 1e-13 * np.abs(K).max()
    hstep = 1e-8
    glob = (4 * conn[:, None] + np.arange(4)[None, :]).ravel()   # local coef -> global coef
    for s in rng.choice(48, 8, replace=False):
        e = np.zeros(48)
        e[3 * glob[s // 3] + s % 3] = hstep
        fp, _ = oracle.element(1, 2, 0, SVK, conn, X, q + e, LWH=LWH, tangent=False)
        fm, _ = oracle.element(1, 2, 0, SVK, conn, X, q - e, LWH=LWH, tangent=False)
        assert np.abs((fp - fm) / (2 * hstep) - K[:, s]).max() < 1e-6 * np.abs(K).max()
