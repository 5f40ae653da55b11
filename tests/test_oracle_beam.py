"""Pins of the oracle's ANCF3243 beam (reading Q23;
P:390): basis interpolation, complex-step
derivatives, exact reproduction of linear geometry, quadrature size,
volume / mass / reference invariants, the affine uniform-stress closed form
against an independent Gauss rule, f = dPi/dx, K = df/dx, rigid motion, the
pattern against brute force and the paper's mesh table. CPU only."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

SVK = dict(synth.SVK_PAPER)
MR = dict(synth.MR_PAPER)
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))
LWH = np.array([0.2, 0.1, 0.1])


def test_beam_rule_and_basis_nodal_values():
    pts, w = oracle.quadrature(3)
    assert len(w) == GOLD["quadrature_sizes"]["ancf_beam_gl"] == 12
    assert np.sum(w) == pytest.approx(8.0, rel=1e-15)
    # at node A (xi = -1) on the axis: r = r_A, dr/dxi = (L/2) r_x^A,
    # dr/deta = (W/2) r_y^A, dr/dzeta = (H/2) r_z^A; likewise at B
    for k, xi in enumerate((-1.0, 1.0)):
        S, dS = oracle.beam_shape([xi, 0.0, 0.0], LWH)
        e = np.zeros(8)
        e[4 * k] = 1.0
        assert np.allclose(S, e, atol=1e-16)
        d = np.zeros((8, 3))
        d[4 * k + 1, 0] = LWH[0] / 2
        d[4 * k + 2, 1] = LWH[1] / 2
        d[4 * k + 3, 2] = LWH[2] / 2
        assert np.allclose(dS, d, atol=1e-16)
    # the two position functions sum to one everywhere (translations)
    for xi in np.linspace(-1, 1, 7):
        S, _ = oracle.beam_shape([xi, 0.3, -0.7], LWH)
        assert S[0] + S[4] == pytest.approx(1.0, rel=1e-15)
    assert len(oracle.beam_shape([0, 0, 0], LWH)[0]) == GOLD["element_block_sizes"]["ancf_beam"] // 3


def test_beam_gradients_complex_step_and_linear_reproduction():
    rng = np.random.default_rng(41)
    A = np.eye(3) + rng.uniform(-0.2, 0.2, (3, 3))
    c = rng.normal(size=3)
    XA, XB = np.array([0.3, -0.1, 0.2]), np.array([0.3 + LWH[0], -0.1, 0.2])
    # coefficients of the affine map phi(X) = A X + c on a straight element
    coef = np.array([A @ XA + c, A[:, 0], A[:, 1], A[:, 2], A @ XB + c, A[:, 0], A[:, 1], A[:, 2]])
    for _ in range(6):
        xi = rng.uniform(-1, 1, 3)
        S, dS = oracle.beam_shape(xi, LWH)
        for dim in range(3):
            assert np.allclose(oracle.beam_shape_csd(xi, LWH, dim), dS[:, dim], rtol=0, atol=1e-14)
        X = np.array([XA[0] + LWH[0] * (xi[0] + 1) / 2, XA[1] + LWH[1] * xi[1] / 2, XA[2] + LWH[2] * xi[2] / 2])
        assert np.allclose(S @ coef, A @ X + c, rtol=0, atol=1e-14)


@pytest.mark.parametrize("rule_mass", [0, 1])
def test_beam_precompute_volume_mass_identity(rule_mass):
    mesh = synth.ancf_beam(3)
    pr = oracle.Problem(mesh, SVK, 3, mass_rule=rule_mass)
    V = mesh.n_el * np.prod(LWH)
    assert pr.J0w.sum() == pytest.approx(V, rel=1e-14)
    # grad_X S at the reference maps the reference coefficients to F = I
    cc = mesh.coef_conn()
    for e in range(mesh.n_el):
        for q in range(pr.nq):
            F = mesh.X[cc[e]].T @ pr.gradN[e, q]
            assert np.allclose(F, np.eye(3), atol=1e-14)
    # translational mass = rho V (position coefficients; both rules exact on it)
    Mpos = sum(pr.M[p] for I in range(0, mesh.n_coef, 4) for p in range(pr.rowptr_c[I], pr.rowptr_c[I + 1])
               if pr.cols_c[p] % 4 == 0)
    assert Mpos == pytest.approx(SVK["rho0"] * V, rel=1e-13)


def test_beam_exact_mass_against_independent_rule():
    # mass_rule 0 (GL 6x2x2) vs an independent 10x4x4 Gauss rule of rho S_a S_b det J
    mesh = synth.ancf_beam(1)
    me = oracle.element_mass(2, 3, 0, SVK["rho0"], mesh.conn[0], mesh.X, LWH=LWH)
    g, w = np.polynomial.legendre.leggauss(10)
    g4, w4 = np.polynomial.legendre.leggauss(4)
    ref = np.zeros((8, 8))
    Xe = mesh.X.reshape(-1, 3)
    for i in range(10):
        for j in range(4):
            for k in range(4):
                S, dS = oracle.beam_shape([g[i], g4[j], g4[k]], LWH)
                J = Xe.T @ dS
                ref += SVK["rho0"] * np.outer(S, S) * np.linalg.det(J) * w[i] * w4[j] * w4[k]
    assert np.abs(me - ref).max() < 1e-13 * np.abs(ref).max()


def test_beam_reference_rigid_motion_and_affine_stress():
    mesh = synth.ancf_beam(1)
    X = mesh.X
    conn = mesh.conn[0]
    scale = SVK["E"] * LWH[1] * LWH[2]
    fe, _ = oracle.element(2, 3, 0, SVK, conn, X, X.ravel(), LWH=LWH, tangent=False)
    assert np.abs(fe).max() < 1e-7 * scale
    rng = np.random.default_rng(42)
    R = synth.random_rotation(rng)
    q = X.reshape(2, 4, 3).copy()
    q[:, 0] = q[:, 0] @ R.T + rng.normal(size=3)
    q[:, 1:] = q[:, 1:] @ R.T
    fr, _ = oracle.element(2, 3, 0, SVK, conn, X, q.ravel(), LWH=LWH, tangent=False)
    assert np.abs(fr).max() < 1e-7 * scale
    # affine coefficients: F = A everywhere, f_a = P(A) int grad_X S_a dV
    A = np.eye(3) + rng.uniform(-0.05, 0.05, (3, 3))
    qa = X.reshape(2, 4, 3) @ A.T
    fa, _ = oracle.element(2, 3, 0, SVK, conn, X, qa.ravel(), LWH=LWH, tangent=False)
    P = oracle.pk1_elastic(0, SVK, A)
    g, w = np.polynomial.legendre.leggauss(8)
    integ = np.zeros((8, 3))
    for i in range(8):
        for j in range(8):
            for k in range(8):
                S, dS = oracle.beam_shape([g[i], g[j], g[k]], LWH)
                J = X.T @ dS
                integ += (dS @ np.linalg.inv(J)) * np.linalg.det(J) * w[i] * w[j] * w[k]
    ref = integ @ P.T
    assert np.abs(fa.reshape(8, 3) - ref).max() < 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("mat", [SVK, MR], ids=["svk", "mr"])
def test_beam_force_energy_gradient_and_tangent_fd(mat):
    mesh = synth.ancf_beam(1)
    X = mesh.X
    conn = mesh.conn[0]
    rng = np.random.default_rng(43)
    q = X.ravel() + rng.normal(0, 1e-3, X.size)
    fe, K = oracle.element(2, 3, mat["model"], mat, conn, X, q, LWH=LWH)
    g = oracle.element_energy_grad_csd(2, 3, mat["model"], mat, conn, X, q, LWH=LWH)
    assert np.abs(g - fe).max() < 1e-11 * np.abs(fe).max()
    assert np.abs(fe.reshape(8, 3)[0::4].sum(0)).max() < 1e-11 * np.abs(fe).max()
    assert np.abs(K - K.T).max() < 1e-12 * np.abs(K).max()
    hstep = 1e-8
    for s in rng.choice(24, 8, replace=False):
        e = np.zeros(24)
        e[s] = hstep
        fp, _ = oracle.element(2, 3, mat["model"], mat, conn, X, q + e, LWH=LWH, tangent=False)
        fm, _ = oracle.element(2, 3, mat["model"], mat, conn, X, q - e, LWH=LWH, tangent=False)
        assert np.abs((fp - fm) / (2 * hstep) - K[:, s]).max() < 1e-6 * np.abs(K).max()


def test_beam_pattern_brute_force_and_paper_table():
    mesh = synth.ancf_beam(4)
    pr = oracle.Problem(mesh, SVK, 3)
    cc = mesh.coef_conn()
    rows = [set() for _ in range(mesh.n_coef)]
    for e in range(mesh.n_el):
        for a in cc[e]:
            rows[a].update(int(b) for b in cc[e])
    for I in range(mesh.n_coef):
        assert pr.cols_c[pr.rowptr_c[I]:pr.rowptr_c[I + 1]].tolist() == sorted(rows[I])
    # coefficient nnz of an n-element chain: 16 [2 (2 nodes) + 3 (n-1 nodes)]... closed form
    n = mesh.n_el
    assert pr.nnz_c == 16 * (2 * 2 + 3 * (n - 1))
    for row in GOLD["ancf3243_mesh_statistics"]["rows"][:3]:
        m = synth.ancf_beam(row["n"])
        assert m.n_el == row["elements"]
        assert m.n_coef // 4 == row["nodes"]
        assert m.n_dof == row["dofs"]
        # the clamped x = 0 end: all 4 coefficient vectors of node 0
        assert synth.clamped_dofs_ancf(m) == row["constrained_dofs"]
