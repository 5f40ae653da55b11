"""Pins of the oracle's quadrature, shape functions and reference precompute
against closed forms (§4.1, §4.3)."""
import math

import numpy as np
import pytest

import oracle
import synth

TET_VERTS = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)


def tet_moment(i, j, k):
    # int over the unit tetrahedron of xi^i eta^j zeta^k = i! j! k! / (i+j+k+3)!
    return math.factorial(i) * math.factorial(j) * math.factorial(k) / math.factorial(i + j + k + 3)


def monomials(deg):
    for i in range(deg + 1):
        for j in range(deg + 1 - i):
            for k in range(deg + 1 - i - j):
                yield i, j, k


@pytest.mark.parametrize("rule,degree", [(0, 2), (1, 3)])
def test_tet_rules_exact_to_degree(rule, degree):
    pts, w = oracle.quadrature(rule)
    assert len(w) == {0: 4, 1: 5}[rule]
    assert abs(w.sum() - 1.0 / 6.0) < 1e-15
    for i, j, k in monomials(degree):
        q = np.sum(w * pts[:, 0] ** i * pts[:, 1] ** j * pts[:, 2] ** k)
        assert abs(q - tet_moment(i, j, k)) < 1e-15, (rule, i, j, k)
    # and NOT exact one degree higher (the rule is the stated one, not better)
    errs = [abs(np.sum(w * pts[:, 0] ** i * pts[:, 1] ** j * pts[:, 2] ** k) - tet_moment(i, j, k))
            for i, j, k in monomials(degree + 1) if i + j + k == degree + 1]
    assert max(errs) > 1e-6


def test_keast_points_and_signed_weight():
    # S:116 / P:390: centroid weight -(4/5)(1/6), four (1/2,1/6,1/6,1/6) points (9/20)(1/6)
    pts, w = oracle.quadrature(1)
    assert np.allclose(pts[0], 0.25) and abs(w[0] + 2.0 / 15.0) < 1e-16
    bary = np.column_stack([1 - pts.sum(1), pts])
    for q in range(1, 5):
        assert np.allclose(np.sort(bary[q]), [1 / 6, 1 / 6, 1 / 6, 0.5], atol=1e-15)
        assert abs(w[q] - 3.0 / 40.0) < 1e-16


def test_gauss_legendre_443():
    pts, w = oracle.quadrature(2)
    assert len(w) == 48            # 4x4x3 = 48 points
    assert abs(w.sum() - 8.0) < 1e-14
    # exact for xi^a eta^b zeta^c, a,b <= 7, c <= 5
    one_d = lambda n: 0.0 if n % 2 else 2.0 / (n + 1)
    for a in range(8):
        for b in range(8):
            for c in range(6):
                q = np.sum(w * pts[:, 0] ** a * pts[:, 1] ** b * pts[:, 2] ** c)
                assert abs(q - one_d(a) * one_d(b) * one_d(c)) < 1e-14
    q = np.sum(w * pts[:, 2] ** 6)
    assert abs(q - 8 * one_d(6) / 2) > 1e-6  # zeta rule is the 3-point one
    # ordering: xi-major, zeta-minor
    assert pts[0, 2] < pts[1, 2] < pts[2, 2] and pts[0, 0] == pts[11, 0] and pts[12, 0] > pts[0, 0]


T10_NODE_XI = np.vstack([TET_VERTS] + [(TET_VERTS[a] + TET_VERTS[b]) / 2 for a, b in synth.T10_EDGES])


def test_t10_kronecker_partition_gradsum():
    for a in range(10):
        N, _ = oracle.t10_shape(T10_NODE_XI[a])
        assert np.allclose(N, np.eye(10)[a], atol=1e-15)
    rng = np.random.default_rng(1)
    for _ in range(20):
        xi = rng.dirichlet(np.ones(4))[1:]
        N, dN = oracle.t10_shape(xi)
        assert abs(N.sum() - 1) < 1e-14
        assert np.abs(dN.sum(0)).max() < 1e-14


def test_t10_centroid_values():
    # at the centroid, corners -1/8, mid-edges 1/4
    N, _ = oracle.t10_shape([0.25, 0.25, 0.25])
    assert np.allclose(N[:4], -0.125, atol=1e-16) and np.allclose(N[4:], 0.25, atol=1e-16)


def test_t10_gradient_vs_complex_step_and_fd():
    rng = np.random.default_rng(2)
    for _ in range(10):
        xi = rng.uniform(-0.2, 0.8, 3)
        _, dN = oracle.t10_shape(xi)
        for d in range(3):
            assert np.abs(oracle.t10_shape_csd(xi, d) - dN[:, d]).max() < 1e-14
            e = np.eye(3)[d] * 1e-6
            fd = (oracle.t10_shape(xi + e)[0] - oracle.t10_shape(xi - e)[0]) / 2e-6
            assert np.abs(fd - dN[:, d]).max() < 1e-8


ANCF_NODE = np.array([[-1, -1], [1, -1], [1, 1], [-1, 1]], float)


def test_ancf_nodal_interpolation_and_gradients():
    LWH = np.array([0.4, 0.2, 0.1])
    for k in range(4):
        S, dS = oracle.ancf_shape([ANCF_NODE[k, 0], ANCF_NODE[k, 1], 0.0], LWH)
        # position functions interpolate, gradient functions vanish at nodes
        for j in range(4):
            assert abs(S[4 * j] - (1.0 if j == k else 0.0)) < 1e-15
            assert abs(S[4 * j + 1]) < 1e-15 and abs(S[4 * j + 2]) < 1e-15
        # x = x_c + (L/2) xi: d/dxi of the r_x function at its node is L/2, etc.
        assert abs(dS[4 * k + 1, 0] - LWH[0] / 2) < 1e-15
        assert abs(dS[4 * k + 2, 1] - LWH[1] / 2) < 1e-15
        assert abs(dS[4 * k + 0, 0]) < 1e-15 and abs(dS[4 * k + 0, 1]) < 1e-15


def test_ancf_reproduces_linear_geometry_and_csd():
    # Flat reference coefficients reproduce X(xi) = center + (L xi, W eta, H zeta)/2
    LWH = np.array([0.3, 0.15, 0.07])
    c = np.array([1.0, 2.0, 0.0])
    coef = np.zeros((16, 3))
    for k in range(4):
        coef[4 * k] = c + np.array([ANCF_NODE[k, 0] * LWH[0] / 2, ANCF_NODE[k, 1] * LWH[1] / 2, 0])
        coef[4 * k + 1] = [1, 0, 0]
        coef[4 * k + 2] = [0, 1, 0]
        coef[4 * k + 3] = [0, 0, 1]
    rng = np.random.default_rng(3)
    for _ in range(10):
        xi = rng.uniform(-1, 1, 3)
        S, dS = oracle.ancf_shape(xi, LWH)
        X = S @ coef
        assert np.allclose(X, c + xi * LWH / 2, atol=1e-15)
        assert abs(S[0::4].sum() - 1) < 1e-14
        for d in range(3):
            assert np.abs(oracle.ancf_shape_csd(xi, LWH, d) - dS[:, d]).max() < 1e-14


def _tet_volumes(mesh):
    X, c = mesh.X, mesh.conn
    D = np.stack([X[c[:, 1]] - X[c[:, 0]], X[c[:, 2]] - X[c[:, 0]], X[c[:, 3]] - X[c[:, 0]]], axis=2)
    return np.linalg.det(D) / 6.0


@pytest.mark.parametrize("rule", [0, 1])
def test_precompute_t10_volume_and_identity(rule):
    mesh = synth.kuhn_t10_box(2, 2, 1, 0.4, 0.3, 0.1)
    # perturb interior geometry slightly so the isoparametric map is exercised
    pr = oracle.Problem(mesh, synth.SVK_PAPER, rule, with_pattern=False)
    assert np.allclose(pr.J0w.sum(1), _tet_volumes(mesh), rtol=1e-13)
    # F(X) = sum_a X_a (x) grad_X N_a = I at every (e,q)
    Xe = mesh.X[mesh.conn]                                   # [e, a, 3]
    F = np.einsum("eai,eqaj->eqij", Xe, pr.gradN)
    assert np.abs(F - np.eye(3)).max() < 1e-13


def test_precompute_ancf_volume_and_identity():
    mesh = synth.ancf_plate(3)
    pr = oracle.Problem(mesh, synth.SVK_PAPER, 2, with_pattern=False)
    L, W, H = mesh.dims[0]
    assert np.allclose(pr.J0w.sum(1), L * W * H, rtol=1e-14)
    Xe = mesh.X[mesh.coef_conn()]
    F = np.einsum("eai,eqaj->eqij", Xe, pr.gradN)
    assert np.abs(F - np.eye(3)).max() < 1e-13


def test_precompute_detects_inverted_element():
    mesh = synth.kuhn_t10_box(1, 1, 1, 1, 1, 1)
    c = mesh.conn.copy()
    c[3, [1, 2]] = c[3, [2, 1]]
    c[3, [4, 5, 6, 7, 8, 9]] = c[3, [6, 5, 4, 7, 9, 8]]   # consistent edge relabel
    bad = synth.Mesh(0, mesh.X, c)
    with pytest.raises(ValueError, match="inverted element 3"):
        oracle.Problem(bad, synth.SVK_PAPER, 1, with_pattern=False)
