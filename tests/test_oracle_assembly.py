"""Pins of the oracle's pattern, slot map, mass, residual and Hessian
assembly (§4.2, §4.4, Eq. residual P:101-113,
Eq. cost, Eq. hessian) against brute force, closed forms,
special cases and finite differences of the augmented cost Phi."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

SVK = dict(synth.SVK_PAPER)
MR = dict(synth.MR_PAPER)
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))


def brute_pattern(mesh):
    cc = mesh.coef_conn()
    rows = [set() for _ in range(mesh.n_coef)]
    for e in range(mesh.n_el):
        for a in cc[e]:
            rows[a].update(int(b) for b in cc[e])
    return rows


@pytest.mark.parametrize("mk", [lambda: synth.kuhn_t10_box(3, 2, 2, 1, 1, 1),
                                lambda: synth.ancf_plate(4)], ids=["t10", "ancf"])
def test_pattern_equals_brute_force_and_lift(mk):
    mesh = mk()
    pr = oracle.Problem(mesh, SVK, 1 if mesh.element == 0 else 2)
    rows = brute_pattern(mesh)
    for I in range(mesh.n_coef):
        cols = pr.cols_c[pr.rowptr_c[I]:pr.rowptr_c[I + 1]]
        assert list(cols) == sorted(rows[I])
    # DOF lift: row 3I+d = [3J+e for J in row I for e in 0..2]
    for I in range(0, mesh.n_coef, 7):
        for d in range(3):
            r = 3 * I + d
            cols = pr.cols[pr.rowptr[r]:pr.rowptr[r + 1]]
            assert list(cols) == [3 * J + e for J in sorted(rows[I]) for e in range(3)]
    assert pr.nnz == 9 * pr.nnz_c


def test_pattern_counts_closed_forms():
    # SURVEY §8(c) pins: cfg1 nnz_H = 82,017; one T10 element: 100 coefficient pairs
    one = synth.Mesh(0, synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).X, synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).conn[:1])
    assert oracle.Problem(one, SVK, 1).nnz_c == 100
    assert oracle.Problem(synth.config(1).mesh, SVK, 0).nnz == 82017
    # ANCF n x n: nnz_H = 144 [(n+1)^2 + 4 n (n+1) + 4 n^2]
    for n in (1, 2, 5):
        assert oracle.Problem(synth.ancf_plate(n), SVK, 2).nnz == 144 * ((n + 1) ** 2 + 4 * n * (n + 1) + 4 * n * n)


def test_slot_map_invariants():
    mesh = synth.kuhn_t10_box(2, 2, 1, 1, 1, 1)
    pr = oracle.Problem(mesh, SVK, 1)
    sl = pr.slot_map()
    cc = mesh.coef_conn()
    for e in range(mesh.n_el):
        for a in range(10):
            for d in range(3):
                r = 3 * cc[e, a] + d
                s = sl[e, 3 * a + d]
                assert np.all((s >= pr.rowptr[r]) & (s < pr.rowptr[r + 1]))
                assert list(pr.cols[s]) == [3 * cc[e, b] + f for b in range(10) for f in range(3)]


def test_t10_exact_mass_closed_form_vs_brute_force():
    """rho V/420 integer matrix (reading Q4) vs an independent conical-product
    Gauss rule (5x5x5, exact to degree 9) over the oracle's shape functions."""
    rng = np.random.default_rng(21)
    X = rng.uniform(0, 1, (4, 3))
    X[1:] += np.eye(3)
    Xf = np.vstack([X] + [(X[a] + X[b]) / 2 for a, b in synth.T10_EDGES])
    conn = np.arange(10, dtype=np.int32)
    me = oracle.element_mass(0, 1, 0, 2700.0, conn, Xf)
    g, w = np.polynomial.legendre.leggauss(5)
    g, w = (g + 1) / 2, w / 2
    V = np.linalg.det(np.stack([X[1] - X[0], X[2] - X[0], X[3] - X[0]], 1)) / 6
    ref = np.zeros((10, 10))
    for i in range(5):
        for j in range(5):
            for k in range(5):
                u, s, t = g[i], g[j], g[k]
                xi = np.array([u, s * (1 - u), t * (1 - u) * (1 - s)])   # Duffy map onto the tet
                jac = (1 - u) ** 2 * (1 - s)
                N, _ = oracle.t10_shape(xi)
                ref += np.outer(N, N) * jac * w[i] * w[j] * w[k] * 6 * V * 2700.0
    assert np.abs(me - ref).max() < 1e-13 * np.abs(ref).max()
    assert abs(me.sum() - 2700.0 * V) < 1e-13 * 2700 * V
    # consistent body-force load: corners -1/20, mid-edges +1/5 of rho V
    rs = me.sum(1) / (2700.0 * V)
    assert np.allclose(rs[:4], -1 / 20, atol=1e-15) and np.allclose(rs[4:], 1 / 5, atol=1e-15)
    assert np.all(np.linalg.eigvalsh(me) > 0)


def test_t10_exact_mass_curved_element():
    """Curved (isoparametric) T10: N_a N_b det J has degree 7; the oracle's
    exact mass must equal an independent 8x8x8 collapsed-Gauss integral
    computed here, and its total must equal rho * volume (det J is cubic, so
    the degree-3 Keast rule gives the volume exactly)."""
    rng = np.random.default_rng(22)
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    Xf = np.vstack([X] + [(X[a] + X[b]) / 2 for a, b in synth.T10_EDGES])
    Xf[4:] += rng.uniform(-0.08, 0.08, (6, 3))                    # bend the edges
    conn = np.arange(10, dtype=np.int32)
    me = oracle.element_mass(0, 1, 0, 1000.0, conn, Xf)
    g, w = np.polynomial.legendre.leggauss(8)
    g, w = (g + 1) / 2, w / 2
    ref = np.zeros((10, 10))
    for i in range(8):
        for j in range(8):
            for k in range(8):
                u, s, t = g[i], g[j], g[k]
                xi = np.array([u, s * (1 - u), t * (1 - u) * (1 - s)])
                N, dN = oracle.t10_shape(xi)
                detJ = np.linalg.det(Xf.T @ dN)
                ref += np.outer(N, N) * detJ * (1 - u) ** 2 * (1 - s) * w[i] * w[j] * w[k] * 1000.0
    assert np.abs(me - ref).max() < 1e-13 * np.abs(ref).max()
    mesh = synth.Mesh(0, Xf, conn[None, :])
    pr = oracle.Problem(mesh, synth.SVK_PAPER, 1, with_pattern=False)
    assert abs(me.sum() - 1000.0 * pr.J0w.sum()) < 1e-13 * 1000.0 * pr.J0w.sum()


def test_t10_force_rule_mass_literal_reading():
    """mass_rule = 1 (P:309-310 literally): 4-point rule gives a rank-4 element
    mass; Keast-5 one negative eigenvalue (reading Q4)."""
    X = synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).X
    conn = synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).conn[0]
    ev4 = np.linalg.eigvalsh(oracle.element_mass(0, 0, 1, 1.0, conn, X))
    ev5 = np.linalg.eigvalsh(oracle.element_mass(0, 1, 1, 1.0, conn, X))
    assert np.sum(np.abs(ev4) > 1e-12 * ev4.max()) == 4
    assert np.sum(ev5 < -1e-12 * ev5.max()) == 1


def test_global_mass_and_force_field():
    mesh = synth.kuhn_t10_box(3, 2, 1, 3, 2, 1)
    g = np.array([0.0, 0.0, -9.81])
    pr = oracle.Problem(mesh, SVK, 1, gravity=g)
    assert abs(pr.M.sum() - 2700.0 * 6.0) < 1e-10 * 2700 * 6     # rho * V_total
    assert abs(pr.fff[2::3].sum() + 9.81 * 2700 * 6.0) < 1e-9 * 2700 * 6 * 9.81
    # ANCF: translational mass of the position coefficients = rho L W H per element
    pa = oracle.Problem(synth.ancf_plate(3), SVK, 2)
    pos = np.zeros(pa.n_coef)
    pos[0::4] = 1.0
    dense = np.zeros((pa.n_coef, pa.n_coef))
    for I in range(pa.n_coef):
        dense[I, pa.cols_c[pa.rowptr_c[I]:pa.rowptr_c[I + 1]]] = pa.M[pa.rowptr_c[I]:pa.rowptr_c[I + 1]]
    assert abs(pos @ dense @ pos - 2700.0 * 4 * 2 * 0.1) < 1e-10 * 2700 * 0.8
    assert np.abs(dense - dense.T).max() < 1e-12 * np.abs(dense).max()


def dense_H(pr, H):
    n = 3 * pr.n_coef
    D = np.zeros((n, n))
    for r in range(n):
        D[r, pr.cols[pr.rowptr[r]:pr.rowptr[r + 1]]] = H[pr.rowptr[r]:pr.rowptr[r + 1]]
    return D


def dense_M(pr):
    D = np.zeros((pr.n_coef, pr.n_coef))
    for I in range(pr.n_coef):
        D[I, pr.cols_c[pr.rowptr_c[I]:pr.rowptr_c[I + 1]]] = pr.M[pr.rowptr_c[I]:pr.rowptr_c[I + 1]]
    return D


def test_inertia_only_limit():
    """Material stubbed to zero (E = 0 -> P = 0, A = 0): H = M/h exactly and
    g = (1/h) M (v - v_n) — against a dense SpMV."""
    mesh = synth.kuhn_t10_box(2, 1, 1, 1, 1, 1)
    zero = dict(SVK, E=0.0)
    pr = oracle.Problem(mesh, zero, 1)
    x, v, vn, _ = synth.t10_state(mesh)
    h = 1e-3
    g, H, f = pr.eval(x, v, vn, None, h)
    assert np.abs(f).max() == 0
    Md = np.kron(dense_M(pr), np.eye(3))
    assert np.abs(dense_H(pr, H) - Md / h).max() < 1e-15 * np.abs(Md).max() / h
    assert np.abs(g - Md @ (v - vn) / h).max() < 1e-13 * np.abs(g).max()


def test_residual_zero_at_rest():
    mesh = synth.kuhn_t10_box(2, 2, 1, 1, 1, 1)
    pr = oracle.Problem(mesh, SVK, 1)
    v = np.random.default_rng(3).normal(size=mesh.n_dof)
    g, H, f = pr.eval(mesh.X.ravel(), v, v, None, 1e-3)
    assert np.abs(g).max() < 1e-6 and np.abs(f).max() < 1e-6


@pytest.mark.parametrize("mat", [SVK, MR], ids=["svk", "mr"])
def test_residual_is_gradient_of_augmented_cost_and_H_its_jacobian(mat):
    """Eq. cost without constraints: Phi(v) = 1/(2h)(v-vn)^T M (v-vn)
    + (1/h) Pi(q_n + h v) - f_ext^T v - f_ff^T v. Central FD of Phi w.r.t. v
    reproduces g; central FD of g reproduces H (no viscosity, Q8)."""
    mesh = synth.kuhn_t10_box(1, 1, 1, 0.2, 0.2, 0.2)
    grav = np.array([0.0, -9.81, 0.0])
    pr = oracle.Problem(mesh, mat, 1, gravity=grav)
    h = 1e-3
    rng = np.random.default_rng(8)
    qn = mesh.X.ravel() + rng.normal(0, 2e-3, mesh.n_dof)
    v = rng.normal(0, 0.5, mesh.n_dof)
    vn = rng.normal(0, 0.5, mesh.n_dof)
    fext = rng.normal(0, 100.0, mesh.n_dof)
    Md = np.kron(dense_M(pr), np.eye(3))
    cc = mesh.coef_conn()

    def Pi(x):
        return sum(oracle.element_energy(0, 1, mat["model"], mat, mesh.conn[e], mesh.X,
                                         x.reshape(-1, 3)[cc[e]].ravel()) for e in range(mesh.n_el))

    def Phi(vv):
        dv = vv - vn
        return dv @ Md @ dv / (2 * h) + Pi(qn + h * vv) / h - fext @ vv - pr.fff @ vv

    g, H, _ = pr.eval(qn + h * v, v, vn, fext, h)
    step = 1e-5
    fd = np.array([(Phi(v + step * e) - Phi(v - step * e)) / (2 * step) for e in np.eye(mesh.n_dof)])
    assert np.abs(fd - g).max() < 1e-6 * np.abs(g).max()
    Hd = dense_H(pr, H)
    assert np.abs(Hd - Hd.T).max() < 1e-12 * np.abs(Hd).max()
    for j in rng.choice(mesh.n_dof, 12, replace=False):
        e = np.zeros(mesh.n_dof)
        e[j] = 1e-4
        gp, _, _ = pr.eval(qn + h * (v + e), v + e, vn, fext, h, hessian=False)
        gm, _, _ = pr.eval(qn + h * (v - e), v - e, vn, fext, h, hessian=False)
        assert np.abs((gp - gm) / 2e-4 - Hd[:, j]).max() < 1e-6 * np.abs(Hd).max()
    # Remark P:507-513: SPD at the paper's h -> Cholesky succeeds
    np.linalg.cholesky(Hd)


def test_hessian_minus_mass_is_h_times_stiffness():
    mesh = synth.kuhn_t10_box(2, 1, 1, 0.4, 0.2, 0.2)
    pr = oracle.Problem(mesh, SVK, 0)
    x, v, vn, _ = synth.t10_state(mesh)
    h = 1e-3
    _, H, _ = pr.eval(x, v, vn, None, h)
    K = np.zeros((mesh.n_dof, mesh.n_dof))
    cc = mesh.coef_conn()
    for e in range(mesh.n_el):
        _, Ke = oracle.element(0, 0, 0, SVK, mesh.conn[e], mesh.X, x)
        idx = (3 * cc[e][:, None] + np.arange(3)[None, :]).ravel()
        K[np.ix_(idx, idx)] += Ke
    Md = np.kron(dense_M(pr), np.eye(3))
    assert np.abs(dense_H(pr, H) - Md / h - h * K).max() < 1e-13 * np.abs(dense_H(pr, H)).max()


def test_stage1_stage2_split_equals_fused():
    mesh = synth.kuhn_t10_box(2, 1, 1, 0.4, 0.2, 0.2)
    mat = dict(MR, eta_damp=5e3, lambda_damp=5e3)
    pr = oracle.Problem(mesh, mat, 1)
    x, v, vn, _ = synth.t10_state(mesh)
    P = pr.stress(x, v)
    f2 = pr.force_from_stress(P)
    _, _, f = pr.eval(x, v, vn, None, 1e-3, hessian=False)
    assert np.abs(f2 - f).max() < 1e-13 * np.abs(f).max()


def test_many_body_invariants():
    mesh, x, v = synth.many_body(n_bodies=3, cells=(2, 1, 1), size=(0.2, 0.1, 0.1))
    pr = oracle.Problem(mesh, synth.TIRE_DROP, 1)
    _, _, f = pr.eval(x, v, v, None, 1e-3, hessian=False)
    f = f.reshape(-1, 3)
    xn = x.reshape(-1, 3)
    per = mesh.n_coef // 3
    for b in range(3):
        fb, xb = f[b * per:(b + 1) * per], xn[b * per:(b + 1) * per]
        s = np.abs(fb).max()
        assert np.abs(fb.sum(0)).max() < 1e-12 * s
        assert np.abs(np.cross(xb, fb).sum(0)).max() < 1e-12 * s * 1.0


def test_eval_rows_matches_full_eval():
    mesh = synth.kuhn_t10_box(3, 2, 2, 0.6, 0.4, 0.4)
    mat = dict(SVK)
    pr = oracle.Problem(mesh, mat, 1)
    x, v, vn, _ = synth.t10_state(mesh)
    h = 1e-3
    _, H, f = pr.eval(x, v, vn, None, h)
    nodes = np.array([0, 5, 17, mesh.n_coef - 1])
    cols, Hr, fr, Mr = oracle.eval_rows(mesh, mat, 1, 0, x, v, h, nodes)
    for s, I in enumerate(nodes):
        c = cols[s][cols[s] >= 0]
        assert list(c) == list(pr.cols_c[pr.rowptr_c[I]:pr.rowptr_c[I + 1]])
        for d in range(3):
            r = 3 * I + d
            row = H[pr.rowptr[r]:pr.rowptr[r + 1]].reshape(-1, 3)
            assert np.abs(row - Hr[s, d, :len(c)]).max() < 1e-13 * np.abs(row).max()
        assert np.abs(fr[s] - f[3 * I:3 * I + 3]).max() < 1e-12 * np.abs(f).max()


# ------------------------------------------------------------ paper tables --

def test_t10_res0_statistics():
    row = GOLD["t10_mesh_statistics"]["RES0"]
    mesh = synth.kuhn_t10_box(3, 2, 1, 3.0, 2.0, 1.0)
    assert (mesh.n_coef, mesh.n_el, mesh.n_dof, synth.clamped_dofs_t10(mesh)) == \
        (row["nodes"], row["elements"], row["dofs"], row["constrained_dofs"])


def test_ancf3443_statistics_all_rows():
    for row in GOLD["ancf3443_mesh_statistics"]["rows"]:
        mesh = synth.ancf_plate(row["n"])
        assert (mesh.n_coef // 4, mesh.n_el, mesh.n_dof, synth.clamped_dofs_ancf(mesh)) == \
            (row["nodes"], row["elements"], row["dofs"], row["constrained_dofs"])


def test_paper_sizes():
    assert len(oracle.quadrature(1)[1]) == GOLD["quadrature_sizes"]["t10_keast"]
    assert len(oracle.quadrature(2)[1]) == GOLD["quadrature_sizes"]["ancf_shell_gl"]
    _, K = oracle.element(0, 1, 0, SVK, np.arange(10, dtype=np.int32), synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).X,
                          synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).X.ravel())
    assert K.shape == (GOLD["element_block_sizes"]["t10"],) * 2
    m = synth.ancf_plate(1)
    _, K = oracle.element(1, 2, 0, SVK, m.conn[0], m.X, m.X.ravel(), LWH=m.dims[0])
    assert K.shape == (GOLD["element_block_sizes"]["ancf_shell"],) * 2
    for k in ("E", "nu", "rho0"):
        assert synth.SVK_PAPER[k] == GOLD["svk_scaling_material"][k]
    for k in ("C10", "C01", "kappa", "rho0"):
        assert synth.MR_PAPER[k] == GOLD["mr_material"][k]


def test_pattern_counts_configs_2_and_3():
    """SURVEY §8(c) pattern pins for the two large Kuhn boxes (config 2:
    nnz_H = 34,979,121; config 3: 1,384,065,801), without building their
    patterns: on a Kuhn box every coefficient pair belongs to an interior,
    face, edge or corner class of the cell lattice, so nnz_c is a trilinear
    polynomial in the cell counts (nx, ny, nz) once each is >= 2 (no two
    boundary layers overlap). Fit it exactly on the 8 boxes {3,4}^3 with the
    oracle's brute-force pattern, check it on boxes outside the fit, evaluate."""
    def nnz_c(n):
        return oracle.Problem(synth.kuhn_t10_box(*n, 1.0, 1.0, 1.0), SVK, 1).nnz_c

    def row(n):
        x, y, z = n
        return [1, x, y, z, x * y, x * z, y * z, x * y * z]

    fit = [(a, b, c) for a in (3, 4) for b in (3, 4) for c in (3, 4)]
    coef = np.linalg.solve(np.array([row(n) for n in fit], float), np.array([nnz_c(n) for n in fit], float))
    coef = np.round(coef * 6) / 6  # the class counts are integers per cell, edge and face
    for n in ((5, 3, 4), (2, 6, 3), (7, 2, 2)):
        assert round(float(np.dot(row(n), coef))) == nnz_c(n), n
    assert 9 * round(float(np.dot(row((42, 28, 14)), coef))) == 34_979_121
    assert 9 * round(float(np.dot(row((144, 96, 48)), coef))) == 1_384_065_801


def test_all_core_oracle_equals_serial():
    """The all-core CPU baseline (OpenMP element loop, thread-private element
    blocks assembled in element order) is bitwise the serial oracle."""
    for mesh, mat, rule in ((synth.kuhn_t10_box(4, 3, 2, 0.8, 0.6, 0.4), SVK, 1),
                            (synth.ancf_plate(3), SVK, 2)):
        pr = oracle.Problem(mesh, mat, rule)
        if mesh.element == 0:
            x, v, vn, fe = synth.t10_state(mesh, with_fext=True)
        else:
            x, v, vn = synth.ancf_state(mesh)
            fe = None
        a = pr.eval(x, v, vn, fe, 1e-3)
        b = pr.eval(x, v, vn, fe, 1e-3, all_cores=True)
        for u, w in zip(a, b):
            assert np.array_equal(u, w)
    assert oracle.max_threads() >= 1
