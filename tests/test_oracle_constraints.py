"""Pins of the oracle's constraint terms (Eq. residual
P:101-113, Eq. cost) with linear
constraints c(q) = C q - b (reading Q22): the pattern union against brute
force, g = grad_v of the augmented cost Phi_rho (central differences), H =
dg/dv, the h^2 rho C^T C closed form and the clamp-row closed form. CPU only."""
import numpy as np
import pytest

import oracle
import synth

SVK = dict(synth.SVK_PAPER)


def dense_C(con, n_dof):
    C = np.zeros((con["b"].size, n_dof))
    for k in range(con["b"].size):
        for p in range(con["rowptr"][k], con["rowptr"][k + 1]):
            C[k, con["cols"][p]] += con["vals"][p]
    return C


def dense_H(pr, H):
    D = np.zeros((pr.n_dof if hasattr(pr, "n_dof") else 3 * pr.n_coef,) * 2)
    for i in range(D.shape[0]):
        D[i, pr.cols[pr.rowptr[i]:pr.rowptr[i + 1]]] = H[pr.rowptr[i]:pr.rowptr[i + 1]]
    return D


def dense_M(pr):
    D = np.zeros((pr.n_coef, pr.n_coef))
    for I in range(pr.n_coef):
        D[I, pr.cols_c[pr.rowptr_c[I]:pr.rowptr_c[I + 1]]] = pr.M[pr.rowptr_c[I]:pr.rowptr_c[I + 1]]
    return D


@pytest.mark.parametrize("mk", [lambda: synth.kuhn_t10_box(3, 2, 1, 0.3, 0.2, 0.1),
                                lambda: synth.ancf_plate(3)], ids=["t10", "ancf"])
def test_pattern_is_union_with_constraint_couplings(mk):
    mesh = mk()
    con = synth.constraint_set(mesh, n_ties=6)
    rule = 1 if mesh.element == 0 else 2
    pr = oracle.Problem(mesh, SVK, rule, constraints=con)
    cc = mesh.coef_conn()
    rows = [set() for _ in range(mesh.n_coef)]
    for e in range(mesh.n_el):
        for a in cc[e]:
            rows[a].update(int(b) for b in cc[e])
    for k in range(con["b"].size):
        coefs = {int(j) // 3 for j in con["cols"][con["rowptr"][k]:con["rowptr"][k + 1]]}
        for I in coefs:
            rows[I] |= coefs
    for I in range(mesh.n_coef):
        assert pr.cols_c[pr.rowptr_c[I]:pr.rowptr_c[I + 1]].tolist() == sorted(rows[I])
    # the ties couple nodes no element couples -> the union is strictly larger
    base = oracle.Problem(mesh, SVK, rule)
    assert pr.nnz_c > base.nnz_c


def test_residual_is_gradient_of_constrained_cost_and_H_its_jacobian():
    """Phi_rho(v) = 1/(2h)(v-vn)^T M (v-vn) + Pi(q_n + h v)/h - (f_ext + f_ff)^T v
    + lam^T c(q_n + h v) + rho/2 ||c(q_n + h v)||^2 (Eq. cost)."""
    mesh = synth.kuhn_t10_box(1, 1, 1, 0.2, 0.2, 0.2)
    con = synth.constraint_set(mesh, n_ties=3)
    grav = np.array([0.0, -9.81, 0.0])
    pr = oracle.Problem(mesh, SVK, 1, gravity=grav, constraints=con)
    h, rho = 1e-3, 3e6
    rng = np.random.default_rng(18)
    qn = mesh.X.ravel() + rng.normal(0, 2e-3, mesh.n_dof)
    v = rng.normal(0, 0.5, mesh.n_dof)
    vn = rng.normal(0, 0.5, mesh.n_dof)
    fext = rng.normal(0, 100.0, mesh.n_dof)
    lam = rng.normal(0, 50.0, con["b"].size)
    Md = np.kron(dense_M(pr), np.eye(3))
    Cd = dense_C(con, mesh.n_dof)
    cc = mesh.coef_conn()

    def Pi(x):
        return sum(oracle.element_energy(0, 1, 0, SVK, mesh.conn[e], mesh.X, x.reshape(-1, 3)[cc[e]].ravel())
                   for e in range(mesh.n_el))

    def Phi(vv):
        dv = vv - vn
        q = qn + h * vv
        c = Cd @ q - con["b"]
        return dv @ Md @ dv / (2 * h) + Pi(q) / h - fext @ vv - pr.fff @ vv + lam @ c + 0.5 * rho * c @ c

    g, H, _ = pr.eval(qn + h * v, v, vn, fext, h, lam=lam, rho=rho)
    step = 1e-5
    fd = np.array([(Phi(v + step * e) - Phi(v - step * e)) / (2 * step) for e in np.eye(mesh.n_dof)])
    assert np.abs(fd - g).max() < 1e-6 * np.abs(g).max()
    Hd = dense_H(pr, H)
    for j in rng.choice(mesh.n_dof, 12, replace=False):
        e = np.zeros(mesh.n_dof)
        e[j] = 1e-4
        gp, _, _ = pr.eval(qn + h * (v + e), v + e, vn, fext, h, hessian=False, lam=lam, rho=rho)
        gm, _, _ = pr.eval(qn + h * (v - e), v - e, vn, fext, h, hessian=False, lam=lam, rho=rho)
        assert np.abs((gp - gm) / 2e-4 - Hd[:, j]).max() < 1e-6 * np.abs(Hd).max()


def test_constraint_terms_closed_forms():
    mesh = synth.kuhn_t10_box(2, 1, 1, 0.2, 0.1, 0.1)
    con = synth.constraint_set(mesh, n_ties=5)
    pr = oracle.Problem(mesh, SVK, 0, constraints=con)
    x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    h, rho = 1e-3, 1e7
    lam = np.random.default_rng(3).normal(0, 10.0, con["b"].size)
    g0, H0, f0 = pr.eval(x, v, vn, fext, h)                      # lam = 0, rho = 0
    g1, H1, f1 = pr.eval(x, v, vn, fext, h, lam=lam, rho=rho)
    assert np.array_equal(f0, f1)
    Cd = dense_C(con, mesh.n_dof)
    c = Cd @ x - con["b"]
    assert np.allclose(pr.constraint_residual(x), c, rtol=0, atol=1e-15)
    # g1 - g0 = h C^T (lam + rho c); H1 - H0 = h^2 rho C^T C (dense, exact)
    assert np.allclose(g1 - g0, h * Cd.T @ (lam + rho * c), rtol=1e-12, atol=1e-12 * np.abs(g1).max())
    dH = dense_H(pr, H1) - dense_H(pr, H0)
    assert np.allclose(dH, h * h * rho * Cd.T @ Cd, rtol=1e-12, atol=1e-9)
    # clamp rows: g_i gains h (lam_k + rho (x_i - b_k)), H_ii gains h^2 rho
    n_clamp = 3 * int(np.count_nonzero(np.abs(mesh.X[:, 0]) < 1e-12))
    for k in range(n_clamp):
        i = int(con["cols"][con["rowptr"][k]])
        ties = [t for t in range(n_clamp, con["b"].size) if i in con["cols"][con["rowptr"][t]:con["rowptr"][t + 1]]]
        if ties:
            continue
        # (g1 - g0 cancels: tolerance relative to |g|)
        assert (g1 - g0)[i] == pytest.approx(h * (lam[k] + rho * (x[i] - con["b"][k])),
                                             rel=0, abs=1e-13 * np.abs(g1).max())
        assert dH[i, i] == pytest.approx(h * h * rho, rel=0, abs=1e-13 * np.abs(H1).max())
