"""Pins of the oracle's constitutive functions (§4.3; the
forms of readings Q5-Q7 / SPEC S:266-303) against closed forms, invariants and
finite differences of the strain energy."""
import numpy as np
import pytest

import oracle
import synth

SVK = dict(synth.SVK_PAPER)
MR = dict(synth.MR_PAPER)
KV = dict(synth.SVK_PAPER, eta_damp=5e3, lambda_damp=7e3)


def lame(mat):
    E, nu = mat["E"], mat["nu"]
    return E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))


def rand_rot(rng):
    return synth.random_rotation(rng)


def rand_F(rng, amp=0.1):
    return np.eye(3) + rng.uniform(-amp, amp, (3, 3))


@pytest.mark.parametrize("mat", [SVK, MR], ids=["svk", "mr"])
def test_stress_free_reference_and_rotation(mat):
    m = mat["model"]
    assert np.abs(oracle.pk1_elastic(m, mat, np.eye(3))).max() < 1e-6 * (mat["E"] or mat["kappa"]) * 1e-9
    rng = np.random.default_rng(4)
    for _ in range(5):
        R = rand_rot(rng)
        scale = mat["E"] or mat["kappa"]
        assert np.abs(oracle.pk1_elastic(m, mat, R)).max() < 1e-15 * scale * 10
        F = rand_F(rng)
        P = oracle.pk1_elastic(m, mat, F)
        assert np.allclose(oracle.pk1_elastic(m, mat, R @ F), R @ P, rtol=0, atol=1e-14 * scale * 10)


def test_svk_uniaxial_closed_form():
    # F = diag(ls,1,1): P11 = ls (lam/2 + mu)(ls^2-1), P22 = P33 = lam (ls^2-1)/2
    lam, mu = lame(SVK)
    for ls in (0.9, 1.05, 1.3):
        P = oracle.pk1_elastic(0, SVK, np.diag([ls, 1.0, 1.0]))
        ref = np.diag([ls * (lam / 2 + mu) * (ls ** 2 - 1), lam * (ls ** 2 - 1) / 2, lam * (ls ** 2 - 1) / 2])
        assert np.allclose(P, ref, rtol=1e-14, atol=1e-6)


def test_mr_pure_dilation_closed_form():
    # F = s I: deviatoric parts vanish; P = kappa (J - 1) s^2 I with J = s^3
    for s in (0.95, 1.02, 1.1):
        P = oracle.pk1_elastic(1, MR, s * np.eye(3))
        J = s ** 3
        assert np.allclose(P, MR["kappa"] * (J - 1) * s * s * np.eye(3), rtol=1e-13, atol=1e-4)


def test_mr_small_strain_shear_modulus():
    # Linearised MR: mu = 2 (C10 + C01) (reading Q6)
    g = 1e-7
    F = np.eye(3)
    F[0, 1] = g
    P = oracle.pk1_elastic(1, MR, F)
    mu = 2 * (MR["C10"] + MR["C01"])
    assert abs(P[0, 1] / g - mu) / mu < 1e-5


@pytest.mark.parametrize("mat", [SVK, MR], ids=["svk", "mr"])
def test_pk1_is_energy_gradient(mat):
    """P = dW/dF: complex step of W (exact to rounding) and central FD (1e-6)."""
    m = mat["model"]
    rng = np.random.default_rng(5)
    for _ in range(20):
        F = rand_F(rng, 0.25)
        P = oracle.pk1_elastic(m, mat, F)
        scale = np.abs(P).max()
        assert np.abs(oracle.energy_grad_csd(m, mat, F) - P).max() < 1e-13 * scale
        fd = np.zeros((3, 3))
        for i in range(3):
            for j in range(3):
                E = np.zeros((3, 3))
                E[i, j] = 1e-6
                fd[i, j] = (oracle.energy(m, mat, F + E) - oracle.energy(m, mat, F - E)) / 2e-6
        assert np.abs(fd - P).max() < 1e-6 * scale


def test_svk_energy_uniaxial():
    lam, mu = lame(SVK)
    ls = 1.1
    Eg = 0.5 * (ls ** 2 - 1)
    assert abs(oracle.energy(0, SVK, np.diag([ls, 1, 1])) - (lam / 2 * Eg ** 2 + mu * Eg ** 2)) < 1e-6


@pytest.mark.parametrize("mat", [SVK, MR], ids=["svk", "mr"])
def test_tangent_fd_and_major_symmetry(mat):
    m = mat["model"]
    rng = np.random.default_rng(6)
    for _ in range(10):
        F = rand_F(rng, 0.2)
        A = oracle.tangent(m, mat, F)
        scale = np.abs(A).max()
        fd = np.zeros((3, 3, 3, 3))
        for k in range(3):
            for L in range(3):
                E = np.zeros((3, 3))
                E[k, L] = 1e-6
                fd[:, :, k, L] = (oracle.pk1_elastic(m, mat, F + E) - oracle.pk1_elastic(m, mat, F - E)) / 2e-6
        assert np.abs(fd - A).max() < 1e-6 * scale
        # hyperelastic: A_iJkL = A_kLiJ
        assert np.abs(A - A.transpose(2, 3, 0, 1)).max() < 1e-13 * scale


def test_svk_tangent_at_identity_is_linear_elastic():
    lam, mu = lame(SVK)
    d = np.eye(3)
    ref = (lam * np.einsum("ij,kl->ijkl", d, d) + mu * (np.einsum("ik,jl->ijkl", d, d)
                                                         + np.einsum("il,jk->ijkl", d, d)))
    assert np.allclose(oracle.tangent(0, SVK, np.eye(3)), ref, rtol=1e-14, atol=1e-3)


def test_kelvin_voigt_closed_forms():
    eta, lamd = KV["eta_damp"], KV["lambda_damp"]
    # F = I, Fdot = diag(a,0,0) -> P_v = diag(2 eta a + lam a, lam a, lam a)
    a = 0.3
    P = oracle.pk1_viscous(KV, np.eye(3), np.diag([a, 0, 0]))
    assert np.allclose(P, np.diag([2 * eta * a + lamd * a, lamd * a, lamd * a]), rtol=1e-15)
    assert np.abs(oracle.pk1_viscous(KV, rand_F(np.random.default_rng(0)), np.zeros((3, 3)))).max() == 0
    rng = np.random.default_rng(7)
    for _ in range(200):
        F = rand_F(rng, 0.3)
        Fd = rng.normal(size=(3, 3))
        Pv = oracle.pk1_viscous(KV, F, Fd)
        # P_v F^T symmetric (Kirchhoff-like stress) and non-negative power P_v : Fdot
        T = Pv @ F.T
        assert np.abs(T - T.T).max() < 1e-12 * np.abs(T).max()
        assert np.sum(Pv * Fd) >= -1e-12 * np.abs(Pv).max()
    # total = elastic + viscous
    F = rand_F(rng)
    Fd = rng.normal(size=(3, 3))
    assert np.allclose(oracle.pk1(0, KV, F, Fd), oracle.pk1_elastic(0, KV, F) + oracle.pk1_viscous(KV, F, Fd),
                       rtol=1e-15, atol=1e-6)
