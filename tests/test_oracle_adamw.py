"""Pins of the oracle's AdamW inner iteration (Alg. 2; SURVEY
§8(f) NEXT-2) against closed forms of the update rule and a descent property
of the whole iteration. CPU only."""
import numpy as np
import pytest

import oracle
import synth

PRM = dict(alpha=2e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=1e-2)


def _vecs(n=57, seed=5):
    rng = np.random.default_rng(seed)
    return rng.normal(size=n), rng.normal(size=n), rng.normal(size=n)


def test_zero_gradient_first_iteration_is_pure_decay():
    # m = s = 0 and g = 0: m_hat = 0, so v <- (1 - alpha wd) v exactly
    v, qn, _ = _vecs()
    z = np.zeros_like(v)
    m, s, v1, q = oracle.adamw_update(1, PRM, z, z, z, v, qn, 1e-3)
    assert np.array_equal(m, z) and np.array_equal(s, z)
    assert np.array_equal(v1, (1 - PRM["alpha"] * PRM["weight_decay"]) * v)
    assert np.allclose(q, qn + 1e-3 * v1, rtol=0, atol=1e-15)


def test_beta_zero_is_normalized_sign_descent():
    # beta1 = beta2 = 0: m_hat = g, s_hat = g^2 -> v <- v - alpha g / (|g| + eps)
    v, qn, g = _vecs(seed=6)
    prm = dict(PRM, beta1=0.0, beta2=0.0, weight_decay=0.0, eps=0.0)
    z = np.zeros_like(v)
    for l in (1, 2, 7):
        _, _, v1, _ = oracle.adamw_update(l, prm, g, z, z, v, qn, 1e-3)
        assert np.allclose(v1, v - prm["alpha"] * np.sign(g), rtol=0, atol=1e-15)


def test_bias_correction_constant_gradient():
    # from zero moments and a constant g: m_l = (1 - b1^l) g, s_l = (1 - b2^l) g^2,
    # so the bias-corrected step is alpha g / (|g| + eps) at EVERY iteration l
    v, qn, g = _vecs(seed=7)
    prm = dict(PRM, weight_decay=0.0)
    m = np.zeros_like(v)
    s = np.zeros_like(v)
    for l in range(1, 8):
        m, s, v1, _ = oracle.adamw_update(l, prm, g, m, s, v, qn, 1e-3)
        step = v - v1
        assert np.allclose(step, prm["alpha"] * g / (np.abs(g) + prm["eps"]), rtol=1e-12, atol=0)
        assert np.allclose(m, (1 - prm["beta1"] ** l) * g, rtol=1e-13, atol=0)
        assert np.allclose(s, (1 - prm["beta2"] ** l) * g * g, rtol=1e-12, atol=0)
        v = v1


@pytest.mark.parametrize("rule", [0, 1])
def test_iteration_descends_inertia_only(rule):
    # E = 0: f_int = 0, so g = M (v - v_n)/h - f_ext - f_ff is the gradient of a
    # strictly convex quadratic; AdamW from v = v_n must drive ||g|| down
    mesh = synth.kuhn_t10_box(3, 2, 1, 0.3, 0.2, 0.1)
    mat = dict(synth.SVK_PAPER, E=0.0)
    pr = oracle.Problem(mesh, mat, rule, gravity=(0.0, 0.0, -9.81))
    x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    h = 1e-3
    qn = x - h * v
    v = vn.copy()
    g, _, f = pr.eval(qn + h * v, v, vn, fext, h, hessian=False)
    assert np.array_equal(f, np.zeros_like(f))
    g0 = np.linalg.norm(g)
    m = np.zeros_like(v)
    s = np.zeros_like(v)
    prm = dict(PRM, alpha=5e-3, weight_decay=0.0)
    for l in range(1, 301):
        v, m, s, g, q, f, gn, vnorm = oracle.adamw_iteration(pr, l, prm, qn, vn, fext, h, v, m, s, g)
        assert gn == pytest.approx(np.linalg.norm(g), rel=1e-15)
    assert np.allclose(q, qn + h * v, rtol=0, atol=1e-15)
    assert gn < 0.1 * g0
