"""CPU tests: the oracle against the committed golden fixtures and the SPEC's known-answer checks.

The reference ships no tests; the KATs below are the SPEC examples for the online path
 plus the operator pin against the reference's own assembler.
"""

import numpy as np
import pytest

from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import affine, synthetic
from paper_1807_11866_b200.model import ReducedModel

from .golden_utils import golden, reference_model


# ---- operator pinned against the reference assembler -------------------------------------------------

def test_reference_operator_pin():
    """Tensor residual/Jacobian == projected high-fidelity forms of rbflow.assemble (assemble.py:86-101)."""
    d = golden("reference_operator")
    model = reference_model()
    for i in range(len(d["mu"])):
        R, J = oracle.reduced_operator(model, d["mu"][i], d["eta"][i])
        assert np.abs(R - d["R_ref"][i]).max() <= 1e-12 * np.abs(d["R_ref"][i]).max()
        assert np.abs(J - d["J_ref"][i]).max() <= 1e-12 * np.abs(d["J_ref"][i]).max()


def test_reference_model_solutions_and_galerkin():
    """Reduced solutions of the reference-assembled model: Galerkin orthogonality (≤1e-7)."""
    d = golden("reference_operator")
    model = reference_model()
    assert np.all(d["galerkin_residual"] <= 1e-10)
    for mu, u_ref, it_ref in zip(d["solve_mu"], d["solve_u"], d["solve_iters"]):
        u, it, st, _ = oracle.solve_sample(model, mu)
        assert st == oracle.CONVERGED and it == it_ref
        assert np.abs(u - u_ref).max() <= 1e-13 * np.abs(u_ref).max()


# ---- synthetic configs: generator drift + oracle reproduces the fixtures --------------------------------

@pytest.mark.parametrize("c", [0, 1, 2, 4])
def test_synthetic_golden(cfg_model, c):
    d = golden(f"synthetic_cfg{c}")
    cfg = synthetic.CONFIGS[c]
    model = cfg_model(c)
    from tests.golden.make_golden import checksums

    np.testing.assert_allclose(checksums(model), d["checksums"], rtol=1e-13, atol=1e-12)
    mu = synthetic.config_mu(cfg, len(d["mu"]))
    np.testing.assert_array_equal(mu, d["mu"])
    u, it, st, _ = oracle.solve_batch(model, mu, tol=cfg.tol, max_iter=cfg.max_iter)
    assert np.all(st == 0) and np.array_equal(it, d["iters"])
    assert np.abs(u - d["u"]).max() <= 1e-12 * np.abs(d["u"]).max()
    if cfg.n_p:
        p = oracle.recover_pressure(model, mu, u)
        assert np.abs(p - d["p"]).max() <= 1e-12 * np.abs(d["p"]).max()


def test_oracle_paths_agree_cfg0_full(cfg_model):
    """Per-sample einsum path == batched GEMM path (the device's formulation) on all of config 0."""
    cfg = synthetic.CONFIGS[0]
    model = cfg_model(0)
    mu = synthetic.config_mu(cfg)
    ub, ib, sb, _ = oracle.solve_batch(model, mu)
    for b in range(len(mu)):
        u, it, st, _ = oracle.solve_sample(model, mu[b])
        assert it == ib[b] and st == sb[b] == 0
        assert np.abs(u - ub[b]).max() <= 1e-13 * np.abs(u).max()


# ---- SPEC known answers for reduced_operator ------------------------------------------

def test_eta_zero_kat(cfg_model):
    """η = 0 → residual = −f(μ), Jacobian = ν A(μ) only."""
    model = cfg_model(1)
    mu = np.array([0.3, 57.0])
    R, J = oracle.reduced_operator(model, mu, np.zeros(model.n))
    th = affine.evaluate_weights(model.theta, mu[None])[0]
    np.testing.assert_allclose(R, -(th @ model.f), rtol=0, atol=1e-14)
    np.testing.assert_allclose(J, np.einsum("q,qij->ij", th, model.A) / mu[1], rtol=0, atol=1e-14)


def test_jacobian_finite_differences(cfg_model):
    """Tensor Jacobian vs central differences, step 1e-6, max rel entry err ≤ 1e-6 (#5)."""
    model = cfg_model(0)
    rng = np.random.default_rng(3)
    mu = np.array([0.4, 80.0])
    eta = rng.standard_normal(model.n)
    _, J = oracle.reduced_operator(model, mu, eta)
    h = 1e-6
    Jfd = np.empty_like(J)
    for m in range(model.n):
        e = np.zeros(model.n)
        e[m] = h
        Rp, _ = oracle.reduced_operator(model, mu, eta + e)
        Rm, _ = oracle.reduced_operator(model, mu, eta - e)
        Jfd[:, m] = (Rp - Rm) / (2 * h)
    assert np.abs(J - Jfd).max() <= 1e-6 * np.abs(J).max()


def test_weight_consistency_monomial():
    """At α = 0 only the φ⁰ monomials survive: residual == the one assembled from k = 0 terms."""
    model = reference_model()
    rng = np.random.default_rng(1)
    eta = rng.standard_normal(model.n)
    mu = np.array([0.0, 1.0])
    R, _ = oracle.reduced_operator(model, mu, eta)
    k0 = ReducedModel(A=model.A[:1], C=model.C[:1], f=model.f[:1], theta=model.theta[:1])
    R0, _ = oracle.reduced_operator(k0, mu, eta)
    np.testing.assert_allclose(R, R0, rtol=0, atol=1e-13)


def test_energy_identity(cfg_model):
    """C antisymmetric in (k,l) ⇒ c(u,u,u) = 0: uᵀR(u) = ν uᵀA(μ)u − uᵀf(μ) (structure of the generators)."""
    model = cfg_model(1)
    rng = np.random.default_rng(2)
    u = rng.standard_normal(model.n)
    mu = np.array([0.2, 150.0])
    R, _ = oracle.reduced_operator(model, mu, u)
    th = affine.evaluate_weights(model.theta, mu[None])[0]
    A = np.einsum("q,qij->ij", th, model.A)
    np.testing.assert_allclose(u @ R, u @ A @ u / mu[1] - u @ (th @ model.f), rtol=1e-12)


# ---- θ families ---------------------------------------------------------------------

def test_theta_families():
    a = np.linspace(0, np.deg2rad(35), 11)
    mu = np.stack([a, np.full_like(a, 50.0)], 1)
    t7 = affine.evaluate_weights(affine.family("trig7"), mu)
    np.testing.assert_allclose(t7[:, 6], t7[:, 3] - t7[:, 4], atol=1e-15)   # cos 2α = cos²α − sin²α
    np.testing.assert_allclose(t7[:, 3] + t7[:, 4], 1.0, atol=1e-15)
    f13 = affine.evaluate_weights(affine.family("fourier13"), mu)
    assert f13.shape == (11, 13)
    np.testing.assert_allclose(f13[:, 11], np.cos(6 * a), atol=1e-15)
    m = affine.monomials([(0, 0), (1, 0), (2, 1)], [2.0, 0.5, -1.0])
    w = affine.evaluate_weights(m, np.array([[0.2, 3.0], [0.0, 1.0]]))
    np.testing.assert_allclose(w[0], [2.0, 0.1, -0.12], atol=1e-15)   # scale·αᵏ·Reᵐ
    np.testing.assert_allclose(w[1], [2.0, 0.0, 0.0])                 # μ=(0,1): k>0 weights vanish


def test_configs_match_baseline():
    import json
    from pathlib import Path

    txt = json.loads((Path(__file__).resolve().parents[1] / "BASELINE.json").read_text())["configs"]
    expect = {0: (10, 3, 64), 1: (50, 7, 16384), 2: (100, 7, 65536), 3: (200, 13, 131072), 4: (100, 7, 65536)}
    for c, (n, q, b) in expect.items():
        cfg = synthetic.CONFIGS[c]
        assert (cfg.n, cfg.q, cfg.batch) == (n, q, b)
        assert f"N={n}" in txt[c] and f"Q={q}" in txt[c]
        assert len(affine.family(cfg.theta_family)) == q
    assert synthetic.CONFIGS[4].n_p == 100


# ---- outcomes: singular / non-finite / non-converged are statuses ---------------------------

def _tiny(n=4, q=1, scale_c=0.0, a_scale=1.0, f_scale=1.0):
    rng = np.random.default_rng(0)
    A = a_scale * np.eye(n)[None].repeat(q, 0)
    C = scale_c * rng.standard_normal((q, n, n, n))
    f = f_scale * rng.standard_normal((q, n))
    return ReducedModel(A=A, C=C, f=f, theta=[affine.ThetaTerm(affine.CONST)] * q)


def test_oracle_outcomes():
    sing = _tiny(a_scale=0.0)
    _, it, st, _ = oracle.solve_sample(sing, np.array([0.1, 10.0]))
    assert st == oracle.SINGULAR_SYSTEM and it == 1
    _, it, st, _ = oracle.solve_batch(sing, np.array([[0.1, 10.0]]))
    assert st[0] == oracle.SINGULAR_SYSTEM
    zero_f = _tiny(f_scale=0.0)
    u, it, st, _ = oracle.solve_sample(zero_f, np.array([0.1, 10.0]))
    assert st == oracle.CONVERGED and it == 1 and not u.any()
    nc = _tiny(scale_c=5.0)
    _, it, st, _ = oracle.solve_sample(nc, np.array([0.1, 10.0]), max_iter=1)
    assert st == oracle.NON_CONVERGED and it == 1


def test_pressure_recovery_oracle(cfg_model):
    model = cfg_model(4)
    rng = np.random.default_rng(4)
    u = rng.standard_normal((3, model.n))
    mu = synthetic.config_mu(4, 3)
    p = oracle.recover_pressure(model, mu, u)
    th = affine.evaluate_weights(model.theta, mu)
    for b in range(3):
        rhs = np.einsum("q,qik,k->i", th[b], model.Bq, u[b])
        np.testing.assert_allclose(model.Mp @ p[b], rhs, rtol=1e-12, atol=1e-12)   # recovery residual
    np.testing.assert_allclose(oracle.recover_pressure(model, mu, 2 * u), 2 * p, rtol=1e-14)  # linearity
