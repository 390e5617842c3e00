"""error_study / timing_study and their offline helpers (pod SPEC.md:436-446, Galerkin
projection SPEC.md:449-457) — SURVEY.md §8(f) row 4.

Stand-in for the reference's high-fidelity stage (offline, out of scope): an algebraic "high-fidelity" model of
the same residual form at n_h = 96 unknowns, its snapshots solved by the CPU oracle (test infrastructure), a POD
basis in the G = A₀ (SPD, H1-semi-like) norm, and the Galerkin-projected ReducedModel solved on the device.
"""

import numpy as np
import pytest


def test_loglog_slope_and_cpu_refusal():
    from paper_1807_11866_b200 import study
    from paper_1807_11866_b200.errors import NativeError

    x = np.array([1e-1, 1e-2, 1e-3])
    assert abs(study.loglog_slope(x, 3 * x) - 1.0) < 1e-12
    with pytest.raises(NativeError):
        study.pod(np.eye(3), device="cpu")


def _hifi(n_h=96, s=24, seed=7):
    from oracle import rbns_oracle as oracle
    from paper_1807_11866_b200 import synthetic

    hifi = synthetic.make_model(n_h, 3, "trig3", seed=seed, kappa_c=2e-4)
    mus = synthetic.make_mu(s, 40.0, seed=seed + 1)
    U, it, st, _ = oracle.solve_batch(hifi, mus)
    assert np.all(st == 0)
    return hifi, mus, U


@pytest.mark.gpu
def test_pod_spec_examples():
    from paper_1807_11866_b200 import study

    # ε = 0.1, spectrum {1, 0.005, 0.004, 0.001} → M = 1
    lam = np.array([1.0, 0.005, 0.004, 0.001])
    Y = np.zeros((4, 10))
    Y[np.arange(4), np.arange(4)] = np.sqrt(lam)
    V, l2, eps = study.pod(Y, eps=0.1)
    assert V.shape == (10, 1) and np.allclose(l2, lam)
    # projection-error identity Σ‖φ_i − P_V φ_i‖² = Σ_{k>M} λ_k, G-orthonormal basis
    rng = np.random.default_rng(0)
    Y = rng.standard_normal((12, 40))
    G = np.eye(40) + 0.1 * np.ones((40, 40))
    V, lam, eps = study.pod(Y, G=G, M=5)
    assert np.abs(V.T @ G @ V - np.eye(5)).max() <= 1e-10
    R = Y - (Y @ G @ V) @ V.T
    proj_err = np.einsum("ij,jk,ik->", R, G, R)
    assert abs(proj_err - lam[5:].sum()) <= 1e-8 * lam[5:].sum()
    with pytest.raises(ValueError, match="rank"):
        study.pod(Y, M=13)


@pytest.mark.gpu
def test_error_study_reproduces_snapshots():
    """Complete basis of the snapshot span (every mode above the numerical-rank cut), test grid =
    training grid → mean errors ≤ 1e-7."""
    from paper_1807_11866_b200 import study

    hifi, mus, U = _hifi()
    G = hifi.A[0]
    V, lam, eps = study.pod(U, G=G, eps=1e-9)
    rm = study.galerkin_project(hifi, V)
    rep = study.error_study(rm, mus, U, V, G=G, expected=eps)
    assert rep.n_unconverged == 0 and rep.n_queries == len(mus)
    assert rep.mean_velocity_error <= 1e-7, rep
    print(study.CSV_HEADER)
    print(rep.row(V.shape[1]))


@pytest.mark.gpu
def test_error_study_convergence_in_m_and_unconverged_queries():
    """Errors on a separate 15 × 15 test grid fall as M grows, paired with the expected ε(M); unconverged
    queries are excluded and counted."""
    from paper_1807_11866_b200 import study

    hifi, mus, U = _hifi(s=48)
    from oracle import rbns_oracle as oracle

    a, re = np.meshgrid(np.linspace(0.0, np.deg2rad(35.0), 15), np.linspace(10.0, 40.0, 15))
    test_mu = np.stack([a.ravel(), re.ravel()], axis=1)
    U_test, _, st, _ = oracle.solve_batch(hifi, test_mu)
    assert np.all(st == 0)
    G = hifi.A[0]
    rows, meas, exp = [], [], []
    for m in (2, 4, 6, 8):
        V, lam, eps = study.pod(U, G=G, M=m)
        rm = study.galerkin_project(hifi, V)
        rep = study.error_study(rm, test_mu, U_test, V, G=G, expected=eps)
        assert rep.n_unconverged == 0
        rows.append(rep.row(m))
        meas.append(rep.mean_velocity_error)
        exp.append(eps)
    assert all(b < a for a, b in zip(meas, meas[1:])), meas
    print(study.CSV_HEADER, *rows, f"log-log slope measured vs expected: {study.loglog_slope(exp, meas):.2f}",
          sep="\n")
    rep = study.error_study(rm, test_mu, U_test, V, G=G, max_iter=1)
    assert rep.n_unconverged == len(test_mu) and np.isnan(rep.mean_velocity_error)


@pytest.mark.gpu
def test_timing_study():
    import torch

    from paper_1807_11866_b200 import online, study, synthetic

    cfg = synthetic.CONFIGS[1]
    m = synthetic.config_model(cfg)
    mus = synthetic.config_mu(cfg, 2048)
    with online.DeviceModel(m, 0) as dm:
        t = study.timing_study({"block": lambda mu: dm.solve(mu, pressure=False)}, mus)
    assert t["block"] > 0.0
