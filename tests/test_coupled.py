"""Naive coupled saddle solvers on the same sm_100a path.

SPEC examples: block vs coupled-stabilised on the same div-conforming model agree in velocity to 1e-8
(SPEC.md:526); unstabilised div-conforming → SINGULAR_SYSTEM or NON_CONVERGED, gracefully;
block wall time < coupled-3M wall time at M ≥ 20.
"""

import numpy as np
import pytest

from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import synthetic
from paper_1807_11866_b200.coupled import COUPLED_TOL, split


def test_embedding_structure():
    cm, blk = synthetic.make_coupled_model(6, 1)
    rm = cm.embedded()
    assert rm.n == 18 and rm.n_stop == 12 and rm.stop_absolute and not rm.nu_linear
    qa, qb = cm.A.shape[0], cm.B.shape[0]
    assert rm.counts == (qa + qb, cm.C.shape[0], cm.f.shape[0], 0)
    np.testing.assert_array_equal(rm.A[qa:, 12:, :12], cm.B)
    np.testing.assert_array_equal(rm.A[qa:, :12, 12:], cm.B.transpose(0, 2, 1))
    assert not rm.C[:, 12:].any() and not rm.C[:, :, 12:].any() and not rm.C[:, :, :, 12:].any()
    np.testing.assert_array_equal(rm.A[:qa, :6, :6], blk.A)      # velocity blocks verbatim


def test_oracle_block_coupled_equivalence():
    cm, blk = synthetic.make_coupled_model(10, 2)
    mu = synthetic.make_lifted_mu(32, seed=4)
    ub, itb, stb, _ = oracle.solve_batch(blk, mu)
    x, itc, stc, _ = oracle.solve_batch(cm.embedded(), mu, tol=COUPLED_TOL)
    u, s, p = split(cm, x)
    assert np.all(stb == 0) and np.all(stc == 0)
    assert np.abs(u - ub).max() <= 1e-8 * np.abs(ub).max()
    assert not s.any()                                            # s = 0 exactly (div-conforming)
    # the supremizer rows of the coupled residual vanish at the solution: Eq. (blocksolve-2) recovers p
    R, _ = oracle.reduced_operator(cm.embedded(), mu[0], x[0])
    assert np.abs(R).max() <= 1e-9 * np.abs(x[0]).max()


def test_oracle_unstabilised_fails_gracefully():
    cm, _ = synthetic.make_coupled_model(8, 1, stabilized=False)
    _, it, st, _ = oracle.solve_batch(cm.embedded(), synthetic.make_lifted_mu(4), tol=COUPLED_TOL)
    assert np.all(st == oracle.SINGULAR_SYSTEM) and np.all(it == 1)


# ---- GPU ------------------------------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("m", [10, 30])
def test_coupled_device_parity(m):
    cm, blk = synthetic.make_coupled_model(m, 2)
    rm = cm.embedded()
    mu = synthetic.make_lifted_mu(256, seed=6)
    from paper_1807_11866_b200.coupled import solve_coupled_batch

    u, s, p, it, st, _ = solve_coupled_batch(cm, mu)
    xr, itr, str_, _ = oracle.solve_batch(rm, mu, tol=COUPLED_TOL)
    ur, sr, pr = split(cm, xr)
    assert np.all(st == 0) and np.all(str_ == 0)
    assert np.abs(u - ur).max() <= 1e-10 * np.abs(ur).max()
    assert np.abs(p - pr).max() <= 1e-10 * np.abs(pr).max()
    assert not s.any()
    assert np.array_equal(it, itr)


@pytest.mark.gpu
def test_coupled_vs_block_device():
    """Velocity equivalence and the timing claim, on the device."""
    import time

    import torch

    from paper_1807_11866_b200 import online
    from paper_1807_11866_b200.coupled import solve_coupled_batch

    m = 30
    cm, blk = synthetic.make_coupled_model(m, 2)
    mu = synthetic.make_lifted_mu(4096, seed=8)
    dm = online.device_model(blk)
    res = dm.solve_host(mu)
    u, s, p, it, st, _ = solve_coupled_batch(cm, mu)
    assert np.all(st == 0) and np.all(res["status"] == 0)
    assert np.abs(u - res["u"]).max() <= 1e-8 * np.abs(res["u"]).max()
    t = []
    for fn in (lambda: dm.solve_host(mu), lambda: solve_coupled_batch(cm, mu)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    assert t[0] < t[1], f"block {t[0]:.4f}s vs coupled {t[1]:.4f}s"


@pytest.mark.gpu
def test_unstabilised_device_singular():
    from paper_1807_11866_b200.coupled import solve_coupled, solve_coupled_batch
    from paper_1807_11866_b200.errors import SingularSystemError

    cm, _ = synthetic.make_coupled_model(12, 1, stabilized=False)
    _, _, _, it, st, _ = solve_coupled_batch(cm, synthetic.make_lifted_mu(64))
    assert np.all(st == oracle.SINGULAR_SYSTEM) and np.all(it == 1)
    with pytest.raises(SingularSystemError):
        solve_coupled(cm, synthetic.make_lifted_mu(1)[0])


@pytest.mark.gpu
def test_timing_study_block_vs_coupled_scaling():
    """SPEC.md:630-638 timing_study examples on the device: block < coupled-3M at every M, and the coupled-3M time
    grows ≈ cubically in M (fitted exponent in [2.2, 3.5] over M ∈ {10, 20, 30, 50}; the dense LU of the
    (3M)-sized saddle system dominates)."""
    import torch

    from paper_1807_11866_b200 import online, study
    from paper_1807_11866_b200.coupled import solve_coupled_batch

    ms, tc = (10, 20, 30, 50), []
    for m in ms:
        cm, blk = synthetic.make_coupled_model(m, 12)
        mu = synthetic.make_lifted_mu(4096, seed=3)
        with online.DeviceModel(blk, 0) as dm:
            t = study.timing_study({"block": lambda x: dm.solve(x, pressure=False),
                                    "coupled": lambda x: solve_coupled_batch(cm, x.cpu().numpy())}, mu)
        assert t["block"] < t["coupled"], (m, t)
        tc.append(t["coupled"])
        torch.cuda.synchronize()
    slope = study.loglog_slope(ms, tc)
    print(f"coupled-3M ms/query {[round(x, 5) for x in tc]}, fitted exponent {slope:.2f}")
    assert 2.2 <= slope <= 3.5, slope
