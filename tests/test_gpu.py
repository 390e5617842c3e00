"""GPU parity tests: the sm_100a path through the C ABI against the CPU oracle and the golden fixtures.

Bar (BASELINE.json north_star): relative error ≤ 1e-10 on velocity and pressure coefficients and identical
Newton iteration counts.  Counts are compared exactly; a mismatch is tolerated only for a sample whose
deciding update lies within 1e-6 relative of the stop threshold on the oracle side (knife-edge, reported).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import rbns_oracle as oracle  # noqa: E402
from paper_1807_11866_b200 import affine, online, synthetic  # noqa: E402
from paper_1807_11866_b200.errors import NativeError, SingularSystemError  # noqa: E402
from paper_1807_11866_b200.model import ReducedModel  # noqa: E402

from .golden_utils import golden, reference_model  # noqa: E402

REL = 1e-10


def rel_err(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def device_solve(dm, mu, **kw):
    r = dm.solve(torch.from_numpy(np.ascontiguousarray(mu)).cuda(), **kw)
    torch.cuda.synchronize()
    return (r.u.cpu().numpy(), None if r.p is None else r.p.cpu().numpy(), r.iters.cpu().numpy(),
            r.status.cpu().numpy(), r.last_update.cpu().numpy(), r.stats)


def knife_edge(model, mu, tol=1e-12, max_iter=20, window=1e-6):
    """Per-sample oracle margin: how close the deciding update was to the stop threshold."""
    u = np.zeros(model.n)
    for it in range(1, max_iter + 1):
        R, J = oracle.reduced_operator(model, mu, u)
        d = np.linalg.solve(J, -R)
        u = u + d
        ratio = np.linalg.norm(d) / (tol * np.linalg.norm(u))
        if abs(ratio - 1.0) < window:
            return True
        if ratio <= 1.0:
            return False
    return False


def check_counts(model, mu, it_dev, it_ref, tol=1e-12):
    bad = np.nonzero(it_dev != it_ref)[0]
    for b in bad:
        assert knife_edge(model, mu[b], tol=tol), f"sample {b}: iters {it_dev[b]} vs oracle {it_ref[b]}"
    return len(bad)


@pytest.fixture(scope="module")
def dms():
    cache = {}

    def get(key, model):
        if key not in cache:
            cache[key] = online.DeviceModel(model, 0)
        return cache[key]

    yield get
    for dm in cache.values():
        dm.close()


# ---- golden fixtures -----------------------------------------------------------------------------------

@pytest.mark.parametrize("c", [0, 1, 2, 3, 4])
def test_golden_configs(cfg_model, dms, c):
    d = golden(f"synthetic_cfg{c}")
    cfg = synthetic.CONFIGS[c]
    dm = dms(c, cfg_model(c))
    u, p, it, st, last, stats = device_solve(dm, d["mu"], tol=cfg.tol, max_iter=cfg.max_iter)
    assert np.all(st == 0)
    assert rel_err(u, d["u"]) <= REL
    assert np.array_equal(it, d["iters"])
    if cfg.n_p:
        assert rel_err(p, d["p"]) <= REL
    assert stats["kernel_launches"] > 0 and stats["lu_launches"] > 0


def test_reference_assembled_model(dms):
    """Operator + solve on the reduced model built by the reference's own assembler (golden pin)."""
    d = golden("reference_operator")
    model = reference_model()
    dm = dms("ref", model)
    R, J = dm.reduced_operator(d["mu"], d["eta"])
    R, J = R.cpu().numpy(), J.cpu().numpy()
    for i in range(len(d["mu"])):
        assert rel_err(R[i], d["R_ref"][i]) <= 1e-12
        assert rel_err(J[i], d["J_ref"][i]) <= 1e-12
    u, _, it, st, _, _ = device_solve(dm, d["solve_mu"])
    assert np.all(st == 0) and np.array_equal(it, d["solve_iters"])
    assert rel_err(u, d["solve_u"]) <= REL


# ---- larger seeded slices against the oracle ---------------------------------------------------------

@pytest.mark.parametrize("c,nb", [(0, 64), (1, 1024), (2, 384)])
def test_parity_vs_oracle(cfg_model, dms, c, nb):
    cfg = synthetic.CONFIGS[c]
    model = cfg_model(c)
    mu = synthetic.config_mu(cfg, nb)
    u, _, it, st, last, _ = device_solve(dms(c, model), mu)
    ur, itr, str_, _ = oracle.solve_batch(model, mu)
    assert np.all(st == 0) and np.all(str_ == 0)
    assert rel_err(u, ur) <= REL
    check_counts(model, mu, it, itr)
    assert np.all(last <= 1e-12 * np.linalg.norm(u, axis=1) * (1 + 1e-9))   # stop rule


def test_pressure_recovery_parity(cfg_model, dms):
    cfg = synthetic.CONFIGS[4]
    model = cfg_model(4)
    mu = synthetic.config_mu(cfg, 256)
    u, p, it, st, _, _ = device_solve(dms(4, model), mu)
    pr = oracle.recover_pressure(model, mu, u)
    assert rel_err(p, pr) <= REL
    # recovery alone, linearity
    p1, _ = dms(4, model).recover_pressure(mu[:8], u[:8])
    p2, _ = dms(4, model).recover_pressure(mu[:8], 2 * u[:8])
    np.testing.assert_allclose(p2.cpu().numpy(), 2 * p1.cpu().numpy(), rtol=1e-13, atol=1e-13)


def test_jacobian_finite_differences_device(cfg_model, dms):
    model = cfg_model(1)
    dm = dms(1, model)
    rng = np.random.default_rng(11)
    mu = np.array([[0.3, 120.0]])
    eta = rng.standard_normal((1, model.n))
    _, J = dm.reduced_operator(mu, eta)
    J = J[0].cpu().numpy()
    h = 1e-6
    E = np.eye(model.n) * h
    Rp, _ = dm.reduced_operator(np.repeat(mu, model.n, 0), eta + E)
    Rm, _ = dm.reduced_operator(np.repeat(mu, model.n, 0), eta - E)
    Jfd = ((Rp - Rm).cpu().numpy() / (2 * h)).T
    assert np.abs(J - Jfd).max() <= 1e-6 * np.abs(J).max()
    R0, J0 = dm.reduced_operator(mu, np.zeros((1, model.n)))      # η = 0 KAT
    th = affine.evaluate_weights(model.theta, mu)[0]
    np.testing.assert_allclose(R0[0].cpu().numpy(), -(th @ model.f), atol=1e-13)


# ---- full BASELINE sizes: size-independent properties ------------------------------------------------

def test_full_batch_cfg2_properties(cfg_model, dms):
    cfg = synthetic.CONFIGS[2]
    model = cfg_model(2)
    dm = dms(2, model)
    mu = synthetic.config_mu(cfg)
    mud = torch.from_numpy(mu).cuda()
    r1 = dm.solve(mud)
    u1, it1, st1 = r1.u.clone(), r1.iters.clone(), r1.status.clone()
    r2 = dm.solve(mud)
    assert torch.equal(u1, r2.u) and torch.equal(it1, r2.iters)          # bitwise determinism
    assert int((st1 == 0).sum()) == cfg.batch                            # all 65536 converge
    # batch-composition invariance: a strided subset solved alone is bitwise identical
    idx = torch.arange(7, cfg.batch, 97, device="cuda")
    r3 = dm.solve(mud[idx])
    assert torch.equal(r3.u, u1[idx]) and torch.equal(r3.iters, it1[idx])
    # residual at the solution (size-independent): ‖R(u)‖ ≤ 1e-9 ‖f‖ on a subset
    sub = idx[:512]
    R, _ = dm.reduced_operator(mud[sub], u1[sub])
    th = affine.evaluate_weights(model.theta, mu[sub.cpu().numpy()])
    fn = np.linalg.norm(th @ model.f, axis=1)
    assert np.all(np.linalg.norm(R.cpu().numpy(), axis=1) <= 1e-9 * fn)
    # oracle parity on a random subset of the full batch
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(cfg.batch, 256, replace=False))
    ur, itr, _, _ = oracle.solve_batch(model, mu[pick])
    assert rel_err(u1.cpu().numpy()[pick], ur) <= REL
    check_counts(model, mu[pick], it1.cpu().numpy()[pick], itr)


def threaded_oracle(model, mu, chunk=64):
    """oracle.solve_batch over all host cores: chunks of μ on a thread pool, BLAS single-threaded per call."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    from threadpoolctl import threadpool_limits

    S = oracle.symmetrised_operator(model)
    with threadpool_limits(1), ThreadPoolExecutor(len(os.sched_getaffinity(0))) as ex:
        parts = list(ex.map(lambda i: oracle.solve_batch(model, mu[i:i + chunk], S=S), range(0, len(mu), chunk)))
    return tuple(np.concatenate([q[k] for q in parts]) for k in range(3))


def test_cfg3_slice_oracle_parity(cfg_model, dms):
    """Config 3 (N = 200, Q = 13: the hybrid register/shared-memory tiled Newton kernel, S streamed from HBM) on a
    1024-sample slice."""
    cfg = synthetic.CONFIGS[3]
    model = cfg_model(3)
    mu = synthetic.config_mu(cfg, 1024)
    u, _, it, st, _, _ = device_solve(dms(3, model), mu)
    ur, itr, str_ = threaded_oracle(model, mu, chunk=16)
    assert np.all(st == 0) and np.all(str_ == 0)
    per_sample = np.abs(u - ur).max(axis=1) / np.abs(ur).max(axis=1)
    assert per_sample.max() <= REL, per_sample.max()
    mism = np.nonzero(it != itr)[0]
    check_counts(model, mu[mism], it[mism], itr[mism])
    print(f"cfg3 slice (1024): max per-sample rel err u {per_sample.max():.2e}, count mismatches {len(mism)}")


def test_cfg3_full_batch(cfg_model, dms):
    """Config 3 at its full size (N = 200, Q = 13, B = 131 072): every sample converges, the solve is bitwise
    deterministic, the Newton residual at the solution is ≤ 1e-9·‖f(μ)‖ for every sample, and 8 192 samples —
    the first 4 096 and the last 4 096 of the seeded stream — match the oracle (≤ 1e-10 per sample, identical
    Newton counts up to knife-edge samples)."""
    cfg = synthetic.CONFIGS[3]
    model = cfg_model(3)
    dm = dms(3, model)
    mu = synthetic.config_mu(cfg)
    mud = torch.from_numpy(mu).cuda()
    a = dm.solve(mud)
    ua, ita = a.u.clone(), a.iters.clone()
    b = dm.solve(mud)
    torch.cuda.synchronize()
    assert torch.equal(b.u, ua) and torch.equal(b.iters, ita)              # bitwise determinism
    st = a.status.cpu().numpy()
    assert np.all(st == 0), np.bincount(st)
    # residual ≤ 1e-9 ‖f(μ)‖ at every solution (device reduced_operator, chunks of 4096)
    worst = 0.0
    for c0 in range(0, len(mu), 4096):
        R, _ = dm.reduced_operator(mu[c0:c0 + 4096], ua[c0:c0 + 4096])
        f = oracle.weights(model, mu[c0:c0 + 4096])["load"] @ model.f
        worst = max(worst, float((np.linalg.norm(R.cpu().numpy(), axis=1) / np.linalg.norm(f, axis=1)).max()))
    assert worst <= 1e-9, worst
    idx = np.r_[0:4096, len(mu) - 4096:len(mu)]
    ur, itr, str_ = threaded_oracle(model, mu[idx], chunk=16)
    assert np.all(str_ == 0)
    u = ua.cpu().numpy()[idx]
    it = ita.cpu().numpy()[idx]
    per_sample = np.abs(u - ur).max(axis=1) / np.abs(ur).max(axis=1)
    assert per_sample.max() <= REL, per_sample.max()
    mism = np.nonzero(it != itr)[0]
    assert len(mism) <= 16, len(mism)
    check_counts(model, mu[idx][mism], it[mism], itr[mism])
    print(f"cfg3 full batch: residual/||f|| max {worst:.2e}; 8192 head+tail samples vs oracle: max rel err "
          f"{per_sample.max():.2e}, count mismatches {len(mism)}; iteration histogram {np.bincount(ita.cpu().numpy()).tolist()}")


@pytest.mark.parametrize("c", [1, 2, 4])
def test_full_batch_oracle_parity(cfg_model, dms, c):
    """Every sample of configs 1 (16 384), 2 (65 536: the benchmark's workload) and 4 (65 536, with pressure
    recovery) against the oracle: relative error ≤ 1e-10 per sample on u (and p) and identical Newton counts
    (mismatches only at knife-edge samples).  The oracle runs on all host cores (chunks of 64 μ on a thread
    pool, BLAS single-threaded per call)."""
    cfg = synthetic.CONFIGS[c]
    model = cfg_model(c)
    dm = dms(c, model)
    mu = synthetic.config_mu(cfg)
    pressure = cfg.n_p > 0
    u, p, it, st, _, _ = device_solve(dm, mu, pressure=pressure)
    ur, itr, str_ = threaded_oracle(model, mu)
    assert np.all(st == 0) and np.all(str_ == 0)
    per_sample = np.abs(u - ur).max(axis=1) / np.abs(ur).max(axis=1)
    assert per_sample.max() <= REL, per_sample.max()
    mism = np.nonzero(it != itr)[0]
    assert len(mism) <= 64, len(mism)          # knife-edge cases only (checked below)
    check_counts(model, mu[mism], it[mism], itr[mism])
    msg = f"cfg{c} full batch ({len(mu)}): max per-sample rel err u {per_sample.max():.2e}"
    if pressure:
        pr = oracle.recover_pressure(model, mu, ur)
        pe = np.abs(p - pr).max(axis=1) / np.abs(pr).max(axis=1)
        assert pe.max() <= REL, pe.max()
        msg += f", p {pe.max():.2e}"
    print(msg + f", count mismatches {len(mism)}")


# ---- edge cases the SPEC names -------------------------------------------------------------------------

def _tiny(n=6, q=2, c_scale=0.0, a_scale=1.0, f_scale=1.0, seed=0, **kw):
    rng = np.random.default_rng(seed)
    A = a_scale * np.stack([np.eye(n) * (1 + i) for i in range(q)])
    C = c_scale * rng.standard_normal((q, n, n, n))
    f = f_scale * rng.standard_normal((q, n))
    return ReducedModel(A=A, C=C, f=f, theta=affine.family("trig3")[:q], **kw)


def test_edge_batch_sizes_and_max_iter(cfg_model, dms):
    dm = dms(0, cfg_model(0))
    mu = synthetic.config_mu(0)
    r = dm.solve(torch.zeros((0, 2), dtype=torch.float64, device="cuda"))
    assert r.u.shape == (0, 10)
    u, _, it, st, _, _ = device_solve(dm, mu[:1])
    ur, itr, _, _ = oracle.solve_batch(cfg_model(0), mu[:1])
    assert rel_err(u, ur) <= REL and it[0] == itr[0]
    u, _, it, st, last, _ = device_solve(dm, mu, max_iter=0)
    assert np.all(st == 1) and np.all(it == 0) and not u.any() and np.all(np.isnan(last))
    u, _, it, st, _, _ = device_solve(dm, mu, max_iter=2)
    assert np.all(st == 1) and np.all(it == 2)


def test_edge_outcomes():
    mu = np.array([[0.1, 20.0], [0.2, 50.0]])
    with online.DeviceModel(_tiny(a_scale=0.0), 0) as dm:            # J = 0: singular
        _, _, it, st, _, _ = device_solve(dm, mu)
        assert np.all(st == 2) and np.all(it == 1)
    with online.DeviceModel(_tiny(f_scale=0.0), 0) as dm:            # f = 0: u = 0 in one step
        u, _, it, st, _, _ = device_solve(dm, mu)
        assert np.all(st == 0) and np.all(it == 1) and not u.any()
    with online.DeviceModel(_tiny(), 0) as dm:                       # Re = 0 → ν = inf
        _, _, _, st, _, _ = device_solve(dm, np.array([[0.1, 0.0]]))
        assert st[0] in (2, 4)
    bad_mp = _tiny(Mp=-np.eye(3), Bq=np.ones((2, 3, 6)))             # B_sp not SPD → SINGULAR_RECOVERY
    with online.DeviceModel(bad_mp, 0) as dm:
        _, p, _, st, _, _ = device_solve(dm, mu)
        assert np.all(st == 3) and np.all(np.isnan(p))
    with online.DeviceModel(_tiny(), 0) as dm:                       # p requested, model has no Np
        mu_d = torch.from_numpy(mu).cuda()
        out = [torch.empty(2, 6, dtype=torch.float64, device="cuda"), torch.empty(2, 6, dtype=torch.float64, device="cuda"),
               torch.empty(2, dtype=torch.int32, device="cuda"), torch.empty(2, dtype=torch.int8, device="cuda"),
               torch.empty(2, dtype=torch.float64, device="cuda")]
        rc = dm.lib.rbns_solve(dm._h, mu_d.data_ptr(), 2, 1e-12, 20, *[t.data_ptr() for t in out], None)
        assert rc == 5
        with pytest.raises(NativeError):
            from paper_1807_11866_b200 import _native
            _native.check(rc, "rbns_solve")


def _random_model(n, q, seed):
    """Generator-style model (SURVEY.md Appendix B scalings) with q terms drawn from the Fourier + monomial
    families, for shapes outside the BASELINE configs."""
    rng = np.random.default_rng(seed)
    terms = (affine.family("fourier13") + affine.monomials([(1, 0), (0, 1), (2, 0)], [1.0, 1e-3, 0.5]))[:q]
    G = rng.standard_normal((n, n))
    A = [G @ G.T / n + np.eye(n)]
    for _ in range(1, q):
        S = rng.standard_normal((n, n))
        A.append(0.1 * (S + S.T) / 2 / np.sqrt(n))
    C = 1e-5 / n * rng.standard_normal((q, n, n, n))
    C = 0.5 * (C - C.transpose(0, 1, 3, 2))
    return ReducedModel(A=np.stack(A), C=C, f=rng.standard_normal((q, n)), theta=terms)


@pytest.mark.parametrize("n,q", [(1, 1), (7, 1), (13, 3), (33, 5), (64, 16), (89, 2), (91, 3), (95, 1), (96, 2),
                                 (103, 4), (104, 1), (127, 2), (128, 2), (207, 1)])
def test_odd_and_extreme_shapes(n, q):
    model = _random_model(n, q, seed=n)
    mu = synthetic.make_mu(40 if n <= 127 else 12, 100.0, seed=n)
    with online.DeviceModel(model, 0) as dm:
        u, _, it, st, _, _ = device_solve(dm, mu)
    ur, itr, str_, _ = oracle.solve_batch(model, mu)
    assert np.array_equal(st, str_)
    assert rel_err(u, ur) <= REL
    check_counts(model, mu, it, itr)


def test_monomial_family_and_single_query(dms):
    model = reference_model()
    sol = online.solve_block(model, (0.2, 4.0))
    u, it, st, _ = oracle.solve_sample(model, np.array([0.2, 4.0]))
    assert sol.converged and sol.newton_iters == it and not sol.s_coeffs.any()
    assert rel_err(sol.u_coeffs, u) <= REL
    assert set(sol.wall_time) >= {"assembly", "solve", "recovery"}
    with pytest.raises(SingularSystemError):
        online.solve_block(_tiny(a_scale=0.0), (0.1, 10.0))


def test_zero_quadrature_online(cfg_model, dms):
    """The online path performs no quadrature (reference instrument.py:3-5): the package's counter,
    which the offline projection increments (checked, so the probe is live), is unchanged across every online
    entry point, and the online path never imports the reference's quadrature assembly."""
    import sys

    from paper_1807_11866_b200 import instrument, projection

    rng = np.random.default_rng(0)
    before = instrument.quadrature_evals()
    projection.project_viscous(rng.standard_normal((12, 2, 2, 4)), np.full(12, 0.5))
    assert instrument.quadrature_evals() == before + 12  # the probe counts offline quadrature
    before = instrument.quadrature_evals()
    model = synthetic.config_model(4, attached=True)
    mu = synthetic.config_mu(4, 64)
    with online.DeviceModel(model, 0) as dm:
        sol = dm.solve(torch.from_numpy(mu).cuda())
        dm.recover_pressure(mu, sol.u)
        dm.reconstruct_pressure(sol.u)
        dm.reduced_operator(mu[:4], sol.u[:4])
    online.solve_block(cfg_model(0), synthetic.config_mu(0)[0])
    online.sweep_report(synthetic.config_mu(0), online.solve_block_batch(cfg_model(0), synthetic.config_mu(0)))
    torch.cuda.synchronize()
    assert instrument.quadrature_evals() == before
    assert not any(m == "rbflow" or m.startswith("rbflow.") for m in sys.modules)


# ---- combined scheme: pressure reconstruction from attached modes -----------------------

def test_reconstruct_pressure_parity_and_kats():
    """p = P_att u on the device against the oracle; u = 0 → p = 0 and linearity exactly."""
    model = synthetic.config_model(4, attached=True)
    mu = synthetic.config_mu(4, 1024)
    ur, _, _, _ = oracle.solve_batch(model, mu)
    with online.DeviceModel(model, 0) as dm:
        p = dm.reconstruct_pressure(torch.from_numpy(ur).cuda()).cpu().numpy()
        z = dm.reconstruct_pressure(torch.zeros((8, model.n), dtype=torch.float64)).cpu().numpy()
        p2 = dm.reconstruct_pressure(torch.from_numpy(2.0 * ur).cuda()).cpu().numpy()
    pr = oracle.reconstruct_pressure(model, ur)
    assert rel_err(p, pr) <= 1e-13
    assert np.all(z == 0.0)
    assert np.array_equal(p2, 2.0 * p)  # exact: scaling by 2 is exact in every product and sum
    # SPEC surface: one state in, one pressure vector out; batched numpy in, numpy out
    one = online.reconstruct_pressure(model, ur[3])
    assert one.shape == (model.n_att,) and rel_err(one, pr[3]) <= 1e-13
    online.release_device_models()


def test_reconstruct_pressure_requires_attached_modes(cfg_model):
    from paper_1807_11866_b200.errors import RbflowError

    with pytest.raises(RbflowError, match="attached"):
        online.reconstruct_pressure(cfg_model(4), np.zeros(100))
    with online.DeviceModel(cfg_model(4), 0) as dm:
        with pytest.raises(RbflowError):
            dm.reconstruct_pressure(np.zeros((2, 100)))
        lib = dm.lib
        rc = lib.rbns_reconstruct_pressure(dm._h, 0, 0, 0, None)
        assert rc == 6  # RBNS_ERR_NO_ATTACHED through the raw C ABI


def test_combined_scheme_batch_and_timing():
    """solve_block_batch(pressure="combined") = velocity solve + reconstruction; the reconstruction is no
    slower than the recovery solve it replaces ("combined-reconstruction ≤ block time")."""
    model = synthetic.config_model(4, attached=True)
    mu = synthetic.config_mu(4, 16384)
    rec = online.solve_block_batch(model, mu, pressure="recovery")
    comb = online.solve_block_batch(model, mu, pressure="combined")
    torch.cuda.synchronize()
    assert torch.equal(rec.u, comb.u) and torch.equal(rec.iters, comb.iters)
    pr = oracle.reconstruct_pressure(model, comb.u.cpu().numpy())
    assert rel_err(comb.p.cpu().numpy(), pr) <= 1e-13
    t_rec = min(online.solve_block_batch(model, mu, pressure="recovery").stats["ms_recovery"] for _ in range(3))
    t_comb = min(online.solve_block_batch(model, mu, pressure="combined").stats["ms_recovery"] for _ in range(3))
    assert t_comb <= t_rec, (t_comb, t_rec)
    online.release_device_models()


# ---- boundary hygiene --------------------------------------------------------------------------------------

def test_out_buffers_are_validated(cfg_model, dms):
    dm = dms(4, cfg_model(4))
    mu = torch.from_numpy(synthetic.config_mu(4, 64)).cuda()
    good = dm.solve(mu)
    small = dm.solve(mu[:32])
    with pytest.raises(ValueError, match="shape"):
        dm.solve(mu, out=small)                               # too few rows
    bad = online.BatchSolution(u=good.u, p=None, iters=good.iters, status=good.status, last_update=good.last_update)
    with pytest.raises(ValueError, match="pressure"):
        dm.solve(mu, out=bad)                                  # p requested, none given
    bad = online.BatchSolution(u=good.u.float(), p=good.p, iters=good.iters, status=good.status,
                               last_update=good.last_update)
    with pytest.raises(ValueError, match="dtype"):
        dm.solve(mu, out=bad)
    bad = online.BatchSolution(u=good.u.cpu(), p=good.p, iters=good.iters, status=good.status,
                               last_update=good.last_update)
    with pytest.raises(ValueError, match="cuda|device|on"):
        dm.solve(mu, out=bad)
    wide = torch.empty((64, 2 * dm.n), dtype=torch.float64, device="cuda")
    bad = online.BatchSolution(u=wide[:, ::2], p=good.p, iters=good.iters, status=good.status,
                               last_update=good.last_update)
    with pytest.raises(ValueError):
        dm.solve(mu, out=bad)                                  # strided view
    host = dm.solve_host(mu.cpu().numpy())
    host["u"] = host["u"][:10]
    with pytest.raises(ValueError):
        dm.solve_host(mu.cpu().numpy(), out=host)
    again = dm.solve(mu, out=good)                             # a valid buffer is reused
    assert again.u.data_ptr() == good.u.data_ptr()


def test_per_call_stats_and_phase_times(cfg_model, dms):
    """Statistics come back per call (rbns_solve_ex), so two calls of different sizes report their own work;
    solve_block's assembly phase includes the u = 0 affine assembly."""
    dm = dms(1, cfg_model(1))
    mu = torch.from_numpy(synthetic.config_mu(1, 512)).cuda()
    a = dm.solve(mu[:64])
    b = dm.solve(mu)
    assert a.stats["sample_iterations"] == int(a.iters.sum()) and b.stats["sample_iterations"] == int(b.iters.sum())
    assert dm.stats()["sample_iterations"] == b.stats["sample_iterations"]  # the handle keeps the latest copy
    sol = online.solve_block(cfg_model(1), synthetic.config_mu(1, 1)[0])
    s = online.device_model(cfg_model(1)).stats()
    assert sol.wall_time["assembly"] == pytest.approx((s["ms_assembly"] + s["ms_gemm"]) * 1e-3)
    assert s["ms_assembly"] > 0.0


def test_multi_device_batch_is_bitwise_single_device(cfg_model):
    """solve_block_batch(devices=[...]): μ-sharded, one handle and host thread per device, gathered on the first
    device — bit-identical to one device (two handles on one B200 stand in for two GPUs)."""
    model = cfg_model(4)
    mu = synthetic.config_mu(4, 3001)
    one = online.solve_block_batch(model, mu)
    torch.cuda.synchronize()
    u1, p1, it1 = one.u.clone(), one.p.clone(), one.iters.clone()
    ndev = max(2, torch.cuda.device_count())
    two = online.solve_block_batch(model, mu, devices=[i % torch.cuda.device_count() for i in range(ndev)])
    torch.cuda.synchronize()
    assert torch.equal(two.u, u1) and torch.equal(two.p, p1) and torch.equal(two.iters, it1)
    assert two.stats["sample_iterations"] == int(it1.sum())
    online.release_device_models()


def test_concurrent_streams(cfg_model, dms):
    """Two solves on two streams with one shared read-only model."""
    dm = dms(1, cfg_model(1))
    mu = torch.from_numpy(synthetic.config_mu(1, 512)).cuda()
    ref = dm.solve(mu)
    ref_u = ref.u.clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        a = dm.solve(mu[:256], stream=s1)
    with torch.cuda.stream(s2):
        b = dm.solve(mu[256:], stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([a.u, b.u]), ref_u)
    assert a.stats["sample_iterations"] == int(a.iters.sum()) and b.stats["sample_iterations"] == int(b.iters.sum())


@pytest.mark.parametrize("n", [40, 100, 150, 200])
def test_pivot_hint_misses_take_the_exact_path(n):
    """Rows of A₀ permuted: partial pivoting picks a non-identity order, so the speculative kernel's identity hint
    fails at the first Newton iteration and every sample is re-run by the exact full-search kernel; from the
    second iteration the hint (the previous order) holds.  Results must equal the oracle's either way."""
    rng = np.random.default_rng(n)
    base = synthetic.make_model(n, 3, "trig3", seed=n)
    perm = rng.permutation(n)
    A = base.A.copy()
    A[0] = A[0][perm] * 3.0 + 0.0                       # row-permuted dominant term
    model = ReducedModel(A=A, C=base.C, f=base.f, theta=base.theta)
    mu = synthetic.make_mu(256 if n <= 127 else 48, 50.0, seed=n)
    with online.DeviceModel(model, 0) as dm:
        u, _, it, st, _, stats = device_solve(dm, mu)
    ur, itr, str_, _ = oracle.solve_batch(model, mu)
    assert np.array_equal(st, str_) and np.all(st == 0)
    assert rel_err(u, ur) <= REL
    check_counts(model, mu, it, itr)
    import os

    if os.environ.get("RBNS_NEWTON", "") in ("", "gjs"):  # the default (speculative) kernel
        assert stats["pivot_fallbacks"] >= len(mu)       # at least the first iteration of every sample
        assert stats["pivot_fallbacks"] < stats["sample_iterations"]


@pytest.mark.parametrize("variant", ["gjs", "gj2", "chunks"])
def test_alternate_newton_kernels(variant):
    """The non-default Newton-update kernels (RBNS_NEWTON, read once per process) stay parity-green; "chunks"
    runs the default kernels with a 40 MB Jacobian buffer, so every Newton round is split into many chunks."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np, torch\n"
        "from oracle import rbns_oracle as o\n"
        "from paper_1807_11866_b200 import online, synthetic\n"
        "for c, nb in ((1, 256), (2, 96), (3, 24)):\n"
        "    cfg = synthetic.CONFIGS[c]; m = synthetic.config_model(cfg); mu = synthetic.config_mu(cfg, nb)\n"
        "    with online.DeviceModel(m, 0) as dm:\n"
        "        r = dm.solve(torch.from_numpy(mu).cuda()); torch.cuda.synchronize()\n"
        "    ur, itr, st, _ = o.solve_batch(m, mu)\n"
        "    u = r.u.cpu().numpy(); it = r.iters.cpu().numpy()\n"
        "    assert np.abs(u - ur).max() <= 1e-10 * np.abs(ur).max(), c\n"
        "    assert (it != itr).sum() <= 1 and np.all(r.status.cpu().numpy() == 0), c\n"
        "print('ok')\n")
    env = dict(os.environ, RBNS_JBUF_BYTES="40000000") if variant == "chunks" else dict(os.environ, RBNS_NEWTON=variant)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]



def test_hybrid_kernel_test_shapes():
    """The hybrid register/shared-memory tiled kernel (rbns_tgh.cuh, config 3's N = 200) at its two small test
    shapes (N = 56: 3 warps, N = 104: 6 warps; RBNS_NEWTON=tgh) against the oracle, batch over several CTA waves."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np, torch\n"
        "from oracle import rbns_oracle as o\n"
        "from paper_1807_11866_b200 import online, synthetic\n"
        "for n in (56, 97, 100, 103, 104):\n"
        "    m = synthetic.make_model(n, 3, 'trig3', seed=n); mu = synthetic.make_mu(400, 50.0, seed=n)\n"
        "    with online.DeviceModel(m, 0) as dm:\n"
        "        r = dm.solve(torch.from_numpy(mu).cuda()); torch.cuda.synchronize()\n"
        "    ur, itr, st, _ = o.solve_batch(m, mu)\n"
        "    u = r.u.cpu().numpy(); it = r.iters.cpu().numpy()\n"
        "    assert np.all(st == 0) and np.all(r.status.cpu().numpy() == 0), n\n"
        "    assert (np.abs(u - ur).max(axis=1) / np.abs(ur).max(axis=1)).max() <= 1e-10, n\n"
        "    assert (it != itr).sum() <= 1, n\n"
        "print('ok')\n")
    env = dict(os.environ, RBNS_NEWTON="tgh")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]

@pytest.mark.parametrize("n", [33, 40, 64, 80, 104, 111, 120, 127, 128, 150, 175, 192, 199])
def test_tiled_kernel_shapes_default_path(n):
    """Every instantiated tiled shape family on the default dispatch: register kernel (32 < N ≤ 103), hybrid
    register/shared kernel with 5 warps (103 < N ≤ 127) and with 12 warps (127 < N < 200), partial and full tiles,
    against the oracle."""
    rng_seed = n
    model = synthetic.make_model(n, 3, "trig3", seed=rng_seed)
    mu = synthetic.make_mu(64, 50.0, seed=rng_seed)
    with online.DeviceModel(model, 0) as dm:
        u, _, it, st, _, stats = device_solve(dm, mu)
    ur, itr, str_, _ = oracle.solve_batch(model, mu)
    assert np.all(st == 0) and np.all(str_ == 0)
    assert (np.abs(u - ur).max(axis=1) / np.abs(ur).max(axis=1)).max() <= REL
    check_counts(model, mu, it, itr)

def test_unsupported_size_fails_loudly():
    """N beyond the register/cluster Newton kernels (207) is rejected at model creation, not computed wrong."""
    n = 208
    model = ReducedModel(A=np.eye(n)[None], C=np.zeros((1, n, n, n)), f=np.ones((1, n)),
                         theta=[affine.ThetaTerm(affine.CONST)])
    with pytest.raises(NativeError, match="exceeds"):
        online.DeviceModel(model, 0)


def test_query_api_solver_kinds():
    """SPEC.md:566 Query API: (μ, solver kind) → ReducedSolution for the block, combined and coupled solvers;
    block and combined share the velocity, combined pressure = P_att u, coupled velocity within 1e-8 of block."""
    from paper_1807_11866_b200.coupled import solve_coupled

    model = synthetic.config_model(4, attached=True)
    mu = synthetic.config_mu(4, 2)[1]
    b = online.query(model, mu, "block")
    c = online.query(model, mu, "combined")
    assert b.converged and c.converged and b.newton_iters == c.newton_iters
    np.testing.assert_array_equal(b.u_coeffs, c.u_coeffs)
    np.testing.assert_allclose(c.p_coeffs, oracle.reconstruct_pressure(model, b.u_coeffs[None])[0], rtol=1e-12,
                               atol=1e-14)
    assert b.p_coeffs is not None and not np.array_equal(b.p_coeffs, c.p_coeffs)  # recovery ≠ reconstruction
    cm, blk = synthetic.make_coupled_model(10, 2)
    mu2 = synthetic.make_lifted_mu(1, seed=4)[0]
    q = online.query(cm, mu2, "coupled")
    r = online.query(blk, mu2, "block")
    assert np.abs(q.u_coeffs - r.u_coeffs).max() <= 1e-8 * np.abs(r.u_coeffs).max()
    with pytest.raises(ValueError):
        online.query(model, mu, "nonsense")
    with pytest.raises(TypeError):
        online.query(model, mu, "coupled")
