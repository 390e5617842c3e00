"""Models with the paper's per-form term families: a + c0 linear terms, c quadratic terms,
d0 u∞¹/u∞² loads, μ = (φ, u∞), ν in the descriptors.

CPU tests pin the oracle and the model contract; ``gpu`` tests run the CUDA path through the C ABI
(rbns_model_create2) against the oracle and the committed fixtures (same bar as test_gpu.py).
"""

import numpy as np
import pytest

from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import affine, synthetic
from paper_1807_11866_b200.model import ReducedModel

from .golden_utils import golden

LIFTED = {"lifted_small": dict(n=12, series=2, n_p=6), "lifted_n12": dict(n=50, series=12, n_p=0)}


def lifted(name):
    spec = LIFTED[name]
    return synthetic.make_lifted_model(spec["n"], spec["series"], n_p=spec["n_p"])


def checksums(model):
    out = []
    for arr in (model.A, model.C, model.f, model.Mp, model.Bq):
        out += [0.0, 0.0] if arr is None else [float(arr.sum()), float((arr * arr).sum())]
    return np.array(out)


# ---- CPU: model contract and oracle --------------------------------------------------------------------

def test_family_structure():
    m = lifted("lifted_n12")
    n = 12
    assert m.counts == (4 * n + 3 + 4 * n + 1, 4 * n + 1, 4 * n + 3 + 4 * n + 1, 0)
    assert not m.nu_linear and not m.shared_theta
    # a-terms carry ν = 1/6; c0 terms are linear in u∞ (m = 1)
    assert m.theta_linear[0].scale == pytest.approx(1 / 6) and m.theta_linear[0].m == 0
    assert all(t.m == 1 for t in m.theta_linear[4 * n + 3:])
    # d0 lift-lift family at u∞ = 20 is 400x its value at u∞ = 1
    w1 = affine.evaluate_weights(m.theta_load, np.array([[0.3, 1.0]]))[0]
    w20 = affine.evaluate_weights(m.theta_load, np.array([[0.3, 20.0]]))[0]
    np.testing.assert_allclose(w20[4 * n + 3:], 400 * w1[4 * n + 3:], rtol=1e-14)
    np.testing.assert_allclose(w20[:4 * n + 3], 20 * w1[:4 * n + 3], rtol=1e-14)


def test_family_validation():
    m = lifted("lifted_small")
    with pytest.raises(ValueError, match="linear terms"):
        ReducedModel(A=m.A, C=m.C, f=m.f, theta_linear=m.theta_linear[:-1], theta_quadratic=m.theta_quadratic,
                     theta_load=m.theta_load)
    with pytest.raises(ValueError, match="quadratic terms"):
        ReducedModel(A=m.A, C=m.C, f=m.f, theta_linear=m.theta_linear, theta_load=m.theta_load)
    with pytest.raises(ValueError, match="at least one"):
        ReducedModel(A=m.A[:0], C=m.C, f=m.f, theta_linear=(), theta_quadratic=m.theta_quadratic,
                     theta_load=m.theta_load)
    # a shared list still works for every family of equal size
    k = ReducedModel(A=m.A[:3], C=m.C[:3], f=m.f[:3], theta=m.theta_quadratic[:3])
    assert k.shared_theta and k.nu_linear


@pytest.mark.parametrize("name", sorted(LIFTED))
def test_lifted_golden_oracle(name):
    d = golden(name)
    m = lifted(name)
    np.testing.assert_allclose(checksums(m), d["checksums"], rtol=1e-12)
    for b in range(min(8, len(d["mu"]))):
        u, it, st, last = oracle.solve_sample(m, d["mu"][b])
        assert st == 0 and it == d["iters"][b]
        np.testing.assert_allclose(u, d["u"][b], rtol=0, atol=1e-12 * np.abs(d["u"][b]).max())


def test_lifted_oracle_paths_agree():
    m = lifted("lifted_small")
    mu = synthetic.make_lifted_mu(64)
    ub, itb, stb, _ = oracle.solve_batch(m, mu)
    d = golden("lifted_small")
    assert np.all(stb == 0) and np.array_equal(itb, d["iters"])
    assert np.abs(ub - d["u"]).max() <= 1e-12 * np.abs(d["u"]).max()
    np.testing.assert_allclose(oracle.recover_pressure(m, mu, ub), d["p"], rtol=1e-11, atol=1e-12)


def test_lifted_operator_identities():
    """η = 0 KAT (residual = −loads, Jacobian = linear blocks) and the FD Jacobian."""
    m = lifted("lifted_small")
    mu = np.array([0.4, 7.0])
    w = oracle.weights(m, mu[None])
    R, J = oracle.reduced_operator(m, mu, np.zeros(m.n))
    np.testing.assert_allclose(R, -(w["load"][0] @ m.f), atol=1e-14)
    np.testing.assert_allclose(J, np.einsum("a,aij->ij", w["linear"][0], m.A), atol=1e-14)
    eta = np.random.default_rng(3).standard_normal(m.n) * 50
    _, J = oracle.reduced_operator(m, mu, eta)
    h = 1e-6 * np.abs(eta).max()
    fd = np.empty_like(J)
    for j in range(m.n):
        e = np.zeros(m.n)
        e[j] = h
        fd[:, j] = (oracle.reduced_operator(m, mu, eta + e)[0] - oracle.reduced_operator(m, mu, eta - e)[0]) / (2 * h)
    assert np.abs(fd - J).max() <= 1e-6 * np.abs(J).max()


# ---- GPU: the CUDA path through rbns_model_create2 ----------------------------------------------------

@pytest.fixture(scope="module")
def dmodels():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1807_11866_b200 import online

    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = online.DeviceModel(lifted(name), 0)
        return cache[name]

    yield get
    for dm in cache.values():
        dm.close()


def _solve(dm, mu, **kw):
    import torch

    r = dm.solve(torch.from_numpy(np.ascontiguousarray(mu)).cuda(), **kw)
    torch.cuda.synchronize()
    return (r.u.cpu().numpy(), None if r.p is None else r.p.cpu().numpy(), r.iters.cpu().numpy(),
            r.status.cpu().numpy())


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.gpu
def test_lifted_term_plan(dmodels):
    """a-terms tie to the c-blocks (μ₁⁰), c0 terms too (μ₁¹): two h groups; a-terms φ^{4n+1}, φ^{4n+2} have
    no c-block and become the two extra contraction blocks."""
    n = 12
    plan = dmodels("lifted_n12").terms()
    assert plan == {"linear": 8 * n + 4, "quadratic": 4 * n + 1, "load": 8 * n + 4, "coupling": 0,
                    "blocks": 4 * n + 3, "groups": 2}
    assert dmodels("lifted_small").terms()["coupling"] == 4 * 2 + 1


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(LIFTED))
def test_lifted_golden_device(dmodels, name):
    d = golden(name)
    u, p, it, st = _solve(dmodels(name), d["mu"], pressure=LIFTED[name]["n_p"] > 0)
    assert np.all(st == 0)
    assert _rel(u, d["u"]) <= 1e-10
    assert np.array_equal(it, d["iters"])
    if LIFTED[name]["n_p"]:
        assert _rel(p, d["p"]) <= 1e-10


@pytest.mark.gpu
def test_lifted_parity_batch(dmodels):
    from .test_gpu import check_counts

    m = lifted("lifted_n12")
    mu = synthetic.make_lifted_mu(1024, seed=5)
    u, _, it, st = _solve(dmodels("lifted_n12"), mu)
    ur, itr, str_, _ = oracle.solve_batch(m, mu)
    assert np.all(st == 0) and np.all(str_ == 0)
    assert _rel(u, ur) <= 1e-10
    check_counts(m, mu, it, itr)


@pytest.mark.gpu
def test_lifted_reduced_operator_device(dmodels):
    m = lifted("lifted_small")
    dm = dmodels("lifted_small")
    rng = np.random.default_rng(11)
    mu = synthetic.make_lifted_mu(16, seed=9)
    eta = rng.standard_normal((16, m.n)) * 30
    R, J = dm.reduced_operator(mu, eta)
    R, J = R.cpu().numpy(), J.cpu().numpy()
    for b in range(16):
        Rr, Jr = oracle.reduced_operator(m, mu[b], eta[b])
        assert _rel(R[b], Rr) <= 1e-12 and _rel(J[b], Jr) <= 1e-12


@pytest.mark.gpu
def test_weight_consistency_phi0_device(dmodels):
    """SPEC.md:508 weight consistency: the residual (and Jacobian) at μ = (φ, u∞) = (0, 1) equals that of the
    model restricted to its φ⁰ terms (every other monomial vanishes there), to 1e-13 — on the device."""
    from paper_1807_11866_b200 import online

    m = lifted("lifted_small")
    keep = {fam: [i for i, t in enumerate(getattr(m, f"theta_{fam}")) if t.k == 0]
            for fam in ("linear", "quadratic", "load")}
    m0 = ReducedModel(A=m.A[keep["linear"]], C=m.C[keep["quadratic"]], f=m.f[keep["load"]],
                      theta_linear=[m.theta_linear[i] for i in keep["linear"]],
                      theta_quadratic=[m.theta_quadratic[i] for i in keep["quadratic"]],
                      theta_load=[m.theta_load[i] for i in keep["load"]], nu_linear=m.nu_linear)
    mu = np.array([[0.0, 1.0]] * 4)
    eta = np.random.default_rng(5).standard_normal((4, m.n)) * 20
    R, J = dmodels("lifted_small").reduced_operator(mu, eta)
    with online.DeviceModel(m0, 0) as dm0:
        R0, J0 = dm0.reduced_operator(mu, eta)
    R, J, R0, J0 = (x.cpu().numpy() for x in (R, J, R0, J0))
    assert _rel(R, R0) <= 1e-13 and _rel(J, J0) <= 1e-13
