"""Affine-term compression (model.compress_affine / affine.dependence): linearly dependent coefficient functions
of a family are merged, X'_i = Σ_q coef[q,i] X_q — an exact rewrite of the affine sums, so the
reduced residual and Jacobian are unchanged up to round-off."""

import numpy as np
import pytest

from paper_1807_11866_b200 import affine, synthetic


def test_trig7_relations_are_found_exactly():
    basis, coef = affine.dependence(affine.family("trig7"))
    assert basis == [0, 1, 2, 3, 5]                      # 1, cos, sin, cos², sin·cos
    assert coef[4].tolist() == [1.0, 0.0, 0.0, -1.0, 0.0]  # sin² = 1 − cos²
    assert coef[6].tolist() == [-1.0, 0.0, 0.0, 2.0, 0.0]  # cos 2α = 2cos² − 1


@pytest.mark.parametrize("fam", ["trig3", "fourier13"])
def test_independent_families_are_left_alone(fam):
    m = synthetic.make_model(6, len(affine.family(fam)), fam, seed=1)
    assert m.compress_affine() is m
    mono = affine.monomials([(k, m_) for k in range(4) for m_ in range(2)])
    assert affine.dependence(mono)[0] == list(range(8))


def test_compressed_operator_matches():
    from oracle import rbns_oracle as oracle

    m = synthetic.make_model(12, 7, "trig7", seed=3, n_p=5)
    mc = m.compress_affine()
    assert mc.C.shape[0] == 5 and mc.A.shape[0] == 5 and mc.f.shape[0] == 5 and mc.Bq.shape[0] == 5
    mu = synthetic.make_mu(16, 200.0, seed=5)
    rng = np.random.default_rng(0)
    for b in range(len(mu)):
        u = 0.3 * rng.standard_normal(12)
        R1, J1 = oracle.reduced_operator(m, mu[b], u)
        R2, J2 = oracle.reduced_operator(mc, mu[b], u)
        assert np.abs(R1 - R2).max() <= 1e-14 * np.abs(R1).max()
        assert np.abs(J1 - J2).max() <= 1e-14 * np.abs(J1).max()
    p1 = oracle.recover_pressure(m, mu, np.ones((len(mu), 12)))
    p2 = oracle.recover_pressure(mc, mu, np.ones((len(mu), 12)))
    assert np.abs(p1 - p2).max() <= 1e-13 * np.abs(p1).max()


def test_compressed_model_store_round_trip(tmp_path):
    from paper_1807_11866_b200 import store

    mc = synthetic.make_model(8, 7, "trig7", seed=2).compress_affine()
    m2 = store.load_model(store.save_model(mc, tmp_path / "c"))
    assert np.array_equal(m2.C, mc.C) and m2.theta_quadratic == mc.theta_quadratic


@pytest.mark.gpu
def test_gpu_compressed_solve_matches():
    """Config 2 slice: the compressed model (Q 7 → 5) solves to the same u as the uncompressed one (≤ 1e-12
    relative, identical counts up to knife-edge samples) and as the oracle on the original model."""
    import torch

    from oracle import rbns_oracle as oracle
    from paper_1807_11866_b200 import online

    from .test_gpu import check_counts

    cfg = synthetic.CONFIGS[2]
    m = synthetic.config_model(cfg)
    mc = m.compress_affine()
    mu = synthetic.config_mu(cfg, 1024)
    res = []
    for model in (m, mc):
        with online.DeviceModel(model, 0) as dm:
            r = dm.solve(torch.from_numpy(mu).cuda(), pressure=False)
            torch.cuda.synchronize()
            res.append((r.u.cpu().numpy(), r.iters.cpu().numpy(), r.status.cpu().numpy()))
    (u1, it1, st1), (u2, it2, st2) = res
    assert np.all(st1 == 0) and np.all(st2 == 0)
    assert (np.abs(u1 - u2).max(axis=1) / np.abs(u1).max(axis=1)).max() <= 1e-12
    mism = np.nonzero(it1 != it2)[0]
    check_counts(m, mu[mism], it2[mism], it1[mism])
    ur, itr, _, _ = oracle.solve_batch(m, mu)
    assert (np.abs(u2 - ur).max(axis=1) / np.abs(ur).max(axis=1)).max() <= 1e-10
