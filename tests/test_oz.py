"""The INT8-sliced contraction (csrc/rbns_oz.cuh): the splitting's arithmetic on the CPU (numpy restatement of
`digits`, exact rational reference) and, on the GPU, the tcgen05 kernel bit for bit against the host emulation
(tools/oz_probe.cu), the sliced path against the FP64 DMMA path on the same models, and the path switch."""

import os
import subprocess
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
KS = 8                                              # RBNS_OZ_SLICES
BAL = 0x0080808080808080                            # 0x80 in every byte below the top one (rbns_oz.cuh kBal)


def digits(v, ks=KS):
    """numpy restatement of rbns::oz::digits: F = rint(v·2^(8s-1)), balanced radix-256 digits = bytes of
    (F + C) xor C; returns the digits (most significant first) and the rounding remainder in units of 2^-(8s-1)."""
    assert ks == 8
    v = np.asarray(v, dtype=np.float64)
    f = v * 2.0 ** 63
    F = np.rint(f)
    rem = f - F
    t = (F.astype(np.int64).astype(np.uint64) + np.uint64(BAL)) ^ np.uint64(BAL)
    out = [((t >> np.uint64(8 * (ks - 1 - i))) & np.uint64(0xFF)).astype(np.uint8).view(np.int8).astype(np.float64)
           for i in range(ks)]
    return np.array(out), rem


def slice_row(v, ks=KS):
    m = np.abs(v).max()
    if m == 0.0:
        return np.zeros((ks, len(v))), 0.0
    e = int(np.floor(np.log2(m))) + 1
    assert 2.0 ** (e - 1) <= m < 2.0 ** e
    d, _ = digits(np.ldexp(v, -(e + 1)), ks)
    return d, np.ldexp(1.0, e - 6)


def test_digits_are_bytes_and_exact():
    rng = np.random.default_rng(0)
    v = rng.uniform(-0.5, 0.5, 400_000)
    v[::3] *= 1e-6
    v[::7] *= 1e-12
    edge = np.array([0.0, 0.5 - 2.0 ** -54, -0.5 + 2.0 ** -54, 127.0 / 255.0 / 128.0, 2.0 ** -64, 2.0 ** -60,
                     -(2.0 ** -60), 0.25, -0.25, 1.0 / 3.0, -1.0 / 3.0])
    v = np.concatenate([v, edge])
    d, r = digits(v)
    assert d[0].min() >= -64 and d[0].max() <= 64
    assert d.min() >= -128 and d.max() <= 127
    assert np.all(np.abs(r) <= 0.5)
    # exact reconstruction: v = Σ d_i 2^{-7-8i} + r·2^{-(8s-1)} in rational arithmetic
    for k in list(range(0, len(v), 9973)) + list(range(len(v) - len(edge), len(v))):
        acc = sum(Fraction(int(d[i][k])) / Fraction(2) ** (7 + 8 * i) for i in range(KS))
        acc += Fraction(float(r[k])) / Fraction(2) ** (8 * KS - 1)
        assert acc == Fraction(float(v[k])), k
    # truncation bound of the kept digits
    w = 2.0 ** -(7.0 + 8.0 * np.arange(KS))
    rec = (d * w[:, None]).sum(axis=0)  # exact in binary64 only for the leading digits; bound checked loosely
    assert np.abs(rec - v).max() <= 2.0 ** -52


def test_sliced_dot_products_reach_binary64_accuracy():
    """Group sums over the kept slice pairs (i + j < s), Horner in binary64, row scales: against the exact
    rational dot product the error stays below that of a plain binary64 dot product's bound."""
    rng = np.random.default_rng(1)
    n, q = 40, 3
    k = n * q
    s_mat = 1e-7 * rng.standard_normal((64, k))
    cexp = np.floor(np.log2(np.abs(s_mat).max(axis=0))).astype(int) + 1
    u = rng.standard_normal(n) * 0.8 ** np.arange(n) * 300.0
    w = rng.uniform(-1, 1, q)
    x = (w[:, None] * u[None, :]).ravel()
    xd, xs = slice_row(np.ldexp(x, cexp))
    worst = 0.0
    for r in range(s_mat.shape[0]):
        sd, ss = slice_row(np.ldexp(s_mat[r], -cexp))
        acc = [0] * KS
        for i in range(KS):
            for j in range(KS - i):
                acc[i + j] += int(np.dot(sd[i].astype(np.int64), xd[j].astype(np.int64)))
        assert max(abs(a) for a in acc) < 2 ** 31
        t = float(acc[KS - 1])
        for g in range(KS - 2, -1, -1):
            t = t * 2.0 ** -8 + float(acc[g])
        got = t * ss * xs
        exact = sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, s_mat[r]))
        mag = float(sum(abs(Fraction(float(a)) * Fraction(float(b))) for a, b in zip(x, s_mat[r])))
        worst = max(worst, abs(float(Fraction(got) - exact)) / mag)
    assert worst <= 2.0 ** -52, worst


# ---- GPU ---------------------------------------------------------------------------------------------------

@pytest.mark.gpu
def test_probe_kernel_is_bit_exact(tmp_path):
    """tools/oz_probe.cu: the tcgen05 kernel's output equals the host emulation of the same splitting for every
    checked (sample, row) pair, on a shape with partial tiles (N = 37: 1406 rows, 300 samples)."""
    from paper_1807_11866_b200 import build

    exe = build.build_probe()
    for args in (["300", "37", "3", "1"], ["4096", "100", "7", "1"]):
        r = subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "0 mismatches vs host emulation" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def _solve(model, mu, mode, pressure=False):
    import torch

    from paper_1807_11866_b200 import online

    prev = os.environ.get("RBNS_CONTRACT")
    os.environ["RBNS_CONTRACT"] = mode
    try:
        dm = online.DeviceModel(model, 0)
    finally:
        if prev is None:
            os.environ.pop("RBNS_CONTRACT", None)
        else:
            os.environ["RBNS_CONTRACT"] = prev
    with dm:
        slices = dm.contraction_slices()
        r = dm.solve(torch.from_numpy(np.ascontiguousarray(mu)).cuda(), pressure=pressure)
        torch.cuda.synchronize()
        return (slices, r.u.cpu().numpy(), r.iters.cpu().numpy(), r.status.cpu().numpy(),
                None if r.p is None else r.p.cpu().numpy(), r.stats)


@pytest.mark.gpu
@pytest.mark.parametrize("c,nb", [(0, 64), (1, 4096), (2, 4096), (3, 512), (4, 2048)])
def test_sliced_contraction_matches_dmma(c, nb):
    """Same model, same μ: the INT8-sliced contraction (default) and the FP64 DMMA contraction
    (RBNS_CONTRACT=dmma, read per model create) give the same iterates to round-off and the same Newton counts."""
    from paper_1807_11866_b200 import synthetic

    cfg = synthetic.CONFIGS[c]
    model = synthetic.config_model(cfg)
    mu = synthetic.config_mu(cfg, nb)
    pressure = cfg.n_p > 0
    s8, u8, it8, st8, p8, stats8 = _solve(model, mu, "i8", pressure)
    s0, u0, it0, st0, p0, stats0 = _solve(model, mu, "dmma", pressure)
    assert s8 == KS and s0 == 0
    assert np.array_equal(st8, st0) and np.all(st8 == 0)
    rel = np.abs(u8 - u0).max(axis=1) / np.abs(u0).max(axis=1)
    assert rel.max() <= 1e-13, rel.max()
    assert np.array_equal(it8, it0)
    if pressure:
        assert (np.abs(p8 - p0).max(axis=1) / np.abs(p0).max(axis=1)).max() <= 1e-12
    # one X-slicing launch more per contraction round after the first
    assert stats8["kernel_launches"] > stats0["kernel_launches"]


@pytest.mark.gpu
@pytest.mark.parametrize("n,q", [(7, 1), (37, 3), (64, 16), (100, 2), (129, 2)])
def test_sliced_contraction_shapes(n, q):
    """Partial row tiles, partial K chunks (Q·Ne not a multiple of 32), Q = 1 and Q = 16 affine columns."""
    from oracle import rbns_oracle as oracle
    from paper_1807_11866_b200 import synthetic

    from .test_gpu import _random_model

    model = _random_model(n, q, seed=n + 1)
    mu = synthetic.make_mu(200, 100.0, seed=5)
    s8, u8, it8, st8, _, _ = _solve(model, mu, "i8")
    assert s8 == KS
    ur, itr, str_, _ = oracle.solve_batch(model, mu)
    ok = (st8 == 0) & (str_ == 0)
    assert ok.sum() >= 100 and np.array_equal(st8, str_)
    rel = np.abs(u8[ok] - ur[ok]).max(axis=1) / np.abs(ur[ok]).max(axis=1)
    assert rel.max() <= 1e-10, rel.max()
    assert np.array_equal(it8[ok], itr[ok])


@pytest.mark.gpu
def test_sliced_contraction_is_deterministic_and_batch_invariant():
    from paper_1807_11866_b200 import synthetic

    cfg = synthetic.CONFIGS[2]
    model = synthetic.config_model(cfg)
    mu = synthetic.config_mu(cfg, 1000)
    _, ua, ita, _, _, _ = _solve(model, mu, "i8")
    _, ub, itb, _, _, _ = _solve(model, mu, "i8")
    _, uc, itc, _, _, _ = _solve(model, mu[37:437], "i8")
    assert np.array_equal(ua, ub) and np.array_equal(ita, itb)
    assert np.array_equal(ua[37:437], uc) and np.array_equal(ita[37:437], itc)


@pytest.mark.gpu
@pytest.mark.parametrize("span", [6.0, 12.0])
def test_sliced_contraction_under_basis_scaling(span):
    """The same model in a basis whose vectors are scaled by d_i = 10^U(−span/2, span/2) (A → D A D,
    C[j,k,l] → d_j d_k d_l C, f → D f, u → D⁻¹u): solution coefficients spread over `span` decades, as POD
    coefficients do.  The column equilibration of the sliced path absorbs the scaling: error against the oracle
    (measured in the unscaled basis) stays at round-off and every Newton count matches."""
    from oracle import rbns_oracle as oracle
    from paper_1807_11866_b200 import synthetic
    from paper_1807_11866_b200.model import ReducedModel

    n, q, nb = 40, 7, 160
    base = synthetic.make_model(n, q, "trig7", seed=3)
    d = 10.0 ** np.random.default_rng(4).uniform(-span / 2, span / 2, n)
    model = ReducedModel(A=base.A * d[None, :, None] * d[None, None, :],
                         C=base.C * d[None, :, None, None] * d[None, None, :, None] * d[None, None, None, :],
                         f=base.f * d[None, :], theta=base.theta)
    mu = synthetic.make_mu(nb, 200.0, seed=9)
    s8, u8, it8, st8, _, _ = _solve(model, mu, "i8")
    assert s8 == KS
    ur, itr, str_, _ = oracle.solve_batch(model, mu)
    assert np.all(st8 == 0) and np.all(str_ == 0)
    err = np.abs((u8 - ur) * d).max(axis=1) / np.abs(ur * d).max(axis=1)
    assert err.max() <= 1e-12, err.max()
    assert np.array_equal(it8, itr)
    assert np.abs(ur).max() / np.abs(ur).min() > 10.0 ** (span - 3)
