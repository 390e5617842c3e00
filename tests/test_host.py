"""CPU tests of the host-side logic (model validation, θ descriptors, generators, sharding)."""

import numpy as np
import pytest

from paper_1807_11866_b200 import affine, sharding, synthetic
from paper_1807_11866_b200.model import ReducedModel


def test_model_validation():
    A = np.zeros((2, 3, 3))
    C = np.zeros((2, 3, 3, 3))
    f = np.zeros((2, 3))
    th = affine.family("trig3")[:2]
    m = ReducedModel(A=A, C=C, f=f, theta=th)
    assert (m.n, m.q, m.n_p) == (3, 2, 0)
    with pytest.raises(ValueError):
        ReducedModel(A=A, C=C[:, :2], f=f, theta=th)
    with pytest.raises(ValueError):
        ReducedModel(A=A, C=C, f=f, theta=th[:1])
    with pytest.raises(ValueError):
        ReducedModel(A=A, C=C, f=f, theta=th, Mp=np.eye(2))
    with pytest.raises(ValueError):
        affine.ThetaTerm(9)
    with pytest.raises(ValueError):
        affine.family("fourier4")
    assert not m.A.flags.writeable      # immutable once built


def test_generators_deterministic_and_pinned():
    a = synthetic.make_model(10, 3, "trig3")
    b = synthetic.make_model(10, 3, "trig3")
    np.testing.assert_array_equal(a.C, b.C)
    np.testing.assert_allclose(a.C, -a.C.transpose(0, 1, 3, 2), atol=0)      # antisymmetric in (k,l)
    np.testing.assert_allclose(a.A[1], a.A[1].T)
    assert np.linalg.eigvalsh(a.A[0]).min() >= 1.0 - 1e-12                  # GGᵀ/N + I
    mu = synthetic.make_mu(1000, 200.0)
    assert mu[:, 0].min() >= 0 and mu[:, 0].max() <= np.deg2rad(35)
    assert mu[:, 1].min() >= 10 and mu[:, 1].max() <= 200


@pytest.mark.parametrize("total,world", [(10, 3), (65536, 8), (5, 8), (0, 2)])
def test_shard_bounds_partition(total, world):
    seen = []
    for r in range(world):
        s, e = sharding.shard_bounds(total, world, r)
        assert 0 <= s <= e <= total
        seen.extend(range(s, e))
    assert seen == list(range(total))
