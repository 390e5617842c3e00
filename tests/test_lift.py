"""lift_solution: SPEC examples + a numpy restatement."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(n_dofs=400, n=12, seed=3):
    rng = np.random.default_rng(seed)
    V, _ = np.linalg.qr(rng.standard_normal((n_dofs, n)))
    ell = rng.standard_normal(n_dofs)
    return V, ell


def test_zero_solution_is_the_lift():
    from paper_1807_11866_b200.lift import Lifter

    V, ell = _setup()
    L = Lifter(V, ell)
    U, _ = L.lift(np.zeros((3, V.shape[1])), np.array([1.0, 7.5, 20.0]))
    np.testing.assert_array_equal(U.cpu().numpy(), np.outer([1.0, 7.5, 20.0], ell))


def test_lift_matches_restatement_and_is_affine():
    from paper_1807_11866_b200.lift import Lifter, lifted_error

    V, ell = _setup()
    rng = np.random.default_rng(5)
    u = rng.standard_normal((64, V.shape[1])) * 10
    uinf = rng.uniform(1, 20, 64)
    L = Lifter(V, ell, P=V[:50])
    U, Ph = L.lift(u, uinf, p=u)
    ref = u @ V.T + uinf[:, None] * ell
    assert np.abs(U.cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()
    np.testing.assert_allclose(Ph.cpu().numpy(), u @ V[:50].T, rtol=1e-13, atol=1e-12)
    U2, _ = L.lift(2 * u, uinf)
    np.testing.assert_allclose((U2 - U).cpu().numpy(), u @ V.T, rtol=1e-12, atol=1e-10)
    err = lifted_error(U, ref).cpu().numpy()
    assert err.max() <= 1e-14
    G = np.eye(V.shape[0]) * 2.0
    np.testing.assert_allclose(lifted_error(U2, U, G).cpu().numpy(),
                               np.linalg.norm(u @ V.T, axis=1) / np.linalg.norm(ref, axis=1), rtol=1e-12)
