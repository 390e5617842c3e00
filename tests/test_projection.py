"""Offline Galerkin projection pinned to the reference's own assembler.

tests/golden/projection_ref.npz holds the reduced basis tabulated at the quadrature points of a deformed
(φ = 20°, Piola) div-conforming mesh and the reference's projected operators V_lᵀ N1(V_j) V_k and Vᵀ A_h V
(assemble.convection_matrices / viscous_matrix, /root/reference/pkg/src/rbflow/assemble.py:60-101).
The GPU side is the hand-written DMMA kernel rbns_project_convection (csrc/rbns_project.cu) and the
multi-term driver projection.build_reduced_model.
"""

import numpy as np
import pytest

from .golden_utils import golden


def _random_terms(n, p, nc=3, na=2, nf=2, seed=0):
    from paper_1807_11866_b200 import affine
    from paper_1807_11866_b200.projection import AffineTerms, ConvectionTerm, LinearTerm, LoadTerm

    rng = np.random.default_rng(seed)
    tab = lambda *s: rng.standard_normal(s) / np.sqrt(n)
    w = rng.uniform(0.1, 1.0, p) / p
    conv = [ConvectionTerm(affine.ThetaTerm(affine.MONOMIAL, k=i), tab(p, 2, n), tab(p, 2, 2, n), tab(p, 2, n), w)
            for i in range(nc)]
    lin = [LinearTerm(affine.ThetaTerm(affine.MONOMIAL, k=i, scale=0.5), tab(p, 2, 2, n), w, scale=1.0 + i)
           for i in range(na)]
    # keep A₀ dominant and SPD (the viscous Gram of the first tabulation)
    lin[0].grad_b = None
    load = [LoadTerm(affine.ThetaTerm(affine.MONOMIAL, m=i), tab(p, 2, n), w, rng.standard_normal((p, 2)))
            for i in range(nf)]
    return AffineTerms(conv, lin, load, nu_linear=False)


def test_quadrature_restatement_matches_reference():
    """The quadrature-sum form the GPU projection evaluates reproduces the reference's sparse projection."""
    from oracle import rbns_oracle as oracle

    d = golden("projection_ref")
    C = oracle.project_convection(d["val"], d["grad"], d["val"], d["w"])
    A = np.einsum("p,pcdj,pcdk->jk", d["w"], d["grad"], d["grad"], optimize=True)
    assert np.abs(C - d["C_ref"]).max() <= 1e-13 * np.abs(d["C_ref"]).max()
    assert np.abs(A - d["A_ref"]).max() <= 1e-13 * np.abs(d["A_ref"]).max()


def test_projection_refuses_cpu():
    from paper_1807_11866_b200 import projection
    from paper_1807_11866_b200.errors import NativeError

    d = golden("projection_ref")
    with pytest.raises(NativeError):
        projection.project_convection(d["val"], d["grad"], d["val"], d["w"], device="cpu")
    with pytest.raises(NativeError):
        projection.build_reduced_model(_random_terms(6, 40), device="cpu")


def test_multi_term_restatement_shapes():
    from oracle import rbns_oracle as oracle

    C, A, f = oracle.project_terms(_random_terms(6, 40))
    assert C.shape == (3, 6, 6, 6) and A.shape == (2, 6, 6) and f.shape == (2, 6)
    assert np.allclose(A[0], A[0].T)


@pytest.mark.gpu
@pytest.mark.parametrize("splits", [0, 1, 3])
def test_gpu_projection_matches_reference(splits):
    from paper_1807_11866_b200 import projection

    d = golden("projection_ref")
    C = projection.project_convection(d["val"], d["grad"], d["val"], d["w"], splits=splits).cpu().numpy()
    A = projection.project_viscous(d["grad"], d["w"]).cpu().numpy()
    assert np.abs(C - d["C_ref"]).max() <= 1e-13 * np.abs(d["C_ref"]).max()
    assert np.abs(A - d["A_ref"]).max() <= 1e-13 * np.abs(d["A_ref"]).max()


@pytest.mark.gpu
@pytest.mark.parametrize("n,p", [(1, 1), (7, 13), (17, 1000), (64, 2051), (100, 777), (131, 300)])
def test_gpu_projection_kernel_shapes(n, p):
    """Ragged N (tile edges in j, k and l) and point counts (partial chunks, split-K edges) against numpy;
    deterministic across calls."""
    from oracle import rbns_oracle as oracle
    from paper_1807_11866_b200 import projection

    rng = np.random.default_rng(n * 1000 + p)
    vu, g, vw = rng.standard_normal((p, 2, n)), rng.standard_normal((p, 2, 2, n)), rng.standard_normal((p, 2, n))
    w = rng.uniform(0, 1, p)
    ref = oracle.project_convection(vu, g, vw, w)
    c1 = projection.project_convection(vu, g, vw, w)
    c2 = projection.project_convection(vu, g, vw, w)
    scale = np.einsum("p,pdj,pcdk,pcl->jkl", w, np.abs(vu), np.abs(g), np.abs(vw), optimize=True).max()
    assert np.abs(c1.cpu().numpy() - ref).max() <= 1e-14 * scale * max(1.0, np.sqrt(p))
    assert bool((c1 == c2).all())


@pytest.mark.gpu
def test_gpu_multi_term_driver_and_store(tmp_path):
    """build_reduced_model (every term on its own stream) against the restatement; the store round trip is
    byte-stable; the projected model feeds the online solver (oracle parity)."""
    import torch

    from oracle import rbns_oracle as oracle
    from paper_1807_11866_b200 import online, projection, store

    terms = _random_terms(24, 3000)
    rm = projection.build_reduced_model(terms, name="projected")
    C, A, f = oracle.project_terms(terms)
    for got, ref in ((rm.C, C), (rm.A, A), (rm.f, f)):
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    path = store.save_model(rm, tmp_path / "projected")
    rm2 = store.load_model(path)
    assert np.array_equal(rm2.C, rm.C) and np.array_equal(rm2.A, rm.A) and np.array_equal(rm2.f, rm.f)
    # a solvable model from the projected families: A dominated by its SPD first term, small convection
    A = rm.A.copy()
    A[0] += 4.0 * np.eye(A.shape[1])
    import dataclasses
    rm3 = dataclasses.replace(rm2, A=A, C=rm2.C * 0.05)
    mu = np.stack([np.linspace(0.1, 0.6, 16), np.linspace(0.5, 2.0, 16)], axis=1)
    with online.DeviceModel(rm3, 0) as dm:
        r = dm.solve(torch.from_numpy(mu).cuda())
        torch.cuda.synchronize()
    ur, itr, st, _ = oracle.solve_batch(rm3, mu)
    assert np.all(st == 0) and np.all(r.status.cpu().numpy() == 0)
    assert np.abs(r.u.cpu().numpy() - ur).max() <= 1e-10 * np.abs(ur).max()
    assert np.array_equal(r.iters.cpu().numpy(), itr)


@pytest.mark.gpu
def test_gpu_projection_feeds_the_solver():
    """Projected operators → ReducedModel → online solve (oracle parity) — the offline→online seam."""
    import torch

    from oracle import rbns_oracle as oracle
    from paper_1807_11866_b200 import affine, online, projection
    from paper_1807_11866_b200.model import ReducedModel

    d = golden("projection_ref")
    C = projection.project_convection(d["val"], d["grad"], d["val"], d["w"]).cpu().numpy()
    A = projection.project_viscous(d["grad"], d["w"]).cpu().numpy()
    n = A.shape[0]
    f = 0.05 * np.random.default_rng(2).standard_normal((1, n))
    rm = ReducedModel(A=A[None], C=C[None] * 10, f=f, theta=[affine.ThetaTerm(affine.CONST)])
    mu = np.array([[0.0, 1.0], [0.0, 3.0], [0.0, 6.0], [0.0, 10.0]])
    with online.DeviceModel(rm, 0) as dm:
        r = dm.solve(torch.from_numpy(mu).cuda())
        torch.cuda.synchronize()
        ur, itr, st, _ = oracle.solve_batch(rm, mu)
        assert np.all(st == 0) and np.array_equal(r.iters.cpu().numpy(), itr)
        assert np.abs(r.u.cpu().numpy() - ur).max() <= 1e-10 * np.abs(ur).max()
