"""Offline Galerkin projection pinned to the reference's own assembler.

tests/golden/projection_ref.npz holds the reduced basis tabulated at the quadrature points of a deformed
(φ = 20°, Piola) div-conforming mesh and the reference's projected operators V_lᵀ N1(V_j) V_k and Vᵀ A_h V
(assemble.convection_matrices / viscous_matrix, /root/reference/pkg/src/rbflow/assemble.py:60-101).
"""

import numpy as np
import pytest

from .golden_utils import golden


def test_quadrature_restatement_matches_reference():
    """The quadrature-sum form the GPU projection evaluates reproduces the reference's sparse projection."""
    d = golden("projection_ref")
    C = np.einsum("p,pdj,pcdk,pcl->jkl", d["w"], d["val"], d["grad"], d["val"], optimize=True)
    A = np.einsum("p,pcdj,pcdk->jk", d["w"], d["grad"], d["grad"], optimize=True)
    assert np.abs(C - d["C_ref"]).max() <= 1e-13 * np.abs(d["C_ref"]).max()
    assert np.abs(A - d["A_ref"]).max() <= 1e-13 * np.abs(d["A_ref"]).max()


def test_projection_refuses_cpu():
    from paper_1807_11866_b200 import projection
    from paper_1807_11866_b200.errors import NativeError

    d = golden("projection_ref")
    with pytest.raises(NativeError):
        projection.project_convection(d["val"], d["grad"], d["val"], d["w"], device="cpu")


@pytest.mark.gpu
def test_gpu_projection_matches_reference():
    from paper_1807_11866_b200 import projection

    d = golden("projection_ref")
    C = projection.project_convection(d["val"], d["grad"], d["val"], d["w"], chunk_bytes=1 << 12).cpu().numpy()
    A = projection.project_viscous(d["grad"], d["w"]).cpu().numpy()
    assert np.abs(C - d["C_ref"]).max() <= 1e-13 * np.abs(d["C_ref"]).max()
    assert np.abs(A - d["A_ref"]).max() <= 1e-13 * np.abs(d["A_ref"]).max()


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
