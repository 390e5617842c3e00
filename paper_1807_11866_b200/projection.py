"""Offline Galerkin projection of the reduced operators on the GPU — SURVEY.md §8(f) row 2.

Produces the online stage's inputs (SPEC.md:449-457 ``build_reduced_model``):

    C[j,k,l] = V_lᵀ N1(V_j) V_k = ∫ (ψ_j·∇) ψ_k · ψ_l dx             (convective tensor, c(u_j, u_k, u_l))
    A[j,k]   = ν ∫ ∇ψ_j : ∇ψ_k dx                                     (viscous a-form)

from the reduced basis ψ_j = Σ V[dof, j] φ_dof tabulated at the quadrature points of the (deformed)
high-fidelity mesh: values ``val[p, c, j]`` (P×2×N), gradients ``grad[p, c, d, j]`` = ∂_d ψ_{j,c} (P×2×2×N) and
weights ``w[p]`` (quadrature weight × |det G|).  This is the same integral the reference evaluates element by
element (assemble.convection_matrices / viscous_matrix, /root/reference/pkg/src/rbflow/assemble.py:60-101) and
then projects with sparse products; here the sum over quadrature points is the GEMM dimension:

    C[j,k,l] = Σ_{p,c} (w_p ψ_{l,c}(p)) · T[(p,c),(j,k)],   T[(p,c),(j,k)] = Σ_d ψ_{j,d}(p) ∂_d ψ_{k,c}(p)

chunked over p so T never exceeds ``chunk_bytes``; the contraction is a cuBLAS DGEMM (a plain library GEMM,
fp64), the per-point outer products are elementwise.  With one tabulation per affine term (the Piola B±-series
pushes of SPEC.md:339-346) the call is repeated per term.  Offline only: the online solve never runs it.
"""

from __future__ import annotations

import torch

from . import instrument
from .errors import NativeError


def _dev(x, device):
    device = torch.device(device)
    if device.type != "cuda":
        raise NativeError("the projection runs on the GPU (no CPU path)")
    return torch.as_tensor(x, dtype=torch.float64, device=device)


def project_convection(val_u, grad, val_w, w, device="cuda", chunk_bytes: int = 1 << 28) -> torch.Tensor:
    """C (N, N, N) with C[j,k,l] = Σ_p w_p Σ_{c,d} val_u[p,d,j] grad[p,c,d,k] val_w[p,c,l] (fp64, on device).

    ``val_u`` tabulates the advecting functions, ``grad`` the advected ones, ``val_w`` the test functions (the
    same basis for the velocity-only tensor; different tabulations for affine terms of the Piola expansion)."""
    vu, g, vw, wt = (_dev(x, device) for x in (val_u, grad, val_w, w))
    p_tot, _, n = vu.shape
    if g.shape != (p_tot, 2, 2, n) or vw.shape != (p_tot, 2, n) or wt.shape != (p_tot,):
        raise ValueError(f"tabulation shapes val_u{tuple(vu.shape)} grad{tuple(g.shape)} val_w{tuple(vw.shape)} "
                         f"w{tuple(wt.shape)}")
    instrument.count_quadrature(p_tot)  # offline quadrature (the online stage must never do this)
    step = max(1, chunk_bytes // (2 * n * n * 8))
    out = torch.zeros((n, n * n), dtype=torch.float64, device=device)       # [l, (j,k)]
    for p0 in range(0, p_tot, step):
        sl = slice(p0, min(p_tot, p0 + step))
        T = torch.einsum("pdj,pcdk->pcjk", vu[sl], g[sl]).reshape(-1, n * n)   # [(p,c), (j,k)]
        W = (wt[sl, None, None] * vw[sl]).reshape(-1, n)                      # [(p,c), l]
        out.addmm_(W.T, T)
    return out.reshape(n, n, n).permute(1, 2, 0).contiguous()


def project_viscous(grad, w, nu: float = 1.0, device="cuda") -> torch.Tensor:
    """A (N, N) = ν Σ_p w_p Σ_{c,d} grad[p,c,d,j] grad[p,c,d,k] (one DGEMM)."""
    g, wt = _dev(grad, device), _dev(w, device)
    p_tot, _, _, n = g.shape
    instrument.count_quadrature(p_tot)
    G = (torch.sqrt(wt)[:, None, None, None] * g).reshape(-1, n) if bool((wt >= 0).all()) else None
    if G is None:
        raise ValueError("negative quadrature weights")
    return nu * (G.T @ G)


def project_load(val_w, w, force, device="cuda") -> torch.Tensor:
    """f (N,) = Σ_p w_p Σ_c force[p,c] val_w[p,c,j] for a body force tabulated at the quadrature points."""
    vw, wt, fo = _dev(val_w, device), _dev(w, device), _dev(force, device)
    instrument.count_quadrature(wt.shape[0])
    return torch.einsum("p,pc,pcj->j", wt, fo, vw)
