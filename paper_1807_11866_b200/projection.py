"""Offline Galerkin projection of the reduced operators on the GPU — SURVEY.md §8(f) row 2.

Produces the online stage's inputs (SPEC.md:449-457 ``build_reduced_model``):

    C[j,k,l] = V_lᵀ N1(V_j) V_k = ∫ (ψ_j·∇) ψ_k · ψ_l dx             (convective tensor, c(u_j, u_k, u_l))
    A[j,k]   = ν ∫ ∇ψ_j : ∇ψ_k dx                                     (viscous a-form)
    f[j]     = ∫ F · ψ_j dx                                           (load)

from the reduced basis ψ_j = Σ V[dof, j] φ_dof tabulated at the quadrature points of the (deformed)
high-fidelity mesh: values ``val[p, c, j]`` (P×2×N), gradients ``grad[p, c, d, j]`` = ∂_d ψ_{j,c} (P×2×2×N) and
weights ``w[p]`` (quadrature weight × |det G|).  This is the same integral the reference evaluates element by
element (assemble.convection_matrices / viscous_matrix, /root/reference/pkg/src/rbflow/assemble.py:60-101) and
then projects with sparse products; here the sum over quadrature points is the GEMM dimension.

* ``project_convection`` runs the hand-written sm_100a kernel ``rbns_project_convection`` (csrc/rbns_project.cu):
  the per-point products T[(p,c),(j,k)] = Σ_d ψ_{j,d} ∂_d ψ_{k,c} are formed in shared memory next to the FP64
  tensor-core (DMMA) GEMM against w_p ψ_{l,c}, so T never reaches HBM; split-K over the points with a
  fixed-order reduction (deterministic).
* ``project_viscous`` / ``project_load`` are one cuBLAS DGEMM / one contraction (plain library work, ≤ 2 % of
  the flops of a c-term at the same P and N).
* ``build_reduced_model`` is the multi-term driver: every affine term of an ``AffineFormSet``
  — c-terms, a-terms, loads, each with its own tabulation (the Piola B±-series pushes give one tabulation per
  term) and its own θ descriptor — projected on its own CUDA stream ("Projection of independent affine terms
  is parallel", SPEC.md Concurrency Model), assembled into a storable ``ReducedModel`` (``store.save_model``).

Offline only: the online solve never runs any of it (zero quadrature online).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _native, instrument
from .affine import ThetaTerm
from .errors import NativeError
from .model import ReducedModel


def _dev(x, device):
    device = torch.device(device)
    if device.type != "cuda":
        raise NativeError("the projection runs on the GPU (no CPU path)")
    return torch.as_tensor(x, dtype=torch.float64, device=device).contiguous()


def project_convection(val_u, grad, val_w, w, device="cuda", splits: int = 0, out: Optional[torch.Tensor] = None
                       ) -> torch.Tensor:
    """C (N, N, N) with C[j,k,l] = Σ_p w_p Σ_{c,d} val_u[p,d,j] grad[p,c,d,k] val_w[p,c,l] (fp64, on device).

    ``val_u`` tabulates the advecting functions, ``grad`` the advected ones, ``val_w`` the test functions (the
    same basis for the velocity-only tensor; different tabulations for affine terms of the Piola expansion).
    ``splits``: split-K slices over the points (0: automatic)."""
    vu, g, vw, wt = (_dev(x, device) for x in (val_u, grad, val_w, w))
    p_tot, _, n = vu.shape
    if g.shape != (p_tot, 2, 2, n) or vw.shape != (p_tot, 2, n) or wt.shape != (p_tot,):
        raise ValueError(f"tabulation shapes val_u{tuple(vu.shape)} grad{tuple(g.shape)} val_w{tuple(vw.shape)} "
                         f"w{tuple(wt.shape)}")
    instrument.count_quadrature(p_tot)  # offline quadrature (the online stage must never do this)
    if out is None:
        out = torch.empty((n, n, n), dtype=torch.float64, device=vu.device)
    elif out.shape != (n, n, n) or out.dtype != torch.float64 or not out.is_contiguous() or out.device != vu.device:
        raise ValueError("out must be a contiguous float64 (N, N, N) tensor on the tabulations' device")
    lib = _native.load()
    with torch.cuda.device(vu.device):
        st = torch.cuda.current_stream(vu.device).cuda_stream
        rc = lib.rbns_project_convection(vu.data_ptr(), g.data_ptr(), vw.data_ptr(), wt.data_ptr(), p_tot, n,
                                         out.data_ptr(), int(splits), ctypes.c_void_p(st))
    _native.check(rc, "rbns_project_convection")
    return out


def project_viscous(grad, w, nu: float = 1.0, device="cuda", grad_b=None) -> torch.Tensor:
    """A (N, N) = ν Σ_p w_p Σ_{c,d} grad[p,c,d,j] grad_b[p,c,d,k] (grad_b defaults to grad; one DGEMM)."""
    g, wt = _dev(grad, device), _dev(w, device)
    gb = g if grad_b is None else _dev(grad_b, device)
    p_tot, _, _, n = g.shape
    if gb.shape != g.shape or wt.shape != (p_tot,):
        raise ValueError("tabulation shapes")
    instrument.count_quadrature(p_tot)
    return nu * ((wt[:, None, None, None] * g).reshape(-1, n).T @ gb.reshape(-1, n))


def project_load(val_w, w, force, device="cuda") -> torch.Tensor:
    """f (N,) = Σ_p w_p Σ_c force[p,c] val_w[p,c,j] for a body force tabulated at the quadrature points."""
    vw, wt, fo = _dev(val_w, device), _dev(w, device), _dev(force, device)
    instrument.count_quadrature(wt.shape[0])
    return torch.einsum("p,pc,pcj->j", wt, fo, vw)


# ---- multi-term driver (SPEC.md:449-457 build_reduced_model) --------------------------------------------------

@dataclass
class ConvectionTerm:
    """One c-term: C = c(ψ_j, ψ_k, ψ_l) with this term's tabulations, weighted online by θ."""
    theta: ThetaTerm
    val_u: object
    grad: object
    val_w: object
    w: object


@dataclass
class LinearTerm:
    """One a-term (or lift c0-term): A[j,k] = scale Σ_p w_p grad_a[p,:,:,j] : grad_b[p,:,:,k]."""
    theta: ThetaTerm
    grad: object
    w: object
    grad_b: object = None
    scale: float = 1.0


@dataclass
class LoadTerm:
    """One load (or lift d0) term: f[j] = Σ_p w_p force[p,c] val_w[p,c,j]."""
    theta: ThetaTerm
    val_w: object
    w: object
    force: object


@dataclass
class AffineTerms:
    """The projected families' inputs (an AffineFormSet's velocity block)."""
    convection: Sequence[ConvectionTerm]
    linear: Sequence[LinearTerm]
    load: Sequence[LoadTerm]
    nu_linear: bool = True
    meta: dict = field(default_factory=dict)


def build_reduced_model(terms: AffineTerms, device="cuda", name: str = "projected-model",
                        splits: int = 0) -> ReducedModel:
    """Project every affine term (each on its own CUDA stream) and assemble the ReducedModel the online stage
    consumes; ``store.save_model`` writes it.  Per-family descriptors follow the terms' own θ."""
    if not terms.convection or not terms.linear:
        raise ValueError("need at least one convection term and one linear term")
    device = torch.device(device)
    if device.type != "cuda":
        raise NativeError("the projection runs on the GPU (no CPU path)")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    streams: List[torch.cuda.Stream] = []
    Cs, As, fs = [], [], []
    main = torch.cuda.current_stream(device)
    for i, t in enumerate(list(terms.convection) + list(terms.linear) + list(terms.load)):
        s = torch.cuda.Stream(device)
        s.wait_stream(main)
        streams.append(s)
        with torch.cuda.stream(s):
            if isinstance(t, ConvectionTerm):
                Cs.append(project_convection(t.val_u, t.grad, t.val_w, t.w, device=device, splits=splits))
            elif isinstance(t, LinearTerm):
                As.append(project_viscous(t.grad, t.w, nu=t.scale, device=device, grad_b=t.grad_b))
            else:
                fs.append(project_load(t.val_w, t.w, t.force, device=device))
    for s in streams:
        main.wait_stream(s)
    n = Cs[0].shape[0]
    C = torch.stack(Cs).cpu().numpy()
    A = torch.stack(As).cpu().numpy()
    f = torch.stack(fs).cpu().numpy() if fs else np.zeros((1, n))
    th_f = [t.theta for t in terms.load] if fs else [ThetaTerm(0, scale=0.0)]
    return ReducedModel(A=A, C=C, f=f, name=name, nu_linear=terms.nu_linear,
                        theta_linear=[t.theta for t in terms.linear],
                        theta_quadratic=[t.theta for t in terms.convection], theta_load=th_f,
                        meta=dict(terms.meta, projected_terms=[len(Cs), len(As), len(fs)]))
