"""High-fidelity expansion of reduced solutions — SPEC ``online.lift_solution``, SURVEY.md §8(f)
row 4.

    u_h(μ_b) = V u_b + u∞,b · ℓ_unit,        p_h(μ_b) = P p_b

(u = u₀ + ℓ with the lift scaled linearly in u∞, "ℓ̂(μ) = u∞ · ℓ̂_unit").  For a
batch this is one tall-skinny DGEMM (n_dofs × N by N × B, cuBLAS: a plain library GEMM) plus a rank-1 update,
on the GPU; the high-fidelity basis stays resident on the device across calls.  ``lifted_error`` gives the
relative error against high-fidelity snapshots in a Gram norm (the ``error_study`` measure).
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from .errors import NativeError


class Lifter:
    """Device-resident V (n_dofs × N), lift ℓ_unit (n_dofs) and optional pressure basis P (n_pdofs × Np)."""

    def __init__(self, V, ell_unit, P=None, device="cuda"):
        device = torch.device(device)
        if device.type != "cuda":
            raise NativeError("lift_solution runs on the GPU (no CPU path)")
        self.device = device
        self.V = torch.as_tensor(np.ascontiguousarray(V), dtype=torch.float64, device=device)
        self.ell = torch.as_tensor(np.ascontiguousarray(ell_unit), dtype=torch.float64, device=device)
        self.P = None if P is None else torch.as_tensor(np.ascontiguousarray(P), dtype=torch.float64, device=device)
        if self.ell.shape != (self.V.shape[0],):
            raise ValueError("lift and basis disagree on the number of dofs")

    def lift(self, u, uinf, p=None):
        """(U_h (B × n_dofs), P_h (B × n_pdofs) or None) for reduced coefficients u (B × N), u∞ (B,)."""
        u = torch.as_tensor(u, dtype=torch.float64, device=self.device)
        uinf = torch.as_tensor(uinf, dtype=torch.float64, device=self.device).reshape(-1)
        if u.ndim != 2 or u.shape[1] != self.V.shape[1] or uinf.shape[0] != u.shape[0]:
            raise ValueError(f"u{tuple(u.shape)} / u_inf{tuple(uinf.shape)} do not match the basis")
        U = torch.outer(uinf, self.ell)
        U.addmm_(u, self.V.T)                       # U = u Vᵀ + u∞ ℓᵀ
        Ph = None
        if p is not None:
            if self.P is None:
                raise ValueError("no pressure basis")
            Ph = torch.as_tensor(p, dtype=torch.float64, device=self.device) @ self.P.T
        return U, Ph


def lifted_error(U, U_ref, G: Optional[np.ndarray] = None, device="cuda"):
    """Relative errors ‖U_b − U_ref,b‖_G / ‖U_ref,b‖_G per sample (G: Gram matrix, default Euclidean)."""
    U = torch.as_tensor(U, dtype=torch.float64, device=device)
    R = torch.as_tensor(U_ref, dtype=torch.float64, device=device)
    D = U - R
    if G is None:
        num, den = (D * D).sum(1), (R * R).sum(1)
    else:
        Gt = torch.as_tensor(np.array(G, dtype=np.float64), dtype=torch.float64, device=device)
        num, den = (D * (D @ Gt)).sum(1), (R * (R @ Gt)).sum(1)
    return torch.sqrt(num / den)
