"""``ReducedModel`` — the hot path's input contract.

Only the fields the velocity-only block solver consumes are carried: per affine term q the projected viscous
matrix A_q (N×N), the convective tensor C_q (N×N×N, C[j,k,l] = c(u_j advecting, u_k advected, u_l test);
PAPER.md:821-827, index convention cross-checked against the reference assembler
``assemble.convection_matrices`` /root/reference/pkg/src/rbflow/assemble.py:86-101 by tests/golden), the load
vector f_q (N) and the θ descriptors.  Optional pressure-recovery operators (BASELINE.json config 4,
SURVEY.md Appendix B #7): an SPD, μ-independent pressure Gramian M_p (Np×Np, the role of B_sp,
PAPER.md:905-908) and coupling operators B_q (Np×N), recovering p = M_p⁻¹ Σ_q θ_q(μ) B_q u.

Immutable after construction and safe to share across concurrent queries.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .affine import MAX_TERMS, ThetaTerm


@dataclass(frozen=True)
class ReducedModel:
    A: np.ndarray                      # (Q, N, N)   projected a-terms (multiplied by ν online)
    C: np.ndarray                      # (Q, N, N, N) convective tensors
    f: np.ndarray                      # (Q, N)      projected loads
    theta: Sequence[ThetaTerm]         # Q descriptors
    Mp: Optional[np.ndarray] = None    # (Np, Np)    SPD pressure Gramian (B_sp)
    Bq: Optional[np.ndarray] = None    # (Q, Np, N)  pressure coupling terms (A_sv role)
    name: str = "reduced-model"
    meta: dict = field(default_factory=dict, compare=False)

    def __post_init__(self):
        A = np.ascontiguousarray(self.A, dtype=np.float64)
        C = np.ascontiguousarray(self.C, dtype=np.float64)
        f = np.ascontiguousarray(self.f, dtype=np.float64)
        object.__setattr__(self, "A", A)
        object.__setattr__(self, "C", C)
        object.__setattr__(self, "f", f)
        object.__setattr__(self, "theta", tuple(self.theta))
        q, n = f.shape
        if A.shape != (q, n, n) or C.shape != (q, n, n, n):
            raise ValueError(f"inconsistent operator shapes A{A.shape} C{C.shape} f{f.shape}")
        if len(self.theta) != q:
            raise ValueError(f"{len(self.theta)} theta descriptors for {q} affine terms")
        if not 1 <= q <= MAX_TERMS:
            raise ValueError(f"Q={q} outside [1, {MAX_TERMS}]")
        if (self.Mp is None) != (self.Bq is None):
            raise ValueError("pressure recovery needs both Mp and Bq")
        if self.Mp is not None:
            Mp = np.ascontiguousarray(self.Mp, dtype=np.float64)
            Bq = np.ascontiguousarray(self.Bq, dtype=np.float64)
            npr = Mp.shape[0]
            if Mp.shape != (npr, npr) or Bq.shape != (q, npr, n):
                raise ValueError(f"inconsistent pressure shapes Mp{Mp.shape} Bq{Bq.shape}")
            object.__setattr__(self, "Mp", Mp)
            object.__setattr__(self, "Bq", Bq)
        for arr in (A, C, f):
            arr.flags.writeable = False

    @property
    def n(self) -> int:
        return self.f.shape[1]

    @property
    def q(self) -> int:
        return self.f.shape[0]

    @property
    def n_p(self) -> int:
        return 0 if self.Mp is None else self.Mp.shape[0]

    @property
    def theta_list(self) -> List[ThetaTerm]:
        return list(self.theta)
