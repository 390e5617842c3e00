"""``ReducedModel`` — the hot path's input contract.

Only the fields the velocity-only block solver consumes are carried, grouped in the SPEC's per-form term
families (``AffineFormSet``) as they enter the reduced residual:

    R(u) = L(μ) u + Σ_c θ_c(μ) C_c(u, u) − Σ_f θ_f(μ) f_f,         L(μ) = [ν] Σ_a θ_a(μ) A_a

* ``A``  (Qa, N, N)    linear family: the viscous a-terms and, for lifted models, the lift-convection
                        c0-terms (everything linear in u);
* ``C``  (Qc, N, N, N) quadratic family: convective tensors C[j,k,l] = c(u_j advecting, u_k advected, u_l test)
                        (index convention pinned against the reference assembler
                        ``assemble.convection_matrices``, /root/reference/pkg/src/rbflow/assemble.py:86-101, by
                        tests/golden);
* ``f``  (Qf, N)       load family: projected loads and the lift's d0 terms (u∞¹ and u∞² families);
* ``Bq`` (Qb, Np, N) + SPD ``Mp`` (Np, Np): optional pressure recovery M_p p = Σ_b θ_b(μ) B_b u
                        (BASELINE.json config 4; the role of B_sp).
* ``P_att`` (n_att, N): optional attached pressure modes of the combined scheme ("optional attached
                        pressure modes for the combined scheme"): column j is the pressure data
                        attached to velocity mode j, so reconstruction is p = P_att u.

Descriptors: ``theta`` is the shared list of the BASELINE configs (one θ per term index for every family);
the ``theta_*`` fields override it per family (the paper's models: a-terms ν·φᵏ, c-terms φᵏ, c0-terms u∞·φᵏ,
d0-terms u∞·φᵏ and u∞²·φᵏ).  ``nu_linear`` multiplies the linear family by ν = 1/μ₁ (the
BASELINE rule); the paper's a-term descriptors carry ν in their scale instead (nu_linear=False).

Immutable after construction and safe to share across concurrent queries.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .affine import MAX_TERMS, ThetaTerm

FAMILIES = ("linear", "quadratic", "load", "coupling")


@dataclass(frozen=True)
class ReducedModel:
    A: np.ndarray                      # (Qa, N, N)     linear family
    C: np.ndarray                      # (Qc, N, N, N)  quadratic family
    f: np.ndarray                      # (Qf, N)        load family
    theta: Sequence[ThetaTerm] = ()    # shared descriptors (every family), BASELINE configs
    Mp: Optional[np.ndarray] = None    # (Np, Np)       SPD pressure Gramian (B_sp)
    Bq: Optional[np.ndarray] = None    # (Qb, Np, N)    pressure coupling terms (A_sv role)
    name: str = "reduced-model"
    meta: dict = field(default_factory=dict, compare=False)
    theta_linear: Optional[Sequence[ThetaTerm]] = None
    theta_quadratic: Optional[Sequence[ThetaTerm]] = None
    theta_load: Optional[Sequence[ThetaTerm]] = None
    theta_coupling: Optional[Sequence[ThetaTerm]] = None
    nu_linear: bool = True
    n_stop: int = 0                    # leading unknowns in the Newton stop norm (0: all N)
    stop_absolute: bool = False        # ‖δ‖ ≤ tol (coupled rule) instead of ‖δ‖ ≤ tol·‖u‖
    P_att: Optional[np.ndarray] = None # (n_att, N)    attached pressure modes (combined scheme), or None

    def __post_init__(self):
        A = np.ascontiguousarray(self.A, dtype=np.float64)
        C = np.ascontiguousarray(self.C, dtype=np.float64)
        f = np.ascontiguousarray(self.f, dtype=np.float64)
        for name, arr in (("A", A), ("C", C), ("f", f)):
            object.__setattr__(self, name, arr)
        object.__setattr__(self, "theta", tuple(self.theta))
        if f.ndim != 2 or A.ndim != 3 or C.ndim != 4:
            raise ValueError(f"operator ranks: A{A.shape} C{C.shape} f{f.shape}")
        n = A.shape[1]
        if A.shape[1:] != (n, n) or C.shape[1:] != (n, n, n) or f.shape[1] != n:
            raise ValueError(f"inconsistent operator shapes A{A.shape} C{C.shape} f{f.shape}")
        if (self.Mp is None) != (self.Bq is None):
            raise ValueError("pressure recovery needs both Mp and Bq")
        if self.Mp is not None:
            Mp = np.ascontiguousarray(self.Mp, dtype=np.float64)
            Bq = np.ascontiguousarray(self.Bq, dtype=np.float64)
            npr = Mp.shape[0]
            if Mp.shape != (npr, npr) or Bq.ndim != 3 or Bq.shape[1:] != (npr, n) or npr < 1:
                raise ValueError(f"inconsistent pressure shapes Mp{Mp.shape} Bq{Bq.shape}")
            object.__setattr__(self, "Mp", Mp)
            object.__setattr__(self, "Bq", Bq)
        if self.P_att is not None:
            P_att = np.ascontiguousarray(self.P_att, dtype=np.float64)
            if P_att.ndim != 2 or P_att.shape[1] != n or P_att.shape[0] < 1:
                raise ValueError(f"attached pressure modes P_att{P_att.shape} must be (n_att >= 1, {n})")
            P_att.flags.writeable = False
            object.__setattr__(self, "P_att", P_att)
        counts = {"linear": A.shape[0], "quadratic": C.shape[0], "load": f.shape[0],
                  "coupling": 0 if self.Bq is None else self.Bq.shape[0]}
        for fam in FAMILIES:
            own = getattr(self, f"theta_{fam}")
            terms = tuple(own) if own is not None else self.theta
            if own is None and fam == "coupling" and self.Bq is None:
                terms = ()
            if len(terms) != counts[fam]:
                raise ValueError(f"{len(terms)} theta descriptors for {counts[fam]} {fam} terms")
            if counts[fam] > MAX_TERMS:
                raise ValueError(f"{counts[fam]} {fam} terms > {MAX_TERMS}")
            object.__setattr__(self, f"theta_{fam}", terms)
        if counts["linear"] < 1:
            raise ValueError("the linear family needs at least one term")
        if self.Bq is not None and counts["coupling"] < 1:
            raise ValueError("pressure recovery needs at least one coupling term")
        object.__setattr__(self, "nu_linear", bool(self.nu_linear))
        object.__setattr__(self, "stop_absolute", bool(self.stop_absolute))
        if not 0 <= int(self.n_stop) <= n:
            raise ValueError(f"n_stop={self.n_stop} outside [0, {n}]")
        object.__setattr__(self, "n_stop", int(self.n_stop))
        for arr in (A, C, f):
            arr.flags.writeable = False

    @property
    def n(self) -> int:
        return self.A.shape[1]

    @property
    def q(self) -> int:
        """Number of quadratic (convective) terms — the Q of BASELINE.json's configs."""
        return self.C.shape[0]

    @property
    def n_p(self) -> int:
        return 0 if self.Mp is None else self.Mp.shape[0]

    @property
    def n_att(self) -> int:
        """Rows of the attached pressure modes (0: the model carries none)."""
        return 0 if self.P_att is None else self.P_att.shape[0]

    @property
    def stop_dim(self) -> int:
        """Number of leading unknowns in the stop norm."""
        return self.n_stop or self.n

    @property
    def counts(self) -> Tuple[int, int, int, int]:
        """(linear, quadratic, load, coupling) term counts."""
        return (self.A.shape[0], self.C.shape[0], self.f.shape[0], 0 if self.Bq is None else self.Bq.shape[0])

    @property
    def shared_theta(self) -> bool:
        """True when every family uses one descriptor list (the BASELINE configs)."""
        fams = [self.theta_linear, self.theta_quadratic, self.theta_load]
        if self.Bq is not None:
            fams.append(self.theta_coupling)
        return all(t == fams[0] for t in fams)

    @property
    def theta_list(self) -> List[ThetaTerm]:
        return list(self.theta)

    def compress_affine(self) -> "ReducedModel":
        """The same model with linearly dependent coefficient functions merged, family by family (an exact
        algebraic rewrite of the affine sums Σ_q θ_q(μ) X_q; round-off aside the reduced
        residual and Jacobian are unchanged): each family keeps a maximal independent subset of its own
        descriptors (``affine.dependence``) and X'_i = Σ_q coef[q, i] X_q.  BASELINE's trig7 family (configs 1, 2
        and 4) has 5 independent functions among its 7, so the convective contraction does 5/7 of the work.
        Returns self when nothing is dependent."""
        from .affine import dependence

        arrays = {"linear": self.A, "quadratic": self.C, "load": self.f, "coupling": self.Bq}
        out, changed, kept = {}, False, {}
        for fam in FAMILIES:
            terms = list(getattr(self, f"theta_{fam}"))
            X = arrays[fam]
            if X is None or not terms:
                out[fam] = (X, terms)
                continue
            basis, coef = dependence(terms)
            kept[fam] = [len(terms), len(basis)]
            if len(basis) == len(terms):
                out[fam] = (X, terms)
                continue
            changed = True
            Xf = X.reshape(X.shape[0], -1)
            out[fam] = ((coef.T @ Xf).reshape((len(basis),) + X.shape[1:]), [terms[i] for i in basis])
        if not changed:
            return self
        from dataclasses import replace

        return replace(self, A=out["linear"][0], C=out["quadratic"][0], f=out["load"][0],
                       Bq=out["coupling"][0] if self.Bq is not None else None, theta=(),
                       theta_linear=out["linear"][1], theta_quadratic=out["quadratic"][1],
                       theta_load=out["load"][1], theta_coupling=out["coupling"][1] if self.Bq is not None else None,
                       name=f"{self.name}-compressed", meta=dict(self.meta, affine_compressed=kept))
