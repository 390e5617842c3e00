"""Affine coefficient functions θ_q(μ) — the reduced-level half of the SPEC ``affine`` module.

Reference: ``CoefficientDescriptor`` ("evaluation is exactly scale·φᵏ·u∞ᵐ") and
``evaluate_weights``.  The reference's paper uses exact φ/u∞ monomials
(PAPER.md:442-474); BASELINE.json's configs use trigonometric families of the angle of attack α.  Both are
expressed here as a list of :class:`ThetaTerm` descriptors whose evaluation rule is shared, term by term, with
the CUDA kernels (``csrc/rbns_common.cuh: eval_theta``) so the host and the device evaluate θ identically.

μ is ``(alpha [rad], Re)`` for the BASELINE configs (viscosity rule ν = 1/Re, BASELINE.json config 0) and
``(φ [rad], u∞)`` for the paper's lifted models, whose descriptors carry ν themselves.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, List, Sequence

import numpy as np

# term kinds — keep in sync with include/rbns.h (RBNS_THETA_*)
CONST = 0          # scale
COS_K = 1          # scale * cos(k α)
SIN_K = 2          # scale * sin(k α)
COS_SIN_POW = 3    # scale * cos(α)^k * sin(α)^m
MONOMIAL = 4       # scale * α^k * Re^m      (the paper's scale·φᵏ·u∞ᵐ)

MAX_TERMS = 256    # RBNS_MAX_TERMS (per term family)


@dataclass(frozen=True)
class ThetaTerm:
    """One coefficient descriptor θ_q(μ) = scale · base_kind(α, Re; k, m)."""

    kind: int
    k: int = 0
    m: int = 0
    scale: float = 1.0

    def __post_init__(self):
        if self.kind not in (CONST, COS_K, SIN_K, COS_SIN_POW, MONOMIAL):
            raise ValueError(f"unknown theta kind {self.kind}")
        if self.k < 0 or self.m < 0:
            raise ValueError("theta exponents must be non-negative")


def _ipow(x: np.ndarray, n: int) -> np.ndarray:
    """x**n by repeated multiplication, in the same order the device uses (eval_theta)."""
    r = np.ones_like(x)
    for _ in range(n):
        r = r * x
    return r


def evaluate_weights(terms: Sequence[ThetaTerm], mu: np.ndarray) -> np.ndarray:
    """θ[b, q] for μ[b] = (α, Re) (exact evaluation, ordering matches the operator list)."""
    mu = np.atleast_2d(np.asarray(mu, dtype=np.float64))
    alpha, re = mu[:, 0], mu[:, 1]
    out = np.empty((mu.shape[0], len(terms)), dtype=np.float64)
    for q, t in enumerate(terms):
        if t.kind == CONST:
            base = np.ones_like(alpha)
        elif t.kind == COS_K:
            base = np.cos(t.k * alpha)
        elif t.kind == SIN_K:
            base = np.sin(t.k * alpha)
        elif t.kind == COS_SIN_POW:
            base = _ipow(np.cos(alpha), t.k) * _ipow(np.sin(alpha), t.m)
        else:
            base = _ipow(alpha, t.k) * _ipow(re, t.m)
        out[:, q] = t.scale * base
    return out


def viscosity(mu: np.ndarray) -> np.ndarray:
    """ν = 1/Re (BASELINE.json config 0)."""
    mu = np.atleast_2d(np.asarray(mu, dtype=np.float64))
    return 1.0 / mu[:, 1]


# ---- the θ families named by BASELINE.json's configs ------------------------------------------------------

def family(name: str) -> List[ThetaTerm]:
    """θ families of BASELINE.json configs (Appendix B #6 for ``fourier13``)."""
    if name == "trig3":        # config 0: (1, cos α, sin α)
        return [ThetaTerm(CONST), ThetaTerm(COS_K, 1), ThetaTerm(SIN_K, 1)]
    if name == "trig7":        # configs 1, 2, 4: (1, cos α, sin α, cos²α, sin²α, sin α cos α, cos 2α)
        return [ThetaTerm(CONST), ThetaTerm(COS_SIN_POW, 1, 0), ThetaTerm(COS_SIN_POW, 0, 1),
                ThetaTerm(COS_SIN_POW, 2, 0), ThetaTerm(COS_SIN_POW, 0, 2), ThetaTerm(COS_SIN_POW, 1, 1),
                ThetaTerm(COS_K, 2)]
    if name.startswith("fourier"):   # config 3: (1, cos kα, sin kα for k = 1..K), Q = 2K+1
        q = int(name[len("fourier"):])
        if q < 1 or q % 2 == 0:
            raise ValueError("fourier families have an odd number of terms")
        terms = [ThetaTerm(CONST)]
        for k in range(1, (q - 1) // 2 + 1):
            terms += [ThetaTerm(COS_K, k), ThetaTerm(SIN_K, k)]
        return terms
    raise ValueError(f"unknown theta family {name!r}")


def dependence(terms: Sequence[ThetaTerm], samples: int = 64, seed: int = 0, rtol: float = 1e-12):
    """Linear dependence among the coefficient functions of one family: returns (basis, coef) with basis the
    indices of a maximal independent subset (first occurrences kept, in order) and coef[q] the exact-to-rounding
    coefficients expressing θ_q in that basis, θ_q(μ) = Σ_i coef[q, i] θ_basis[i](μ) for every μ.

    The functions are sampled at random μ (α ∈ [−π, π], μ₁ ∈ [0.5, 2]: any point set in general position
    determines a dependence among these analytic functions); a term joins the basis when its least-squares
    residual against the current basis exceeds rtol relative.  E.g. BASELINE's trig7 list (1, cos α, sin α, cos²α,
    sin²α, sin α cos α, cos 2α) spans only 5 functions: sin²α = 1 − cos²α, cos 2α = 2cos²α − 1."""
    terms = list(terms)
    rng = np.random.default_rng(seed)
    mu = np.stack([rng.uniform(-np.pi, np.pi, samples), rng.uniform(0.5, 2.0, samples)], axis=1)
    Th = evaluate_weights(terms, mu)
    basis: List[int] = []
    coef = np.zeros((len(terms), len(terms)))
    for q in range(len(terms)):
        col = Th[:, q]
        if basis:
            c, *_ = np.linalg.lstsq(Th[:, basis], col, rcond=None)
            snap = np.round(c * 2.0 ** 20) / 2.0 ** 20  # dyadic relations (±1, 2, ½ …) exactly
            c = np.where(np.abs(c - snap) <= 1e-12 * np.maximum(1.0, np.abs(c)), snap, c)
            res = np.linalg.norm(Th[:, basis] @ c - col)
            if res <= rtol * max(np.linalg.norm(col), 1e-300):
                coef[q, :len(basis)] = c
                continue
        basis.append(q)
        coef[q, len(basis) - 1] = 1.0
    return basis, coef[:, :len(basis)]


def monomials(powers: Iterable[tuple], scales: Iterable[float] | None = None) -> List[ThetaTerm]:
    """The paper's exact monomial family scale·αᵏ·Reᵐ from (k, m) pairs."""
    powers = list(powers)
    scales = [1.0] * len(powers) if scales is None else list(scales)
    return [ThetaTerm(MONOMIAL, int(k), int(m), float(s)) for (k, m), s in zip(powers, scales)]
