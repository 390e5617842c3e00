"""Naive coupled saddle-point solvers — SPEC ``online.solve_coupled``, SURVEY.md §8(f) row 3.

The paper's comparison baseline: Newton on the full reduced saddle system instead of the velocity-only block
(PAPER.md:725-734 Eq. (sys-instab), :926-929 Eq. (block)),

    R_v = A(μ) v + C(μ)(v, v) + B(μ)ᵀ p − f_v(μ)           v = u (unstabilised, size M)
    R_p = B(μ) v − f_p(μ)                                 v = (u, s) (supremizer-stabilised, size 2M)

of size 2M or 3M.  It runs on the same sm_100a path as the block solver: the saddle system is embedded as one
:class:`ReducedModel` of size N = N_v + N_p — the linear family holds A (top-left) and the divergence terms
(B in the pressure rows, Bᵀ in the pressure columns, own descriptors θ_b), the quadratic family the convective
tensors on the velocity unknowns, the load family f_v and f_p — and ``rbns_model_create2`` gets
``n_stop = N_v`` with the absolute stop rule of SPEC.md:513 ("velocity-block update Euclidean norm ≤ 1e−10").
Dense LU with partial pivoting handles the zero pressure block; a machine-zero inf-sup constant (unstabilised
div-conforming models, Table 1) surfaces as SINGULAR_SYSTEM or NON_CONVERGED per sample, never as a
crash.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .affine import ThetaTerm
from .model import ReducedModel

COUPLED_TOL = 1e-10


@dataclass(frozen=True)
class CoupledModel:
    """Blocks of the reduced saddle system (v = velocity unknowns, u or (u, s); p = pressure)."""

    A: np.ndarray                       # (Qa, Nv, Nv)
    B: np.ndarray                       # (Qb, Np, Nv)   b(v, q) divergence terms
    C: np.ndarray                       # (Qc, Nv, Nv, Nv)
    f: np.ndarray                       # (Qf, Nv)
    theta_linear: Sequence[ThetaTerm]
    theta_div: Sequence[ThetaTerm]
    theta_quadratic: Sequence[ThetaTerm]
    theta_load: Sequence[ThetaTerm]
    fp: Optional[np.ndarray] = None     # (Qd, Np) pressure-equation loads (the lift's d1 terms)
    theta_pload: Sequence[ThetaTerm] = ()
    nu_linear: bool = True
    stabilized: bool = True
    name: str = "coupled"

    @property
    def n_v(self) -> int:
        return self.A.shape[1]

    @property
    def n_p(self) -> int:
        return self.B.shape[1]

    def embedded(self) -> ReducedModel:
        """The saddle system as one ReducedModel of size Nv + Np (zero-padded operators)."""
        nv, npr = self.n_v, self.n_p
        n = nv + npr
        qa, qb = self.A.shape[0], self.B.shape[0]
        A = np.zeros((qa + qb, n, n))
        A[:qa, :nv, :nv] = self.A
        A[qa:, nv:, :nv] = self.B
        A[qa:, :nv, nv:] = self.B.transpose(0, 2, 1)
        C = np.zeros((self.C.shape[0], n, n, n))
        C[:, :nv, :nv, :nv] = self.C
        loads = [np.pad(self.f, ((0, 0), (0, npr)))]
        theta_load = list(self.theta_load)
        if self.fp is not None:
            loads.append(np.pad(self.fp, ((0, 0), (nv, 0))))
            theta_load += list(self.theta_pload)
        # ν multiplies A only: fold it into the divergence descriptors' absence by scaling θ_b / ν is not
        # expressible, so the embedding requires the descriptors to carry ν (nu_linear=False) when B is present
        if self.nu_linear:
            raise ValueError("embed with nu in the a-term descriptors (nu_linear=False): the divergence "
                             "terms are not scaled by ν")
        return ReducedModel(A=A, C=C, f=np.concatenate(loads), name=self.name,
                            theta_linear=list(self.theta_linear) + list(self.theta_div),
                            theta_quadratic=self.theta_quadratic, theta_load=theta_load, nu_linear=False,
                            n_stop=nv, stop_absolute=True,
                            meta={"coupled": True, "n_v": nv, "n_p": npr, "stabilized": self.stabilized})


def split(model: CoupledModel, x: np.ndarray):
    """(u, s, p) coefficient blocks of embedded solutions x (…, Nv + Np)."""
    nv = model.n_v
    m = nv // 2 if model.stabilized else nv
    u = x[..., :m]
    s = x[..., m:nv] if model.stabilized else np.zeros_like(u)
    return u, s, x[..., nv:]


def solve_coupled_batch(model: CoupledModel, mus, tol: float = COUPLED_TOL, max_iter: int = 20, device: int = 0):
    """Batched naive coupled Newton on the GPU; returns (u, s, p, iters, status) as numpy."""
    from . import online

    rm = _embedded_cache(model)
    res = online.device_model(rm, device).solve_host(np.ascontiguousarray(mus, dtype=np.float64), tol=tol,
                                                      max_iter=max_iter, pressure=False)
    u, s, p = split(model, res["u"])
    return u, s, p, res["iters"], res["status"], res["stats"]


def solve_coupled(model: CoupledModel, mu, tol: float = COUPLED_TOL, max_iter: int = 20, device: int = 0):
    """Single query → ReducedSolution; SINGULAR_SYSTEM raises SingularSystemError."""
    import time

    from . import online
    from .errors import SingularSystemError

    t0 = time.perf_counter()
    u, s, p, it, st, stats = solve_coupled_batch(model, np.reshape(mu, (1, 2)), tol, max_iter, device)
    wall = time.perf_counter() - t0
    if st[0] == online.SINGULAR_SYSTEM:
        raise SingularSystemError(f"SINGULAR_SYSTEM in the coupled system at mu={tuple(np.ravel(mu))}")
    return online.ReducedSolution(
        mu=tuple(float(x) for x in np.ravel(mu)), u_coeffs=u[0], s_coeffs=s[0], p_coeffs=p[0],
        newton_iters=int(it[0]), wall_time={"assembly": stats["ms_gemm"] * 1e-3, "solve": stats["ms_lu"] * 1e-3,
                                            "recovery": 0.0, "total": wall},
        converged=int(st[0]) == online.CONVERGED, status=int(st[0]))


_emb: dict = {}


def _embedded_cache(model: CoupledModel) -> ReducedModel:
    rm = _emb.get(id(model))
    if rm is None or rm[0] is not model:
        rm = (model, model.embedded())
        _emb[id(model)] = rm
    return rm[1]
