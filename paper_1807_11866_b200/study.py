"""Accuracy and timing studies over the batched device solver — SPEC.md:620-638 ``error_study`` /
``timing_study``, SURVEY.md §8(f) row 4 (with ``lift.Lifter``).

``error_study`` takes the high-fidelity side as a *reference ensemble* ("reference ensemble or
on-the-fly high-fidelity"): high-fidelity solutions U_ref at the test parameters, the reduced basis V and the
Gram matrix G of the error norm (H1-semi for velocity).  The reference's high-fidelity solver and
POD stage are offline and out of this repo's scope (SURVEY.md §8 / DESIGN.md §8), so the studies here consume
their outputs; ``pod`` and ``galerkin_project`` are the small offline helpers (method of snapshots, SPEC.md:436-446;
Galerkin projection of an algebraic high-fidelity system) that turn a high-fidelity model and
its snapshots into a ReducedModel, all on the GPU.

    error_study:  solve the reduced model on the test grid (one batched device solve), lift through V
                  (u_h = V u [+ u∞ ℓ]), relative G-norm errors per query, mean over the converged queries,
                  unconverged queries excluded and counted, paired with the expected error ε(M)
                  of the basis (PAPER Eq. (error)).
    timing_study: per-solver mean device wall time per query over the same grid (block vs
                  combined vs coupled, the latter via coupled.solve_coupled_batch).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Callable, Dict, Optional, Sequence

import numpy as np
import torch

from .errors import NativeError
from .lift import Lifter, lifted_error
from .model import ReducedModel


def _cuda(device) -> torch.device:
    d = torch.device(device if not isinstance(device, int) else f"cuda:{device}")
    if d.type != "cuda":
        raise NativeError("the studies run on the GPU (no CPU path)")
    return d


def _t(x, device) -> torch.Tensor:
    return torch.as_tensor(np.array(x, dtype=np.float64) if isinstance(x, np.ndarray) else x,
                           dtype=torch.float64, device=device)


def pod(snapshots, G=None, M: Optional[int] = None, eps: Optional[float] = None, device=0):
    """Method of snapshots: covariance K = Y G Yᵀ of the S snapshots (rows of Y), K = Σ λ v vᵀ,
    ψ_j = λ_j^{-1/2} Σ_i v_ji Y_i (G-orthonormal).  Fixed-M mode keeps M modes; energy mode (eps) the smallest M
    with Σ_{j≤M} λ_j ≥ (1−ε²) Σ λ_j.  Returns (V (n_h × M) numpy, λ (descending), realized ε(M))."""
    dev = _cuda(device)
    Y = _t(snapshots, dev)
    YG = Y if G is None else Y @ _t(G, dev)
    K = YG @ Y.T
    K = 0.5 * (K + K.T)
    lam, vec = torch.linalg.eigh(K)
    order = torch.argsort(-lam, stable=True)  # descending, ties by ascending index (SPEC.md: determinism)
    lam, vec = lam[order], vec[:, order]
    total = float(lam.clamp(min=0).sum())
    rank = int((lam > 1e-14 * lam[0]).sum())
    if M is None:
        if eps is None:
            raise ValueError("give M or eps")
        cum = torch.cumsum(lam.clamp(min=0), 0)
        M = min(int((cum < (1.0 - eps * eps) * total).sum()) + 1, rank)  # ε below round-off: every mode kept
    if M > rank:
        raise ValueError(f"requested M = {M} exceeds the numerical rank {rank}")
    V = (Y.T @ vec[:, :M]) / torch.sqrt(lam[:M])[None, :]
    tail = float(lam[M:].clamp(min=0).sum())
    return V.cpu().numpy(), lam.cpu().numpy(), math.sqrt(max(tail, 0.0) / total)


def galerkin_project(hifi: ReducedModel, V, device=0, name: Optional[str] = None) -> ReducedModel:
    """Galerkin projection of an algebraic high-fidelity model of the same form (linear, quadratic and load
    families with their descriptors) onto the basis V (n_h × M): A_r = Vᵀ A V, C_r[j,k,l] = Σ C[a,b,c] V_aj V_bk V_cl,
    f_r = Vᵀ f (cuBLAS DGEMMs on the GPU)."""
    dev = _cuda(device)
    Vt = _t(V, dev)
    nh, m = Vt.shape
    if hifi.n != nh:
        raise ValueError(f"basis rows {nh} != high-fidelity dimension {hifi.n}")
    A = torch.stack([Vt.T @ _t(a, dev) @ Vt for a in hifi.A])
    Cs = []
    for c in hifi.C:
        ct = _t(c, dev).reshape(nh, nh * nh)
        t1 = (Vt.T @ ct).reshape(m, nh, nh)                          # [j, b, c]
        t2 = torch.einsum("jbc,bk->jkc", t1, Vt)                     # [j, k, c]
        Cs.append(torch.einsum("jkc,cl->jkl", t2, Vt))
    f = _t(hifi.f, dev) @ Vt
    return replace(hifi, A=A.cpu().numpy(), C=torch.stack(Cs).cpu().numpy(), f=f.cpu().numpy(),
                   Mp=None, Bq=None, P_att=None, name=name or f"{hifi.name}-galerkin{m}",
                   meta=dict(hifi.meta, galerkin_basis=m))


@dataclass
class ErrorReport:
    n_queries: int
    n_unconverged: int
    mean_velocity_error: float
    max_velocity_error: float
    expected_error: Optional[float]
    mean_pressure_error: Optional[float] = None
    velocity_errors: np.ndarray = field(default_factory=lambda: np.zeros(0), repr=False)
    mean_ms_per_query: float = 0.0

    def row(self, m: int) -> str:
        pe = "" if self.mean_pressure_error is None else f"{self.mean_pressure_error:.6e}"
        ex = "" if self.expected_error is None else f"{self.expected_error:.6e}"
        return (f"{m},{self.n_queries},{self.n_unconverged},{self.mean_velocity_error:.6e},{pe},{ex},"
                f"{self.mean_ms_per_query:.6f}")


CSV_HEADER = "M,queries,unconverged,mean_rel_velocity_error,mean_rel_pressure_error,expected_error,ms_per_query"


def error_study(rm: ReducedModel, mus, U_ref, V, G=None, ell=None, P_ref=None, P_basis=None, Gp=None,
                expected: Optional[float] = None, device=0, tol: float = 1e-12, max_iter: int = 20) -> ErrorReport:
    """Mean relative G-norm velocity error (and L2/Gp pressure error when P_ref and P_basis are given) of the
    reduced model against the high-fidelity reference ensemble U_ref (B × n_h) at μ = mus (B × 2)."""
    from .online import DeviceModel  # the device solver (C ABI)

    dev = _cuda(device)
    mus = np.ascontiguousarray(mus, dtype=np.float64)
    U_ref = np.asarray(U_ref, dtype=np.float64)
    if U_ref.shape != (len(mus), np.asarray(V).shape[0]):
        raise ValueError("U_ref must be (queries × high-fidelity dofs)")
    want_p = P_ref is not None and P_basis is not None and rm.n_p > 0
    with torch.cuda.device(dev), DeviceModel(rm, dev.index) as dm:
        mu_d = _t(mus, dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sol = dm.solve(mu_d, tol=tol, max_iter=max_iter, pressure=want_p)
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        ok = sol.status == 0
        lifter = Lifter(V, np.zeros(np.asarray(V).shape[0]) if ell is None else ell, P_basis, device=dev)
        uinf = mu_d[:, 1] if ell is not None else torch.zeros(len(mus), dtype=torch.float64, device=dev)
        U, Ph = lifter.lift(sol.u[ok], uinf[ok], sol.p[ok] if want_p else None)
        err = lifted_error(U, _t(U_ref, dev)[ok], G, device=dev)
        perr = None
        if want_p:
            perr = float(lifted_error(Ph, _t(P_ref, dev)[ok], Gp, device=dev).mean())
    n_bad = int((~ok).sum())
    errs = err.cpu().numpy()
    return ErrorReport(len(mus), n_bad, float(errs.mean()) if errs.size else float("nan"),
                       float(errs.max()) if errs.size else float("nan"), expected, perr, errs, ms / len(mus))


def timing_study(solvers: Dict[str, Callable[[torch.Tensor], object]], mus, device=0, repeats: int = 3
                 ) -> Dict[str, float]:
    """Mean device wall time per query (ms) of each solver callable over the same μ grid:
    one warm-up call, then the best of ``repeats`` timed calls, CUDA events on the current stream."""
    dev = _cuda(device)
    mu_d = _t(mus, dev)
    out = {}
    for name, fn in solvers.items():
        fn(mu_d)
        best = float("inf")
        for _ in range(repeats):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record()
            fn(mu_d)
            e1.record()
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1))
        out[name] = best / len(mus)
    return out


def loglog_slope(x: Sequence[float], y: Sequence[float]) -> float:
    """Least-squares slope of log y against log x (measured vs expected error)."""
    lx, ly = np.log(np.asarray(x, dtype=float)), np.log(np.asarray(y, dtype=float))
    return float(np.polyfit(lx, ly, 1)[0])
