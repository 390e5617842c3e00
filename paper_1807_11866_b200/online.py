"""Online velocity-only reduced Newton solver on B200 — the SPEC ``online`` module surface.

Host code is Python + PyTorch (device memory, streams); all arithmetic runs in the sm_100a kernels of
``librbns.so`` through the C ABI (include/rbns.h).  There is no CPU fallback: a missing library raises
:class:`~paper_1807_11866_b200.errors.NativeError`.

Public API (names and meaning follow the SPEC):

* :class:`ReducedSolution` — SPEC.md:493-496 (μ, u_coeffs, s_coeffs = 0 for the block solver, p_coeffs,
  newton_iters, wall_time per phase, converged).
* :func:`solve_block` (rm, μ) → ReducedSolution — SPEC.md:520-528; raises SingularSystemError for
  SINGULAR_SYSTEM / SINGULAR_RECOVERY; NON_CONVERGED is reported, not raised.
* :func:`solve_block_batch` (rm, μ[B,2]) → :class:`BatchSolution` — the batch sweep API.
* :func:`reduced_operator` (rm, μ, η) → (residual, Jacobian) — SPEC.md:500-508.
* :func:`reconstruct_pressure` — recovery alone for given velocities (SPEC.md:523 step 2).
* :func:`sweep_report` — the batch sweep's tabular (CSV) report.
* :class:`DeviceModel` — the uploaded, immutable operator handle (one per device), for callers that keep
  tensors on the GPU.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import Dict, Optional, Tuple

import numpy as np
import torch

from . import _native
from .errors import NativeError, SingularSystemError
from .model import ReducedModel

CONVERGED, NON_CONVERGED, SINGULAR_SYSTEM, SINGULAR_RECOVERY, NONFINITE = 0, 1, 2, 3, 4

DEFAULT_TOL = 1e-12       # BASELINE.json: "tolerance 1e-12 relative"
DEFAULT_MAX_ITER = 20     # BASELINE.json: "at most 20 iterations"


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_handle(stream: Optional[torch.cuda.Stream], device: torch.device) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


@dataclass
class ReducedSolution:
    """SPEC.md:493-496."""

    mu: Tuple[float, float]
    u_coeffs: np.ndarray
    s_coeffs: np.ndarray
    p_coeffs: Optional[np.ndarray]
    newton_iters: int
    wall_time: Dict[str, float]
    converged: bool
    status: int = CONVERGED
    last_update: float = float("nan")


@dataclass
class BatchSolution:
    """Batched result; tensors live on the model's device unless produced by the host path."""

    u: torch.Tensor                 # (B, N) fp64
    p: Optional[torch.Tensor]       # (B, Np) fp64 or None
    iters: torch.Tensor             # (B,) int32
    status: torch.Tensor            # (B,) int8
    last_update: torch.Tensor       # (B,) fp64
    stats: Dict[str, float] = field(default_factory=dict)


def _native_desc(model: ReducedModel):
    """rbns_model_desc2 for a model (per-family descriptors, include/rbns.h); returns (desc, keep-alive list)."""
    desc = _native.ModelDesc2C()
    desc.n, desc.n_p = model.n, model.n_p
    desc.flags = ((_native.NU_LINEAR if model.nu_linear else 0)
                  | (_native.STOP_ABSOLUTE if model.stop_absolute else 0))
    desc.n_stop = model.n_stop
    keep = []
    fams = (("linear", model.A), ("quadratic", model.C), ("load", model.f), ("coupling", model.Bq))
    for name, data in fams:
        terms = getattr(model, f"theta_{name}")
        arr = (_native.ThetaTermC * max(1, len(terms)))()
        for i, t in enumerate(terms):
            arr[i] = _native.ThetaTermC(t.kind, t.k, t.m, 0, t.scale)
        keep.append(arr)
        fam = getattr(desc, name)
        fam.count = len(terms) if data is not None else 0
        fam.data = data.ctypes.data if data is not None else None
        fam.theta = arr
    desc.Mp = model.Mp.ctypes.data if model.Mp is not None else None
    return desc, keep


class DeviceModel:
    """Operators of a :class:`ReducedModel` resident on one GPU (rbns_model_create2)."""

    def __init__(self, model: ReducedModel, device: int | torch.device = 0):
        self.lib = _native.load()
        dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        if dev.type != "cuda":
            raise NativeError("DeviceModel needs a CUDA device")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.model = model
        desc, keep = _native_desc(model)
        handle = ctypes.c_void_p()
        _native.check(self.lib.rbns_model_create2(ctypes.byref(desc), dev.index, ctypes.byref(handle)),
                      "rbns_model_create2")
        self._keep = keep
        self._h = handle

    # -- lifecycle --------------------------------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.rbns_model_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def n(self) -> int:
        return self.model.n

    @property
    def n_p(self) -> int:
        return self.model.n_p

    def terms(self) -> dict:
        """Term plan of the device handle: family sizes, contraction blocks, h groups (rbns_model_terms)."""
        c = (ctypes.c_int32 * 6)()
        _native.check(self.lib.rbns_model_terms(self._h, c), "rbns_model_terms")
        return dict(zip(("linear", "quadratic", "load", "coupling", "blocks", "groups"), list(c)))

    def device_bytes(self) -> int:
        return int(self.lib.rbns_model_device_bytes(self._h))

    def stats(self) -> dict:
        st = _native.StatsC()
        _native.check(self.lib.rbns_get_stats(self._h, ctypes.byref(st)), "rbns_get_stats")
        return st.as_dict()

    # -- device-buffer API ------------------------------------------------------------------------------
    def _mu_tensor(self, mu) -> torch.Tensor:
        mu = torch.as_tensor(mu, dtype=torch.float64)
        if mu.ndim == 1:
            mu = mu.reshape(1, 2)
        if mu.ndim != 2 or mu.shape[1] != 2:
            raise ValueError("mu must have shape (B, 2) = (alpha [rad], Re)")
        return mu.to(self.device).contiguous()

    def solve(self, mu, tol: float = DEFAULT_TOL, max_iter: int = DEFAULT_MAX_ITER, pressure: bool = True,
              stream: Optional[torch.cuda.Stream] = None, out: Optional[BatchSolution] = None) -> BatchSolution:
        """Batched solve with device tensors (rbns_solve)."""
        mu = self._mu_tensor(mu)
        b = mu.shape[0]
        want_p = pressure and self.n_p > 0
        if out is None:
            kw = dict(device=self.device)
            out = BatchSolution(
                u=torch.empty((b, self.n), dtype=torch.float64, **kw),
                p=torch.empty((b, self.n_p), dtype=torch.float64, **kw) if want_p else None,
                iters=torch.empty(b, dtype=torch.int32, **kw),
                status=torch.empty(b, dtype=torch.int8, **kw),
                last_update=torch.empty(b, dtype=torch.float64, **kw))
        rc = self.lib.rbns_solve(self._h, mu.data_ptr(), b, float(tol), int(max_iter), out.u.data_ptr(),
                                 _ptr(out.p) if want_p else None, out.iters.data_ptr(), out.status.data_ptr(),
                                 out.last_update.data_ptr(), _stream_handle(stream, self.device))
        _native.check(rc, "rbns_solve")
        out.stats = self.stats()
        return out

    def solve_host(self, mu: np.ndarray, tol: float = DEFAULT_TOL, max_iter: int = DEFAULT_MAX_ITER,
                   pressure: bool = True, stream: Optional[torch.cuda.Stream] = None,
                   out: Optional[dict] = None) -> dict:
        """Batched solve with HOST numpy buffers (rbns_solve_host; copies inside the call)."""
        mu = np.ascontiguousarray(np.atleast_2d(mu), dtype=np.float64)
        b = mu.shape[0]
        want_p = pressure and self.n_p > 0
        if out is None:
            out = dict(u=np.empty((b, self.n)), p=np.empty((b, self.n_p)) if want_p else None,
                       iters=np.empty(b, dtype=np.int32), status=np.empty(b, dtype=np.int8),
                       last_update=np.empty(b))
        rc = self.lib.rbns_solve_host(self._h, mu.ctypes.data, b, float(tol), int(max_iter),
                                      out["u"].ctypes.data, out["p"].ctypes.data if want_p else None,
                                      out["iters"].ctypes.data, out["status"].ctypes.data,
                                      out["last_update"].ctypes.data, _stream_handle(stream, self.device))
        _native.check(rc, "rbns_solve_host")
        out["stats"] = self.stats()
        return out

    def reduced_operator(self, mu, eta, stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
        mu = self._mu_tensor(mu)
        eta = torch.as_tensor(eta, dtype=torch.float64).reshape(mu.shape[0], self.n).to(self.device).contiguous()
        b = mu.shape[0]
        res = torch.empty((b, self.n), dtype=torch.float64, device=self.device)
        jac = torch.empty((b, self.n, self.n), dtype=torch.float64, device=self.device)
        _native.check(self.lib.rbns_reduced_operator(self._h, mu.data_ptr(), eta.data_ptr(), b, res.data_ptr(),
                                                     jac.data_ptr(), _stream_handle(stream, self.device)),
                      "rbns_reduced_operator")
        return res, jac

    def recover_pressure(self, mu, u, stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
        mu = self._mu_tensor(mu)
        b = mu.shape[0]
        u = torch.as_tensor(u, dtype=torch.float64).reshape(b, self.n).to(self.device).contiguous()
        p = torch.empty((b, self.n_p), dtype=torch.float64, device=self.device)
        st = torch.zeros(b, dtype=torch.int8, device=self.device)
        _native.check(self.lib.rbns_recover_pressure(self._h, mu.data_ptr(), u.data_ptr(), b, p.data_ptr(),
                                                     st.data_ptr(), _stream_handle(stream, self.device)),
                      "rbns_recover_pressure")
        return p, st


# ---- model-level convenience API (SPEC names) ------------------------------------------------------------

_cache: Dict[Tuple[int, int], DeviceModel] = {}


def device_model(rm: ReducedModel, device: int = 0) -> DeviceModel:
    """Upload once per (model, device) and reuse (the ReducedModel is immutable)."""
    key = (id(rm), device)
    dm = _cache.get(key)
    if dm is None or dm.model is not rm:
        dm = DeviceModel(rm, device)
        _cache[key] = dm
    return dm


def release_device_models() -> None:
    for dm in _cache.values():
        dm.close()
    _cache.clear()


def solve_block_batch(rm: ReducedModel, mus, tol: float = DEFAULT_TOL, max_iter: int = DEFAULT_MAX_ITER,
                      pressure: bool = True, device: int = 0) -> BatchSolution:
    """Batch sweep over μ samples on the GPU; returns device tensors."""
    return device_model(rm, device).solve(mus, tol=tol, max_iter=max_iter, pressure=pressure)


def solve_block(rm: ReducedModel, mu, tol: float = DEFAULT_TOL, max_iter: int = DEFAULT_MAX_ITER,
                device: int = 0) -> ReducedSolution:
    """Single query.  s = 0 exactly; phase timings from the device events."""
    dm = device_model(rm, device)
    mu_np = np.asarray(mu, dtype=np.float64).reshape(2)
    t0 = time.perf_counter()
    res = dm.solve_host(mu_np.reshape(1, 2), tol=tol, max_iter=max_iter, pressure=rm.n_p > 0)
    wall = time.perf_counter() - t0
    st = int(res["status"][0])
    if st == SINGULAR_SYSTEM:
        raise SingularSystemError(f"SINGULAR_SYSTEM at mu={tuple(mu_np)} after {int(res['iters'][0])} iterations")
    if st == SINGULAR_RECOVERY:
        raise SingularSystemError(f"SINGULAR_RECOVERY at mu={tuple(mu_np)}: pressure Gramian not SPD")
    s = res["stats"]
    return ReducedSolution(
        mu=(float(mu_np[0]), float(mu_np[1])), u_coeffs=res["u"][0].copy(), s_coeffs=np.zeros(rm.n),
        p_coeffs=None if res["p"] is None else res["p"][0].copy(), newton_iters=int(res["iters"][0]),
        wall_time={"assembly": s["ms_gemm"] * 1e-3, "solve": s["ms_lu"] * 1e-3,
                   "recovery": s["ms_recovery"] * 1e-3, "total": wall},
        converged=st == CONVERGED, status=st, last_update=float(res["last_update"][0]))


def reduced_operator(rm: ReducedModel, mu, eta, device: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """(residual, Jacobian) at η, computed by the device contraction."""
    r, j = device_model(rm, device).reduced_operator(np.reshape(mu, (1, 2)), np.reshape(eta, (1, -1)))
    return r[0].cpu().numpy(), j[0].cpu().numpy()


def reconstruct_pressure(rm: ReducedModel, mus, u, device: int = 0) -> torch.Tensor:
    """Pressure recovery for given velocity coefficients."""
    p, _ = device_model(rm, device).recover_pressure(mus, u)
    return p


SWEEP_COLUMNS = ("phi", "u_inf", "solver", "iters", "status", "last_update", "converged",
                 "t_assembly_s", "t_solve_s", "t_recovery_s")


def sweep_report(mus, sol: BatchSolution, path=None, solver: str = "block") -> str:
    """Tabular report of a batch sweep ("batch sweep API over parameter grids returning a tabular
    report (CSV columns: φ, u∞, solver, iters, errors if reference available, phase timings)").  Phase timings
    are the batch's device times divided evenly over its samples.  Deterministic text (fixed column order,
    repr-exact floats); written to ``path`` when given, returned either way."""
    import csv
    import io

    mus = np.asarray(mus.cpu() if isinstance(mus, torch.Tensor) else mus, dtype=np.float64).reshape(-1, 2)
    it = sol.iters.cpu().numpy()
    st = sol.status.cpu().numpy()
    last = sol.last_update.cpu().numpy()
    b = max(1, len(mus))
    per = {k: sol.stats.get(f"ms_{k}", 0.0) * 1e-3 / b for k in ("gemm", "lu", "recovery")}
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    buf.write("# rbflow batch sweep report v1\n")
    w.writerow(SWEEP_COLUMNS)
    names = {CONVERGED: "CONVERGED", NON_CONVERGED: "NON_CONVERGED", SINGULAR_SYSTEM: "SINGULAR_SYSTEM",
             SINGULAR_RECOVERY: "SINGULAR_RECOVERY", NONFINITE: "NONFINITE"}
    for i in range(len(mus)):
        w.writerow([repr(float(mus[i, 0])), repr(float(mus[i, 1])), solver, int(it[i]), names.get(int(st[i]), int(st[i])),
                    repr(float(last[i])), int(st[i]) == CONVERGED, repr(per["gemm"]), repr(per["lu"]),
                    repr(per["recovery"])])
    text = buf.getvalue()
    if path is not None:
        with open(path, "w") as fh:
            fh.write(text)
    return text
