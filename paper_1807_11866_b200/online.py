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
* :func:`query` (model, μ, solver) → :class:`ReducedSolution` — the query API over the block,
  combined (:func:`solve_combined`) and coupled solvers.
* :func:`reduced_operator` (rm, μ, η) → (residual, Jacobian) — SPEC.md:500-508.
* :func:`recover_pressure` — a-posteriori recovery alone for given velocities (SPEC.md:523 step 2).
* :func:`reconstruct_pressure` (rm, u_coeffs) → p_coeffs — the combined scheme's reconstruction from the
  model's attached pressure modes, p = P_att u.
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
from .errors import NativeError, RbflowError, SingularSystemError
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
    desc.n_att = model.n_att
    desc.P_att = model.P_att.ctypes.data if model.P_att is not None else None
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

    @property
    def n_att(self) -> int:
        return self.model.n_att

    def terms(self) -> dict:
        """Term plan of the device handle: family sizes, contraction blocks, h groups (rbns_model_terms)."""
        c = (ctypes.c_int32 * 6)()
        _native.check(self.lib.rbns_model_terms(self._h, c), "rbns_model_terms")
        return dict(zip(("linear", "quadratic", "load", "coupling", "blocks", "groups"), list(c)))

    def device_bytes(self) -> int:
        return int(self.lib.rbns_model_device_bytes(self._h))

    def contraction_slices(self) -> int:
        """0: the FP64 DMMA contraction; s > 0: the tcgen05 INT8 contraction over s slices per entry (default)."""
        return int(self.lib.rbns_model_contraction_slices(self._h))

    def stats(self) -> dict:
        """Statistics of the most recent solve on this handle (per-call numbers are in BatchSolution.stats)."""
        st = _native.StatsC()
        _native.check(self.lib.rbns_get_stats(self._h, ctypes.byref(st)), "rbns_get_stats")
        return st.as_dict()

    def _check_out(self, out: BatchSolution, b: int, want_p: bool) -> None:
        """A caller-supplied ``out`` must hold the batch: shapes, dtypes, this device, contiguous; p when
        pressure is requested (the kernels write every row, so a short or strided buffer would be overrun)."""
        specs = (("u", out.u, (self.n,), torch.float64), ("iters", out.iters, (), torch.int32),
                 ("status", out.status, (), torch.int8), ("last_update", out.last_update, (), torch.float64))
        if want_p:
            if out.p is None:
                raise ValueError("pressure requested but out.p is None")
            specs += (("p", out.p, (self.n_p,), torch.float64),)
        for name, t, tail, dt in specs:
            if not isinstance(t, torch.Tensor):
                raise ValueError(f"out.{name} must be a torch tensor")
            if t.dim() != 1 + len(tail) or t.shape[0] < b or tuple(t.shape[1:]) != tail:
                raise ValueError(f"out.{name} has shape {tuple(t.shape)}, need ({b}+{''.join(', ' + str(x) for x in tail)})")
            if t.dtype != dt:
                raise ValueError(f"out.{name} has dtype {t.dtype}, need {dt}")
            if t.device != self.device:
                raise ValueError(f"out.{name} is on {t.device}, the model is on {self.device}")
            if not t.is_contiguous():
                raise ValueError(f"out.{name} must be contiguous")

    def _check_host_out(self, out: dict, b: int, want_p: bool) -> None:
        specs = (("u", (self.n,), np.float64), ("iters", (), np.int32), ("status", (), np.int8),
                 ("last_update", (), np.float64))
        if want_p:
            specs += (("p", (self.n_p,), np.float64),)
        for name, tail, dt in specs:
            a = out.get(name)
            if not isinstance(a, np.ndarray):
                raise ValueError(f"out[{name!r}] must be a numpy array")
            if a.ndim != 1 + len(tail) or a.shape[0] < b or tuple(a.shape[1:]) != tail or a.dtype != dt:
                raise ValueError(f"out[{name!r}] is {a.dtype}{a.shape}, need {np.dtype(dt)}({b}, ...{tail})")
            if not a.flags.c_contiguous:
                raise ValueError(f"out[{name!r}] must be C-contiguous")

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
        else:
            self._check_out(out, b, want_p)
        st = _native.StatsC()
        rc = self.lib.rbns_solve_ex(self._h, mu.data_ptr(), b, float(tol), int(max_iter), out.u.data_ptr(),
                                    _ptr(out.p) if want_p else None, out.iters.data_ptr(), out.status.data_ptr(),
                                    out.last_update.data_ptr(), ctypes.byref(st), _stream_handle(stream, self.device))
        _native.check(rc, "rbns_solve_ex")
        out.stats = st.as_dict()
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
        else:
            self._check_host_out(out, b, want_p)
        st = _native.StatsC()
        rc = self.lib.rbns_solve_host_ex(self._h, mu.ctypes.data, b, float(tol), int(max_iter),
                                         out["u"].ctypes.data, out["p"].ctypes.data if want_p else None,
                                         out["iters"].ctypes.data, out["status"].ctypes.data,
                                         out["last_update"].ctypes.data, ctypes.byref(st),
                                         _stream_handle(stream, self.device))
        _native.check(rc, "rbns_solve_host_ex")
        out["stats"] = st.as_dict()
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

    def reconstruct_pressure(self, u, stream=None) -> torch.Tensor:
        """Combined-scheme reconstruction p = P_att u (rbns_reconstruct_pressure)."""
        if not self.n_att:
            raise RbflowError("reconstruct_pressure: the reduced model carries no attached pressure modes "
                              "(combined scheme, SPEC.md:530-538)")
        u = torch.as_tensor(u, dtype=torch.float64).to(self.device)
        u = u.reshape(-1, self.n).contiguous()
        b = u.shape[0]
        p = torch.empty((b, self.n_att), dtype=torch.float64, device=self.device)
        _native.check(self.lib.rbns_reconstruct_pressure(self._h, u.data_ptr(), b, p.data_ptr(),
                                                         _stream_handle(stream, self.device)),
                      "rbns_reconstruct_pressure")
        return p


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


def _phase_times(stats: dict) -> Dict[str, float]:
    """SPEC phase timings (seconds) from one call's device statistics: assembly = the u = 0 affine assembly plus
    the contraction launches (θ-weighted assembly of J fused with the convective contraction), solve = the
    Newton-update kernels, recovery = pressure recovery / reconstruction."""
    return {"assembly": (stats.get("ms_assembly", 0.0) + stats.get("ms_gemm", 0.0)) * 1e-3,
            "solve": stats.get("ms_lu", 0.0) * 1e-3, "recovery": stats.get("ms_recovery", 0.0) * 1e-3}


def _merge_stats(parts) -> dict:
    out = {}
    for st in parts:
        for k, v in st.items():
            if k.startswith("ms_") or k == "newton_rounds":
                out[k] = max(out.get(k, 0), v)  # devices run concurrently: wall-clock phase = slowest device
            else:
                out[k] = out.get(k, 0) + v
    return out


def solve_block_batch(rm: ReducedModel, mus, tol: float = DEFAULT_TOL, max_iter: int = DEFAULT_MAX_ITER,
                      pressure: bool | str = True, device: int = 0, devices=None) -> BatchSolution:
    """Batch sweep over μ samples on the GPU; returns device tensors.

    ``pressure``: True / "recovery" (the block solver's a-posteriori recovery), "combined" (the
    combined scheme: velocity solve, then p = P_att u from the attached modes), False / "none".
    ``devices``: several GPUs (μ-sharded, one host thread and one model handle per device, no collective;
    SURVEY.md §8(e)); the result is gathered on ``devices[0]``.  Per-sample results are bit-identical to a
    single-device solve (each sample's arithmetic is independent of the batch it is in)."""
    mode = {True: "recovery", False: "none", None: "none"}.get(pressure, pressure)
    if mode not in ("recovery", "combined", "none"):
        raise ValueError(f"pressure={pressure!r}: use 'recovery', 'combined' or 'none'")
    devs = list(devices) if devices else [device]
    mus_t = torch.as_tensor(mus, dtype=torch.float64).reshape(-1, 2)

    def run(dev, mu_part):
        dm = device_model(rm, dev)
        sol = dm.solve(mu_part.to(dm.device), tol=tol, max_iter=max_iter, pressure=mode == "recovery")
        if mode == "combined":
            stream = torch.cuda.current_stream(dm.device)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sol.p = dm.reconstruct_pressure(sol.u, stream=stream)
            e1.record(stream)
            e1.synchronize()
            sol.stats["ms_recovery"] = e0.elapsed_time(e1)
        return sol

    if len(devs) == 1:
        return run(devs[0], mus_t)
    from concurrent.futures import ThreadPoolExecutor

    from .sharding import shard_bounds

    bounds = [shard_bounds(mus_t.shape[0], len(devs), r) for r in range(len(devs))]
    with ThreadPoolExecutor(len(devs)) as ex:  # ctypes releases the GIL during every library call
        parts = list(ex.map(lambda i: run(devs[i], mus_t[bounds[i][0]:bounds[i][1]]), range(len(devs))))
    home = torch.device("cuda", devs[0])
    cat = lambda name: torch.cat([getattr(s, name).to(home) for s in parts])  # noqa: E731  (NVLink peer copies)
    return BatchSolution(u=cat("u"), p=None if parts[0].p is None else cat("p"), iters=cat("iters"),
                         status=cat("status"), last_update=cat("last_update"),
                         stats=_merge_stats([s.stats for s in parts]))


def solve_block(rm: ReducedModel, mu, tol: float = DEFAULT_TOL, max_iter: int = DEFAULT_MAX_ITER,
                device: int = 0) -> ReducedSolution:
    """Single query.  s = 0 exactly; phase timings from the device events of this call."""
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
    wt = _phase_times(res["stats"])
    wt["total"] = wall
    return ReducedSolution(
        mu=(float(mu_np[0]), float(mu_np[1])), u_coeffs=res["u"][0].copy(), s_coeffs=np.zeros(rm.n),
        p_coeffs=None if res["p"] is None else res["p"][0].copy(), newton_iters=int(res["iters"][0]),
        wall_time=wt, converged=st == CONVERGED, status=st, last_update=float(res["last_update"][0]))


def solve_combined(rm: ReducedModel, mu, tol: float = DEFAULT_TOL, max_iter: int = DEFAULT_MAX_ITER,
                   device: int = 0) -> ReducedSolution:
    """Single query of the combined scheme: the block velocity solve without
    the recovery solve, then p = P_att u from the model's attached pressure modes."""
    if rm.P_att is None:
        raise RbflowError("solve_combined: the reduced model carries no attached pressure modes "
                          "(built without the combined flag, SPEC.md:449)")
    dm = device_model(rm, device)
    mu_np = np.asarray(mu, dtype=np.float64).reshape(2)
    t0 = time.perf_counter()
    res = dm.solve_host(mu_np.reshape(1, 2), tol=tol, max_iter=max_iter, pressure=False)
    t1 = time.perf_counter()
    st = int(res["status"][0])
    if st == SINGULAR_SYSTEM:
        raise SingularSystemError(f"SINGULAR_SYSTEM at mu={tuple(mu_np)} after {int(res['iters'][0])} iterations")
    p = reconstruct_pressure(rm, res["u"][0], device)
    wt = _phase_times(res["stats"])
    wt["recovery"] = time.perf_counter() - t1
    wt["total"] = time.perf_counter() - t0
    return ReducedSolution(
        mu=(float(mu_np[0]), float(mu_np[1])), u_coeffs=res["u"][0].copy(), s_coeffs=np.zeros(rm.n),
        p_coeffs=p, newton_iters=int(res["iters"][0]), wall_time=wt, converged=st == CONVERGED, status=st,
        last_update=float(res["last_update"][0]))


SOLVERS = ("block", "combined", "coupled")


def query(model, mu, solver: str = "block", device: int = 0, **kw) -> ReducedSolution:
    """The Query API: (μ, solver kind) → ReducedSolution.  ``solver``: "block" (velocity-only
    Newton + a-posteriori pressure recovery), "combined" (block velocity + reconstruction from the
    attached modes) or "coupled" (the stabilised coupled-3M system; ``model`` is then
    a ``coupled.CoupledModel``)."""
    if solver == "block":
        return solve_block(model, mu, device=device, **kw)
    if solver == "combined":
        return solve_combined(model, mu, device=device, **kw)
    if solver == "coupled":
        from .coupled import CoupledModel, solve_coupled

        if not isinstance(model, CoupledModel):
            raise TypeError("solver='coupled' needs a coupled.CoupledModel")
        return solve_coupled(model, mu, device=device, **kw)
    raise ValueError(f"solver={solver!r}: use one of {SOLVERS}")


def reduced_operator(rm: ReducedModel, mu, eta, device: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """(residual, Jacobian) at η, computed by the device contraction."""
    r, j = device_model(rm, device).reduced_operator(np.reshape(mu, (1, 2)), np.reshape(eta, (1, -1)))
    return r[0].cpu().numpy(), j[0].cpu().numpy()


def recover_pressure(rm: ReducedModel, mus, u, device: int = 0) -> torch.Tensor:
    """A-posteriori pressure recovery for given velocity coefficients: B_sp p = f_s − A_sv u (SPEC.md:523,
    PAPER.md:905-908); the config-4 form M_p p = Σ_q θ_q(μ) B_q u."""
    p, _ = device_model(rm, device).recover_pressure(mus, u)
    return p


def reconstruct_pressure(rm: ReducedModel, u_coeffs, device: int = 0):
    """p_coeffs = u_coeffs applied to the model's attached pressure modes (combined scheme,
    PAPER.md:941-986), p = P_att u, on the device.  One state (N,) gives (n_att,) numpy; a batch (B, N) gives
    (B, n_att) — numpy for numpy input, a device tensor for tensor input.  Raises RbflowError when the model
    carries no attached modes ("errors: rm lacks attached modes")."""
    if rm.P_att is None:
        raise RbflowError("reconstruct_pressure: the reduced model carries no attached pressure modes "
                          "(built without the combined flag, SPEC.md:449)")
    p = device_model(rm, device).reconstruct_pressure(u_coeffs)
    if isinstance(u_coeffs, torch.Tensor):
        return p if u_coeffs.dim() > 1 else p[0]
    out = p.cpu().numpy()
    return out if np.ndim(u_coeffs) > 1 else out[0]


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
    per = {k: v / b for k, v in _phase_times(sol.stats).items()}
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    buf.write("# rbflow batch sweep report v1\n")
    w.writerow(SWEEP_COLUMNS)
    names = {CONVERGED: "CONVERGED", NON_CONVERGED: "NON_CONVERGED", SINGULAR_SYSTEM: "SINGULAR_SYSTEM",
             SINGULAR_RECOVERY: "SINGULAR_RECOVERY", NONFINITE: "NONFINITE"}
    for i in range(len(mus)):
        w.writerow([repr(float(mus[i, 0])), repr(float(mus[i, 1])), solver, int(it[i]), names.get(int(st[i]), int(st[i])),
                    repr(float(last[i])), int(st[i]) == CONVERGED, repr(per["assembly"]), repr(per["solve"]),
                    repr(per["recovery"])])
    text = buf.getvalue()
    if path is not None:
        with open(path, "w") as fh:
            fh.write(text)
    return text
