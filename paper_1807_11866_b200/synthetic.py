"""Seeded synthetic reduced models and μ batches for BASELINE.json's configs (no dataset exists for this path).

Generators follow BASELINE.json ``configs`` with the pins of SURVEY.md Appendix B (each a documented
deviation):

* numpy ``default_rng`` (PCG64); operator seed 0, μ seed 1;
* generation order A₀(G) → A₁…A_{Q−1} → C → f [→ H → B_q];
* A₀ = GGᵀ/N + I;  A_{q≥1} = 0.1·(S+Sᵀ)/2/√N  (Appendix B #2: the literal scaling makes A(μ) indefinite);
* C_q = κ_C·N(0,1)/N, then antisymmetrised in (k, l): C ← ½(C − C^{(kl)})  (#1, #3; κ_C = 1e-5);
* f_q ~ N(0,1);  config 4: M_p = HHᵀ/Np + I, B_q ~ N(0,1)/√N  (#7);
* α ~ U[0°, 35°] (radians), Re ~ U[10, 100] (config 0) or U[10, 200] (configs 1–4, #5).
"""

from __future__ import annotations

from dataclasses import dataclass
from math import factorial

import numpy as np

from .affine import MONOMIAL, ThetaTerm, family
from .model import ReducedModel


@dataclass(frozen=True)
class Config:
    index: int
    n: int
    q: int
    batch: int
    theta_family: str
    re_max: float
    n_p: int = 0
    tol: float = 1e-12
    max_iter: int = 20
    kappa_c: float = 1e-5

    @property
    def name(self) -> str:
        s = f"cfg{self.index}: N={self.n}, Q={self.q}, B={self.batch}"
        return s + (f", Np={self.n_p}" if self.n_p else "")


CONFIGS = {
    0: Config(0, 10, 3, 64, "trig3", 100.0),
    1: Config(1, 50, 7, 16384, "trig7", 200.0),
    2: Config(2, 100, 7, 65536, "trig7", 200.0),
    3: Config(3, 200, 13, 131072, "fourier13", 200.0),
    4: Config(4, 100, 7, 65536, "trig7", 200.0, n_p=100),
}


def make_model(n: int, q: int, theta_family: str, n_p: int = 0, seed: int = 0,
               kappa_c: float = 1e-5, name: str = "synthetic", attached: int = 0) -> ReducedModel:
    """BASELINE.json generators (SURVEY.md Appendix B pins).  ``attached`` > 0 adds combined-scheme attached
    pressure modes P_att (attached × n, N(0,1)/√n), drawn after every other array so the other operators are
    unchanged."""
    rng = np.random.default_rng(seed)
    A = np.empty((q, n, n))
    G = rng.standard_normal((n, n))
    A[0] = G @ G.T / n + np.eye(n)
    for i in range(1, q):
        S = rng.standard_normal((n, n))
        A[i] = 0.1 * (S + S.T) / 2.0 / np.sqrt(n)
    C = rng.standard_normal((q, n, n, n))
    C *= kappa_c / n
    C = 0.5 * (C - C.transpose(0, 1, 3, 2))
    f = rng.standard_normal((q, n))
    Mp = Bq = None
    if n_p:
        H = rng.standard_normal((n_p, n_p))
        Mp = H @ H.T / n_p + np.eye(n_p)
        Bq = rng.standard_normal((q, n_p, n)) / np.sqrt(n)
    P_att = rng.standard_normal((attached, n)) / np.sqrt(n) if attached else None
    return ReducedModel(A=A, C=C, f=f, theta=family(theta_family), Mp=Mp, Bq=Bq, name=name, P_att=P_att,
                        meta={"seed": seed, "kappa_c": kappa_c, "family": theta_family, "attached": attached})


def make_mu(batch: int, re_max: float, seed: int = 1, re_min: float = 10.0,
            alpha_max_deg: float = 35.0) -> np.ndarray:
    """μ[b] = (α [rad], Re): α ~ U[0, 35°], Re ~ U[10, re_max] (α drawn first, then Re)."""
    rng = np.random.default_rng(seed)
    alpha = rng.uniform(0.0, np.deg2rad(alpha_max_deg), batch)
    re = rng.uniform(re_min, re_max, batch)
    return np.ascontiguousarray(np.stack([alpha, re], axis=1))


def config_model(cfg: Config | int, attached: bool = False) -> ReducedModel:
    """The config's model; ``attached`` adds n_p (or N) combined-scheme attached pressure modes."""
    cfg = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    return make_model(cfg.n, cfg.q, cfg.theta_family, n_p=cfg.n_p, kappa_c=cfg.kappa_c, name=cfg.name,
                      attached=(cfg.n_p or cfg.n) if attached else 0)


def config_mu(cfg: Config | int, batch: int | None = None) -> np.ndarray:
    """The config's μ batch; ``batch`` < cfg.batch gives the leading slice of the same seeded stream only
    when drawn with the full size, so slices are always taken from the full draw."""
    cfg = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    mu = make_mu(cfg.batch, cfg.re_max)
    return mu if batch is None else mu[:batch].copy()


# ---- the paper's term structure (lifted, Piola formulation) ------------------------------------------------

NU_PAPER = 1.0 / 6.0  # SPEC.md:237 "viscosity was set at ν = 1/6"


def lifted_families(series: int, nu: float = NU_PAPER):
    """Descriptor families of a lifted Piola model at series order n (§5.2):
    linear = a-terms ν·φᵏ/k! (k = 0..4n+2) + c0-terms u∞·φᵏ/k! (k = 0..4n); quadratic = c-terms φᵏ/k!
    (k = 0..4n); load = d0 viscous-lift u∞·φᵏ/k! (k = 0..4n+2) + lift-lift u∞²·φᵏ/k! (k = 0..4n).
    μ = (φ, u∞); the 1/k! scales mirror the truncated rotation series the affine terms come from."""
    ka, kc = 4 * series + 3, 4 * series + 1
    lin = [ThetaTerm(MONOMIAL, k, 0, nu / factorial(k)) for k in range(ka)]
    lin += [ThetaTerm(MONOMIAL, k, 1, 1.0 / factorial(k)) for k in range(kc)]
    quad = [ThetaTerm(MONOMIAL, k, 0, 1.0 / factorial(k)) for k in range(kc)]
    load = [ThetaTerm(MONOMIAL, k, 1, 1.0 / factorial(k)) for k in range(ka)]
    load += [ThetaTerm(MONOMIAL, k, 2, 1.0 / factorial(k)) for k in range(kc)]
    return lin, quad, load


def make_lifted_model(n: int, series: int, seed: int = 0, nu: float = NU_PAPER, kappa_c: float = 5e-5,
                      kappa_0: float = 1e-3, lift2: float = 0.05, n_p: int = 0,
                      name: str = "lifted") -> ReducedModel:
    """Seeded model with the paper's per-form families (no real reduced model ships with the reference; the
    operator values are synthetic, the term structure and μ = (φ, u∞) rules are the paper's).

    Generation order (PCG64 ``seed``): G → A_{k≥1} → c0 terms → C → f (u∞ family, then u∞²) [→ H → B].
    A₀ = GGᵀ/N + I, A_{k≥1} = 0.1·sym(N(0,1))/√N; c0 terms κ₀·N(0,1)/√N (non-symmetric: c(ℓ,u,w)+c(u,ℓ,w));
    C_c = κ_C·N(0,1)/N antisymmetrised in (k,l); u∞ loads N(0,1), u∞² loads lift2·N(0,1)."""
    rng = np.random.default_rng(seed)
    lin_t, quad_t, load_t = lifted_families(series, nu)
    ka, kc = 4 * series + 3, 4 * series + 1
    A = np.empty((ka + kc, n, n))
    G = rng.standard_normal((n, n))
    A[0] = G @ G.T / n + np.eye(n)
    for i in range(1, ka):
        S = rng.standard_normal((n, n))
        A[i] = 0.1 * (S + S.T) / 2.0 / np.sqrt(n)
    A[ka:] = kappa_0 * rng.standard_normal((kc, n, n)) / np.sqrt(n)
    C = rng.standard_normal((kc, n, n, n))
    C *= kappa_c / n
    C = 0.5 * (C - C.transpose(0, 1, 3, 2))
    f = np.concatenate([rng.standard_normal((ka, n)), lift2 * rng.standard_normal((kc, n))])
    Mp = Bq = None
    coupling = None
    if n_p:
        H = rng.standard_normal((n_p, n_p))
        Mp = H @ H.T / n_p + np.eye(n_p)
        Bq = rng.standard_normal((kc, n_p, n)) / np.sqrt(n)
        coupling = quad_t
    return ReducedModel(A=A, C=C, f=f, Mp=Mp, Bq=Bq, name=name, theta_linear=lin_t, theta_quadratic=quad_t,
                        theta_load=load_t, theta_coupling=coupling, nu_linear=False,
                        meta={"seed": seed, "series": series, "nu": nu, "kappa_c": kappa_c, "kappa_0": kappa_0,
                              "lift2": lift2, "form": "lifted-piola"})


def make_lifted_mu(batch: int, seed: int = 1, phi_max_deg: float = 35.0, uinf=(1.0, 20.0)) -> np.ndarray:
    """μ[b] = (φ [rad], u∞): φ ~ U[−35°, 35°], u∞ ~ U[1, 20] (the paper's parameter box)."""
    rng = np.random.default_rng(seed)
    phi = rng.uniform(-np.deg2rad(phi_max_deg), np.deg2rad(phi_max_deg), batch)
    u = rng.uniform(uinf[0], uinf[1], batch)
    return np.ascontiguousarray(np.stack([phi, u], axis=1))


def make_coupled_model(m: int, series: int, stabilized: bool = True, seed: int = 0, kappa_s: float = 0.1):
    """Saddle-system blocks for the naive coupled solvers around the lifted velocity model
    ``make_lifted_model(m, series, seed)`` — its (A, C, f) are the velocity-velocity blocks verbatim.

    Div-conforming structure (Eq. (piolablock)): the velocity modes are solenoidal, so the
    velocity-pressure block B_pu is exactly zero; the supremizer-pressure block B_ps (Np = m) is regular.
    Stabilised (v = (u, s), size 3m): extra supremizer blocks A_us, A_su, A_ss (A_ss[0] = HHᵀ/m + I), mixed
    convective entries κ_C-sized, supremizer loads f_s; b-terms φᵏ/k! (k = 0..4n) with B_ps[0] = I + 0.3·G/√m.
    Unstabilised (v = u, size 2m): B = B_pu = 0 — the machine-zero inf-sup case that must fail gracefully.
    Returns (CoupledModel, the block ReducedModel)."""
    from .coupled import CoupledModel

    block = make_lifted_model(m, series, seed=seed)
    lin_t, quad_t, load_t = block.theta_linear, block.theta_quadratic, block.theta_load
    qa, qc, qf = block.counts[:3]
    div_t = [ThetaTerm(MONOMIAL, k, 0, 1.0 / factorial(k)) for k in range(4 * series + 1)]
    rng = np.random.default_rng(seed + 1000)
    if not stabilized:
        return CoupledModel(A=block.A, B=np.zeros((len(div_t), m, m)), C=block.C, f=block.f, theta_linear=lin_t,
                            theta_div=div_t, theta_quadratic=quad_t, theta_load=load_t, nu_linear=False,
                            stabilized=False, name=f"coupled-2M-{m}"), block
    nv = 2 * m
    A = np.zeros((qa, nv, nv))
    A[:, :m, :m] = block.A
    A[:, :m, m:] = kappa_s * rng.standard_normal((qa, m, m)) / np.sqrt(m) * 0.1
    A[:, m:, :m] = A[:, :m, m:].transpose(0, 2, 1)
    H = rng.standard_normal((m, m))
    A[0, m:, m:] = H @ H.T / m + np.eye(m)
    A[1:, m:, m:] = 0.1 * kappa_s * rng.standard_normal((qa - 1, m, m)) / np.sqrt(m)
    kc = block.meta["kappa_c"]
    C = rng.standard_normal((qc, nv, nv, nv)) * (kc / nv)
    C = 0.5 * (C - C.transpose(0, 1, 3, 2))
    C[:, :m, :m, :m] = block.C
    f = np.concatenate([block.f, rng.standard_normal((qf, m))], axis=1)
    B = np.zeros((len(div_t), m, nv))
    B[:, :, m:] = 0.1 * rng.standard_normal((len(div_t), m, m)) / np.sqrt(m)
    B[0, :, m:] = np.eye(m) + 0.3 * rng.standard_normal((m, m)) / np.sqrt(m)
    return CoupledModel(A=A, B=B, C=C, f=f, theta_linear=lin_t, theta_div=div_t, theta_quadratic=quad_t,
                        theta_load=load_t, nu_linear=False, stabilized=True, name=f"coupled-3M-{m}"), block
