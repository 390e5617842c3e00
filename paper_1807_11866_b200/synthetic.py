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

import numpy as np

from .affine import family
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
               kappa_c: float = 1e-5, name: str = "synthetic") -> ReducedModel:
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
    return ReducedModel(A=A, C=C, f=f, theta=family(theta_family), Mp=Mp, Bq=Bq, name=name,
                        meta={"seed": seed, "kappa_c": kappa_c, "family": theta_family})


def make_mu(batch: int, re_max: float, seed: int = 1, re_min: float = 10.0,
            alpha_max_deg: float = 35.0) -> np.ndarray:
    """μ[b] = (α [rad], Re): α ~ U[0, 35°], Re ~ U[10, re_max] (α drawn first, then Re)."""
    rng = np.random.default_rng(seed)
    alpha = rng.uniform(0.0, np.deg2rad(alpha_max_deg), batch)
    re = rng.uniform(re_min, re_max, batch)
    return np.ascontiguousarray(np.stack([alpha, re], axis=1))


def config_model(cfg: Config | int) -> ReducedModel:
    cfg = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    return make_model(cfg.n, cfg.q, cfg.theta_family, n_p=cfg.n_p, kappa_c=cfg.kappa_c, name=cfg.name)


def config_mu(cfg: Config | int, batch: int | None = None) -> np.ndarray:
    """The config's μ batch; ``batch`` < cfg.batch gives the leading slice of the same seeded stream only
    when drawn with the full size, so slices are always taken from the full draw."""
    cfg = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    mu = make_mu(cfg.batch, cfg.re_max)
    return mu if batch is None else mu[:batch].copy()
