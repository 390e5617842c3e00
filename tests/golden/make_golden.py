"""Generate the committed golden fixtures (run in the development container, where /root/reference exists).

    python tests/golden/make_golden.py

1. ``reference_operator.npz`` — pins the oracle's reduced operator to the REFERENCE's own code.  A small reduced
   model is assembled with the reference package's quadrature assembler (/root/reference/pkg/src/rbflow:
   geometry.build_omesh, spaces.build_space_pair(DIV_CONFORMING), assemble.deformed_tables "piola",
   assemble.viscous_matrix, assemble.convection_matrices) and a random orthonormal reduced basis V:
       A_q = Vᵀ A_h(φ_q) V,  C_q[j,k,l] = V_lᵀ N1_h(φ_q; V_j) V_k   (assemble.py:86-101)
   with two affine terms, θ = (1, α/φ₁) (monomials) interpolating the direct assembly at
   φ₀ = 0 and φ₁ = 20°, so the reduced model is exact at α ∈ {0, φ₁}.  At those α the fixture stores the
   reference-side reduced residual and Jacobian computed from the HIGH-FIDELITY forms:
       R = ν Vᵀ A_h V η + Vᵀ N1_h(Vη) V η − f(μ),   J = ν Vᵀ A_h V + Vᵀ (N1_h + N2_h)(Vη) V
   (assemble.py:86-101 docstring: "the Newton Jacobian block is their sum, the residual contribution N1 @ coeffs").
2. ``synthetic_cfg{0..4}.npz`` — seeded BASELINE.json configs (SURVEY.md Appendix B pins): μ slices, oracle
   velocity/pressure, Newton counts and statuses, plus operator checksums that detect generator drift.
4. ``projection_ref.npz`` — reduced-basis tabulations at the quadrature points of a small deformed mesh (from the
   reference's ``deformed_tables`` / ``field_at_quadrature``) and the reference's own projected operators
   V_lᵀ N1(V_j) V_k and Vᵀ A_h V (``convection_matrices`` / ``viscous_matrix`` + sparse products): the pin for
   the GPU projection (paper_1807_11866_b200/projection.py).
3. ``lifted_small.npz`` / ``lifted_n12.npz`` — seeded models with the paper's per-form term families
   (synthetic.make_lifted_model: a + c0 linear, c quadratic, d0 u∞/u∞² loads; μ = (φ, u∞)), the small one with
   pressure recovery on its own coupling family.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
REF_SRC = Path("/root/reference/pkg/src")

from oracle import rbns_oracle as oracle  # noqa: E402
from paper_1807_11866_b200 import affine, synthetic  # noqa: E402
from paper_1807_11866_b200.model import ReducedModel  # noqa: E402


def reference_operator_fixture(m: int = 8, seed: int = 7) -> None:
    sys.path.insert(0, str(REF_SRC))
    from rbflow import assemble, geometry, instrument, spaces  # the reference package (read-only import)

    prof = geometry.naca_profile(0.15, 24)
    mesh = geometry.build_omesh(prof, 6.0, 24, 8, 1.15)
    space = spaces.build_space_pair(mesh, spaces.DIV_CONFORMING)
    geom = geometry.DeformedGeometry()
    rng = np.random.default_rng(seed)
    free = space.free_v
    V = np.zeros((space.n_vdofs, m))
    Qm, _ = np.linalg.qr(rng.standard_normal((free.size, m)))
    V[free] = Qm

    phis = [0.0, math.radians(20.0)]
    tables = [assemble.deformed_tables(space, geom, ph, "piola") for ph in phis]
    A_h = [assemble.viscous_matrix(space, dg, 1.0) for (_, dg) in tables]

    def conv(tab, coeffs):
        dval, dgrad = tab
        return assemble.convection_matrices(space, dval, dgrad, coeffs)

    # reduced operators per angle, then the two affine terms (value at φ0, difference to φ1)
    Ar = [V.T @ (A @ V) for A in A_h]
    Cr = []
    for tab in tables:
        C = np.empty((m, m, m))
        for j in range(m):
            N1, _ = conv(tab, V[:, j])
            C[j] = (V.T @ (N1 @ V)).T          # C[j, k, l] = V_lᵀ N1(V_j) V_k
        Cr.append(C)
    f_h = rng.standard_normal((2, space.n_vdofs))
    f_h[:, ~np.isin(np.arange(space.n_vdofs), free)] = 0.0
    fr = [V.T @ f_h[0], V.T @ f_h[1]]
    A = np.stack([Ar[0], Ar[1] - Ar[0]])
    C = np.stack([Cr[0], Cr[1] - Cr[0]])
    f = 0.3 * np.stack([fr[0], fr[1] - fr[0]])
    theta = [affine.ThetaTerm(affine.MONOMIAL, 0, 0, 1.0), affine.ThetaTerm(affine.MONOMIAL, 1, 0, 1.0 / phis[1])]
    model = ReducedModel(A=A, C=C, f=f, theta=theta, name="reference-assembled")

    mus, etas, Rs, Js = [], [], [], []
    for ai, alpha in enumerate(phis):
        for re in (2.0, 10.0):
            for _ in range(2):
                eta = 0.5 * rng.standard_normal(m)
                nu = 1.0 / re
                U = V @ eta
                N1, N2 = conv(tables[ai], U)
                th = affine.evaluate_weights(theta, np.array([[alpha, re]]))[0]
                fmu = th @ f
                R = nu * (V.T @ (A_h[ai] @ U)) + V.T @ (N1 @ U) - fmu
                J = nu * (V.T @ (A_h[ai] @ V)) + V.T @ ((N1 + N2) @ V)
                mus.append([alpha, re]), etas.append(eta), Rs.append(R), Js.append(J)
    # reduced Newton solutions (oracle) and the Galerkin-orthogonality residual from the direct assembly
    solve_mu = np.array([[phis[0], 3.0], [phis[1], 3.0], [phis[1], 8.0], [phis[0], 8.0]])
    us, its, sts, gal = [], [], [], []
    for mu in solve_mu:
        u, it, st, _ = oracle.solve_sample(model, mu)
        ai = phis.index(mu[0])
        U = V @ u
        N1, _ = conv(tables[ai], U)
        th = affine.evaluate_weights(theta, mu[None])[0]
        r = (1.0 / mu[1]) * (V.T @ (A_h[ai] @ U)) + V.T @ (N1 @ U) - th @ f
        us.append(u), its.append(it), sts.append(st), gal.append(np.linalg.norm(r))
    np.savez_compressed(
        HERE / "reference_operator.npz", A=A, C=C, f=f,
        theta=np.array([[t.kind, t.k, t.m, t.scale] for t in theta]),
        mu=np.array(mus), eta=np.array(etas), R_ref=np.array(Rs), J_ref=np.array(Js),
        solve_mu=solve_mu, solve_u=np.array(us), solve_iters=np.array(its), solve_status=np.array(sts),
        galerkin_residual=np.array(gal), quadrature_evals=instrument.quadrature_evals(),
        mesh=np.array([24, 8]), n_vdofs=space.n_vdofs)
    print("reference_operator.npz:", "iters", its, "status", sts, "galerkin", np.array(gal))


def checksums(model) -> np.ndarray:
    out = []
    for arr in (model.A, model.C, model.f, model.Mp, model.Bq):
        if arr is None:
            out += [0.0, 0.0]
        else:
            out += [float(arr.sum()), float((arr * arr).sum())]
    return np.array(out)


SLICES = {0: 64, 1: 48, 2: 12, 3: 3, 4: 12}


def synthetic_fixtures() -> None:
    for c, nb in SLICES.items():
        cfg = synthetic.CONFIGS[c]
        model = synthetic.config_model(cfg)
        mu = synthetic.config_mu(cfg, nb)
        res = [oracle.solve_sample(model, mu[b], tol=cfg.tol, max_iter=cfg.max_iter) for b in range(nb)]
        u = np.array([r[0] for r in res])
        data = dict(mu=mu, u=u, iters=np.array([r[1] for r in res]), status=np.array([r[2] for r in res]),
                    last=np.array([r[3] for r in res]), checksums=checksums(model))
        if cfg.n_p:
            data["p"] = oracle.recover_pressure(model, mu, u)
        np.savez_compressed(HERE / f"synthetic_cfg{c}.npz", **data)
        print(f"synthetic_cfg{c}.npz: B={nb} iters={np.bincount(data['iters']).tolist()}")


LIFTED = {"lifted_small": dict(n=12, series=2, n_p=6, nb=64), "lifted_n12": dict(n=50, series=12, n_p=0, nb=8)}


def lifted_fixtures() -> None:
    for name, spec in LIFTED.items():
        model = synthetic.make_lifted_model(spec["n"], spec["series"], n_p=spec["n_p"])
        mu = synthetic.make_lifted_mu(spec["nb"])
        res = [oracle.solve_sample(model, mu[b]) for b in range(spec["nb"])]
        u = np.array([r[0] for r in res])
        data = dict(mu=mu, u=u, iters=np.array([r[1] for r in res]), status=np.array([r[2] for r in res]),
                    last=np.array([r[3] for r in res]), checksums=checksums(model))
        if spec["n_p"]:
            data["p"] = oracle.recover_pressure(model, mu, u)
        np.savez_compressed(HERE / f"{name}.npz", **data)
        print(f"{name}.npz: B={spec['nb']} iters={np.bincount(data['iters']).tolist()}")


def projection_fixture(m: int = 6, seed: int = 11) -> None:
    sys.path.insert(0, str(REF_SRC))
    from rbflow import assemble, geometry, spaces  # the reference package (read-only import)

    prof = geometry.naca_profile(0.15, 12)
    mesh = geometry.build_omesh(prof, 6.0, 12, 4, 1.2)
    space = spaces.build_space_pair(mesh, spaces.DIV_CONFORMING)
    geom = geometry.DeformedGeometry()
    rng = np.random.default_rng(seed)
    V = np.zeros((space.n_vdofs, m))
    Qm, _ = np.linalg.qr(rng.standard_normal((space.free_v.size, m)))
    V[space.free_v] = Qm
    dval, dgrad = assemble.deformed_tables(space, geom, math.radians(20.0), "piola")
    vals, grads = [], []
    for j in range(m):
        v, g = assemble.field_at_quadrature(space, dval, dgrad, V[:, j])   # (nel,nq,2), (nel,nq,2,2)
        vals.append(v.reshape(-1, 2)), grads.append(g.reshape(-1, 2, 2))
    val = np.stack(vals, axis=-1)                                            # (P, 2, m)
    grad = np.stack(grads, axis=-1)                                          # (P, 2, 2, m): [c, d] = ∂_d u_c
    w = space.qp_w.reshape(-1)
    C = np.empty((m, m, m))
    for j in range(m):
        N1, _ = assemble.convection_matrices(space, dval, dgrad, V[:, j])
        C[j] = (V.T @ (N1 @ V)).T                                            # C[j,k,l] = V_lᵀ N1(V_j) V_k
    A = V.T @ (assemble.viscous_matrix(space, dgrad, 1.0) @ V)
    np.savez_compressed(HERE / "projection_ref.npz", val=val, grad=grad, w=w, C_ref=C, A_ref=A,
                        mesh=np.array([12, 4]), phi=math.radians(20.0))
    print("projection_ref.npz: P", val.shape[0], "m", m, "|C|", np.abs(C).max(), "|A|", np.abs(A).max())


if __name__ == "__main__":
    if "--lifted" not in sys.argv and "--projection" not in sys.argv:
        reference_operator_fixture()
        synthetic_fixtures()
    if "--projection" not in sys.argv:
        lifted_fixtures()
    projection_fixture()
