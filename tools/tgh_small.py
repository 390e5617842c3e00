"""RBNS_NEWTON=tgh: the hybrid tiled kernel at its small test shapes (N = 56, 104) and N = 200 against numpy,
one to three Newton steps on a few samples."""
import os, sys
os.environ.setdefault("RBNS_NEWTON", "tgh")
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import online, synthetic
for n in (56, 97, 100, 103, 104, 200):
    m = synthetic.make_model(n, 3, "trig3", seed=n)
    mu = synthetic.make_mu(4, 50.0, seed=n)
    with online.DeviceModel(m, 0) as dm:
        for iters in (1, 2):
            r = dm.solve(torch.from_numpy(mu).cuda(), max_iter=iters, pressure=False, tol=0.0)
            u = r.u.cpu().numpy()
            b = 0
            ur = np.zeros(m.n)
            for it in range(iters):
                R, J = oracle.reduced_operator(m, mu[b], ur)
                ur = ur + np.linalg.solve(J, -R)
            err = np.abs(u[b] - ur)
            print("  ratio u/u_ref (first 10):", np.round(u[b][:10] / ur[:10], 4))
            per_tile = [float(err[8 * i:8 * i + 8].max() / np.abs(ur).max()) for i in range((m.n + 7) // 8)]
            print(f"N={n} iters={iters} rel={err.max() / np.abs(ur).max():.2e} fallbacks={r.stats['pivot_fallbacks']} per-row-tile:", " ".join(f"{x:.0e}" for x in per_tile))
