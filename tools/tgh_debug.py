"""One and two Newton steps on a few config-3 samples (N = 200: the hybrid tiled kernel): device δ against numpy,
per row tile.  Optional argv[1]: number of samples (default 4)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import online, synthetic
cfg = synthetic.CONFIGS[3]
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 4
m = synthetic.config_model(cfg); mu = synthetic.config_mu(cfg, nb)
with online.DeviceModel(m, 0) as dm:
    for iters in (1, 2, 3):
        r = dm.solve(torch.from_numpy(mu).cuda(), max_iter=iters, pressure=False, tol=0.0)
        u = r.u.cpu().numpy()
        for b in range(min(nb, 3)):
            ur = np.zeros(m.n)
            for it in range(iters):
                R, J = oracle.reduced_operator(m, mu[b], ur)
                ur = ur + np.linalg.solve(J, -R)
            err = np.abs(u[b] - ur)
            per_tile = [float(err[8 * i:8 * i + 8].max() / np.abs(ur).max()) for i in range((m.n + 7) // 8)]
            print(f"iters={iters} b={b} rel={err.max() / np.abs(ur).max():.2e} per-row-tile:", " ".join(f"{x:.0e}" for x in per_tile))
        print(r.stats)
