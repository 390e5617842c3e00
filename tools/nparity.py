"""Oracle parity for arbitrary N (trig3 model, 64 samples): python tools/nparity.py N [N ...]."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import rbns_oracle as o
from paper_1807_11866_b200 import online, synthetic
for n in map(int, sys.argv[1:]):
    m = synthetic.make_model(n, 3, "trig3", seed=n)
    mu = synthetic.make_mu(64, 50.0, seed=n)
    with online.DeviceModel(m, 0) as dm:
        r = dm.solve(torch.from_numpy(mu).cuda(), pressure=False)
        torch.cuda.synchronize()
    ur, itr, st, _ = o.solve_batch(m, mu)
    rel = (np.abs(r.u.cpu().numpy() - ur).max(axis=1) / np.abs(ur).max(axis=1)).max()
    print(f"N={n}: rel {rel:.2e}, count mismatches {(r.iters.cpu().numpy() != itr).sum()}, status {np.bincount(r.status.cpu().numpy()).tolist()}, fallbacks {r.stats['pivot_fallbacks']}")
