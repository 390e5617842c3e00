"""SPEC acceptance #10: block solver time < naive coupled-3M time at every M, ratio growing with M.
Desk scale M ∈ {5, 10, 15, 20} plus the larger M = 30, 50; B μ per call (φ, u∞ box), same lifted model family.

    python tools/coupled_speed.py [B]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1807_11866_b200 import online, synthetic  # noqa: E402
from paper_1807_11866_b200.coupled import solve_coupled_batch  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
print(f"{'M':>4} {'block ms':>10} {'coupled-3M ms':>14} {'ratio':>7}  (B = {B}, series n = 12)")
prev = 0.0
for m in (5, 10, 15, 20, 30, 50):
    cm, blk = synthetic.make_coupled_model(m, 12)
    mu = synthetic.make_lifted_mu(B, seed=3)
    dm = online.device_model(blk)
    dm.solve_host(mu)
    solve_coupled_batch(cm, mu)
    tb, tc = [], []
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter(); dm.solve_host(mu); torch.cuda.synchronize()
        tb.append(time.perf_counter() - t)
        t = time.perf_counter(); r = solve_coupled_batch(cm, mu); torch.cuda.synchronize()
        tc.append(time.perf_counter() - t)
        assert np.all(r[4] == 0)
    b, c = min(tb) * 1e3, min(tc) * 1e3
    print(f"{m:>4} {b:>10.2f} {c:>14.2f} {c / b:>7.1f}", flush=True)
    online.release_device_models()
