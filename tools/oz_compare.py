"""INT8-sliced contraction against the DMMA contraction on the same model and μ (RBNS_CONTRACT is read per model
create): max relative difference of u, Newton-count mismatches, and the contraction time of both.

    python tools/oz_compare.py [config] [batch]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_11866_b200 import online, synthetic  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cfg = synthetic.CONFIGS[cfg_id]
model = synthetic.config_model(cfg)
mu = torch.from_numpy(synthetic.config_mu(cfg, B)).cuda()
out = {}
for mode in ("dmma", "i8"):
    os.environ["RBNS_CONTRACT"] = mode
    with online.DeviceModel(model, 0) as dm:
        for _ in range(2):
            r = dm.solve(mu, pressure=False)
            torch.cuda.synchronize()
        out[mode] = (r.u.cpu().numpy(), r.iters.cpu().numpy(), r.status.cpu().numpy(), dict(dm.last_stats) if hasattr(dm, "last_stats") else {})
        try:
            st = dm.stats()
            print(mode, {k: round(v, 3) if isinstance(v, float) else v for k, v in st.items() if k.startswith("ms_") or "launch" in k})
        except Exception as e:  # noqa: BLE001
            print(mode, "stats unavailable", e)
(u1, it1, s1, _), (u2, it2, s2, _) = out["dmma"], out["i8"]
rel = np.abs(u1 - u2).max(axis=1) / np.abs(u1).max(axis=1)
print(f"cfg {cfg_id} B={B}: status nonzero dmma {int((s1 != 0).sum())} i8 {int((s2 != 0).sum())}; "
      f"max rel diff u {rel.max():.3e} (median {np.median(rel):.3e}); count mismatches {int((it1 != it2).sum())}; "
      f"mean iters {it1.mean():.3f} / {it2.mean():.3f}")
