"""Per-call statistics of one cfg solve (device times per phase, launches, Newton rounds, hint misses)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_1807_11866_b200 import online, synthetic  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = synthetic.CONFIGS[c]
m = synthetic.config_model(cfg)
mu = torch.from_numpy(synthetic.config_mu(cfg)).cuda()
with online.DeviceModel(m, 0) as dm:
    r = dm.solve(mu, pressure=cfg.n_p > 0)
    r = dm.solve(mu, pressure=cfg.n_p > 0, out=r)
    torch.cuda.synchronize()
    for k, v in r.stats.items():
        print(f"{k:24s} {v}")
