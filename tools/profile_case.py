"""Small fixed workload for ncu captures: cfg C, B samples, two solves (first warms up)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1807_11866_b200 import online, synthetic
c = int(sys.argv[1]); nb = int(sys.argv[2])
cfg = synthetic.CONFIGS[c]
m = synthetic.config_model(cfg); mu = torch.from_numpy(synthetic.config_mu(cfg, nb)).cuda()
with online.DeviceModel(m, 0) as dm:
    for _ in range(2):
        r = dm.solve(mu, pressure=cfg.n_p > 0)
    torch.cuda.synchronize()
    print(r.stats)
