"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): config 0, a 128-sample slice of the
headline config 2 (TMA-staged tiled Gauss–Jordan kernel + DMMA contraction), config 4 with recovery and the
combined-scheme reconstruction, and a 32-sample config-3 slice (2-CTA cluster kernel), each checked against the
oracle so a silent corruption also fails the run."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import online, synthetic

for c, nb, att in ((0, 64, False), (2, 128, False), (4, 64, True), (3, 32, False)):
    cfg = synthetic.CONFIGS[c]
    model = synthetic.config_model(cfg, attached=att)
    mu = synthetic.config_mu(cfg, nb)
    with online.DeviceModel(model, 0) as dm:
        r = dm.solve(torch.from_numpy(mu).cuda(), tol=cfg.tol, max_iter=cfg.max_iter)
        if att:
            p_att = dm.reconstruct_pressure(r.u).cpu().numpy()
        torch.cuda.synchronize()
        u = r.u.cpu().numpy()
    ur, itr, st, _ = oracle.solve_batch(model, mu, tol=cfg.tol, max_iter=cfg.max_iter)
    rel = np.abs(u - ur).max() / np.abs(ur).max()
    assert rel <= 1e-10 and np.array_equal(r.iters.cpu().numpy(), itr), (c, rel)
    if att:
        assert np.abs(p_att - oracle.reconstruct_pressure(model, u)).max() <= 1e-12 * np.abs(p_att).max()
    print(f"cfg{c} B={nb}: rel={rel:.2e} ok", flush=True)
