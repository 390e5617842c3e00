"""Bitwise run-to-run determinism probe for the contraction and the full solve."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1807_11866_b200 import online, synthetic

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
cfg = synthetic.CONFIGS[c]
m = synthetic.config_model(cfg); mu = synthetic.config_mu(cfg, nb)
rng = np.random.default_rng(5)
eta = rng.standard_normal((min(nb, 2048), cfg.n))
with online.DeviceModel(m, 0) as dm:
    ref = None
    for rep in range(4):
        R, J = dm.reduced_operator(mu[:len(eta)], eta)
        J = J.cpu().numpy()
        if ref is None: ref = J
        else:
            bad = np.argwhere(J != ref)
            print(f"op rep {rep}: mismatching entries {len(bad)}", (np.unique(bad[:, 0]).tolist()[:20] if len(bad) else ""))
    mud = torch.from_numpy(mu).cuda()
    refs = None
    for rep in range(4):
        r = dm.solve(mud, pressure=False)
        u = r.u.cpu().numpy(); it = r.iters.cpu().numpy()
        if refs is None: refs = (u, it)
        else:
            print(f"solve rep {rep}: u mismatch samples {(np.any(u != refs[0], axis=1)).sum()}, iters mismatch {(it != refs[1]).sum()}, sample_it {r.stats['sample_iterations']}")
