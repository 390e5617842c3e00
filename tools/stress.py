"""Run-to-run bitwise determinism stress: repeated GEMM-only (reduced_operator) and full solves."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1807_11866_b200 import online, synthetic

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = synthetic.CONFIGS[c]
m = synthetic.config_model(cfg); mu = synthetic.config_mu(cfg, nb)
mud = torch.from_numpy(mu).cuda()
rng = np.random.default_rng(5)
with online.DeviceModel(m, 0) as dm:
    ne = min(nb, 8192)
    eta = torch.from_numpy(rng.standard_normal((ne, cfg.n)) * 0.3).cuda()
    ref = None
    for rep in range(reps):
        R, J = dm.reduced_operator(mud[:ne], eta)
        if ref is None: ref = (R.clone(), J.clone())
        else:
            bad = (J != ref[1]).any(dim=2).any(dim=1).nonzero().flatten().tolist()
            print(f"op rep {rep}: samples with differing J: {len(bad)} {bad[:10]}", flush=True)
    refs = None
    r = None
    press = len(sys.argv) > 4 and sys.argv[4] == "p"
    for rep in range(reps):
        r = dm.solve(mud, pressure=press, out=r)
        u = r.u.cpu().numpy(); it = r.iters.cpu().numpy()
        if refs is None: refs = (u, it)
        else:
            bad = np.nonzero(np.any(u != refs[0], axis=1))[0]
            print(f"solve rep {rep}: sample_it {r.stats['sample_iterations']} differing samples {len(bad)} iters {[(int(b), int(refs[1][b]), int(it[b])) for b in bad[:12]]}", flush=True)
