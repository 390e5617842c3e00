"""Solve throughput for an arbitrary N (trig7 model, Re ~ U[10, 200]): python tools/ntime.py N [B] [reps]."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1807_11866_b200 import online, synthetic
n = int(sys.argv[1]); nb = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
m = synthetic.make_model(n, 7, "trig7", seed=n)
mu = torch.from_numpy(synthetic.make_mu(nb, 200.0, seed=n)).cuda()
with online.DeviceModel(m, 0) as dm:
    r = dm.solve(mu, pressure=False)
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = dm.solve(mu, pressure=False, out=r)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    s = r.stats
    print(f"N={n} B={nb}: {dt * 1e3:.1f} ms, {nb / dt:.0f} solves/s, gemm {s['ms_gemm']:.1f} ms, lu {s['ms_lu']:.1f} ms, "
          f"sample_it {s['sample_iterations']}, fallbacks {s['pivot_fallbacks']}")
