import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_11866_b200 import online, synthetic
from paper_1807_11866_b200.model import ReducedModel
n = 100
rng = np.random.default_rng(n)
base = synthetic.make_model(n, 7, "trig7", seed=n)
A = base.A.copy(); A[0] = A[0][rng.permutation(n)] * 3.0
m = ReducedModel(A=A, C=base.C, f=base.f, theta=base.theta)
mu = torch.from_numpy(synthetic.make_mu(65536, 50.0, seed=3)).cuda()
with online.DeviceModel(m, 0) as dm:
    r = dm.solve(mu)
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter(); r = dm.solve(mu, out=r); torch.cuda.synchronize()
        s = r.stats
        print(f"permuted N=100: {1e3*(time.perf_counter()-t):.1f} ms lu {s['ms_lu']:.1f} gemm {s['ms_gemm']:.1f} fallbacks {s['pivot_fallbacks']} its {s['sample_iterations']} status {np.bincount(r.status.cpu().numpy())}")
