"""Projection kernel throughput: C (N³) from P quadrature points, fp64; prints TF/s of the main contraction
(4·P·N³ flop: K = 2P, 2 flop per FMA) and the fraction of the live cuBLAS DGEMM peak.
    python tools/projection_perf.py [N] [P]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1807_11866_b200 import projection
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
p = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 18
g = torch.Generator(device="cuda").manual_seed(0)
vu = torch.randn(p, 2, n, dtype=torch.float64, device="cuda", generator=g)
gr = torch.randn(p, 2, 2, n, dtype=torch.float64, device="cuda", generator=g)
vw = torch.randn(p, 2, n, dtype=torch.float64, device="cuda", generator=g)
w = torch.rand(p, dtype=torch.float64, device="cuda", generator=g)
out = torch.empty(n, n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    projection.project_convection(vu, gr, vw, w, out=out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    projection.project_convection(vu, gr, vw, w, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
tf = 4.0 * p * n ** 3 / (ms * 1e-3) / 1e12
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2):
    a @ a
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    a @ a
e1.record()
torch.cuda.synchronize()
peak = 2 * 8192 ** 3 / (e0.elapsed_time(e1) / 5 * 1e-3) / 1e12
print(f"projection N={n} P={p}: {ms:.3f} ms, {tf:.2f} TF/s algorithmic, DGEMM peak {peak:.2f} TF/s, frac {tf / peak:.3f}")
