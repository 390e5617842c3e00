"""Numpy emulation of the tiled Gauss–Jordan elimination (unscaled rows, block pivots) for one sample's first
Newton step, compared with the kernel's dump (RBNS_TGJ_DEBUG=1): W_P per panel and the final column y."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import online, synthetic, _native
cfg = synthetic.CONFIGS[2]
m = synthetic.config_model(cfg); mu = synthetic.config_mu(cfg, 8)
with online.DeviceModel(m, 0) as dm:
    r = dm.solve(torch.from_numpy(mu).cuda(), max_iter=1, pressure=False, tol=0.0)
    torch.cuda.synchronize()
    buf = (ctypes.c_double * 32768)()
    print("dump rc", _native.load().rbns_debug_dump(buf, 32768))
d = np.array(buf[:13 * 64 + 104])
slot = lambda r, c: ((r ^ ((r >> 1) & 1)) << 3) + (c ^ (((r >> 2) & 1) << 2))
Wk = [np.array([[d[P * 64 + slot(r, c)] for c in range(8)] for r in range(8)]) for P in range(13)]
y_k = d[13 * 64:13 * 64 + 104]
# emulation on sample act[0] of the last launch = sample 0
R, J = oracle.reduced_operator(m, mu[0], np.zeros(m.n))
N = m.n
A = np.zeros((104, 104)); A[:N, :N] = J; A[:N, N] = -R
full = np.array(buf[:32768])
def frag(base):  # lane (g,t) pair -> matrix [2t+s][g]
    Mx = np.zeros((8, 8))
    for lane in range(32):
        g, t = lane >> 2, lane & 3
        Mx[2 * t, g] = full[base + 2 * lane]; Mx[2 * t + 1, g] = full[base + 2 * lane + 1]
    return Mx
for P in range(13):
    nc = 8 if P < 12 else N - 96
    D = np.eye(8); D[:nc, :nc] = A[8 * P:8 * P + nc, 8 * P:8 * P + nc]
    if P >= 1:
        Dk = frag(1024 + P * 64)
        print(f"   q (pivot tile in) rel diff {np.abs(Dk[:nc,:nc]-D[:nc,:nc]).max()/np.abs(D).max():.2e}"
              f"  X diff {np.abs(frag(2048 + P * 64) - Xprev[:, 8*P:8*P+8]).max()/np.abs(Xprev).max():.2e}"
              f"  M diff {np.abs(frag(3072 + P * 64).T - Mprev[8*P:8*P+8, :]).max()/np.abs(Mprev).max():.2e}")
    W = np.linalg.inv(D)
    err = np.abs(W - Wk[P]).max() / np.abs(W).max()
    print(f"panel {P}: W rel diff {err:.2e}")
    if P == 3: A2 = A.copy()
    X = W @ A[8 * P:8 * P + 8, :]
    Aprev = A.copy(); Xprev = X.copy()
    Mcol = A[:, 8 * P:8 * P + 8].copy(); Mcol[:, nc:] = 0; Mcol[8 * P:8 * P + 8, :] = 0
    Mprev = -Mcol
    cols = np.arange(104) >= 8 * P + 8
    if P == 12: cols = np.arange(104) >= 96
    A[:, cols] -= Mcol @ X[:, cols]
    if P == 3:
        for nm, base in (("before invert(5)", 16384), ("after invert(5)", 17408), ("before deferred P3", 20480)):
            tk = np.vstack([frag(base + i * 64) for i in range(13)])
            print(f"   tile 9 {nm}: diff vs after-panel-2 {np.abs(tk[:N] - A2[:N, 72:80]).max():.2e}")
        Wd = np.array([[full[24576 + slot(r, c)] for c in range(8)] for r in range(8)])
        print("   W3 as applied by warp 0:", np.abs(Wd - W).max() / np.abs(W).max())
        for i in range(13):
            Md = np.array([[full[24576 + 64 + i * 64 + slot(r, c)] for c in range(8)] for r in range(8)])
            print(f"     M3[{i}] diff", np.abs(Md - (-Mcol[8*i:8*i+8, :])).max())
    if P < 9:
        tk = np.vstack([frag(8192 + P * 1024 + i * 64) for i in range(13)])  # rows 104 x cols 8 of tile 9
        print(f"   tile 9 after panel {P}: rel diff {np.abs(tk[:N] - A[:N, 72:80]).max()/np.abs(A[:N,72:80]).max():.2e}")
y = A[:, N]
print("y rel diff per row tile:", " ".join(f"{np.abs(y[8*i:8*i+8]-y_k[8*i:8*i+8]).max()/np.abs(y).max():.0e}" for i in range(13)))
