"""Per-step clock64 trace of block 0 of the last Newton-update launch (gj kernel; trace build)."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1807_11866_b200 import online, synthetic, _native
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
cfg = synthetic.CONFIGS[c]
m = synthetic.config_model(cfg); mu = torch.from_numpy(synthetic.config_mu(cfg, nb)).cuda()
with online.DeviceModel(m, 0) as dm:
    dm.solve(mu, max_iter=3, pressure=False); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 256)(); _native.load().rbns_debug_trace(buf, 256)
    t0 = buf[0]
    for k in range(0, 60):
        a, b1, b2, nxt = buf[4 * k], buf[4 * k + 1], buf[4 * k + 2], buf[4 * k + 4] if k < 59 else 0
        if a == 0: break
        print(f"k={k:2d} start {a - t0:8d}  owner->bar1 {b1 - a:5d}  bar1->bar2 {b2 - b1:5d}  bar2->next {(nxt - b2) if nxt else 0:5d}")
