"""clock64 trace of sample 0 of the last tiled Gauss–Jordan launch (python -m paper_1807_11866_b200.build --trace;
RBNS_LIB=build/librbns_trace.so python tools/trace_tgj.py [cfg] [B])."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1807_11866_b200 import online, synthetic, _native
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
cfg = synthetic.CONFIGS[c]
m = synthetic.config_model(cfg); mu = torch.from_numpy(synthetic.config_mu(cfg, nb)).cuda()
with online.DeviceModel(m, 0) as dm:
    r = dm.solve(mu, max_iter=2, pressure=False)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 256)()
    _native.load().rbns_debug_trace(buf, 256)
names = {0: "sample start", 1: "J landed", 2: "rhs + M0 ready", 3: "staging consumed", 4: "panel 0 published",
         250: "sample done", 5: "tiles loaded", 6: "row sums reduced", 7: "row-sum barrier", 8: "rhs computed", 9: "hint checked"}
for P in range(16):
    names[192 + P] = f"P{P}: owner starts invert"; names[208 + P] = f"P{P}: invert done"
    names[224 + P] = f"P{P}: published"
    for w in range(4):
        names[128 + 4 * P + w] = f"    w{w} has panel {P}"; names[64 + 4 * P + w] = f"    w{w} done panel {P}"
for w in range(4):
    names[240 + w] = f"w{w} loop end"
t0 = buf[0]
rows = sorted((buf[i] - t0, names.get(i, str(i))) for i in range(256) if buf[i] >= t0 and buf[i] != 0)
prev = 0
for tt, nm in rows:
    print(f"{tt:8d} (+{tt - prev:6d})  {nm}")
    prev = tt
