"""Print the clock64 trace of block 0 of the last Newton-update launch (build with --trace, RBNS_LIB=...)."""
import ctypes, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1807_11866_b200 import online, synthetic, _native
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
cfg = synthetic.CONFIGS[c]
m = synthetic.config_model(cfg); mu = torch.from_numpy(synthetic.config_mu(cfg, nb)).cuda()
with online.DeviceModel(m, 0) as dm:
    r = dm.solve(mu, max_iter=3, pressure=False)
    torch.cuda.synchronize()
    lib = _native.load()
    buf = (ctypes.c_ulonglong * 256)()
    lib.rbns_debug_trace(buf, 256)
    t0 = buf[0]
    names = {0: "start", 1: "loaded", 2: "rhs", 3: "panel0", 200: "end-gj(ok)", 201: "end-gj(FAIL)", 202: "done",
             101: "loaded(piv)", 102: "rhs(piv)", 103: "panel0(piv)"}
    for c in range(8):
        names[120 + 4 * c] = f"  col{c}: start"; names[121 + 4 * c] = f"  col{c}: prow"
        names[122 + 4 * c] = f"  col{c}: rcp"; names[123 + 4 * c] = f"  col{c}: updated"
    for P in range(16):
        names[8 + 4 * P] = f"P{P}: lookahead-start"; names[9 + 4 * P] = f"P{P}: lookahead-done"
        names[10 + 4 * P] = f"P{P}: factor-done"; names[11 + 4 * P] = f"P{P}: barrier"
        names[160 + P] = f"P{P}: lookahead-update-done (copy next)"
    rows = sorted((buf[i] - t0, names.get(i, str(i))) for i in range(256) if buf[i] >= t0 and buf[i] != 0)
    prev = 0
    for tt, nm in rows:
        print(f"{tt:10d} (+{tt - prev:7d})  {nm}", flush=True)
        prev = tt
