"""Development: one Newton step (u0 = 0) of one N = 56 sample through the RBNS_TGH_DUMP build of the hybrid
kernel: its right-hand side, final y column and δ against numpy."""
import ctypes, os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
os.environ["RBNS_LIB"] = str(ROOT / "build" / "librbns_rbns_tgh_dump.so")
os.environ.setdefault("RBNS_NEWTON", "tgh")
sys.path.insert(0, str(ROOT))
import numpy as np, torch
from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import online, synthetic, _native
n = int(sys.argv[1]) if len(sys.argv) > 1 else 56
m = synthetic.make_model(n, 3, "trig3", seed=n)
mu = synthetic.make_mu(1, 50.0, seed=n)
with online.DeviceModel(m, 0) as dm:
    r = dm.solve(torch.from_numpy(mu).cuda(), max_iter=1, pressure=False, tol=0.0)
    torch.cuda.synchronize()
    buf = (ctypes.c_double * 1024)()
    lib = ctypes.CDLL(os.environ["RBNS_LIB"])
    assert lib.rbns_debug_tgh(buf) == 0
    d = np.array(buf).reshape(4, 256)[:, :n]
R, J = oracle.reduced_operator(m, mu[0], np.zeros(n))
delta = np.linalg.solve(J, -R)
np.set_printoptions(precision=4, linewidth=200)
print("rhs / (-R):", (d[0] / -R)[:16])
print("x / delta :", (d[2] / delta)[:16])
print("col1 of rhs tile (should be 0):", d[3][:16])
print("u / delta:", (r.u.cpu().numpy()[0] / delta)[:16])
# y = unscaled: y_i = J_ii^(i) delta_i — report y / delta for reference
print("y/delta:", (d[1] / delta)[:16])
