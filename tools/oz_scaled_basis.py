"""Robustness of the INT8-sliced contraction to basis scaling: the same reduced model written in a basis whose vectors
are scaled by d_i = 10^U(-span/2, span/2) (A -> D A D, C[j,k,l] -> d_j d_k d_l C, f -> D f; u -> D^-1 u), i.e. solution
coefficients spread over `span` decades as POD coefficients do.  Sliced path against the DMMA path and the oracle.

    python tools/oz_scaled_basis.py [n] [q] [span_decades] [batch]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import rbns_oracle as oracle  # noqa: E402
from paper_1807_11866_b200 import online, synthetic  # noqa: E402
from paper_1807_11866_b200.model import ReducedModel  # noqa: E402


def scaled_model(n, q, span, seed=3):
    base = synthetic.make_model(n, q, "trig7" if q == 7 else "trig3", seed=seed)
    rng = np.random.default_rng(seed + 1)
    d = 10.0 ** rng.uniform(-span / 2, span / 2, n)
    A = base.A * d[None, :, None] * d[None, None, :]
    C = base.C * d[None, :, None, None] * d[None, None, :, None] * d[None, None, None, :]
    f = base.f * d[None, :]
    return ReducedModel(A=A, C=C, f=f, theta=base.theta), d


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    q = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    span = float(sys.argv[3]) if len(sys.argv) > 3 else 6.0
    nb = int(sys.argv[4]) if len(sys.argv) > 4 else 512
    model, d = scaled_model(n, q, span)
    mu = synthetic.make_mu(nb, 200.0, seed=9)
    out = {}
    for mode in ("dmma", "i8"):
        os.environ["RBNS_CONTRACT"] = mode
        with online.DeviceModel(model, 0) as dm:
            r = dm.solve(torch.from_numpy(mu).cuda(), pressure=False)
            torch.cuda.synchronize()
            out[mode] = (r.u.cpu().numpy(), r.iters.cpu().numpy(), r.status.cpu().numpy())
    ur, itr, str_, _ = oracle.solve_batch(model, mu)
    for mode in ("dmma", "i8"):
        u, it, st = out[mode]
        ok = (st == 0) & (str_ == 0)
        # error measured in the unscaled basis (u_i d_i): componentwise relative to the sample's largest entry
        e = np.abs((u - ur) * d).max(axis=1) / np.abs(ur * d).max(axis=1)
        print(f"{mode}: n={n} q={q} span={span} decades: status!=0 {int((st != 0).sum())} (oracle {int((str_ != 0).sum())}); "
              f"max err vs oracle {e[ok].max():.3e}; count mismatches vs oracle {int((it[ok] != itr[ok]).sum())}; "
              f"|u| range {np.abs(ur[ok]).min():.2e}..{np.abs(ur[ok]).max():.2e}")
    print("i8 vs dmma count mismatches", int((out['i8'][1] != out['dmma'][1]).sum()))


if __name__ == "__main__":
    main()
