"""Checked build (compute-sanitizer substitute; the pool refuses compute-sanitizer, see
profiles/r02_compute_sanitizer_refused.txt): build/librbns_checked.so compiles the kernels with -DRBNS_CHECKED,
so every hot kernel checks its sample ids, J-block offsets, TMA source ranges, staging sizes, epilogue rows and
compaction positions on the device and counts failures.  Small cases of every kernel path run through it (in a
subprocess, RBNS_LIB) with oracle parity, and the failure count must be 0."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "build", "librbns_checked.so")

CODE = r"""
import ctypes, os, numpy as np, torch
from oracle import rbns_oracle as o
from paper_1807_11866_b200 import online, synthetic, _native
from paper_1807_11866_b200.model import ReducedModel
cases = [(synthetic.config_model(c), synthetic.config_mu(c, nb)) for c, nb in ((0, None), (1, 256), (2, 200), (3, 40), (4, 128))]
for n in (7, 33, 91, 150):  # odd sizes: the rank-1, tiled-edge and cluster kernels
    cases.append((synthetic.make_model(n, 3, "trig3", seed=n), synthetic.make_mu(64, 50.0, seed=n)))
for n in (100, 200):  # row-permuted A0: every sample misses the pivot hint at the first iteration
    base = synthetic.make_model(n, 3, "trig3", seed=n)
    A = base.A.copy(); A[0] = A[0][np.random.default_rng(n).permutation(n)] * 3.0
    cases.append((ReducedModel(A=A, C=base.C, f=base.f, theta=base.theta), synthetic.make_mu(48, 50.0, seed=n)))
for m, mu in cases:
    with online.DeviceModel(m, 0) as dm:
        r = dm.solve(torch.from_numpy(mu).cuda(), pressure=m.n_p > 0)
        R, J = dm.reduced_operator(mu[:4], r.u[:4])
        torch.cuda.synchronize()
    ur, itr, st, _ = o.solve_batch(m, mu)
    u = r.u.cpu().numpy()
    assert np.all(st == 0) and np.all(r.status.cpu().numpy() == 0), m.n
    assert np.abs(u - ur).max() <= 1e-10 * np.abs(ur).max(), m.n
line_m, line_n, cnt = ctypes.c_int(), ctypes.c_int(), ctypes.c_ulonglong()
lib = _native.load()
assert lib.rbns_debug_checks(ctypes.byref(line_m), ctypes.byref(line_n), ctypes.byref(cnt)) == 0
print(f"checks failed: {cnt.value} (first lines {line_m.value}/{line_n.value}) over {len(cases)} cases")
assert cnt.value == 0
print("ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("newton", ["", "tgh", "gj2"])
def test_checked_build_has_no_failed_checks(newton):
    if not os.path.exists(LIB):
        pytest.fail(f"{LIB} missing: run __graft_entry__.build()")
    env = dict(os.environ, RBNS_LIB=LIB, RBNS_NEWTON=newton)
    out = subprocess.run([sys.executable, "-c", CODE], env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    print(out.stdout[-500:])
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stdout[-1000:] + out.stderr[-2000:]
