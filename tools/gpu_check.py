"""Quick on-box parity + timing probe (development aid; the real gates are tests/ and bench.py)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import rbns_oracle as oracle
from paper_1807_11866_b200 import online, synthetic

def check(c, nb, pressure=False):
    cfg = synthetic.CONFIGS[c]
    m = synthetic.config_model(cfg); mu = synthetic.config_mu(cfg, nb)
    with online.DeviceModel(m, 0) as dm:
        r = dm.solve(torch.from_numpy(mu).cuda(), pressure=pressure)
        torch.cuda.synchronize()
        u = r.u.cpu().numpy(); it = r.iters.cpu().numpy(); st = r.status.cpu().numpy()
        ur, itr, str_, _ = oracle.solve_batch(m, mu)
        rel = np.abs(u-ur).max()/np.abs(ur).max()
        msg = f"cfg{c} B={nb}: rel={rel:.2e} iters_mismatch={(it!=itr).sum()} status={np.bincount(st).tolist()} hist={np.bincount(it).tolist()} stats={r.stats}"
        if pressure:
            pr = oracle.recover_pressure(m, mu, ur)
            p = r.p.cpu().numpy()
            msg += f" p_rel={np.abs(p-pr).max()/np.abs(pr).max():.2e}"
        print(msg, flush=True)
        R, J = dm.reduced_operator(mu[:4], ur[:4])
        for b in range(4):
            Rr, Jr = oracle.reduced_operator(m, mu[b], ur[b])
            print("  op", b, np.abs(R[b].cpu().numpy()-Rr).max(), np.abs(J[b].cpu().numpy()-Jr).max()/np.abs(Jr).max())

def timing(c, nb=None, reps=3):
    cfg = synthetic.CONFIGS[c]
    m = synthetic.config_model(cfg); mu = synthetic.config_mu(cfg, nb)
    mud = torch.from_numpy(mu).cuda()
    with online.DeviceModel(m, 0) as dm:
        r = dm.solve(mud, pressure=cfg.n_p > 0)
        for _ in range(reps):
            torch.cuda.synchronize(); t = time.perf_counter()
            r = dm.solve(mud, pressure=cfg.n_p > 0, out=r)
            torch.cuda.synchronize(); dt = time.perf_counter() - t
            s = r.stats
            fl = s['contraction_iterations'] * 2 * cfg.q * cfg.n**3
            print(f"cfg{c} B={len(mu)}: {dt*1e3:.1f} ms, {len(mu)/dt:.0f} solves/s, gemm {s['ms_gemm']:.1f} ms ({fl/s['ms_gemm']/1e9:.1f} TF/s), lu {s['ms_lu']:.1f} ms, rec {s['ms_recovery']:.1f} ms, total {s['ms_total']:.1f}, sample_it {s['sample_iterations']}", flush=True)

if __name__ == "__main__" and not {"lifted", "coupled"} & set(sys.argv):
    check(0, 64)
    check(1, 512)
    check(2, 256)
    check(4, 256, pressure=True)
    timing(1)
    timing(2)
    timing(4)
    if "cfg3" in sys.argv:
        check(3, 64)
        timing(3, reps=1)

def lifted_timing(n=50, series=12, nb=65536, reps=2):
    """Paper-structured model (a+c0 linear, c quadratic, d0 loads; synthetic.make_lifted_model)."""
    m = synthetic.make_lifted_model(n, series); mu = synthetic.make_lifted_mu(nb)
    mud = torch.from_numpy(mu).cuda()
    with online.DeviceModel(m, 0) as dm:
        r = dm.solve(mud)
        ur, itr, _, _ = oracle.solve_batch(m, mu[:256])
        print(f"lifted N={n} series={series}: plan {dm.terms()} rel={np.abs(r.u[:256].cpu().numpy()-ur).max()/np.abs(ur).max():.2e} "
              f"iters_mismatch={(r.iters[:256].cpu().numpy()!=itr).sum()}", flush=True)
        for _ in range(reps):
            torch.cuda.synchronize(); t = time.perf_counter()
            r = dm.solve(mud, out=r)
            torch.cuda.synchronize(); dt = time.perf_counter() - t
            s = r.stats
            fl = s['contraction_iterations'] * 2 * m.q * n**3
            print(f"lifted B={nb}: {dt*1e3:.1f} ms, {nb/dt:.0f} solves/s, gemm {s['ms_gemm']:.1f} ms ({fl/s['ms_gemm']/1e9:.1f} TF/s algorithmic over Qc), lu {s['ms_lu']:.1f} ms, sample_it {s['sample_iterations']}", flush=True)

if __name__ == "__main__" and "lifted" in sys.argv:
    lifted_timing()

def coupled_timing(m=50, series=12, nb=16384):
    """Block (velocity-only, size M) vs naive coupled-3M on the same lifted model."""
    from paper_1807_11866_b200.coupled import solve_coupled_batch
    cm, blk = synthetic.make_coupled_model(m, series)
    mu = synthetic.make_lifted_mu(nb)
    dm = online.device_model(blk)
    dm.solve_host(mu); solve_coupled_batch(cm, mu)
    for name, fn in (("block", lambda: dm.solve_host(mu)), ("coupled-3M", lambda: solve_coupled_batch(cm, mu))):
        torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(f"{name} M={m} B={nb}: {dt*1e3:.1f} ms, {nb/dt:.0f} solves/s", flush=True)

if __name__ == "__main__" and "coupled" in sys.argv:
    coupled_timing()
