"""Copy one GPU session's evidence (tools/profile_round.sh output in gpurun_out/) into profiles/ under a round tag.

    python tools/export_profiles.py r01

Writes profiles/<tag>_bench.json, <tag>_bench_ref.json, <tag>_bench_step_launches.csv, <tag>_ncu_full_details.csv,
<tag>_ncu_full_raw.csv, <tag>_launch_summary.txt and refreshes profiles/contract_traffic.json from the full capture.
"""
import csv
import io
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT, PROF = ROOT / "gpurun_out", ROOT / "profiles"


def ncu_csv(rep, page):
    r = subprocess.run(["ncu", "-i", str(rep), "--page", page, "--csv"], capture_output=True, text=True, check=True)
    return r.stdout


def launch_summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[14]) / 1e6
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>6s}"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:60]:60s} {n:8d} {ms:10.3f} {ms / tot:6.1%}")
    lines.append(f"{'total':60s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")
    # the solver's own kernels only (the step): the cutlass DGEMMs are bench.py's in-run FP64 peak measurement,
    # the at:: kernels its input generation and L2 flush
    own = {k: v for k, v in agg.items() if k.startswith(("rbns::", "oz::"))}
    tot_own = sum(v[1] for v in own.values())
    lines += ["", "solver kernels only (shares of the solve; bench.py's cutlass DGEMMs measure the FP64 peak):",
              f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>6s}"]
    for k, (n, ms) in sorted(own.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:60]:60s} {n:8d} {ms:10.3f} {ms / tot_own:6.1%}")
    return "\n".join(lines) + "\n"


def main():
    tag = sys.argv[1]
    for src, dst in [("bench.json", "bench.json"), ("bench_ref.json", "bench_ref.json"),
                     ("launches.csv", "bench_step_launches.csv")]:
        if (OUT / src).exists():
            shutil.copy(OUT / src, PROF / f"{tag}_{dst}")
    if (OUT / "launches.csv").exists():
        (PROF / f"{tag}_launch_summary.txt").write_text(launch_summary(OUT / "launches.csv"))
    rep_lu = OUT / "full_lu.ncu-rep"
    if rep_lu.exists():
        (PROF / f"{tag}_ncu_full_lu_details.csv").write_text(ncu_csv(rep_lu, "details"))
        (PROF / f"{tag}_ncu_full_lu_raw.csv").write_text(ncu_csv(rep_lu, "raw"))
    rep = OUT / "full.ncu-rep"
    if rep.exists():
        (PROF / f"{tag}_ncu_full_details.csv").write_text(ncu_csv(rep, "details"))
        raw = ncu_csv(rep, "raw")
        (PROF / f"{tag}_ncu_full_raw.csv").write_text(raw)
        rows = list(csv.reader(io.StringIO(raw)))
        hdr = rows[0]
        for r in rows[2:]:
            kname = r[hdr.index("Kernel Name")]
            if "contract_kernel" not in kname and "oz_gemm_kernel" not in kname:
                continue
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= units.get(rows[1][hdr.index("dram__bytes_read.sum")], 1)  # ncu scales each metric's unit
            wr *= units.get(rows[1][hdr.index("dram__bytes_write.sum")], 1)  # separately (Mbyte vs Gbyte)
            scale = 1
            json.dump({"cfg2": {
                "dram_bytes_per_launch": int((rd + wr) * scale), "dram_read_bytes": int(rd * scale),
                "dram_write_bytes": int(wr * scale),
                "launch": f"{r[hdr.index('Kernel Name')]} grid {r[hdr.index('Grid Size')]} = full 65536-sample Newton round",
                "source": f"profiles/{tag}_ncu_full_raw.csv (ncu --set full, cold cache; .ncu-rep kept out of git)",
                "note": ("reads = the sliced X images (8 x 65536 x 704 B, re-read per row tile through L2) + the "
                         "sliced S (52 MB, L2-resident); writes = the Jacobians J (65536 x 10112 x 8 B)")
                if "oz_gemm" in kname else
                "reads = S (56 MB, L2-resident) + u tiles; writes = the Jacobians J (65536 x 10112 x 8 B)"}},
                open(PROF / "contract_traffic.json", "w"), indent=1)
            break
    print(sorted(p.name for p in PROF.iterdir() if p.name.startswith(tag)))


if __name__ == "__main__":
    main()
