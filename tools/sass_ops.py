"""Executed SASS instructions per opcode in an ncu report (source page), optionally per unit of work.
    python tools/sass_ops.py REPORT.ncu-rep [units] [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
hdr, tot = None, {}
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        src = r[hdr.index("Source")].split()
        if not src:
            continue
        op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
        try:
            tot[op] = tot.get(op, 0) + int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            pass
allv = sum(tot.values())
print(f"total {allv} ({allv / units:.1f} per unit)")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{k:10s} {v:12d} {v / units:10.1f} {100 * v / allv:5.1f}%")
