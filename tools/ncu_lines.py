"""Aggregate an ncu source page (cuda,sass) to per-source-line stall samples and executed instructions."""
import csv, subprocess, sys
rep, kern = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
if kern: cmd += ["-k", f"regex:{kern}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; lines = []; fname = ""
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and r[0] and r[0] != "Function Name":
        try:
            lines.append((fname, int(r[0]), r[1][:90], int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0),
                          int(r[hdr.index("Instructions Executed")] or 0)))
        except ValueError:
            pass
tot_s = sum(l[3] for l in lines) or 1; tot_e = sum(l[4] for l in lines) or 1
print(f"total stall samples {tot_s}, instructions {tot_e}")
for l in sorted(lines, key=lambda x: -x[3])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{l[3]*100/tot_s:5.1f}% stall {l[4]*100/tot_e:5.1f}% inst  {l[0]}:{l[1]}  {l[2]}")
