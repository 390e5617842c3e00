"""Per-source-line stall samples broken down by reason, from an ncu source page (cuda,sass).
usage: python tools/ncu_reasons.py REPORT [KERNEL_REGEX] [REASON ...]"""
import csv, subprocess, sys
rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
reasons = sys.argv[3:] or ["stall_wait", "stall_long_sb", "stall_short_sb", "stall_math", "stall_no_inst",
                           "stall_branch_resolving", "stall_barrier", "stall_selected"]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"]
if kern:
    cmd += ["-k", f"regex:{kern}"]
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
hdr, fname, lines = None, "", []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0] != "Function Name":
        try:
            lines.append((fname, int(r[0]), r[1][:80], {k: int(r[hdr.index(k)] or 0) for k in reasons}))
        except (ValueError, IndexError):
            pass
for k in reasons:
    tot = sum(l[3][k] for l in lines) or 1
    print(f"== {k}: {tot} samples")
    for l in sorted(lines, key=lambda x: -x[3][k])[:8]:
        if l[3][k]:
            print(f"  {l[3][k]*100/tot:5.1f}%  {l[0]}:{l[1]}  {l[2]}")
