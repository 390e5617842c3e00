"""Instruction count per source line for one kernel (nvdisasm -gi of the cubin)."""
import collections, re, subprocess, sys
cubin, kern = sys.argv[1], sys.argv[2]
txt = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.splitlines()
inside = False; cur = None; c = collections.Counter(); n = 0
for line in txt:
    if line.startswith(".text."):
        inside = kern in line
        continue
    if not inside: continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line): c[cur] += 1; n += 1
print("total instructions", n)
for k, v in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25): print(f"{v:7d} {k[0]}:{k[1]}")
