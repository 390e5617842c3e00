"""A/B timing of library builds on config 2 (development aid): python tools/ab_lib.py LIB_A LIB_B [cfg].
A variant is a library path, optionally with environment settings: path.so:RBNS_NEWTON=bgj2.
Each variant runs in its own process (alternating A, B, A, B); prints gpu_check.timing lines."""
import os, subprocess, sys
libs = [a for a in sys.argv[1:] if ".so" in a]
rest = [a for a in sys.argv[1:] if ".so" not in a]
cfg = rest[0] if rest else "2"
for rnd in range(2):
    for lib in libs:
        path, *envs = lib.split(":")
        env = dict(os.environ, RBNS_LIB=path, **dict(e.split("=", 1) for e in envs))
        out = subprocess.run([sys.executable, "-c", f"import sys; sys.argv=['x']; sys.path.insert(0,'tools'); "
                              f"import gpu_check as g; g.timing({cfg})"], env=env, capture_output=True, text=True)
        print(lib, out.stdout.strip().replace("\n", "\n    "), out.stderr[-1500:], flush=True)
