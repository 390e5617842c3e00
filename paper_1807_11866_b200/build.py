"""In-tree build of librbns.so for sm_100a (nvcc, no torch JIT cache).

    python -m paper_1807_11866_b200.build

Sources: paper_1807_11866_b200/csrc/*.cu (one translation unit per file, compiled in parallel), header
include/rbns.h.  Flags: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "librbns.so"
OBJ = ROOT / "build" / "obj"

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}", f"-I{CSRC}"]


def _nvcc() -> str:
    cand = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda")) / "bin" / "nvcc"
    return str(cand) if cand.exists() else "nvcc"


def build(verbose: bool = False, force: bool = False, out: Path = OUT, extra=()) -> Path:
    """Compile csrc/*.cu into ``out`` (default: the in-tree librbns.so); ``extra`` adds nvcc flags
    (e.g. -DRBNS_TRACE for the instrumented development build)."""
    OUT_ = Path(out)
    srcs = sorted(CSRC.glob("*.cu"))
    deps = srcs + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "rbns.h"]
    if OUT_.exists() and not force and all(OUT_.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return OUT_
    obj_dir = OBJ if not extra else OBJ.parent / ("obj_" + "_".join(x.strip("-D").lower() for x in extra))
    obj_dir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(src: Path) -> Path:
        obj = obj_dir / (src.stem + ".o")
        flags = NVCC_FLAGS
        if "_shapes_" in src.name:  # coverage instantiations: no line tables (3x the object size); the
            flags = [f for f in NVCC_FLAGS if f != "-lineinfo"]  # profiled shapes are in rbns_tiled_main.cu
        cmd = [nvcc, *flags, *extra, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = OUT_.with_suffix(".so.tmp")
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
                        *map(str, objs)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, OUT_)
    return OUT_


CHECKED = ROOT / "build" / "librbns_checked.so"


def build_checked(force: bool = False) -> Path:
    """The checked development build (-DRBNS_CHECKED: device-side bounds / protocol checks, readout through
    rbns_debug_checks) used by tests/test_checked.py in place of compute-sanitizer."""
    return build(force=force, out=CHECKED, extra=("-DRBNS_CHECKED",))


PROBE = ROOT / "build" / "oz_probe"


def build_probe(force: bool = False) -> Path:
    """tools/oz_probe.cu: the INT8-sliced contraction kernel against a host emulation of the same splitting, bit
    for bit (tests/test_oz.py runs it on the GPU)."""
    src = ROOT / "tools" / "oz_probe.cu"
    deps = [src, CSRC / "rbns_oz.cuh", CSRC / "rbns_common.cuh", ROOT / "include" / "rbns.h"]
    if PROBE.exists() and not force and all(PROBE.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return PROBE
    PROBE.parent.mkdir(parents=True, exist_ok=True)
    r = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
                        f"-I{ROOT / 'include'}", f"-I{CSRC}", str(src), "-o", str(PROBE)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
    return PROBE


if __name__ == "__main__":
    if "--define" in sys.argv:  # development variant: python -m ...build --define NAME=VAL  -> build/librbns_NAME.so
        d = sys.argv[sys.argv.index("--define") + 1]
        print(build(force=True, out=ROOT / "build" / f"librbns_{d.replace('=', '_').replace(',', '_').lower()}.so", extra=tuple(f"-D{x}" for x in d.split(','))))
    elif "--trace" in sys.argv:
        print(build(force="-f" in sys.argv, out=ROOT / "build" / "librbns_trace.so", extra=("-DRBNS_TRACE",)))
    else:
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
