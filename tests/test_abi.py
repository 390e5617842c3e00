"""CPU tests of the C-ABI boundary: the library builds, loads, exports every symbol include/rbns.h declares,
and rejects bad arguments without touching a GPU."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_1807_11866_b200 import build, _native

    build.build()
    return _native.load()


def header_functions():
    txt = (ROOT / "include" / "rbns.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(rbns_\w+)\s*\(", txt, re.M)))


def test_header_lists_functions():
    fns = header_functions()
    assert "rbns_solve" in fns and "rbns_model_create" in fns and len(fns) >= 10


def test_all_header_symbols_exported(lib):
    from paper_1807_11866_b200 import _native

    for name in header_functions():
        assert hasattr(lib, name), f"{name} not exported"
    assert set(header_functions()) == set(_native.EXPORTED_SYMBOLS)


def test_abi_version_and_errors(lib):
    assert lib.rbns_abi_version() == 3
    assert lib.rbns_error_string(0) == b"ok"
    assert b"invalid" in lib.rbns_error_string(1)
    assert lib.rbns_error_string(99) == b"unknown error"


def test_invalid_arguments_rejected_without_gpu(lib):
    from paper_1807_11866_b200 import _native

    out = ctypes.c_void_p()
    assert lib.rbns_model_create(None, 0, ctypes.byref(out)) == 1
    desc = _native.ModelDescC()
    desc.n, desc.q = 0, 1
    assert lib.rbns_model_create(ctypes.byref(desc), 0, ctypes.byref(out)) == 1
    assert b"N >= 1" in lib.rbns_last_error_message()
    desc.n, desc.q = 10, 257
    assert lib.rbns_model_create(ctypes.byref(desc), 0, ctypes.byref(out)) == 1
    assert b"count outside" in lib.rbns_last_error_message()
    desc.n, desc.q = 10, 2  # NULL operators
    assert lib.rbns_model_create(ctypes.byref(desc), 0, ctypes.byref(out)) == 1
    assert b"NULL" in lib.rbns_last_error_message()
    d2 = _native.ModelDesc2C()
    d2.n = 10
    assert lib.rbns_model_create2(ctypes.byref(d2), 0, ctypes.byref(out)) == 1
    assert b"linear family" in lib.rbns_last_error_message()
    terms = (_native.ThetaTermC * 1)(_native.ThetaTermC(9, 0, 0, 0, 1.0))
    a = (ctypes.c_double * 100)()
    d2.linear.count, d2.linear.data, d2.linear.theta = 1, ctypes.addressof(a), terms
    assert lib.rbns_model_create2(ctypes.byref(d2), 0, ctypes.byref(out)) == 1
    assert b"bad theta descriptor" in lib.rbns_last_error_message()
    assert lib.rbns_solve(None, None, 0, 1e-12, 20, None, None, None, None, None, None) == 1
    assert lib.rbns_model_destroy(None) == 0


def test_missing_library_fails_loudly(tmp_path):
    from paper_1807_11866_b200 import _native
    from paper_1807_11866_b200.errors import NativeError

    with pytest.raises(NativeError, match="not built"):
        _native.load(tmp_path / "librbns.so")


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the header structs: sizes and every field offset, checked against the C compiler."""
    import shutil
    import subprocess

    from paper_1807_11866_b200 import _native

    structs = {"rbns_theta_term": _native.ThetaTermC, "rbns_model_desc": _native.ModelDescC,
               "rbns_term_family": _native.TermFamilyC, "rbns_model_desc2": _native.ModelDesc2C,
               "rbns_stats": _native.StatsC}
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "rbns.h"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run([cc, f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        c, f, v = ln.split()
        got[(c, f)] = int(v)
    for cname, cls in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, f"{cname}.{fname}"
