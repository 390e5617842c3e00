"""ReducedModel store: structured-text manifest + raw little-endian float64 arrays.

Format ("ReducedModel file: manifest (term descriptors, basis sizes, formulation tags, provenance hash)
+ raw arrays; round-trip bit-exact"; "Binary store: structured-text manifest plus raw little-endian
64-bit float arrays, row-major, shapes and names in the manifest; … zero-copy loads"):

    <model>.rbm/
        manifest.json        sorted keys, 1-space indent, trailing newline (byte-stable)
        A.f64 C.f64 f.f64    raw '<f8', C order
        [Mp.f64 Bq.f64]

The manifest lists every array (file, shape, sha256), the four term families with their descriptors (kind, k, m
and the scale both as a decimal and as its exact IEEE hex form, which is what the loader reads), the viscosity
rule, the formulation tags and a provenance hash over arrays + descriptors.  Loading verifies sizes and digests
and raises ``StoreError`` (reference errors.py:20-21) on anything missing, corrupt or inconsistent.  Write →
read → write reproduces the files byte for byte.  This is an offline/ingestion path: the online
solver never reads files.
"""

from __future__ import annotations

import hashlib
import json
import os
from pathlib import Path
from typing import Dict

import numpy as np

from .affine import ThetaTerm
from .errors import StoreError
from .model import FAMILIES, ReducedModel

FORMAT = "rbflow-reduced-model"
VERSION = 1
_FAMILY_ARRAY = {"linear": "A", "quadratic": "C", "load": "f", "coupling": "Bq"}


def _term_record(t: ThetaTerm) -> dict:
    return {"kind": int(t.kind), "k": int(t.k), "m": int(t.m), "scale": float(t.scale),
            "scale_hex": float(t.scale).hex()}


def _json_safe(meta: dict) -> dict:
    out = {}
    for k, v in sorted(meta.items()):
        if isinstance(v, (bool, int, str)) or v is None:
            out[str(k)] = v
        elif isinstance(v, float):
            out[str(k)] = v
        elif isinstance(v, (np.integer, np.floating)):
            out[str(k)] = v.item()
    return out


def _digest(arrays: Dict[str, np.ndarray], families: dict, nu_linear: bool, stop: dict) -> str:
    h = hashlib.sha256()
    for name in sorted(arrays):
        a = arrays[name]
        h.update(name.encode())
        h.update(repr(tuple(a.shape)).encode())
        h.update(np.ascontiguousarray(a, dtype="<f8").tobytes())
    h.update(json.dumps(families, sort_keys=True).encode())
    h.update(b"nu_linear" if nu_linear else b"nu_none")
    h.update(json.dumps(stop, sort_keys=True).encode())
    return h.hexdigest()


def save_model(model: ReducedModel, path: os.PathLike) -> Path:
    """Write ``model`` to the directory ``path`` (created; existing files of the same names are replaced)."""
    path = Path(path)
    path.mkdir(parents=True, exist_ok=True)
    arrays = {"A": model.A, "C": model.C, "f": model.f}
    if model.Mp is not None:
        arrays["Mp"] = model.Mp
        arrays["Bq"] = model.Bq
    if model.P_att is not None:  # attached pressure modes of the combined scheme
        arrays["P_att"] = model.P_att
    families = {}
    for fam in FAMILIES:
        if fam == "coupling" and model.Bq is None:
            continue
        families[fam] = {"array": _FAMILY_ARRAY[fam],
                         "terms": [_term_record(t) for t in getattr(model, f"theta_{fam}")]}
    records = {}
    for name, a in arrays.items():
        raw = np.ascontiguousarray(a, dtype="<f8").tobytes()
        (path / f"{name}.f64").write_bytes(raw)
        records[name] = {"file": f"{name}.f64", "shape": list(a.shape), "dtype": "<f8",
                         "sha256": hashlib.sha256(raw).hexdigest()}
    manifest = {
        "format": FORMAT, "version": VERSION, "name": model.name,
        "kind": "velocity-only block (div-conforming, Piola)" if not model.shared_theta else "velocity-only block",
        "basis": {"n_velocity": model.n, "n_pressure": model.n_p, "n_attached_pressure": model.n_att},
        "viscosity": "nu = 1/mu1 multiplies the linear family" if model.nu_linear else "in the descriptors",
        "nu_linear": model.nu_linear,
        "stop": {"n_stop": model.n_stop, "absolute": model.stop_absolute},
        "families": families,
        "arrays": records,
        "provenance": _json_safe(model.meta),
        "hash": _digest(arrays, families, model.nu_linear, {"n_stop": model.n_stop, "absolute": model.stop_absolute}),
    }
    text = json.dumps(manifest, sort_keys=True, indent=1) + "\n"
    (path / "manifest.json").write_text(text)
    return path


def _read_array(path: Path, rec: dict, mmap: bool) -> np.ndarray:
    f = path / rec["file"]
    if not f.is_file():
        raise StoreError(f"{f}: missing array file")
    shape = tuple(int(s) for s in rec["shape"])
    want = int(np.prod(shape)) * 8
    if f.stat().st_size != want:
        raise StoreError(f"{f}: {f.stat().st_size} bytes, manifest shape {shape} needs {want}")
    if rec.get("dtype", "<f8") != "<f8":
        raise StoreError(f"{f}: unsupported dtype {rec.get('dtype')}")
    if mmap:
        a = np.memmap(f, dtype="<f8", mode="r", shape=shape)
        digest = hashlib.sha256(memoryview(a).cast("B")).hexdigest()
    else:
        raw = f.read_bytes()
        digest = hashlib.sha256(raw).hexdigest()
        a = np.frombuffer(raw, dtype="<f8").reshape(shape)
    if digest != rec["sha256"]:
        raise StoreError(f"{f}: sha256 mismatch (corrupt store)")
    return np.asarray(a, dtype=np.float64)


def load_model(path: os.PathLike, mmap: bool = False) -> ReducedModel:
    """Read a store written by :func:`save_model`; verifies every digest.  ``mmap`` maps the arrays (zero-copy
    reads; the model keeps read-only views)."""
    path = Path(path)
    mf = path / "manifest.json"
    if not mf.is_file():
        raise StoreError(f"{path}: no manifest.json")
    try:
        man = json.loads(mf.read_text())
    except json.JSONDecodeError as exc:
        raise StoreError(f"{mf}: not valid JSON ({exc})") from exc
    if man.get("format") != FORMAT or man.get("version") != VERSION:
        raise StoreError(f"{mf}: format {man.get('format')!r} v{man.get('version')!r} not supported")
    try:
        arrays = {name: _read_array(path, rec, mmap) for name, rec in man["arrays"].items()}
        fams = man["families"]
        thetas = {fam: [ThetaTerm(int(t["kind"]), int(t["k"]), int(t["m"]), float.fromhex(t["scale_hex"]))
                        for t in rec["terms"]] for fam, rec in fams.items()}
        nu_linear = bool(man["nu_linear"])
        stop = man.get("stop", {"n_stop": 0, "absolute": False})
    except (KeyError, TypeError, ValueError) as exc:
        raise StoreError(f"{mf}: inconsistent manifest ({exc})") from exc
    if _digest(arrays, fams, nu_linear, stop) != man.get("hash"):
        raise StoreError(f"{mf}: provenance hash mismatch")
    try:
        return ReducedModel(A=arrays["A"], C=arrays["C"], f=arrays["f"], Mp=arrays.get("Mp"), Bq=arrays.get("Bq"),
                            name=man.get("name", "reduced-model"), meta=dict(man.get("provenance", {})),
                            theta_linear=thetas["linear"], theta_quadratic=thetas["quadratic"],
                            theta_load=thetas["load"], theta_coupling=thetas.get("coupling"), nu_linear=nu_linear,
                            n_stop=int(stop["n_stop"]), stop_absolute=bool(stop["absolute"]),
                            P_att=arrays.get("P_att"))
    except (KeyError, ValueError) as exc:
        raise StoreError(f"{path}: arrays inconsistent with the families ({exc})") from exc
