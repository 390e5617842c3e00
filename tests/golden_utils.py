"""Loaders for the committed golden fixtures (tests/golden/*.npz)."""

from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_1807_11866_b200 import affine
from paper_1807_11866_b200.model import ReducedModel

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def golden(name: str):
    with np.load(GOLDEN / f"{name}.npz") as d:
        return {k: d[k] for k in d.files}


def reference_model() -> ReducedModel:
    """The reduced model assembled by the reference package's own quadrature code (make_golden.py)."""
    d = golden("reference_operator")
    theta = [affine.ThetaTerm(int(k), int(a), int(b), float(s)) for k, a, b, s in d["theta"]]
    return ReducedModel(A=d["A"], C=d["C"], f=d["f"], theta=theta, name="reference-assembled")
