"""Quadrature-evaluation counter (mirror of /root/reference/pkg/src/rbflow/instrument.py:1-17).

The offline projection (projection.py) counts its quadrature points here; the online solvers never perform
quadrature, and the tests assert that this counter is unchanged across every online call while a projection
call does increment it, and — where the reference package is importable — that the reference's
own counter is unchanged by the package's host-side online code.
"""

QUADRATURE_EVALS = 0


def count_quadrature(n: int) -> None:
    global QUADRATURE_EVALS
    QUADRATURE_EVALS += int(n)


def quadrature_evals() -> int:
    return QUADRATURE_EVALS
