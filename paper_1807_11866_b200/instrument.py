"""Quadrature-evaluation counter (mirror of /root/reference/pkg/src/rbflow/instrument.py:1-17).

The online solvers of this package never perform quadrature; tests assert that this counter (and, in the
development container, the reference's own counter) is unchanged across online calls.
"""

QUADRATURE_EVALS = 0


def count_quadrature(n: int) -> None:
    global QUADRATURE_EVALS
    QUADRATURE_EVALS += int(n)


def quadrature_evals() -> int:
    return QUADRATURE_EVALS
