"""Exception hierarchy of the online-solve API.

Mirrors the reference's ``rbflow.errors`` (/root/reference/pkg/src/rbflow/errors.py:4-21) so callers written
against the reference catch the same types.  ``SingularSystemError`` is what the reference declares for the
SPEC's ``SINGULAR_SYSTEM`` / ``SINGULAR_RECOVERY`` outcomes; ``NativeError`` is new
here and wraps a nonzero return code from the C-ABI library (``include/rbns.h``).
"""


class RbflowError(Exception):
    """Base class for package errors (reference errors.py:4-5)."""


class MeshError(RbflowError):
    """Kept for API parity with the reference (errors.py:8-9); never raised on the online path."""


class OutOfDomainError(RbflowError):
    """A parameter lies outside the supported domain (reference errors.py:12-13)."""


class SingularSystemError(RbflowError):
    """A linear system that should be regular turned out singular (reference errors.py:16-17)."""


class StoreError(RbflowError):
    """Persistent store is missing, corrupt or inconsistent (reference errors.py:20-21)."""


class NativeError(RbflowError):
    """The CUDA library returned an error code (API misuse, CUDA fault, missing extension)."""
