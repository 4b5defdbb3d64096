"""Error types of the stencil hot path.

Mirrors the reference's two contract errors (``lattice.py:22-27``):
``UsageError(ValueError)`` for operands that violate a contract and
``ResourceError(RuntimeError)`` for exceeded resource limits.  A third,
``DeviceError``, carries CUDA failures reported by the C-ABI (status 3).
"""
from __future__ import annotations


class UsageError(ValueError):
    """An operation was called with operands that violate its contract."""


class ResourceError(RuntimeError):
    """A configured resource limit was exceeded (shared memory, box count)."""


class DeviceError(RuntimeError):
    """The CUDA runtime reported a failure inside the C-ABI library."""
