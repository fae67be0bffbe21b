"""Error types and the (accepted, ignored) execution plan of the reference's
`tissuemix.linalg` (reference linalg.py:46-64, 301-328).

The CUDA engine always reduces with a fixed tree (deterministic for any
worker or GPU count), so `ExecPlan` is kept only for signature parity.
`install()` in `vb.py` swaps these classes for the reference's own so that
callers catching `tissuemix.linalg.NumericError` keep working.
"""

from __future__ import annotations

from dataclasses import dataclass


class BatchItemError(ValueError):
    """A batched operation failed on specific items (reference linalg.py:46-60)."""

    def __init__(self, msg, indices, pivots=None):
        super().__init__(f"{msg} (items {list(indices)})")
        self.indices = list(indices)
        self.pivots = list(pivots) if pivots is not None else None


class NumericError(RuntimeError):
    """Numerical failure that survived the jitter-once retry (reference linalg.py:63-64)."""


DEFAULT_CHUNK = 1024


@dataclass(frozen=True)
class ExecPlan:
    """Signature-compatible stand-in for reference linalg.ExecPlan (ignored by the engine)."""

    workers: int = 1
    chunk_size: int = DEFAULT_CHUNK
    deterministic: bool = True
