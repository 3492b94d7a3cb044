"""B200-native improved GenASM (arXiv 2203.15561): windowed GenASM-DC + GenASM-TB.

Drop-in for the hot path of the reference package ``bitalign``
(pkg/src/bitalign/__init__.py:40-48): the same ``align`` / ``align_batch``
API and result types, computed by hand-written sm_100a CUDA kernels behind
the C-ABI in include/genasm.h.
"""

from .window import (
    DEFAULT_OVERLAP,
    DEFAULT_PRIORITY,
    DEFAULT_WINDOW,
    OP_COST,
    AccessCounters,
    AlignmentResult,
    BatchOutcome,
    EmptyPattern,
    StuckTraceback,
    WindowConfig,
    WindowFailed,
    align,
    align_batch,
    validate_priority,
)

__version__ = "0.1.0"

__all__ = [
    "AccessCounters",
    "AlignmentResult",
    "BatchOutcome",
    "DEFAULT_OVERLAP",
    "DEFAULT_PRIORITY",
    "DEFAULT_WINDOW",
    "EmptyPattern",
    "OP_COST",
    "StuckTraceback",
    "WindowConfig",
    "WindowFailed",
    "align",
    "align_batch",
    "validate_priority",
]
