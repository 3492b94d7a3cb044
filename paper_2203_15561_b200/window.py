"""Drop-in alignment API: the reference's windowed driver names, on the GPU.

Mirrors ``bitalign.window`` (pkg/src/bitalign/window.py) name for name --
``WindowConfig``, ``AlignmentResult``, ``BatchOutcome``, ``EmptyPattern``,
``WindowFailed``, ``align``, ``align_batch`` -- with identical validation,
field values and error strings.  Underneath, every alignment runs in the
fused GenASM-DC + GenASM-TB sm_100a kernel through the C-ABI in
include/genasm.h; there is no CPU fallback.  Two inputs the reference
accepts are rejected with ``ValueError`` because they have no GPU path:
``mode="baseline"`` (the unimproved engine) and ``window > 128``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import _abi
from ._abi import PackedBatch, PackedResults

DEFAULT_WINDOW = 64
DEFAULT_OVERLAP = 24
DEFAULT_PRIORITY = "MSID"
MODES = ("improved", "baseline")
OP_COST = {"=": 0, "X": 1, "I": 1, "D": 1}


class EmptyPattern(ValueError):
    """Alignment of an empty pattern was requested (window.py:31-32)."""


class WindowFailed(RuntimeError):
    """A window's distance exceeded the configured threshold (window.py:35-41)."""

    def __init__(self, window_index: int, k: int):
        super().__init__(f"window {window_index} found no alignment within k={k}")
        self.window_index = window_index
        self.k = k


class StuckTraceback(RuntimeError):
    """No edge bit active at a traceback state (backtrace.py:30-35); the kernel's
    tripwire for a corrupt table.  Never raised on tables the DC produced."""


def validate_priority(priority: str) -> str:
    """backtrace.py:64-67."""
    if sorted(priority) != sorted(DEFAULT_PRIORITY):
        raise ValueError(f"priority must be a permutation of 'MSID', got {priority!r}")
    return priority


@dataclass
class AccessCounters:
    """Persistent-table traffic counters (dptable.py:85-105), computed by the
    kernel with the reference's stored-column predicate (dptable.py:62-82)."""

    entry_reads: int = 0
    entry_writes: int = 0
    words_allocated: int = 0

    @property
    def total_accesses(self) -> int:
        return self.entry_reads + self.entry_writes

    def absorb(self, other: "AccessCounters") -> None:
        self.entry_reads += other.entry_reads
        self.entry_writes += other.entry_writes
        self.words_allocated += other.words_allocated


@dataclass(frozen=True)
class WindowConfig:
    """Driver parameters (window.py:44-70); same defaults and messages."""

    window: int = DEFAULT_WINDOW
    overlap: int = DEFAULT_OVERLAP
    k: int | None = None
    priority: str = DEFAULT_PRIORITY
    mode: str = "improved"

    def __post_init__(self):
        if self.window < 1:
            raise ValueError(f"window must be >= 1, got {self.window}")
        if not 0 <= self.overlap < self.window:
            raise ValueError(
                f"overlap must be in [0, window), got {self.overlap} for window {self.window}")
        if self.k is None:
            object.__setattr__(self, "k", self.window)
        if not 1 <= self.k <= self.window:
            raise ValueError(f"k must be in [1, {self.window}], got {self.k}")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        validate_priority(self.priority)


@dataclass(frozen=True)
class AlignmentResult:
    """Full-pattern alignment (window.py:73-82)."""

    cigar: str
    cost: int
    text_consumed: int
    window_distances: tuple[int, ...]
    counters: AccessCounters
    rows_computed: int


@dataclass(frozen=True)
class BatchOutcome:
    """One slot of a batch (window.py:132-141)."""

    result: AlignmentResult | None = None
    error: str | None = field(default=None)

    @property
    def ok(self) -> bool:
        return self.error is None


def _require_gpu_config(cfg: WindowConfig) -> None:
    if cfg.window > _abi.GA_MAX_WINDOW:
        raise ValueError(
            f"window {cfg.window} exceeds the kernel maximum of {_abi.GA_MAX_WINDOW}")


def outcomes_from_packed(batch: PackedBatch, out: PackedResults,
                         cfg: WindowConfig) -> list[BatchOutcome]:
    """Rebuild the reference's per-slot objects from the C-ABI records
    (window.py:144-149: failures become ``"{type}: {message}"`` strings)."""
    res = out.results
    outcomes: list[BatchOutcome] = []
    status = res["status"].tolist()
    for q in range(batch.n_pairs):
        st = status[q]
        if st == _abi.GA_OK:
            r = res[q]
            outcomes.append(BatchOutcome(result=AlignmentResult(
                cigar=out.cigar(q),
                cost=int(r["cost"]),
                text_consumed=int(r["text_consumed"]),
                window_distances=out.distances(q, int(batch.pat_len[q]), cfg.window, cfg.overlap),
                counters=AccessCounters(int(r["entry_reads"]), int(r["entry_writes"]),
                                        int(r["words_allocated"])),
                rows_computed=int(r["rows_computed"]),
            )))
        elif st == _abi.GA_WINDOW_FAILED:
            exc = WindowFailed(int(res["fail_window"][q]), cfg.k)
            outcomes.append(BatchOutcome(error=f"{type(exc).__name__}: {exc}"))
        elif st == _abi.GA_EMPTY_PATTERN:
            exc = EmptyPattern("pattern must not be empty")
            outcomes.append(BatchOutcome(error=f"{type(exc).__name__}: {exc}"))
        else:
            raise StuckTraceback(
                f"pair {q}: traceback tripwire fired in window {int(res['fail_window'][q])}")
    return outcomes


def align(pattern: str, text: str, cfg: WindowConfig = WindowConfig()) -> AlignmentResult:
    """Align the whole pattern against a prefix of the text (window.py:85-129)."""
    if not pattern:
        raise EmptyPattern("pattern must not be empty")
    _require_gpu_config(cfg)
    from .engine import run_batch
    batch = PackedBatch.from_pairs([(pattern, text)])
    out = run_batch(batch, cfg)
    st = int(out.results["status"][0])
    if st == _abi.GA_WINDOW_FAILED:
        raise WindowFailed(int(out.results["fail_window"][0]), cfg.k)
    return outcomes_from_packed(batch, out, cfg)[0].result


def align_batch(pairs: list[tuple[str, str]], cfg: WindowConfig,
                parallelism: int = 1, *, devices=None) -> list[BatchOutcome]:
    """Align many pairs; results in input order, bit-identical at any
    parallelism degree or device count (window.py:152-163).

    ``parallelism`` is accepted for signature compatibility (the reference's
    process-pool width); GPU parallelism comes from the kernel.  ``devices``
    (an int count or a list of CUDA ordinals) shards the pairs across GPUs.
    """
    _require_gpu_config(cfg)
    if not pairs:
        return []
    from .engine import run_batch
    batch = PackedBatch.from_pairs(pairs)
    out = run_batch(batch, cfg, devices=devices)
    return outcomes_from_packed(batch, out, cfg)
