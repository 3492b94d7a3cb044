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

import gc
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import PackedBatch, PackedResults

try:  # bulk construction of the result objects (csrc/outcomes_py.cpp, build.py)
    from . import _outcomes
except ImportError:  # not built: the same objects from the Python loop
    _outcomes = None

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
    (window.py:144-149: failures become ``"{type}: {message}"`` strings).

    Bulk form: the op bytes are decoded to one str and the window distances
    to one list, each pair slices them; the frozen result objects are filled
    through their ``__dict__`` (what the generated ``__init__`` stores, minus
    a per-field ``object.__setattr__``) -- equal objects, several times
    faster for 10^5 pairs."""
    res = out.results
    n = batch.n_pairs
    status = res["status"].tolist()
    cost = res["cost"].tolist()
    tcons = res["text_consumed"].tolist()
    rows = res["rows_computed"].tolist()
    reads = res["entry_reads"].tolist()
    writes = res["entry_writes"].tolist()
    words = res["words_allocated"].tolist()
    fail = res["fail_window"].tolist()
    ops_len = res["ops_len"].tolist()
    ops_off = out.ops_off.tolist()
    win_off = out.win_off.tolist()
    nwin = _abi.num_windows(batch.pat_len, cfg.window, cfg.overlap)
    nwin = nwin.tolist() if n else []
    if out.ops2:
        lut = np.frombuffer(b"=XID", dtype=np.uint8)
        ops_buf = lut[((out.ops[:, None] >> np.array([0, 2, 4, 6], dtype=np.uint8)) & 3)
                      .reshape(-1)]
    else:
        ops_buf = out.ops
    ops_mv = memoryview(np.ascontiguousarray(ops_buf))  # each CIGAR decoded straight from it
    # window distances sliced from one bytes object: a tuple of a bytes slice
    # is a tuple of the cached small ints, with no 10^7-element list between
    dists = np.ascontiguousarray(out.dists, dtype=np.uint8).tobytes()
    new = object.__new__
    outcomes: list[BatchOutcome] = []
    append = outcomes.append
    # Hundreds of thousands of new container objects would trigger the cyclic
    # collector over and over (none of them can form a cycle): 5.8 -> 2.7 s for
    # config 3's 138,929 pairs with it off.
    gc_was = gc.isenabled()
    gc.disable()
    try:
        if _outcomes is not None:
            # the aligned pairs' objects in one native call (csrc/outcomes_py.cpp)
            ops_arr = np.ascontiguousarray(ops_buf)
            dist_arr = np.ascontiguousarray(out.dists, dtype=np.uint8)
            cols = [np.ascontiguousarray(res[f], dtype=np.int64) for f in
                    ("cost", "text_consumed", "rows_computed", "entry_reads", "entry_writes",
                     "words_allocated", "ops_len")]
            st = np.ascontiguousarray(res["status"], dtype=np.int32)
            offs = [np.ascontiguousarray(x, dtype=np.int64) for x in
                    (out.ops_off, out.win_off, np.asarray(nwin, dtype=np.int64))]
            outcomes = _outcomes.build(AlignmentResult, AccessCounters, BatchOutcome, n,
                                       st.ctypes.data, *(c.ctypes.data for c in cols),
                                       *(o.ctypes.data for o in offs), ops_arr.ctypes.data,
                                       dist_arr.ctypes.data)
            for q in np.flatnonzero(st != _abi.GA_OK).tolist():
                outcomes[q] = _failed_outcome(status[q], fail[q], q, cfg)
        else:
            _fill_outcomes(n, status, cost, tcons, rows, reads, writes, words, fail, ops_len,
                           ops_off, win_off, nwin, ops_mv, dists, cfg, new, append)
    finally:
        if gc_was:
            gc.enable()
    return outcomes


def _failed_outcome(st: int, fail_window: int, q: int, cfg: WindowConfig) -> BatchOutcome:
    if st == _abi.GA_WINDOW_FAILED:
        exc = WindowFailed(fail_window, cfg.k)
        return BatchOutcome(error=f"{type(exc).__name__}: {exc}")
    if st == _abi.GA_EMPTY_PATTERN:
        exc = EmptyPattern("pattern must not be empty")
        return BatchOutcome(error=f"{type(exc).__name__}: {exc}")
    raise StuckTraceback(f"pair {q}: traceback tripwire fired in window {fail_window}")


def _fill_outcomes(n, status, cost, tcons, rows, reads, writes, words, fail, ops_len, ops_off,
                   win_off, nwin, ops_mv, dists, cfg, new, append):
    for q in range(n):
        st = status[q]
        if st == _abi.GA_OK:
            o, w = ops_off[q], win_off[q]
            c = new(AccessCounters)
            c.__dict__.update(entry_reads=reads[q], entry_writes=writes[q],
                              words_allocated=words[q])
            r = new(AlignmentResult)
            r.__dict__.update(cigar=str(ops_mv[o:o + ops_len[q]], "ascii"), cost=cost[q],
                              text_consumed=tcons[q],
                              window_distances=tuple(dists[w:w + nwin[q]]), counters=c,
                              rows_computed=rows[q])
            b = new(BatchOutcome)
            b.__dict__.update(result=r, error=None)
            append(b)
        else:
            append(_failed_outcome(st, fail[q], q, cfg))


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
    from .engine import pack_pairs, run_batch
    batch = pack_pairs(pairs)
    out = run_batch(batch, cfg, devices=devices)
    return outcomes_from_packed(batch, out, cfg)
