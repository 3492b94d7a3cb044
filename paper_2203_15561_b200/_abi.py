"""ctypes mirror of include/genasm.h plus host-side batch packing (H1).

Packing turns the reference's ``pairs: list[tuple[str, str]]`` argument of
``align_batch`` (pkg/src/bitalign/window.py:152-163) into one code array plus
offsets, and unpacks the C-ABI's per-pair records back into the reference's
result objects.  Symbol coding follows the reference's masks exactly
(pkg/src/bitalign/distance.py:70-79): only the uppercase code units 'A', 'C',
'G', 'T' have a mask; every other code unit -- lowercase, 'N', non-ASCII --
maps to code 4 and never matches anything, itself included.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

GA_OK = 0
GA_WINDOW_FAILED = 1
GA_EMPTY_PATTERN = 2
GA_STUCK = 3
GA_MAX_WINDOW = 128


class GaConfig(C.Structure):
    _fields_ = [("window", C.c_int32), ("overlap", C.c_int32), ("k", C.c_int32),
                ("priority", C.c_char * 4), ("mode", C.c_int32)]


class GaBatchIn(C.Structure):
    _fields_ = [("n_pairs", C.c_int64), ("codes", C.c_void_p), ("codes_len", C.c_int64),
                ("pat_off", C.c_void_p), ("pat_len", C.c_void_p),
                ("txt_off", C.c_void_p), ("txt_len", C.c_void_p), ("order", C.c_void_p),
                ("packed2", C.c_int32), ("n_exceptions", C.c_int64),
                ("exceptions", C.c_void_p)]


# ga_batch_in.packed2 (include/genasm.h)
GA_PACK_NONE, GA_PACK_CALLER, GA_PACK_HOST = 0, 1, 2


class GaBatchOut(C.Structure):
    _fields_ = [("results", C.c_void_p), ("ops_off", C.c_void_p), ("ops", C.c_void_p),
                ("ops_capacity", C.c_int64), ("win_off", C.c_void_p),
                ("window_distances", C.c_void_p), ("win_capacity", C.c_int64),
                ("ops2", C.c_int32)]


class GaPairs(C.Structure):
    """ga_pairs (include/genasm_io.h): a parsed pair-list TSV."""
    _fields_ = [("n_pairs", C.c_int64), ("codes", C.c_void_p), ("codes_len", C.c_int64),
                ("pat_off", C.c_void_p), ("pat_len", C.c_void_p), ("txt_off", C.c_void_p),
                ("txt_len", C.c_void_p), ("ids", C.c_void_p), ("id_off", C.c_void_p),
                ("syms", C.c_void_p), ("impl", C.c_void_p)]


GA_IO_OK, GA_IO_PARSE, GA_IO_NONASCII, GA_IO_NOMEM = 0, 1, 2, 3
GA_ROWS_COLLAPSE_M, GA_ROWS_STATS = 1, 2
GA_PARSE_SYMBOLS = 1


# ga_pair_result, 64 bytes
RESULT_DTYPE = np.dtype([
    ("status", np.int32), ("fail_window", np.int32), ("cost", np.int64),
    ("text_consumed", np.int64), ("rows_computed", np.int64), ("ops_len", np.int64),
    ("entry_reads", np.int64), ("entry_writes", np.int64), ("words_allocated", np.int64),
])
assert RESULT_DTYPE.itemsize == 64

_LUT = np.full(256, 4, dtype=np.uint8)
for _code, _sym in enumerate(b"ACGT"):
    _LUT[_sym] = _code


def encode(seq: str) -> np.ndarray:
    """Code units of one sequence -> uint8 codes (0..3 = ACGT, 4 = other)."""
    if seq.isascii():
        return _LUT[np.frombuffer(seq.encode("ascii"), dtype=np.uint8)]
    units = np.frombuffer(seq.encode("utf-32-le"), dtype=np.uint32)
    return np.where(units < 128, _LUT[np.minimum(units, 255)], 4).astype(np.uint8)


def num_windows(pattern_len: np.ndarray | int, window: int, overlap: int):
    """#windows align() walks: 1 + ceil(max(0, |P| - W) / (W - O)); 0 if |P| == 0
    (pkg/src/bitalign/window.py:95-120)."""
    lp = np.asarray(pattern_len, dtype=np.int64)
    step = window - overlap
    extra = np.maximum(lp - window, 0)
    out = np.where(lp > 0, 1 + (extra + step - 1) // step, 0)
    return out if out.ndim else int(out)


@dataclass
class PackedBatch:
    """Host-side packed pairs: the ``ga_batch_in`` arrays."""

    codes: np.ndarray     # uint8
    pat_off: np.ndarray   # int64
    pat_len: np.ndarray   # int32
    txt_off: np.ndarray   # int64
    txt_len: np.ndarray   # int32

    @property
    def n_pairs(self) -> int:
        return int(self.pat_len.shape[0])

    @classmethod
    def from_pairs(cls, pairs) -> "PackedBatch":
        n = len(pairs)
        parts: list[np.ndarray] = []
        pat_len = np.empty(n, dtype=np.int32)
        txt_len = np.empty(n, dtype=np.int32)
        all_ascii = all(p.isascii() and t.isascii() for p, t in pairs)
        if all_ascii:
            # one join + one table lookup for the whole batch
            blob = "".join(p + t for p, t in pairs).encode("ascii")
            codes = _LUT[np.frombuffer(blob, dtype=np.uint8)] if blob else np.zeros(0, np.uint8)
            for q, (p, t) in enumerate(pairs):
                pat_len[q] = len(p)
                txt_len[q] = len(t)
        else:
            for q, (p, t) in enumerate(pairs):
                parts.append(encode(p))
                parts.append(encode(t))
                pat_len[q] = len(p)
                txt_len[q] = len(t)
            codes = np.concatenate(parts) if parts else np.zeros(0, np.uint8)
        lens = np.empty(2 * n, dtype=np.int64)
        lens[0::2] = pat_len
        lens[1::2] = txt_len
        starts = np.zeros(2 * n, dtype=np.int64)
        if n:
            np.cumsum(lens[:-1], out=starts[1:])
        return cls(codes=np.ascontiguousarray(codes, dtype=np.uint8),
                   pat_off=starts[0::2].copy(), pat_len=pat_len,
                   txt_off=starts[1::2].copy(), txt_len=txt_len)

    def struct(self, order: np.ndarray | None = None,
               packed: "Packed2 | None" = None) -> GaBatchIn:
        """ga_batch_in over these arrays; with `packed`, the sequences travel
        as 2-bit symbols plus the exception list (offsets stay in symbols)."""
        s = GaBatchIn(self.n_pairs, self.codes.ctypes.data, int(self.codes.shape[0]),
                      self.pat_off.ctypes.data, self.pat_len.ctypes.data,
                      self.txt_off.ctypes.data, self.txt_len.ctypes.data,
                      None if order is None else order.ctypes.data)
        if packed is not None:
            s.codes = packed.data.ctypes.data
            s.packed2 = GA_PACK_CALLER
            s.n_exceptions = int(packed.exceptions.shape[0])
            s.exceptions = packed.exceptions.ctypes.data if packed.exceptions.shape[0] else None
        return s


@dataclass
class Packed2:
    """2-bit transfer form of a code array (ga_batch_in.packed2): symbol x in
    bits 2(x%4).. of byte x/4, code-4 positions listed in `exceptions`."""

    data: np.ndarray        # uint8, ceil(n/4)
    exceptions: np.ndarray  # int64, ascending


_OPS_LUT = np.frombuffer(b"=XID", dtype=np.uint8)


@dataclass
class PackedResults:
    """Host-side outputs: the ``ga_batch_out`` arrays."""

    results: np.ndarray   # RESULT_DTYPE
    ops_off: np.ndarray   # int64, in ops
    ops: np.ndarray       # uint8: ASCII ops, or 2-bit ops (four per byte) when ops2
    win_off: np.ndarray   # int64
    dists: np.ndarray     # uint8
    ops2: bool = False
    n_ops: int = 0        # ops capacity

    @classmethod
    def allocate(cls, batch: PackedBatch, window: int, overlap: int,
                 ops2: bool = False) -> "PackedResults":
        n = batch.n_pairs
        cap = batch.pat_len.astype(np.int64) + batch.txt_len.astype(np.int64)
        if ops2:  # every pair's ops start on a byte boundary
            cap = (cap + 3) & ~np.int64(3)
        ops_off = np.zeros(n, dtype=np.int64)
        if n:
            np.cumsum(cap[:-1], out=ops_off[1:])
        nwin = num_windows(batch.pat_len, window, overlap)
        win_off = np.zeros(n, dtype=np.int64)
        if n:
            np.cumsum(nwin[:-1], out=win_off[1:])
        total = int(cap.sum())
        nbytes = (total + 3) // 4 if ops2 else total
        return cls(results=np.zeros(n, dtype=RESULT_DTYPE), ops_off=ops_off,
                   ops=np.zeros(max(1, nbytes), dtype=np.uint8), win_off=win_off,
                   dists=np.zeros(max(1, int(nwin.sum())), dtype=np.uint8), ops2=ops2,
                   n_ops=total)

    def struct(self) -> GaBatchOut:
        return GaBatchOut(self.results.ctypes.data, self.ops_off.ctypes.data,
                          self.ops.ctypes.data, self.n_ops, self.win_off.ctypes.data,
                          self.dists.ctypes.data, int(self.dists.nbytes), int(self.ops2))

    def cigar(self, q: int) -> str:
        off = int(self.ops_off[q])
        n_ops = int(self.results["ops_len"][q])
        if self.ops2:
            b = self.ops[off // 4:(off + n_ops + 3) // 4]
            codes = (b[:, None] >> np.array([0, 2, 4, 6], dtype=np.uint8)) & 3
            return _OPS_LUT[codes.reshape(-1)[:n_ops]].tobytes().decode("ascii")
        return self.ops[off:off + n_ops].tobytes().decode("ascii")

    def distances(self, q: int, pattern_len: int, window: int, overlap: int) -> tuple[int, ...]:
        off = int(self.win_off[q])
        count = num_windows(pattern_len, window, overlap)
        return tuple(self.dists[off:off + count].tolist())


GA_MODE_IMPROVED, GA_MODE_BASELINE = 0, 1
MODE_IDS = {"improved": GA_MODE_IMPROVED, "baseline": GA_MODE_BASELINE}


def make_config(window: int, overlap: int, k: int, priority: str,
                mode: str = "improved") -> GaConfig:
    return GaConfig(window, overlap, k, priority.encode("ascii"), MODE_IDS[mode])
