"""File formats of the ``bitalign`` front-end (pkg/src/bitalign/io.py): FASTA,
the pair-list TSV the aligner reads, run-length CIGAR text.

The record types, readers/writers and CIGAR helpers keep the reference's
names, semantics and error texts.  ``load_pairs`` / ``format_align_rows`` are
the fast path the CLI uses: the TSV goes straight from the file image into
the ``ga_batch_in`` arrays and the result rows are written by native code
(``include/genasm_io.h``), multithreaded.  Files with non-ASCII bytes take
the Python reader, whose decoding and ``str.upper()`` are Unicode-aware like
the reference's.
"""

from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass
from typing import IO, Iterable

import numpy as np

from . import _abi
from ._abi import PackedBatch, PackedResults

FASTA_LINE_WIDTH = 60
_ACGT = frozenset("ACGT")
_OPS = "=XID"


class MalformedFasta(ValueError):
    """io.py:23-24"""


class PairParseError(ValueError):
    """io.py:26-29: ``line {n}: {message}``."""

    def __init__(self, line_no: int, message: str):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


class CigarError(ValueError):
    """io.py:32-33"""


@dataclass(frozen=True)
class FastaRecord:
    """io.py:36-50: upper-cased sequence; symbols outside ACGT are kept and
    never match."""

    id: str
    sequence: str

    @property
    def nonstandard(self) -> frozenset[str]:
        return frozenset(self.sequence).difference(_ACGT)


@dataclass(frozen=True)
class PairRecord:
    """io.py:53-59: a read and its candidate reference region."""

    id: str
    pattern: str
    text: str


def read_fasta(stream: IO[str]) -> list[FastaRecord]:
    """io.py:62-89: blank lines ignored, the id is the first header word."""
    records: list[FastaRecord] = []
    name: str | None = None
    seq: list[str] = []

    def close() -> None:
        if name is None:
            return
        joined = "".join(seq)
        if not joined:
            raise MalformedFasta(f"record {name!r} has an empty sequence")
        records.append(FastaRecord(id=name, sequence=joined))

    for raw in stream:
        line = raw.strip()
        if not line:
            continue
        if line[0] == ">":
            close()
            words = line[1:].split()
            if not words:
                raise MalformedFasta("header line with an empty id")
            name, seq = words[0], []
        elif name is None:
            raise MalformedFasta("sequence data before any '>' header")
        else:
            seq.append(line.upper())
    close()
    return records


def write_fasta(records: Iterable[FastaRecord], stream: IO[str],
                line_width: int = FASTA_LINE_WIDTH) -> None:
    """io.py:92-98"""
    for rec in records:
        body = rec.sequence
        stream.write(">" + rec.id + "\n")
        stream.writelines(body[a:a + line_width] + "\n" for a in range(0, len(body), line_width))


def read_pairs(stream: IO[str]) -> list[PairRecord]:
    """io.py:98-113: ``id<TAB>pattern<TAB>text`` rows; blank and '#' lines
    skipped (still counted for line numbers); sequences upper-cased."""
    out: list[PairRecord] = []
    for line_no, raw in enumerate(stream, 1):
        line = raw.rstrip("\n").rstrip("\r")
        if not line.strip() or line.lstrip().startswith("#"):
            continue
        cols = line.split("\t")
        if len(cols) != 3:
            raise PairParseError(line_no, f"expected 3 tab-separated columns, got {len(cols)}")
        if cols[1] == "":
            raise PairParseError(line_no, "empty pattern column")
        out.append(PairRecord(id=cols[0], pattern=cols[1].upper(), text=cols[2].upper()))
    return out


def write_pairs(records: Iterable[PairRecord], stream: IO[str]) -> None:
    """io.py:116-118"""
    stream.writelines(f"{r.id}\t{r.pattern}\t{r.text}\n" for r in records)


def _runs(ops: str) -> str:
    parts: list[str] = []
    a = 0
    n = len(ops)
    while a < n:
        b = a + 1
        while b < n and ops[b] == ops[a]:
            b += 1
        parts.append(f"{b - a}{ops[a]}")
        a = b
    return "".join(parts)


def _check_ops(ops: str) -> None:
    for op in ops:
        if op not in _OPS:
            raise CigarError(f"unknown operator {op!r}")


def format_cigar(ops: str) -> str:
    """io.py:137-142: '====XX=' -> '4=2X1='."""
    _check_ops(ops)
    return _runs(ops)


def parse_cigar(text: str) -> str:
    """io.py:145-160: '2=1I' -> '==I'; CigarError on anything else."""
    out: list[str] = []
    pos = 0
    n = len(text)
    while pos < n:
        d = pos
        while d < n and text[d].isdecimal():
            d += 1
        if d == pos or d == n or text[d] not in _OPS:
            # the reference's regex scan: the junk runs to the next valid run
            nxt = _next_run(text, pos + 1)
            raise CigarError(f"unparsable CIGAR near {text[pos:nxt]!r}")
        count = int(text[pos:d])
        if count == 0:
            raise CigarError(f"zero-length run {text[pos:d + 1]!r}")
        out.append(text[d] * count)
        pos = d + 1
    return "".join(out)


def _next_run(text: str, start: int) -> int:
    """Start of the first ``\\d+[=XID]`` match at or after ``start`` (or len)."""
    n = len(text)
    for a in range(start, n):
        if not text[a].isdecimal():
            continue
        d = a
        while d < n and text[d].isdecimal():
            d += 1
        if d < n and text[d] in _OPS:
            return a
    return n


def collapse_matches(ops: str) -> str:
    """io.py:163-165: '=' and 'X' become classic 'M'."""
    return ops.translate(str.maketrans("=X", "MM"))


def format_classic_cigar(ops: str) -> str:
    """io.py:168-173"""
    _check_ops(ops)
    return _runs(collapse_matches(ops))


# ---------------------------------------------------------------- fast path

@dataclass
class LoadedPairs:
    """A pair-list TSV ready for the device: the packed batch plus the ids."""

    batch: PackedBatch
    ids: bytes            # concatenated UTF-8 ids
    id_off: np.ndarray    # int64, n_pairs + 1
    syms: np.ndarray | None = None  # symbols=True: per-character ids (equal <=> same character)

    @property
    def n_pairs(self) -> int:
        return self.batch.n_pairs

    def id(self, q: int) -> str:
        return self.ids[int(self.id_off[q]):int(self.id_off[q + 1])].decode("utf-8")


def _arr(ptr: int, n: int, dtype) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=dtype)
    item = np.dtype(dtype).itemsize
    return np.frombuffer((C.c_char * (n * item)).from_address(ptr), dtype=dtype).copy()


def parse_pairs_bytes(data: bytes, threads: int = 0, symbols: bool = False) -> LoadedPairs:
    """``read_pairs`` over a whole file image, natively (ASCII files).
    symbols=True also returns per-character symbol ids (for the DP oracle,
    where equal characters match whatever they are)."""
    from .engine import lib
    L = lib()
    out = C.POINTER(_abi.GaPairs)()
    err = C.create_string_buffer(256)
    rc = L.ga_parse_pairs_tsv(data, len(data), threads, _abi.GA_PARSE_SYMBOLS if symbols else 0,
                              C.byref(out), err, 256)
    if rc == _abi.GA_IO_NONASCII:
        import io as _stdio
        return _from_records(read_pairs(_stdio.StringIO(data.decode("utf-8"), newline=None)),
                             symbols)
    if rc == _abi.GA_IO_PARSE:
        msg = err.value.decode()
        head, _, rest = msg.partition(": ")
        if head.startswith("line "):
            raise PairParseError(int(head[5:]), rest)
        raise ValueError(msg)
    if rc != _abi.GA_IO_OK:
        raise MemoryError(err.value.decode() or "ga_parse_pairs_tsv failed")
    try:
        v = out.contents
        n = int(v.n_pairs)
        batch = PackedBatch(codes=_arr(v.codes, max(int(v.codes_len), 1), np.uint8)
                            if v.codes_len else np.zeros(1, np.uint8),
                            pat_off=_arr(v.pat_off, n, np.int64), pat_len=_arr(v.pat_len, n, np.int32),
                            txt_off=_arr(v.txt_off, n, np.int64), txt_len=_arr(v.txt_len, n, np.int32))
        id_off = _arr(v.id_off, n + 1, np.int64)
        ids = C.string_at(v.ids, int(id_off[-1])) if n else b""
        syms = None
        if symbols:
            syms = _arr(v.syms, int(v.codes_len), np.uint8) if v.codes_len else np.zeros(1, np.uint8)
    finally:
        L.ga_pairs_free(out)
    return LoadedPairs(batch=batch, ids=ids, id_off=id_off, syms=syms)


def _from_records(recs: list[PairRecord], symbols: bool = False) -> LoadedPairs:
    enc = [r.id.encode("utf-8") for r in recs]
    id_off = np.zeros(len(recs) + 1, dtype=np.int64)
    if recs:
        np.cumsum([len(e) for e in enc], out=id_off[1:])
    batch = PackedBatch.from_pairs([(r.pattern, r.text) for r in recs])
    syms = None
    if symbols:  # ids by code point: ACGT 0..3, every other character its own id
        table = {"A": 0, "C": 1, "G": 2, "T": 3}
        seq = "".join(r.pattern + r.text for r in recs)
        for ch in set(seq) - set(table):
            table[ch] = len(table)
        if len(table) > 256:
            raise ValueError("more than 252 distinct non-ACGT characters: no symbol ids")
        syms = np.fromiter((table[ch] for ch in seq), dtype=np.uint8, count=len(seq))
        if syms.shape[0] == 0:
            syms = np.zeros(1, np.uint8)
    return LoadedPairs(batch=batch, ids=b"".join(enc), id_off=id_off, syms=syms)


def load_pairs(path: str, threads: int = 0, symbols: bool = False) -> LoadedPairs:
    """``read_pairs(open(path))`` into device-ready arrays.  Raises what the
    reference's loader raises: FileNotFoundError, PairParseError,
    UnicodeDecodeError."""
    with open(path, "rb") as fh:
        data = fh.read()
    return parse_pairs_bytes(data, threads, symbols)


def format_align_rows(pairs: LoadedPairs, out: PackedResults, k: int, collapse_m: bool = False,
                      stats: bool = False, threads: int = 0) -> tuple[bytes, int]:
    """The stdout of ``bitalign align`` (cli.py:104-118) for these results,
    and the number of failed slots."""
    from .engine import lib
    from .window import StuckTraceback
    n = pairs.n_pairs
    if n == 0:
        return b"", 0
    res = out.results
    lens = res["ops_len"].astype(np.int64)
    cap = 200 * n + len(pairs.ids) + 2 * int(lens.sum()) + 64
    buf = np.empty(cap, dtype=np.uint8)
    ids = np.frombuffer(pairs.ids, dtype=np.uint8) if pairs.ids else np.zeros(1, np.uint8)
    flags = (_abi.GA_ROWS_COLLAPSE_M if collapse_m else 0) | (_abi.GA_ROWS_STATS if stats else 0)
    got = lib().ga_format_align_rows(n, ids.ctypes.data, pairs.id_off.ctypes.data, res.ctypes.data,
                                     out.ops.ctypes.data, out.ops_off.ctypes.data, int(out.ops2),
                                     int(k), flags, threads, buf.ctypes.data, cap)
    if got == -2:
        q = int(np.flatnonzero(res["status"] == _abi.GA_STUCK)[0])
        raise StuckTraceback(f"pair {q}: traceback tripwire fired in window "
                             f"{int(res['fail_window'][q])}")
    if got < 0:
        raise RuntimeError("ga_format_align_rows: output buffer too small")
    failed = int(np.count_nonzero(res["status"] != _abi.GA_OK))
    return buf[:got].tobytes(), failed


def write_bytes(data: bytes, stream=None) -> None:
    """Write raw row bytes to a text stream (its binary buffer when it has one)."""
    stream = stream or sys.stdout
    raw = getattr(stream, "buffer", None)
    if raw is not None:
        stream.flush()
        raw.write(data)
        raw.flush()
    else:
        stream.write(data.decode("utf-8"))
