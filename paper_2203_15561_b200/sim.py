"""Synthetic workloads: the reference simulator's recipe, bit-exact, in C++.

``make_reference`` / ``simulate_read`` reproduce pkg/src/bitalign/sim.py:60-103
and ``recipe_pairs`` reproduces ``bitalign simulate --emit-pairs``
(pkg/src/bitalign/cli.py:139-169): same seeds, same MT19937 stream, same
reads, so every bench/parity input is a pair set the reference's own tools
generate.  ``CONFIGS`` are the five BASELINE.json shapes with the seeds of
SURVEY.md 8(d).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import random
from dataclasses import dataclass

import numpy as np

from ._abi import PackedBatch

_ALPHA = np.frombuffer(b"ACGT", dtype=np.uint8)
_sim_lib = None


def _lib():
    # GA_SIM_SO: the generator built on its own (oracle/_oracle_sim.so), for
    # bench.py's CPU reference arm, which must not load the product library
    global _sim_lib
    if _sim_lib is None:
        path = os.environ.get("GA_SIM_SO")
        if path:
            _sim_lib = C.CDLL(path)
        else:
            from .engine import lib
            _sim_lib = lib()
    L = _sim_lib
    if not getattr(L, "_sim_sigs", False):
        L.ga_sim_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ga_sim_derive_seed.restype = C.c_uint64
        L.ga_sim_reference.argtypes = [C.c_int64, C.c_uint64, C.c_void_p]
        L.ga_sim_reference.restype = None
        L.ga_sim_read.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_double,
                                  C.c_double, C.c_uint64, C.c_void_p]
        L.ga_sim_read.restype = C.c_int64
        L.ga_sim_read_truth.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_int64)]
        L.ga_sim_read_truth.restype = C.c_int64
        L.ga_sim_positions.argtypes = [C.c_int64, C.c_int64, C.c_void_p, C.c_uint64, C.c_void_p]
        L.ga_sim_positions.restype = None
        L.ga_sim_read_lengths.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                          C.c_double, C.c_double, C.c_double, C.c_uint64,
                                          C.c_int, C.c_void_p]
        L.ga_sim_read_lengths.restype = None
        L.ga_sim_fill_pairs.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
        L.ga_sim_fill_pairs.restype = None
        L._sim_sigs = True
    return L


def derive_seed(seed: int, *salts: int) -> int:
    """sim.py:53-57."""
    mixed = seed & ((1 << 64) - 1)
    for salt in salts:
        mixed = _lib().ga_sim_derive_seed(mixed, salt & ((1 << 64) - 1))
    return int(mixed)


def make_reference(length: int, seed: int) -> np.ndarray:
    """Codes (0..3) of ``bitalign.sim.make_reference(length, seed)``."""
    if length < 1:
        raise ValueError(f"reference length must be >= 1, got {length}")
    out = np.empty(length, dtype=np.uint8)
    _lib().ga_sim_reference(length, seed & ((1 << 64) - 1), out.ctypes.data)
    return out


def codes_to_str(codes: np.ndarray) -> str:
    return _ALPHA[codes].tobytes().decode("ascii")


def simulate_read(ref: np.ndarray, pos: int, length: int, sub: float, ins: float, dele: float,
                  seed: int) -> np.ndarray:
    """Codes of ``simulate_read(reference, pos, length, ErrorProfile(sub, ins, del, seed)).read``."""
    ref = np.ascontiguousarray(ref, dtype=np.uint8)
    if pos < 0 or length < 1 or pos + length > ref.shape[0]:
        raise ValueError("slice out of range")
    out = np.empty(2 * length, dtype=np.uint8)
    n = _lib().ga_sim_read(ref.ctypes.data, pos, length, sub, ins, dele, seed, out.ctypes.data)
    return out[:n].copy()


def simulate_read_truth(ref: np.ndarray, pos: int, length: int, sub: float, ins: float,
                        dele: float, seed: int) -> tuple[np.ndarray, str]:
    """``simulate_read(...)`` (sim.py:68-103) as (read codes, edit script): the
    script's run-length form is ``SimRecord.truth_cigar`` and its non-'=' count
    ``truth_cost``."""
    ref = np.ascontiguousarray(ref, dtype=np.uint8)
    if pos < 0 or length < 1 or pos + length > ref.shape[0]:
        raise ValueError("slice out of range")
    out = np.empty(2 * length, dtype=np.uint8)
    ops = C.create_string_buffer(2 * length)
    k = C.c_int64(0)
    n = _lib().ga_sim_read_truth(ref.ctypes.data, pos, length, sub, ins, dele, seed,
                                 out.ctypes.data, ops, C.byref(k))
    return out[:n].copy(), ops.raw[:k.value].decode("ascii")


def recipe_pairs(ref: np.ndarray, count: int, read_lens, sub: float, ins: float, dele: float,
                 seed: int, threads: int | None = None) -> tuple[PackedBatch, np.ndarray]:
    """``simulate --emit-pairs`` (cli.py:139-169) as a packed batch: pair i is
    (read i, reference[pos_i : pos_i + read_len_i]).  ``read_lens`` is an int
    (the CLI's --read-len) or one length per read.  Returns (batch, positions)."""
    ref = np.ascontiguousarray(ref, dtype=np.uint8)
    L = _lib()
    threads = threads or os.cpu_count() or 1
    rl = np.full(count, read_lens, dtype=np.int32) if np.isscalar(read_lens) else \
        np.ascontiguousarray(read_lens, dtype=np.int32)
    if count and (rl.min() < 1 or rl.max() > ref.shape[0]):
        raise ValueError("read length out of range")
    pos = np.empty(count, dtype=np.int64)
    L.ga_sim_positions(ref.shape[0], count, rl.ctypes.data, seed, pos.ctypes.data)
    plen = np.empty(count, dtype=np.int32)
    L.ga_sim_read_lengths(ref.ctypes.data, count, pos.ctypes.data, rl.ctypes.data, sub, ins, dele,
                          seed, threads, plen.ctypes.data)
    lens = np.empty(2 * count, dtype=np.int64)
    lens[0::2] = plen
    lens[1::2] = rl
    starts = np.zeros(2 * count, dtype=np.int64)
    if count:
        np.cumsum(lens[:-1], out=starts[1:])
    total = int(lens.sum())
    codes = np.empty(max(total, 1), dtype=np.uint8)
    pat_off = starts[0::2].copy()
    txt_off = starts[1::2].copy()
    L.ga_sim_fill_pairs(ref.ctypes.data, count, pos.ctypes.data, rl.ctypes.data, sub, ins, dele,
                        seed, threads, pat_off.ctypes.data, txt_off.ctypes.data, codes.ctypes.data)
    return PackedBatch(codes=codes, pat_off=pat_off, pat_len=plen, txt_off=txt_off,
                       txt_len=rl.copy()), pos


@dataclass(frozen=True)
class Recipe:
    """One BASELINE.json configuration."""

    name: str
    ref_len: int
    count: int
    read_len: int          # 0 = per-read log-uniform lengths (config 5)
    sub: float
    ins: float
    dele: float
    seed: int


CONFIGS = {
    1: Recipe("150bp_2pct", 2_000_000, 10_000, 150, 0.01, 0.005, 0.005, 1501),
    2: Recipe("250bp_5pct_illumina", 5_000_000, 100_000, 250, 0.04, 0.005, 0.005, 2502),
    3: Recipe("10kb_15pct_pbsim2", 20_000_000, 138_929, 10_000, 0.01, 0.07, 0.07, 10003),
    4: Recipe("100kb_10pct_ont", 50_000_000, 20_000, 100_000, 0.04, 0.02, 0.04, 100004),
    5: Recipe("mixed_100bp_50kb", 5_000_000, 8_192, 0, 0.04, 0.03, 0.03, 5005),
}

# config-5 sweep points: W in {32, 64, 128}, O = 3W/8, k in {W/4, W/2, W}
SWEEP5 = [(w, 3 * w // 8, k) for w in (32, 64, 128) for k in (w // 4, w // 2, w)]


def mixed_lengths(count: int, seed: int, lo: int = 100, hi: int = 50_000) -> np.ndarray:
    """Config-5 read lengths: log-uniform in [lo, hi] from random.Random(seed)."""
    rng = random.Random(seed)
    a, b = math.log(lo), math.log(hi)
    return np.array([int(round(math.exp(rng.uniform(a, b)))) for _ in range(count)],
                    dtype=np.int32)


def config_pairs(cfg_id: int, count: int | None = None, threads: int | None = None,
                 ref: np.ndarray | None = None) -> tuple[PackedBatch, np.ndarray]:
    """The first ``count`` pairs (default: all) of BASELINE config ``cfg_id``."""
    r = CONFIGS[cfg_id]
    n = r.count if count is None else min(count, r.count)
    if ref is None:
        ref = make_reference(r.ref_len, r.seed)
    if r.read_len:
        lens = r.read_len
    else:
        lens = mixed_lengths(r.count, r.seed)[:n]
    return recipe_pairs(ref, n, lens, r.sub, r.ins, r.dele, r.seed, threads)
