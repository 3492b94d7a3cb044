"""Ground-truth edit distances on the GPU (the reference's ``bitalign.oracle``
distances, pkg/src/bitalign/oracle.py:24-74), for the accuracy columns of
``bench``: the classical DP's values computed by a bit-vector kernel
(``ga_edit_distance``, csrc/genasm_dp.cu), many pairs per launch.

Characters are compared as characters: unlike the aligner, 'N' matches 'N'
here, exactly as in the reference's DP.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._abi import PackedBatch


def _symbol_batch(pairs: list[tuple[str, str]]) -> PackedBatch:
    table = {"A": 0, "C": 1, "G": 2, "T": 3}
    seq = "".join(p + t for p, t in pairs)
    for ch in set(seq) - set(table):
        table[ch] = len(table)
    if len(table) > 256:
        raise ValueError("more than 252 distinct non-ACGT characters")
    ids = np.fromiter((table[ch] for ch in seq), dtype=np.uint8, count=len(seq))
    n = len(pairs)
    lens = np.empty(2 * n, dtype=np.int64)
    lens[0::2] = [len(p) for p, _ in pairs]
    lens[1::2] = [len(t) for _, t in pairs]
    starts = np.zeros(2 * n, dtype=np.int64)
    if n:
        np.cumsum(lens[:-1], out=starts[1:])
    return PackedBatch(codes=ids if ids.size else np.zeros(1, np.uint8),
                       pat_off=starts[0::2].copy(), pat_len=lens[0::2].astype(np.int32),
                       txt_off=starts[1::2].copy(), txt_len=lens[1::2].astype(np.int32))


def edit_distances(batch: PackedBatch, semiglobal: bool = False, device: int | None = None,
                   symbols: np.ndarray | None = None) -> np.ndarray:
    """Distances of every pair of ``batch`` (int64; -1 for an empty pattern
    when semiglobal).  ``symbols`` replaces ``batch.codes`` with per-character
    ids (``io.load_pairs(..., symbols=True)``); with aligner codes, every
    non-ACGT character compares equal to every other."""
    from .engine import _ctx_locks, _default_device, context, lib
    dev = _default_device() if device is None else int(device)
    ctx = context(dev)
    out = np.zeros(batch.n_pairs, dtype=np.int64)
    if batch.n_pairs == 0:
        return out
    src = batch if symbols is None else PackedBatch(codes=symbols, pat_off=batch.pat_off,
                                                    pat_len=batch.pat_len, txt_off=batch.txt_off,
                                                    txt_len=batch.txt_len)
    bin_ = src.struct()
    with _ctx_locks[dev]:
        rc = lib().ga_edit_distance(ctx, C.byref(bin_), int(bool(semiglobal)), out.ctypes.data)
        if rc != 0:
            raise RuntimeError(f"ga_edit_distance failed ({rc}): {lib().ga_last_error(ctx).decode()}")
    return out


def global_distances(pairs: list[tuple[str, str]], device: int | None = None) -> list[int]:
    """[oracle.global_distance(p, t) for p, t in pairs] (oracle.py:68-72)."""
    return edit_distances(_symbol_batch(pairs), False, device).tolist()


def semiglobal_distances(pairs: list[tuple[str, str]], device: int | None = None) -> list[int]:
    """[oracle.semiglobal_distance(p, t) ...] (oracle.py:59-65); raises
    ValueError for an empty pattern like the reference."""
    if any(not p for p, _ in pairs):
        raise ValueError("pattern must not be empty")
    return edit_distances(_symbol_batch(pairs), True, device).tolist()
