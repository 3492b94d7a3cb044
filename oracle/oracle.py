"""TEST INFRASTRUCTURE ONLY: ctypes front-end of the C oracle (genasm_oracle.c).

The oracle is the CPU restatement of the reference's windowed improved-GenASM
path used as the parity checker (tests/, __graft_entry__.smoke()) and as the
CPU baseline (bench.py cpu_baseline, bench.py --impl reference).  The product
package never imports this module.

It reuses the product's ABI structs and packing (paper_2203_15561_b200._abi),
so the oracle and the kernel consume byte-identical inputs and fill
byte-identical output records; only the engine differs.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

from paper_2203_15561_b200 import _abi
from paper_2203_15561_b200._abi import PackedBatch, PackedResults

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = C.CDLL(_SO)
        _lib.oracle_align_batch.argtypes = [C.POINTER(_abi.GaBatchIn), C.POINTER(_abi.GaConfig),
                                            C.POINTER(_abi.GaBatchOut), C.c_int]
        _lib.oracle_align_batch.restype = C.c_int
    return _lib


def align_packed(batch: PackedBatch, window: int, overlap: int, k: int,
                 priority: str = "MSID", threads: int = 1, mode: str = "improved") -> PackedResults:
    out = PackedResults.allocate(batch, window, overlap)
    cfg = _abi.make_config(window, overlap, k, priority, mode)
    bin_ = batch.struct()
    bout = out.struct()
    rc = lib().oracle_align_batch(C.byref(bin_), C.byref(cfg), C.byref(bout), int(threads))
    if rc != 0:
        raise RuntimeError(f"oracle_align_batch failed: {rc}")
    return out


def align_batch(pairs, cfg, threads: int = 1):
    """Reference-shaped outcomes (list of BatchOutcome) computed by the oracle."""
    from paper_2203_15561_b200.window import outcomes_from_packed
    batch = PackedBatch.from_pairs(pairs)
    out = align_packed(batch, cfg.window, cfg.overlap, cfg.k, cfg.priority, threads, cfg.mode)
    return outcomes_from_packed(batch, out, cfg)
