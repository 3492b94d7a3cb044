"""Device engine: loads the in-tree sm_100a library and runs packed batches.

There is no CPU fallback.  If ``_genasm.so`` is missing or no CUDA device is
visible, every call raises -- the product path never routes around the
kernel.  One ``ga_ctx`` (stream + device buffers) is kept per device; a
multi-device batch is split longest-first across devices and each device is
driven from its own host thread (ctypes releases the GIL during the call).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _abi
from ._abi import PackedBatch, PackedResults

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("GA_SO") or os.path.join(_HERE, "_genasm.so")

_lib = None
_lib_lock = threading.Lock()
_ctxs: dict[int, C.c_void_p] = {}
_ctx_locks: dict[int, threading.Lock] = {}


class ExtensionMissing(RuntimeError):
    """The CUDA extension is not built; there is deliberately no fallback."""


def lib():
    """Load _genasm.so (declaring every C-ABI signature); raise if absent."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SO_PATH):
            raise ExtensionMissing(
                f"{SO_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the GPU path has no CPU fallback)")
        L = C.CDLL(SO_PATH)
        B = C.POINTER(_abi.GaBatchIn)
        O = C.POINTER(_abi.GaBatchOut)
        F = C.POINTER(_abi.GaConfig)
        sigs = {
            "ga_version": ([], C.c_char_p),
            "ga_num_windows": ([C.c_int64, C.c_int32, C.c_int32], C.c_int64),
            "ga_check_config": ([F, C.c_char_p, C.c_int], C.c_int),
            "ga_encode_ascii": ([C.c_char_p, C.c_int64, C.c_void_p], None),
            "ga_encode_ascii_mt": ([C.c_char_p, C.c_int64, C.c_void_p, C.c_int32], None),
            "ga_encode_ascii_gather": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32],
                                       None),
            "ga_create": ([C.c_int, C.POINTER(C.c_void_p)], C.c_int),
            "ga_destroy": ([C.c_void_p], None),
            "ga_last_error": ([C.c_void_p], C.c_char_p),
            "ga_align_batch": ([C.c_void_p, B, F, O], C.c_int),
            "ga_align_batch_device": ([C.c_void_p, B, F, O, C.c_void_p], C.c_int),
            "ga_last_launch_count": ([C.c_void_p], C.c_int64),
            "ga_lpt_order": ([C.c_int64, C.c_void_p, C.c_void_p], None),
            "ga_pack2": ([C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64], C.c_int64),
            "ga_unpack_ops": ([C.c_void_p, C.c_int64, C.c_int64, C.c_void_p], None),
            "ga_host_alloc": ([C.c_int64], C.c_void_p),
            "ga_host_free": ([C.c_void_p], None),
            "ga_parse_pairs_tsv": ([C.c_char_p, C.c_int64, C.c_int, C.c_int32,
                                    C.POINTER(C.POINTER(_abi.GaPairs)), C.c_char_p, C.c_int64],
                                   C.c_int),
            "ga_pairs_free": ([C.POINTER(_abi.GaPairs)], None),
            "ga_edit_distance": ([C.c_void_p, B, C.c_int32, C.c_void_p], C.c_int),
            "ga_format_align_rows": ([C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int,
                                      C.c_void_p, C.c_int64], C.c_int64),
        }
        for name, (args, res) in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def context(device: int = 0) -> C.c_void_p:
    """The per-device ga_ctx (created on first use)."""
    L = lib()
    with _lib_lock:
        ctx = _ctxs.get(device)
        if ctx is None:
            ctx = C.c_void_p()
            rc = L.ga_create(int(device), C.byref(ctx))
            if rc != 0:
                raise RuntimeError(
                    f"ga_create(device={device}) failed with CUDA error {rc}: no usable CUDA "
                    "device (the GPU path has no CPU fallback)")
            _ctxs[device] = ctx
            _ctx_locks[device] = threading.Lock()
        return ctx


def _default_device() -> int:
    env = os.environ.get("LOCAL_RANK")
    return int(env) if env is not None and env.isdigit() else 0


def lpt_order(pat_len: np.ndarray) -> np.ndarray:
    """Longest-first order (host length bucketing)."""
    order = np.empty(pat_len.shape[0], dtype=np.int32)
    lib().ga_lpt_order(int(pat_len.shape[0]), np.ascontiguousarray(pat_len, np.int32).ctypes.data,
                       order.ctypes.data)
    return order


def pack2(codes: np.ndarray) -> _abi.Packed2:
    """2-bit transfer form of a code array (ga_pack2, multithreaded)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n = int(codes.shape[0])
    data = np.zeros(max(1, (n + 3) // 4), dtype=np.uint8)
    L = lib()
    exc = np.empty(1024, dtype=np.int64)
    n_exc = L.ga_pack2(codes.ctypes.data, n, data.ctypes.data, exc.ctypes.data, exc.shape[0])
    if n_exc > exc.shape[0]:
        exc = np.empty(n_exc, dtype=np.int64)
        L.ga_pack2(codes.ctypes.data, n, data.ctypes.data, exc.ctypes.data, n_exc)
    exc = exc[:n_exc].copy()
    return _abi.Packed2(data=data, exceptions=exc)


def run_packed(batch: PackedBatch, window: int, overlap: int, k: int, priority: str,
               device: int | None = None, *, packed2: bool = False,
               ops2: bool = False, mode: str = "improved",
               host_pack: bool = False) -> PackedResults:
    """One ga_align_batch call on one device (host buffers in and out).
    packed2 / ops2 select the 2-bit transfer formats of include/genasm.h
    (packed2: packed here first, GA_PACK_CALLER); host_pack: the call packs
    each pipeline chunk itself (GA_PACK_HOST); mode="baseline" runs the
    unimproved engine (dense edge tables)."""
    dev = _default_device() if device is None else int(device)
    ctx = context(dev)
    out = PackedResults.allocate(batch, window, overlap, ops2=ops2)
    if batch.n_pairs == 0:
        return out
    cfg = _abi.make_config(window, overlap, k, priority, mode)
    packed = pack2(batch.codes) if packed2 else None  # must outlive the call
    bin_ = batch.struct(packed=packed)
    if host_pack and not packed2:
        bin_.packed2 = _abi.GA_PACK_HOST
    bout = out.struct()
    with _ctx_locks[dev]:
        rc = lib().ga_align_batch(ctx, C.byref(bin_), C.byref(cfg), C.byref(bout))
        if rc != 0:
            raise RuntimeError(f"ga_align_batch failed ({rc}): "
                               f"{lib().ga_last_error(ctx).decode(errors='replace')}")
    return out


def _str_data_offset() -> int | None:
    """Byte offset of a compact ASCII ``str``'s characters from its address
    (CPython lays them out right after the PyASCIIObject header,
    ``sys.getsizeof("") - 1`` bytes), checked on a probe string; None if the
    running interpreter does not lay strings out that way."""
    import sys
    off = sys.getsizeof("") - 1
    probe = "ACGTNacgt" * 7
    try:
        if C.string_at(id(probe) + off, len(probe)) == probe.encode("ascii"):
            return off
    except Exception:  # noqa: BLE001 -- any failure means: do not use it
        pass
    return None


_STR_OFF = _str_data_offset()


def pack_pairs(pairs) -> PackedBatch:
    """``PackedBatch.from_pairs`` for the drop-in ``align_batch``: the pair
    strings encoded by the native multithreaded encoder instead of a numpy
    table lookup -- read in place from the ``str`` objects
    (ga_encode_ascii_gather; CPython's compact ASCII layout, verified at
    import) or, elsewhere, joined once (ga_encode_ascii_mt).  Non-ASCII input
    (Unicode code units, never a match) takes the exact Python path."""
    import itertools
    n = len(pairs)
    lens = np.fromiter(map(len, itertools.chain.from_iterable(pairs)), dtype=np.int64,
                       count=2 * n)
    if _STR_OFF is not None and all(type(a) is str and type(b) is str and a.isascii() and b.isascii()
                                   for a, b in pairs):
        ptrs = np.fromiter((id(x) + _STR_OFF for x in itertools.chain.from_iterable(pairs)),
                           dtype=np.uint64, count=2 * n)
        total = int(lens.sum())
        codes = np.empty(max(1, total), dtype=np.uint8)
        lib().ga_encode_ascii_gather(ptrs.ctypes.data, lens.ctypes.data, 2 * n,
                                     codes.ctypes.data, 0)
        starts = np.zeros(2 * n, dtype=np.int64)
        if n:
            np.cumsum(lens[:-1], out=starts[1:])
        return PackedBatch(codes=codes[:total], pat_off=starts[0::2].copy(),
                           pat_len=lens[0::2].astype(np.int32), txt_off=starts[1::2].copy(),
                           txt_len=lens[1::2].astype(np.int32))
    blob = "".join(itertools.chain.from_iterable(pairs))
    if not blob.isascii():
        return PackedBatch.from_pairs(pairs)
    raw = blob.encode("ascii")
    codes = np.empty(max(1, len(raw)), dtype=np.uint8)
    lib().ga_encode_ascii_mt(raw, len(raw), codes.ctypes.data, 0)
    starts = np.zeros(2 * n, dtype=np.int64)
    if n:
        np.cumsum(lens[:-1], out=starts[1:])
    return PackedBatch(codes=codes[:len(raw)] if len(raw) else codes[:0],
                       pat_off=starts[0::2].copy(), pat_len=lens[0::2].astype(np.int32),
                       txt_off=starts[1::2].copy(), txt_len=lens[1::2].astype(np.int32))


def split_lpt(pat_len: np.ndarray, window: int, overlap: int, n_shards: int) -> list[np.ndarray]:
    """Greedy LPT partition of pair indices by window count (the exact cost
    proxy: #windows follows from |P| alone)."""
    cost = _abi.num_windows(pat_len, window, overlap).astype(np.int64)
    order = np.argsort(-cost, kind="stable")
    loads = np.zeros(n_shards, dtype=np.int64)
    owner = np.empty(pat_len.shape[0], dtype=np.int64)
    for idx in order:
        s = int(np.argmin(loads))
        owner[idx] = s
        loads[s] += max(1, int(cost[idx]))
    return [np.nonzero(owner == s)[0] for s in range(n_shards)]


def _subset(batch: PackedBatch, idx: np.ndarray) -> PackedBatch:
    return PackedBatch(codes=batch.codes, pat_off=batch.pat_off[idx], pat_len=batch.pat_len[idx],
                       txt_off=batch.txt_off[idx], txt_len=batch.txt_len[idx])


def _scatter(full: PackedResults, part: PackedResults, idx: np.ndarray, batch: PackedBatch,
             window: int, overlap: int) -> None:
    """Copy one shard's records, ops and window distances to their input
    positions in `full` (the reference returns slots in input order,
    window.py:152-163)."""
    full.results[idx] = part.results
    n_win = _abi.num_windows(batch.pat_len[idx], window, overlap)
    for local, q in enumerate(idx.tolist()):
        n_ops = int(part.results["ops_len"][local])
        src = int(part.ops_off[local])
        dst = int(full.ops_off[q])
        if part.ops2:  # both layouts start every pair on a byte boundary
            nb = (n_ops + 3) // 4
            full.ops[dst // 4:dst // 4 + nb] = part.ops[src // 4:src // 4 + nb]
        else:
            full.ops[dst:dst + n_ops] = part.ops[src:src + n_ops]
        # the pair's own window count (App. A.4), not the distance to the next
        # offset: allocate() pads an all-empty shard's distance array to 1
        w_src = int(part.win_off[local])
        w_dst = int(full.win_off[q])
        w_n = int(n_win[local])
        full.dists[w_dst:w_dst + w_n] = part.dists[w_src:w_src + w_n]


def run_batch(batch: PackedBatch, cfg, devices=None) -> PackedResults:
    """align_batch on one or more devices; results always in input order."""
    if devices is None or (isinstance(devices, int) and devices <= 1):
        dev = None if devices is None else 0
        return run_packed(batch, cfg.window, cfg.overlap, cfg.k, cfg.priority, dev,
                          mode=cfg.mode)
    dev_list = list(range(devices)) if isinstance(devices, int) else [int(d) for d in devices]
    if len(dev_list) == 1:
        return run_packed(batch, cfg.window, cfg.overlap, cfg.k, cfg.priority, dev_list[0],
                          mode=cfg.mode)
    shards = split_lpt(batch.pat_len, cfg.window, cfg.overlap, len(dev_list))
    parts: list[PackedResults | None] = [None] * len(dev_list)
    errors: list[BaseException] = []

    def work(s: int) -> None:
        try:
            parts[s] = run_packed(_subset(batch, shards[s]), cfg.window, cfg.overlap, cfg.k,
                                  cfg.priority, dev_list[s], mode=cfg.mode)
        except BaseException as exc:  # re-raised on the caller's thread
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(s,)) for s in range(len(dev_list))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    full = PackedResults.allocate(batch, cfg.window, cfg.overlap)
    for s, idx in enumerate(shards):
        if len(idx):
            _scatter(full, parts[s], idx, batch, cfg.window, cfg.overlap)
    return full
