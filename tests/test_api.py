"""Host-side API (CPU only): the drop-in names, validation, packing and the
C-ABI library's exports.  No compute call needs a GPU here."""

from __future__ import annotations

import ctypes as C
import os
import random
import re

import numpy as np
import pytest

import paper_2203_15561_b200 as ga
from paper_2203_15561_b200 import _abi, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_names_exported():
    for name in ("align", "align_batch", "WindowConfig", "AlignmentResult", "BatchOutcome",
                 "WindowFailed", "EmptyPattern", "AccessCounters"):
        assert hasattr(ga, name)


def test_config_defaults_and_validation():
    cfg = ga.WindowConfig()
    assert (cfg.window, cfg.overlap, cfg.k, cfg.mode, cfg.priority) == (64, 24, 64, "improved",
                                                                         "MSID")
    assert ga.WindowConfig(window=32).k == 32
    for kwargs in (dict(window=8, overlap=8), dict(window=8, overlap=-1), dict(window=8, k=9),
                   dict(window=8, k=0), dict(mode="turbo"), dict(priority="MMSS"),
                   dict(window=0)):
        with pytest.raises(ValueError):
            ga.WindowConfig(**kwargs)


@pytest.mark.reference
def test_validation_messages_match_reference(reference):
    from bitalign.window import WindowConfig as RefConfig
    for kwargs in (dict(window=8, overlap=8), dict(window=8, overlap=-1), dict(window=8, k=9),
                   dict(window=8, k=0), dict(mode="turbo"), dict(priority="MMSS"),
                   dict(window=0)):
        with pytest.raises(ValueError) as a:
            RefConfig(**kwargs)
        with pytest.raises(ValueError) as b:
            ga.WindowConfig(**kwargs)
        assert str(a.value) == str(b.value)


def test_errors_before_any_device_work():
    with pytest.raises(ga.EmptyPattern, match="pattern must not be empty"):
        ga.align("", "ACGT")
    with pytest.raises(ValueError, match="kernel maximum"):
        ga.align_batch([("ACGT", "ACGT")], ga.WindowConfig(window=129))
    e = ga.WindowFailed(3, 16)
    assert str(e) == "window 3 found no alignment within k=16"
    assert (e.window_index, e.k) == (3, 16)


def test_encode_symbols():
    assert _abi.encode("ACGTacgtNX").tolist() == [0, 1, 2, 3, 4, 4, 4, 4, 4, 4]
    assert _abi.encode("AÇG").tolist() == [0, 4, 2]


def test_packing_roundtrip():
    pairs = [("ACGT", "AC"), ("", "T"), ("GG", ""), ("AÇG", "ng")]
    b = _abi.PackedBatch.from_pairs(pairs)
    assert b.n_pairs == 4
    assert b.pat_len.tolist() == [4, 0, 2, 3] and b.txt_len.tolist() == [2, 1, 0, 2]
    for q, (p, t) in enumerate(pairs):
        assert b.codes[b.pat_off[q]:b.pat_off[q] + len(p)].tolist() == _abi.encode(p).tolist()
        assert b.codes[b.txt_off[q]:b.txt_off[q] + len(t)].tolist() == _abi.encode(t).tolist()


@pytest.mark.parametrize("in_place", [True, False])
def test_pack_pairs_matches_from_pairs(monkeypatch, in_place):
    # align_batch's native packer: in place from the str objects (CPython's
    # compact ASCII layout) or from one joined copy; non-ASCII takes the
    # exact Python path.  Same codes and offsets as PackedBatch.from_pairs.
    if not in_place:
        monkeypatch.setattr(engine, "_STR_OFF", None)
    else:
        assert engine._STR_OFF is not None  # the layout probe holds on this interpreter
    rng = random.Random(5)
    cases = [[], [("", "")], [("ACGT", "AC"), ("", "T"), ("GG", "")], [("AÇG", "ng"), ("ACGT", "A")]]
    for _ in range(40):
        cases.append([("".join(rng.choice("ACGTNacgtx") for _ in range(rng.randrange(0, 2000))),
                       "".join(rng.choice("ACGT") for _ in range(rng.randrange(0, 40))))
                      for _ in range(rng.randrange(1, 25))])
    big = "".join(rng.choice("ACGTN") for _ in range(5000))
    cases.append([(big[i % 97:], big[:4000 + i]) for i in range(400)])  # > 1 MB: threaded ranges
    for pairs in cases:
        a, b = engine.pack_pairs(pairs), _abi.PackedBatch.from_pairs(pairs)
        for f in ("codes", "pat_off", "pat_len", "txt_off", "txt_len"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_num_windows_formula():
    # 4 windows for 150 bp, 6 for 250 bp, 250 for 10 kb
    assert [_abi.num_windows(x, 64, 24) for x in (0, 1, 64, 65, 150, 250, 10_000)] == \
        [0, 1, 1, 2, 4, 6, 250]


def test_outcomes_from_packed_shapes():
    b = _abi.PackedBatch.from_pairs([("ACGT", "ACGT"), ("AAAA", "TTTT"), ("", "A")])
    out = _abi.PackedResults.allocate(b, 64, 24)
    out.results[0] = (0, -1, 0, 4, 1, 4, 3, 4, 4)
    out.ops[out.ops_off[0]:out.ops_off[0] + 4] = np.frombuffer(b"====", np.uint8)
    out.dists[out.win_off[0]] = 0
    out.results[1] = (1, 0, 0, 0, 0, 0, 0, 0, 0)
    out.results[2] = (2, -1, 0, 0, 0, 0, 0, 0, 0)
    outs = ga.window.outcomes_from_packed(b, out, ga.WindowConfig(window=64, k=2))
    assert outs[0].ok and outs[0].result.cigar == "====" and outs[0].result.window_distances == (0,)
    assert outs[1].error == "WindowFailed: window 0 found no alignment within k=2"
    assert outs[2].error == "EmptyPattern: pattern must not be empty"


def test_outcomes_native_builder_matches_python_loop(monkeypatch):
    # csrc/outcomes_py.cpp builds the same objects as the Python loop:
    # equal outcomes, the dataclass's field order in every result's __dict__
    from paper_2203_15561_b200 import window
    if window._outcomes is None:
        pytest.skip("_outcomes not built (build.py builds it)")
    rng = np.random.default_rng(1)
    prng = random.Random(2)
    pairs = [("".join(prng.choice("ACGT") for _ in range(prng.randrange(0, 900))),
              "ACGT" * prng.randrange(0, 50)) for _ in range(300)]
    b = _abi.PackedBatch.from_pairs(pairs)
    out = _abi.PackedResults.allocate(b, 64, 24)
    n, res = b.n_pairs, out.results
    res["status"] = rng.choice([0, 0, 0, 1, 2], n)
    for f in ("cost", "text_consumed", "rows_computed", "entry_reads", "entry_writes",
              "words_allocated"):
        res[f] = rng.integers(0, 10**9, n)
    res["fail_window"] = rng.integers(0, 5, n)
    cap = np.diff(np.append(out.ops_off, out.ops.shape[0]))
    res["ops_len"] = [rng.integers(0, c + 1) for c in cap]
    out.ops[:] = rng.choice(np.frombuffer(b"=XID", np.uint8), out.ops.shape[0])
    out.dists[:] = rng.integers(0, 64, out.dists.shape[0])
    cfg = ga.WindowConfig(window=64, overlap=24, k=64)
    native = window.outcomes_from_packed(b, out, cfg)
    monkeypatch.setattr(window, "_outcomes", None)
    loop = window.outcomes_from_packed(b, out, cfg)
    assert native == loop and sum(x.ok for x in native) > 100
    for x, y in zip(native, loop):
        if x.ok:
            assert list(vars(x.result)) == list(vars(y.result))
            assert vars(x.result.counters) == vars(y.result.counters)


def test_lpt_split_balances_and_partitions():
    rng = np.random.default_rng(0)
    lens = rng.integers(100, 50_000, size=1000).astype(np.int32)
    shards = engine.split_lpt(lens, 64, 24, 8)
    allidx = np.sort(np.concatenate(shards))
    assert np.array_equal(allidx, np.arange(1000))
    loads = [int(_abi.num_windows(lens[s], 64, 24).sum()) for s in shards]
    assert max(loads) - min(loads) <= int(_abi.num_windows(lens, 64, 24).max())


# ---------------------------------------------------------------------------
# C-ABI library: loads without a GPU and exports every symbol include/genasm.h declares


def _header_functions():
    inc = os.path.join(ROOT, "include")
    text = "".join(open(os.path.join(inc, h)).read()
                   for h in sorted(os.listdir(inc)) if h.endswith(".h"))
    return sorted(set(re.findall(r"\b(ga_[a-z0-9_]+)\s*\(", text)))


def test_capi_exports_every_declared_symbol():
    L = engine.lib()
    names = _header_functions()
    assert len(names) >= 19
    for name in names:
        assert hasattr(L, name), name


def test_capi_host_functions():
    L = engine.lib()
    assert L.ga_version().decode().startswith("genasm-b200")
    for n, w, o in ((0, 64, 24), (150, 64, 24), (10_000, 64, 24), (333, 32, 12), (64, 64, 0)):
        assert L.ga_num_windows(n, w, o) == _abi.num_windows(n, w, o)
    msg = C.create_string_buffer(160)
    assert L.ga_check_config(C.byref(_abi.make_config(64, 24, 64, "MSID")), msg, 160) == 0
    assert L.ga_check_config(C.byref(_abi.make_config(8, 8, 8, "MSID")), msg, 160) == 1
    assert msg.value.decode() == "overlap must be in [0, window), got 8 for window 8"
    assert L.ga_check_config(C.byref(_abi.make_config(8, 2, 9, "MSID")), msg, 160) == 1
    assert msg.value.decode() == "k must be in [1, 8], got 9"
    assert L.ga_check_config(C.byref(_abi.make_config(256, 2, 9, "MSID")), msg, 160) == 1
    out = np.zeros(6, np.uint8)
    L.ga_encode_ascii(b"ACGTNa", 6, out.ctypes.data)
    assert out.tolist() == [0, 1, 2, 3, 4, 4]
    lens = np.array([5, 9, 1, 9], np.int32)
    assert engine.lpt_order(lens).tolist() == [1, 3, 0, 2]


def test_transfer_formats_host_side():
    """ga_pack2 (2-bit input + exception list) and the ops2 decoders."""
    rng = np.random.default_rng(3)
    for n in (0, 1, 3, 4, 5, 31, 32, 33, 1023, 100_003, 2_000_003, 3_000_064):
        codes = rng.integers(0, 4, n).astype(np.uint8)
        codes[rng.random(n) < 0.01] = 4
        codes[n // 3:n // 3 + 70] = 4  # whole 32-symbol blocks of code 4 (vector path)
        p = engine.pack2(codes)
        assert p.data.shape[0] == max(1, (n + 3) // 4)
        unpacked = ((p.data[:, None] >> np.array([0, 2, 4, 6], np.uint8)) & 3).reshape(-1)[:n]
        assert np.array_equal(unpacked, codes & 3)
        assert np.array_equal(p.exceptions, np.nonzero(codes == 4)[0])
    # 2-bit ops -> ASCII, both the C decoder and PackedResults.cigar
    ops = rng.integers(0, 4, 37).astype(np.uint8)
    ops2 = np.zeros(10, np.uint8)
    for x, v in enumerate(ops):
        ops2[x // 4] |= v << (2 * (x % 4))
    out = C.create_string_buffer(37 - 5)
    engine.lib().ga_unpack_ops(ops2.ctypes.data, 5, 37 - 5, out)
    expect = bytes(b"=XID"[v] for v in ops)
    assert out.raw == expect[5:]
    batch = _abi.PackedBatch.from_pairs([("ACGTACGTAC", "ACGTACGTACGTACGTACGTACGTACGT")])
    res = _abi.PackedResults.allocate(batch, 64, 24, ops2=True)
    assert res.n_ops == 40 and res.ops.shape[0] == 10
    res.ops[:] = ops2
    res.results["ops_len"][0] = 37
    assert res.cigar(0) == expect.decode()


def test_no_cpu_fallback_when_extension_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(engine, "SO_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(engine, "_lib", None)
    with pytest.raises(engine.ExtensionMissing):
        engine.lib()
