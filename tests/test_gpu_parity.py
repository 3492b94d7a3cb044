"""GPU parity: the sm_100a kernel (through the C-ABI) vs the reference's outputs.

Three anchors, strongest first:
  * golden fixtures produced by the reference itself (tests/golden/, made by
    make_golden.py): known-answer vectors, a randomized corpus, and per-pair
    digests of the BASELINE configs' recipe pairs;
  * the C oracle (oracle/, pinned to the same fixtures by test_oracle.py) on
    larger sets the reference is too slow to pre-compute, up to the full
    138,929-pair config 3;
  * size-independent properties at full size (replay validity, cost and span
    consistency, batch-composition invariance).
Equality is exact on every field: cigar, cost, text_consumed,
window_distances, rows_computed, the three access counters, error strings.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import corpus

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


@pytest.fixture(scope="module")
def gpu():
    import paper_2203_15561_b200 as ga
    from paper_2203_15561_b200 import engine
    engine.context(0)  # raises (no fallback) if the extension or device is missing
    return ga


def _cfg(ga, w, o, k, prio="MSID"):
    return ga.WindowConfig(window=w, overlap=o, k=k, priority=prio)


def _gpu_outcomes(ga, batch, cfg):
    from paper_2203_15561_b200.engine import run_batch
    from paper_2203_15561_b200.window import outcomes_from_packed
    return outcomes_from_packed(batch, run_batch(batch, cfg), cfg)


def test_extension_is_native(gpu):
    from paper_2203_15561_b200 import engine
    assert engine.lib().ga_version().decode().startswith("genasm-b200")


def test_known_vectors(gpu):
    with open(os.path.join(GOLD, "known.json")) as f:
        known = json.load(f)
    for case in known:
        cfg = _cfg(gpu, case["window"], case["overlap"], case["k"], case["priority"])
        got = gpu.align_batch([(case["pattern"], case["text"])], cfg)[0]
        assert corpus.outcome_key(got) == case["key"], case


def test_align_errors_and_types(gpu):
    with pytest.raises(gpu.EmptyPattern):
        gpu.align("", "ACGT")
    with pytest.raises(gpu.WindowFailed) as info:
        gpu.align("AAAAAAAA", "TTTTTTTT", gpu.WindowConfig(window=8, overlap=2, k=2))
    assert info.value.window_index == 0 and info.value.k == 2
    r = gpu.align("ACGTACGT", "ACGTACGT", gpu.WindowConfig(window=4, overlap=2, k=4))
    assert r.cigar == "========" and r.window_distances == (0, 0, 0)
    with pytest.raises(AttributeError):
        r.cost = 7
    assert gpu.align_batch([], gpu.WindowConfig()) == []
    rb = gpu.align("ACGT", "AGGT", gpu.WindowConfig(mode="baseline"))  # the unimproved engine
    assert (rb.cigar, rb.cost, rb.rows_computed) == ("=X==", 1, 65)


def test_fuzz_vs_reference_golden(gpu):
    with open(os.path.join(GOLD, "fuzz.json")) as f:
        gold = json.load(f)
    for (case, ((w, o, k, prio), pairs)) in zip(gold["cases"],
                                               corpus.fuzz_cases(gold["seed"], gold["batches"])):
        assert case["cfg"] == [w, o, k, prio]
        outs = gpu.align_batch(pairs, _cfg(gpu, w, o, k, prio))
        got = [str(corpus.digest(x)) for x in outs]
        bad = [q for q, (a, b) in enumerate(zip(got, case["digests"])) if a != b]
        assert not bad, (case["cfg"], [pairs[q] for q in bad[:2]])


def test_fuzz_vs_oracle(gpu, oracle_mod):
    for (w, o, k, prio), pairs in corpus.fuzz_cases(777, 150, pairs_per_batch=16, max_len=700):
        cfg = _cfg(gpu, w, o, k, prio)
        got = [corpus.outcome_key(x) for x in gpu.align_batch(pairs, cfg)]
        exp = [corpus.outcome_key(x) for x in oracle_mod.align_batch(pairs, cfg, threads=4)]
        bad = [q for q in range(len(pairs)) if got[q] != exp[q]]
        assert not bad, ((w, o, k, prio), pairs[bad[0]], got[bad[0]], exp[bad[0]])


def _config_digest_check(gpu, cfg_id, key, w=64, o=24, k=64, count=None):
    from paper_2203_15561_b200 import sim
    gold = np.load(os.path.join(GOLD, "configs.npz"))[key]
    n = len(gold) if count is None else count
    batch, _ = sim.config_pairs(cfg_id, count=n)
    outs = _gpu_outcomes(gpu, batch, _cfg(gpu, w, o, k))
    got = np.array([corpus.digest(x) for x in outs], dtype=np.uint64)
    bad = np.nonzero(got != gold[:n])[0]
    assert bad.size == 0, f"{key}: {bad.size} mismatching pairs, first {bad[:5].tolist()}"


def test_config1_all_pairs_vs_reference(gpu):
    _config_digest_check(gpu, 1, "cfg1")


def test_config2_all_pairs_vs_reference(gpu):
    _config_digest_check(gpu, 2, "cfg2")


def test_config3_prefix_vs_reference(gpu):
    _config_digest_check(gpu, 3, "cfg3")


def test_config4_prefix_vs_reference(gpu):
    _config_digest_check(gpu, 4, "cfg4")


@pytest.mark.parametrize("w,o,k", [(w, 3 * w // 8, k) for w in (32, 64, 128)
                                   for k in (w // 4, w // 2, w)])
def test_config5_sweep_vs_reference(gpu, w, o, k):
    _config_digest_check(gpu, 5, f"cfg5_w{w}_k{k}", w=w, o=o, k=k)


def _packed_equal(a, b, tag=""):
    if not np.array_equal(a.results, b.results):
        bad = np.nonzero(a.results != b.results)[0]
        raise AssertionError(f"{tag}: {bad.size} result records differ; first {bad[:4].tolist()}: "
                             f"gpu={a.results[bad[0]]} oracle={b.results[bad[0]]}")
    for q in range(a.results.shape[0]):
        n = int(a.results["ops_len"][q])
        oa, ob = int(a.ops_off[q]), int(b.ops_off[q])
        assert np.array_equal(a.ops[oa:oa + n], b.ops[ob:ob + n]), q
    assert np.array_equal(a.dists, b.dists)


def test_config3_vs_oracle_4096(gpu, oracle_mod):
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    batch, _ = sim.config_pairs(3, count=4096)
    got = run_packed(batch, 64, 24, 64, "MSID")
    exp = oracle_mod.align_packed(batch, 64, 24, 64, "MSID", threads=os.cpu_count())
    _packed_equal(got, exp)


def test_config5_vs_oracle_all_pairs(gpu, oracle_mod):
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    batch, _ = sim.config_pairs(5)
    for (w, o, k) in [(64, 24, 16), (128, 48, 128), (32, 12, 8)]:
        got = run_packed(batch, w, o, k, "MSID")
        exp = oracle_mod.align_packed(batch, w, o, k, "MSID", threads=os.cpu_count())
        _packed_equal(got, exp, (w, o, k))


def test_batch_composition_invariance(gpu):
    """Results of a pair do not depend on its batch (sharding correctness)."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed, split_lpt, _subset
    batch, _ = sim.config_pairs(5, count=600)
    full = run_packed(batch, 64, 24, 64, "MSID")
    for idx in split_lpt(batch.pat_len, 64, 24, 3):
        part = run_packed(_subset(batch, idx), 64, 24, 64, "MSID")
        assert np.array_equal(part.results, full.results[idx])


def _with_exceptions(batch, rate=0.002, seed=5):
    """A copy of `batch` with some symbols replaced by code 4 (non-ACGT)."""
    from paper_2203_15561_b200._abi import PackedBatch
    rng = np.random.default_rng(seed)
    codes = batch.codes.copy()
    hit = rng.random(codes.shape[0]) < rate
    codes[hit] = 4
    return PackedBatch(codes=codes, pat_off=batch.pat_off, pat_len=batch.pat_len,
                       txt_off=batch.txt_off, txt_len=batch.txt_len)


@pytest.mark.parametrize("packed2,ops2", [(True, False), (False, True), (True, True)])
def test_transfer_formats(gpu, oracle_mod, packed2, ops2):
    """2-bit input (with code-4 exceptions) and 2-bit ops give identical results."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    batch, _ = sim.config_pairs(5, count=2000)
    batch = _with_exceptions(batch)
    got = run_packed(batch, 64, 24, 64, "MSID", packed2=packed2, ops2=ops2)
    exp = oracle_mod.align_packed(batch, 64, 24, 64, "MSID", threads=os.cpu_count())
    assert np.array_equal(got.results, exp.results)
    assert np.array_equal(got.dists, exp.dists)
    for q in range(batch.n_pairs):
        n = int(exp.results["ops_len"][q])
        o = int(exp.ops_off[q])
        assert got.cigar(q) == exp.ops[o:o + n].tobytes().decode(), q


@pytest.mark.parametrize("chunks", [1, 3, 8])
def test_host_pack(gpu, oracle_mod, monkeypatch, chunks):
    """GA_PACK_HOST: byte codes (with code-4 symbols) packed per chunk by the
    call itself give the oracle's results; bad packed2 values are refused."""
    import ctypes as C
    from paper_2203_15561_b200 import _abi, engine, sim
    from paper_2203_15561_b200.engine import run_packed
    batch, _ = sim.config_pairs(5, count=2000)
    batch = _with_exceptions(batch)
    monkeypatch.setenv("GA_CHUNKS", str(chunks))
    exp = oracle_mod.align_packed(batch, 64, 24, 64, "MSID", threads=os.cpu_count())
    for ops2 in (False, True):
        got = run_packed(batch, 64, 24, 64, "MSID", host_pack=True, ops2=ops2)
        assert np.array_equal(got.results, exp.results)
        assert np.array_equal(got.dists, exp.dists)
        for q in range(batch.n_pairs):
            n = int(exp.results["ops_len"][q])
            o = int(exp.ops_off[q])
            assert got.cigar(q) == exp.ops[o:o + n].tobytes().decode(), q
    out = _abi.PackedResults.allocate(batch, 64, 24)
    bin_, bout = batch.struct(), out.struct()
    bin_.packed2 = 3
    cfg = _abi.make_config(64, 24, 64, "MSID")
    L, ctx = engine.lib(), engine.context(0)
    assert L.ga_align_batch(ctx, C.byref(bin_), C.byref(cfg), C.byref(bout)) == -3
    assert b"packed2" in L.ga_last_error(ctx)


@pytest.mark.parametrize("chunks", [1, 2, 3, 7])
def test_chunked_pipeline(gpu, monkeypatch, chunks):
    """Chunked, stream-overlapped host path == one-shot path (ga_align_batch)."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    batch, _ = sim.config_pairs(5, count=1500)
    monkeypatch.setenv("GA_CHUNKS", "1")
    ref = run_packed(batch, 64, 24, 64, "MSID")
    monkeypatch.setenv("GA_CHUNKS", str(chunks))
    for packed2, ops2, hp in [(False, False, False), (True, True, False), (False, True, True)]:
        got = run_packed(batch, 64, 24, 64, "MSID", packed2=packed2, ops2=ops2, host_pack=hp)
        assert np.array_equal(got.results, ref.results)
        assert np.array_equal(got.dists, ref.dists)
        for q in range(0, batch.n_pairs, 7):
            assert got.cigar(q) == ref.cigar(q)


def _all_ops_equal(got, exp, tag="", chunk=4096):
    """Every op byte of every pair, compared in vectorised chunks of pairs;
    `got` may hold 2-bit ops (ops2: offsets rounded to 4, its own layout)."""
    n = exp.results.shape[0]
    ln_all = exp.results["ops_len"].astype(np.int64)
    assert np.array_equal(got.results["ops_len"], exp.results["ops_len"]), tag
    total = 0
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        ln = ln_all[a:b]
        m = int(ln.sum())
        if m == 0:
            continue
        # position k of pair q -> (offset + k), for every pair of the chunk
        rank = np.arange(m, dtype=np.int64) - np.repeat(np.cumsum(ln) - ln, ln)
        e_pos = np.repeat(exp.ops_off[a:b], ln) + rank
        g_pos = np.repeat(got.ops_off[a:b], ln) + rank
        e = exp.ops[e_pos]
        if got.ops2:
            g = np.frombuffer(b"=XID", dtype=np.uint8)[(got.ops[g_pos >> 2] >> ((g_pos & 3) * 2).astype(np.uint8)) & 3]
        else:
            g = got.ops[g_pos]
        bad = np.nonzero(g != e)[0]
        if bad.size:
            q = a + int(np.searchsorted(np.cumsum(ln), bad[0], side="right"))
            raise AssertionError(f"{tag}: {bad.size} op bytes differ in pairs {a}..{b}, first in pair {q}")
        total += m
    return total


def test_config3_full_vs_oracle(gpu, oracle_mod):
    """The bench workload itself: all 138,929 pairs of config 3, every field
    and EVERY CIGAR byte against the oracle (the reference's golden digests pin
    the prefix)."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    batch, _ = sim.config_pairs(3)
    got = run_packed(batch, 64, 24, 64, "MSID", packed2=True, ops2=True)
    exp = oracle_mod.align_packed(batch, 64, 24, 64, "MSID", threads=os.cpu_count())
    assert np.array_equal(got.results, exp.results)
    assert np.array_equal(got.dists, exp.dists)
    n_ops = _all_ops_equal(got, exp, "config3")
    assert n_ops == int(exp.results["ops_len"].sum()) > 1_300_000_000
    assert (got.results["status"] == 0).all()  # k = W: every window aligns


def test_config3_shard_on_lane_groups(gpu, oracle_mod, monkeypatch):
    """An 8-GPU shard of config 3 (17,367 pairs) forced onto the 16-lane group
    kernel (two waves of groups, hard windows, the lingering warps), every
    field and every op byte against the oracle."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    monkeypatch.setenv("GA_LANE_GROUPS", "1")
    batch, _ = sim.config_pairs(3, count=17_367)
    got = run_packed(batch, 64, 24, 64, "MSID")
    exp = oracle_mod.align_packed(batch, 64, 24, 64, "MSID", threads=os.cpu_count())
    assert np.array_equal(got.results, exp.results)
    assert np.array_equal(got.dists, exp.dists)
    assert _all_ops_equal(got, exp, "config3 shard, lane groups") > 100_000_000


def test_config4_full_vs_oracle(gpu, oracle_mod):
    """All 20,000 ultra-long config-4 pairs (~2,450-window chains, the
    reference's window loop pkg/src/bitalign/window.py:95-120), every field and
    every op byte against the oracle; the reference's own digests pin the
    first four (test_config4_prefix_vs_reference)."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    batch, _ = sim.config_pairs(4, threads=os.cpu_count())
    got = run_packed(batch, 64, 24, 64, "MSID", packed2=True)
    exp = oracle_mod.align_packed(batch, 64, 24, 64, "MSID", threads=os.cpu_count())
    assert np.array_equal(got.results, exp.results)
    assert np.array_equal(got.dists, exp.dists)
    _all_ops_equal(got, exp, "config4")
    assert (got.results["status"] == 0).all()


@pytest.mark.parametrize("w,o,k", [(w, 3 * w // 8, k) for w in (32, 64, 128)
                                   for k in (w // 4, w // 2, w)])
def test_config5_sweep_full_vs_oracle(gpu, oracle_mod, w, o, k):
    """Config 5 (8,192 mixed 100 bp - 50 kb pairs) at every W x k sweep point,
    every pair, every field and op byte against the oracle -- including the
    WindowFailed-heavy k = W/4 points."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    batch, _ = sim.config_pairs(5)
    got = run_packed(batch, w, o, k, "MSID")
    exp = oracle_mod.align_packed(batch, w, o, k, "MSID", threads=os.cpu_count())
    _packed_equal(got, exp, (w, o, k))
    _all_ops_equal(got, exp, (w, o, k))


def test_full_tier_beyond_level_63(gpu, oracle_mod):
    """Windows at d_min = m = 64 (runs of 'N' or lowercase longer than W: no
    symbol matches): the full tier's third pass holds level
    64 alone and must stay inside the warp's table region.  Every
    pair of the batch -- including the neighbours whose tables follow in
    memory -- against the oracle."""
    import random

    from paper_2203_15561_b200._abi import PackedBatch
    from paper_2203_15561_b200.engine import run_packed
    rng = random.Random(64)
    pairs = []
    for q in range(96):
        core = "".join(rng.choice("ACGT") for _ in range(rng.randrange(100, 900)))
        cut = rng.randrange(0, len(core))
        run = ("N" if q % 2 else "a") * rng.randrange(64, 260)
        pairs.append((core[:cut] + run + core[cut:], corpus.noisy_copy(rng, core, 0.05)))
    batch = PackedBatch.from_pairs(pairs)
    for prio in ("MSID", "IDSM"):
        got = run_packed(batch, 64, 24, 64, prio)
        exp = oracle_mod.align_packed(batch, 64, 24, 64, prio, threads=os.cpu_count())
        _packed_equal(got, exp, ("deep", prio))


@pytest.mark.parametrize("kernel", ["thread", "lanegroups", "lockstep"])
def test_both_kernels_vs_oracle(gpu, oracle_mod, monkeypatch, kernel):
    """Each kernel on its own, whatever the batch size would pick: the
    lane-per-pair kernel with its band / full tiers and hand-over
    (GA_LANE_GROUPS=0), the 16-lane group kernel (GA_LANE_GROUPS=1) and the
    lockstep kernel (GA_KERNEL=lockstep)."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    if kernel == "lockstep":
        monkeypatch.setenv("GA_KERNEL", "lockstep")
    else:
        monkeypatch.setenv("GA_LANE_GROUPS", "1" if kernel == "lanegroups" else "0")
    batch, _ = sim.config_pairs(5)
    for (w, o, k, prio) in [(64, 24, 64, "MSID"), (64, 24, 16, "DISM"), (32, 12, 32, "SMDI"),
                            (48, 18, 30, "IDSM")]:
        got = run_packed(batch, w, o, k, prio)
        exp = oracle_mod.align_packed(batch, w, o, k, prio, threads=os.cpu_count())
        _packed_equal(got, exp, (kernel, w, o, k, prio))
    for (w, o, k, prio), pairs in corpus.fuzz_cases(99, 60, pairs_per_batch=16, max_len=500):
        cfg = _cfg(gpu, w, o, k, prio)
        got = [corpus.outcome_key(x) for x in gpu.align_batch(pairs, cfg)]
        exp = [corpus.outcome_key(x) for x in oracle_mod.align_batch(pairs, cfg, threads=4)]
        assert got == exp, (kernel, (w, o, k, prio))


def test_unrelated_pairs_full_tier(gpu, oracle_mod):
    """Pairs whose windows all exceed the band tier (unrelated sequences, d_min
    often above 31): the lane-per-pair kernel's cooperative full tier with
    several 32-level passes."""
    from paper_2203_15561_b200._abi import PackedBatch
    from paper_2203_15561_b200.engine import run_packed
    rng = np.random.default_rng(12)
    pairs = []
    for q in range(300):
        p = "".join(rng.choice(list("ACGT"), 3000))
        t = "".join(rng.choice(list("ACGT"), 3000)) if q % 3 == 0 else p
        pairs.append((p, t))
    batch = PackedBatch.from_pairs(pairs)
    got = run_packed(batch, 64, 24, 64, "MSID")
    exp = oracle_mod.align_packed(batch, 64, 24, 64, "MSID", threads=os.cpu_count())
    _packed_equal(got, exp, "full tier")


def test_device_call_vs_oracle(gpu, oracle_mod):
    """ga_align_batch_device on torch-owned device buffers, asynchronous on a
    caller stream (the bench's device-resident path), against the oracle."""
    import ctypes as C

    import torch

    from paper_2203_15561_b200 import _abi, engine, sim
    batch, _ = sim.config_pairs(5, count=1200)
    host = _abi.PackedResults.allocate(batch, 64, 24)
    order = engine.lpt_order(batch.pat_len)
    dev = torch.device("cuda:0")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d = [up(x) for x in (batch.codes, batch.pat_off, batch.pat_len, batch.txt_off, batch.txt_len,
                         order, host.ops_off, host.win_off)]
    res = torch.zeros(batch.n_pairs * 64, dtype=torch.uint8, device=dev)
    ops = torch.zeros(host.ops.shape[0], dtype=torch.uint8, device=dev)
    dst = torch.zeros(host.dists.shape[0], dtype=torch.uint8, device=dev)
    din = _abi.GaBatchIn(batch.n_pairs, d[0].data_ptr(), int(batch.codes.shape[0]), d[1].data_ptr(),
                         d[2].data_ptr(), d[3].data_ptr(), d[4].data_ptr(), d[5].data_ptr())
    dout = _abi.GaBatchOut(res.data_ptr(), d[6].data_ptr(), ops.data_ptr(), host.n_ops,
                           d[7].data_ptr(), dst.data_ptr(), int(host.dists.shape[0]))
    stream = torch.cuda.Stream(dev)
    L, ctx = engine.lib(), engine.context(0)
    cfg = _abi.make_config(64, 24, 64, "MSID")
    assert L.ga_align_batch_device(ctx, C.byref(din), C.byref(cfg), C.byref(dout),
                                   C.c_void_p(stream.cuda_stream)) == 0
    assert L.ga_last_launch_count(ctx) >= 1
    stream.synchronize()
    got = _abi.PackedResults(results=res.cpu().numpy().view(_abi.RESULT_DTYPE),
                             ops_off=host.ops_off, ops=ops.cpu().numpy(), win_off=host.win_off,
                             dists=dst.cpu().numpy(), n_ops=host.n_ops)
    exp = oracle_mod.align_packed(batch, 64, 24, 64, "MSID", threads=os.cpu_count())
    _packed_equal(got, exp, "device call")
    # the 2-bit transfer formats belong to the host-buffer call
    din.packed2 = 1
    assert L.ga_align_batch_device(ctx, C.byref(din), C.byref(cfg), C.byref(dout), None) == -3
    assert b"packed2" in L.ga_last_error(ctx)


def test_baseline_mode_vs_oracle(gpu, oracle_mod):
    """mode="baseline": the unimproved engine (all k+1 levels, dense 4-edge
    tables, traceback over stored edges) against the oracle field for field
    -- ops, distances and its own counters -- and against the reference's
    digests (tests/golden/baseline.json)."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.engine import run_packed
    with open(os.path.join(os.path.dirname(__file__), "golden", "baseline.json")) as f:
        gold = json.load(f)
    cases = corpus.fuzz_cases(gold["seed"], gold["batches"], pairs_per_batch=gold["pairs_per_batch"],
                              max_len=gold["max_len"])
    for case, ((w, o, k, prio), pairs) in zip(gold["cases"], cases):
        cfg = gpu.WindowConfig(window=w, overlap=o, k=k, priority=prio, mode="baseline")
        got = [str(corpus.digest(x)) for x in gpu.align_batch(pairs, cfg)]
        assert got == case["digests"], case["cfg"]
    for cfg_id, count, (w, o, k, prio) in [(1, 2000, (64, 24, 64, "MSID")),
                                           (5, 64, (128, 48, 64, "SMDI")),
                                           (5, 64, (32, 12, 8, "IDSM"))]:
        batch, _ = sim.config_pairs(cfg_id, count=count)
        got = run_packed(batch, w, o, k, prio, mode="baseline")
        exp = oracle_mod.align_packed(batch, w, o, k, prio, threads=os.cpu_count(), mode="baseline")
        _packed_equal(got, exp, ("baseline", cfg_id, w, o, k, prio))
    # same alignments as the improved engine, different counters
    batch, _ = sim.config_pairs(1, count=500)
    imp = run_packed(batch, 64, 24, 64, "MSID")
    base = run_packed(batch, 64, 24, 64, "MSID", mode="baseline")
    for f in ("status", "cost", "text_consumed", "ops_len"):
        assert np.array_equal(imp.results[f], base.results[f]), f
    assert (base.results["rows_computed"] > imp.results["rows_computed"]).all()
