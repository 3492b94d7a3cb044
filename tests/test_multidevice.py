"""The in-process multi-device path of ``engine.run_batch(devices=N)`` on CPU.

Each device's ``run_packed`` is replaced by the oracle (no GPU here); what is
under test is the host logic around it: the LPT split, one host thread per
device, and ``_scatter`` putting every shard's records, ops and window
distances back at their input positions.  The contract is the reference's
parallelism invariance (pkg/tests/test_window.py:161-169): the slots equal
the single-device run slot for slot, whatever the shard layout -- uneven
shards, a shard with only empty patterns, more devices than pairs.
"""

from __future__ import annotations

import random
import threading

import numpy as np
import pytest

from paper_2203_15561_b200 import WindowConfig, engine
from paper_2203_15561_b200._abi import PackedBatch


@pytest.fixture
def oracle_devices(monkeypatch, oracle_mod):
    calls = []
    lock = threading.Lock()

    def fake_run_packed(batch, window, overlap, k, priority, device=None, *, packed2=False,
                        ops2=False, mode="improved", host_pack=False):
        with lock:
            calls.append((device, batch.n_pairs, threading.get_ident()))
        return oracle_mod.align_packed(batch, window, overlap, k, priority, 1, mode)

    monkeypatch.setattr(engine, "run_packed", fake_run_packed)
    return calls


def _pairs(seed, n, maxlen=700, empty_every=0):
    import corpus
    rng = random.Random(seed)
    out = []
    for q in range(n):
        if empty_every and q % empty_every == 0:
            out.append(("", "ACGT" * rng.randrange(0, 4)))
            continue
        p = "".join(rng.choice("ACGTN") for _ in range(rng.randrange(1, maxlen)))
        out.append((p, corpus.noisy_copy(rng, p, 0.12)))
    return out


def _equal(a, b, batch):
    assert np.array_equal(a.results, b.results)
    for q in range(batch.n_pairs):
        assert a.cigar(q) == b.cigar(q)
        n = int(batch.pat_len[q])
        assert a.distances(q, n, 32, 8) == b.distances(q, n, 32, 8)
    assert np.array_equal(a.dists, b.dists)


@pytest.mark.parametrize("devices", [2, 3, 8])
def test_run_batch_devices_matches_single(oracle_devices, oracle_mod, devices):
    cfg = WindowConfig(window=32, overlap=8, k=16)
    pairs = _pairs(7 + devices, 37, empty_every=9)
    batch = PackedBatch.from_pairs(pairs)
    got = engine.run_batch(batch, cfg, devices=devices)
    exp = oracle_mod.align_packed(batch, 32, 8, 16, "MSID")
    _equal(got, exp, batch)
    used = {c[0] for c in oracle_devices}
    assert used == set(range(devices))
    # each device is driven from its own host thread, not the caller's
    assert threading.main_thread().ident not in {c[2] for c in oracle_devices}


def test_shard_of_only_empty_patterns(oracle_devices, oracle_mod):
    # the ADVICE r1 case: device 1's shard holds only an empty pattern
    cfg = WindowConfig(window=4, overlap=2, k=4)
    hard = ("ACGTACGT", "TGCATGCA")  # every window at distance > 0
    for pairs in ([("", "A"), hard], [hard, ("", "A")], [("", ""), hard, ("", "C")]):
        batch = PackedBatch.from_pairs(pairs)
        got = engine.run_batch(batch, cfg, devices=2)
        exp = oracle_mod.align_packed(batch, 4, 2, 4, "MSID")
        assert np.array_equal(got.results, exp.results)
        assert np.array_equal(got.dists, exp.dists)
        assert min(got.dists.tolist()[:3]) > 0


def test_more_devices_than_pairs(oracle_devices, oracle_mod):
    cfg = WindowConfig(window=32, overlap=8, k=32)
    pairs = _pairs(3, 3)
    batch = PackedBatch.from_pairs(pairs)
    got = engine.run_batch(batch, cfg, devices=8)
    exp = oracle_mod.align_packed(batch, 32, 8, 32, "MSID")
    _equal(got, exp, batch)


def test_uneven_lengths_keep_order(oracle_devices, oracle_mod):
    # one long pair and many short ones: LPT gives one device a single pair
    cfg = WindowConfig(window=32, overlap=8, k=16)
    pairs = _pairs(11, 20, maxlen=120)
    p = "ACGT" * 900
    pairs.insert(5, (p, p[:1500] + "TT" + p[1500:]))
    batch = PackedBatch.from_pairs(pairs)
    shards = engine.split_lpt(batch.pat_len, 32, 8, 3)
    assert any(len(s) == 1 and s[0] == 5 for s in shards)
    got = engine.run_batch(batch, cfg, devices=3)
    exp = oracle_mod.align_packed(batch, 32, 8, 16, "MSID")
    _equal(got, exp, batch)
