"""Pin the C oracle to the reference (CPU only).

The oracle is the checker for the GPU path, so it is itself checked against
(1) the reference's known-answer vectors, (2) golden fixtures produced by
running the reference (tests/golden/make_golden.py), and (3) when the
reference checkout is present, a live differential run.
"""

from __future__ import annotations

import json
import os
import random

import numpy as np
import pytest

import corpus
from paper_2203_15561_b200 import WindowConfig

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _cfg(w, o, k, prio="MSID"):
    return WindowConfig(window=w, overlap=o, k=k, priority=prio)


def test_known_answer_vectors(oracle_mod):
    with open(os.path.join(GOLD, "known.json")) as f:
        known = json.load(f)
    assert len(known) == len(corpus.KNOWN)
    for case in known:
        cfg = _cfg(case["window"], case["overlap"], case["k"], case["priority"])
        got = oracle_mod.align_batch([(case["pattern"], case["text"])], cfg)[0]
        assert corpus.outcome_key(got) == case["key"], case


def test_reference_test_expectations(oracle_mod):
    """Literal expectations from pkg/tests/test_window.py:62-88 and
    pkg/tests/test_backtrace.py:33-59 (CIGARs in expanded form)."""
    def one(p, t, cfg=None):
        return oracle_mod.align_batch([(p, t)], cfg or WindowConfig())[0]
    r = one("ACGTACGT", "ACGTACGT", _cfg(4, 2, 4)).result
    assert (r.cigar, r.cost, r.text_consumed, r.window_distances) == ("=" * 8, 0, 8, (0, 0, 0))
    r = one("ACGT", "AC").result
    assert (r.cigar, r.cost, r.text_consumed) == ("==II", 2, 2)
    r = one("ACGT", "").result
    assert (r.cigar, r.cost) == ("IIII", 4)
    assert one("AAAAAAAA", "TTTTTTTT", _cfg(8, 2, 2)).error == \
        "WindowFailed: window 0 found no alignment within k=2"
    assert one("", "ACGT").error == "EmptyPattern: pattern must not be empty"
    assert one("ACGT", "AGGT").result.cigar == "=X=="
    assert one("ACGT", "ACT").result.cigar == "==I="
    # windowed align anchors the text at 0 (window.py:1-13), so the free prefix of
    # the DC frame (traceback ("ACG","TTACG") -> "===") becomes leading deletions
    r = one("ACG", "TTACG").result
    assert (r.cigar, r.text_consumed) == ("DD===", 5)
    # symbol corner cases: lowercase and 'N' never match
    r = one("acgt", "acgt").result
    assert (r.cigar, r.cost, r.window_distances, r.rows_computed) == ("XXXX", 4, (4,), 5)
    assert (r.counters.entry_reads, r.counters.entry_writes, r.counters.words_allocated) == \
        (10, 20, 20)
    assert one("ANGT", "ANGT").result.cigar == "=X=="
    assert one("NNNN", "NNNN").result.cigar == "XXXX"


def test_fuzz_golden(oracle_mod):
    with open(os.path.join(GOLD, "fuzz.json")) as f:
        gold = json.load(f)
    for case, ((w, o, k, prio), pairs) in zip(gold["cases"],
                                             corpus.fuzz_cases(gold["seed"], gold["batches"])):
        assert case["cfg"] == [w, o, k, prio]
        got = [str(corpus.digest(x)) for x in oracle_mod.align_batch(pairs, _cfg(w, o, k, prio))]
        assert got == case["digests"], case["cfg"]


@pytest.mark.parametrize("key,cfg_id,w,o,k", [
    ("cfg1", 1, 64, 24, 64), ("cfg3", 3, 64, 24, 64), ("cfg4", 4, 64, 24, 64),
    ("cfg5_w32_k8", 5, 32, 12, 8), ("cfg5_w64_k16", 5, 64, 24, 16),
    ("cfg5_w128_k128", 5, 128, 48, 128),
])
def test_config_digests(oracle_mod, key, cfg_id, w, o, k):
    """Oracle vs the reference's own outputs on the BASELINE recipe pairs."""
    from paper_2203_15561_b200 import sim
    from paper_2203_15561_b200.window import outcomes_from_packed
    gold = np.load(os.path.join(GOLD, "configs.npz"))[key]
    batch, _ = sim.config_pairs(cfg_id, count=len(gold), threads=4)
    cfg = _cfg(w, o, k)
    out = oracle_mod.align_packed(batch, w, o, k, "MSID", threads=os.cpu_count())
    got = np.array([corpus.digest(x) for x in outcomes_from_packed(batch, out, cfg)],
                   dtype=np.uint64)
    assert np.array_equal(got, gold)


def test_thread_count_invariance(oracle_mod):
    rng = random.Random(5)
    pairs = [("".join(rng.choice("ACGT") for _ in range(rng.randrange(1, 300))),
              "".join(rng.choice("ACGT") for _ in range(rng.randrange(0, 300))))
             for _ in range(64)]
    cfg = _cfg(32, 8, 32)
    a = [corpus.outcome_key(x) for x in oracle_mod.align_batch(pairs, cfg, threads=1)]
    b = [corpus.outcome_key(x) for x in oracle_mod.align_batch(pairs, cfg, threads=7)]
    assert a == b


@pytest.mark.reference
def test_live_differential_vs_reference(oracle_mod, reference):
    from bitalign.window import WindowConfig as RefConfig
    from bitalign.window import align_batch as ref_batch
    for (w, o, k, prio), pairs in corpus.fuzz_cases(31337, 25, pairs_per_batch=6, max_len=300):
        ref = ref_batch(pairs, RefConfig(window=w, overlap=o, k=k, priority=prio))
        got = oracle_mod.align_batch(pairs, _cfg(w, o, k, prio))
        assert [corpus.outcome_key(x) for x in got] == [corpus.outcome_key(x) for x in ref]


def _baseline_gold():
    with open(os.path.join(GOLD, "baseline.json")) as f:
        return json.load(f)


def _cfg1_pairs(count):
    from paper_2203_15561_b200 import sim
    batch, _ = sim.config_pairs(1, count=count)
    return [(sim.codes_to_str(batch.codes[batch.pat_off[q]:batch.pat_off[q] + batch.pat_len[q]]),
             sim.codes_to_str(batch.codes[batch.txt_off[q]:batch.txt_off[q] + batch.txt_len[q]]))
            for q in range(batch.n_pairs)]


def test_baseline_mode_golden(oracle_mod):
    """The unimproved engine (dc_baseline + stored-edge traceback) against the
    reference's mode="baseline" outcomes, counters included
    (tests/golden/make_baseline_golden.py)."""
    gold = _baseline_gold()
    cases = corpus.fuzz_cases(gold["seed"], gold["batches"], pairs_per_batch=gold["pairs_per_batch"],
                              max_len=gold["max_len"])
    for case, ((w, o, k, prio), pairs) in zip(gold["cases"], cases):
        cfg = WindowConfig(window=w, overlap=o, k=k, priority=prio, mode="baseline")
        got = [str(corpus.digest(x)) for x in oracle_mod.align_batch(pairs, cfg, threads=4)]
        assert got == case["digests"], case["cfg"]
    cfg = WindowConfig(mode="baseline")
    got = [str(corpus.digest(x)) for x in oracle_mod.align_batch(_cfg1_pairs(200), cfg, threads=4)]
    assert got == gold["cfg1_first200"]


def test_baseline_known_counters(oracle_mod):
    """cli.json's --mode baseline --stats rows: rows_computed k+1 per window,
    4(k+1)n writes, 1 read per level-0 step and 4 above."""
    r = oracle_mod.align_batch([("ACGT", "AGGT")], WindowConfig(mode="baseline"))[0].result
    assert (r.cigar, r.cost, r.rows_computed) == ("=X==", 1, 65)
    assert (r.counters.entry_reads, r.counters.entry_writes, r.counters.words_allocated) == \
        (10, 1040, 1040)
