"""The C++ workload generator reproduces the reference simulator bit-for-bit
(fixtures recorded from pkg/src/bitalign/sim.py and cli.py by make_golden.py)."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2203_15561_b200 import sim

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sdig(s: str) -> str:
    return hashlib.sha1(s.encode()).hexdigest()[:16]


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLD, "sim.json")) as f:
        return json.load(f)


def test_make_reference(gold):
    for length, seed, dig in gold["reference"]:
        assert sdig(sim.codes_to_str(sim.make_reference(length, seed))) == dig, seed


def test_simulate_read(gold):
    ref = sim.make_reference(20000, 42)
    for pos, ln, sub, ins, dele, seed, dig in gold["reads"]:
        read = sim.simulate_read(ref, pos, ln, sub, ins, dele, int(seed))
        assert sdig(sim.codes_to_str(read)) == dig


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 5])
def test_config_recipes(gold, cfg_id):
    expect = gold["recipes"][str(cfg_id)]
    batch, _ = sim.config_pairs(cfg_id, count=len(expect), threads=2)
    for q, dig in enumerate(expect):
        p = sim.codes_to_str(batch.codes[batch.pat_off[q]:batch.pat_off[q] + batch.pat_len[q]])
        t = sim.codes_to_str(batch.codes[batch.txt_off[q]:batch.txt_off[q] + batch.txt_len[q]])
        assert sdig(p + "|" + t) == dig, q


def test_derive_seed_matches_formula():
    m = (1 << 64) - 1
    s = 12345
    for salt in (7, 0xB0B):
        s = (s * 6364136223846793005 + salt + 1442695040888963407) & m
    assert sim.derive_seed(12345, 7, 0xB0B) == s


def test_thread_count_invariance():
    ref = sim.make_reference(100_000, 3)
    a, pa = sim.recipe_pairs(ref, 200, 1000, 0.05, 0.05, 0.05, 9, threads=1)
    b, pb = sim.recipe_pairs(ref, 200, 1000, 0.05, 0.05, 0.05, 9, threads=8)
    assert np.array_equal(a.codes, b.codes) and np.array_equal(pa, pb)
