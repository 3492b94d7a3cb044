"""Deterministic test corpora shared by the golden generator and the parity tests.

Shapes follow the reference's own randomized tests: noisy copies and
independent strings (pkg/tests/test_acceptance.py:41-64,
pkg/tests/test_window.py:19-32), plus the symbol corner cases of SURVEY 8(c)
(lowercase, 'N', empty text, short text, k-failures, every priority).
"""

from __future__ import annotations

import hashlib
import itertools
import random

PRIORITIES = ["".join(p) for p in itertools.permutations("MSID")]

# Known-answer vectors from the reference's tests:
#   pkg/tests/test_window.py:62-88, pkg/tests/test_backtrace.py:33-59, test_cli.py:25-61,
#   and symbol corner cases run through the reference (SURVEY 8c last rows).
KNOWN = [
    # (pattern, text, window, overlap, k, priority)
    ("ACGTACGT", "ACGTACGT", 4, 2, 4, "MSID"),
    ("ACGT", "AC", 64, 24, None, "MSID"),
    ("ACGT", "", 64, 24, None, "MSID"),
    ("AAAAAAAA", "TTTTTTTT", 8, 2, 2, "MSID"),
    ("ACGT", "ACGT", 64, 24, None, "MSID"),
    ("ACGT", "AGGT", 64, 24, None, "MSID"),
    ("AAAA", "", 64, 24, None, "MSID"),
    ("ACGT", "ACT", 64, 24, None, "MSID"),
    ("ACG", "TTACG", 64, 24, None, "MSID"),
    ("acgt", "acgt", 64, 24, None, "MSID"),
    ("ANGT", "ANGT", 64, 24, None, "MSID"),
    ("NNNN", "NNNN", 64, 24, None, "MSID"),
    ("", "ACGT", 64, 24, None, "MSID"),
    ("ACGT" * 40, "ACGT" * 4, 16, 4, None, "MSID"),
    ("AAAA", "TTTT", 4, 1, 2, "MSID"),
]


def noisy_copy(rng: random.Random, seq: str, rate: float, alphabet: str = "ACGT") -> str:
    out = []
    for symbol in seq:
        r = rng.random()
        if r < rate / 3:
            continue
        if r < 2 * rate / 3:
            out.append(rng.choice(alphabet))
        elif r < rate:
            out.append(symbol)
            out.append(rng.choice(alphabet))
        else:
            out.append(symbol)
    return "".join(out)


def fuzz_cases(seed: int, n_batches: int, pairs_per_batch: int = 8, max_len: int = 400,
               windows=(4, 8, 16, 31, 32, 33, 40, 63, 64, 65, 100, 128)):
    """Yields (cfg_tuple, pairs) batches: random W, O, k, priority and pairs
    mixing noisy copies, unrelated strings, non-ACGT symbols and empty texts."""
    rng = random.Random(seed)
    for _ in range(n_batches):
        W = rng.choice(windows)
        O = rng.randrange(0, W)
        k = rng.choice([None, max(1, W // 4), max(1, W // 2), W, rng.randrange(1, W + 1)])
        prio = rng.choice(PRIORITIES) if rng.random() < 0.5 else "MSID"
        pairs = []
        for _ in range(pairs_per_batch):
            L = rng.randrange(0, max_len)
            alpha = "ACGT" if rng.random() < 0.8 else "ACGTNacgt"
            p = "".join(rng.choice(alpha) for _ in range(L))
            if rng.random() < 0.8:
                t = noisy_copy(rng, p, rng.choice([0.0, 0.02, 0.05, 0.15, 0.3, 0.5]))
            else:
                t = "".join(rng.choice(alpha) for _ in range(rng.randrange(0, max_len)))
            pairs.append((p, t))
        yield (W, O, k, prio), pairs


def outcome_key(o) -> str:
    """Canonical text of one BatchOutcome: every field the parity contract names."""
    if not o.ok:
        return "ERR|" + o.error
    r = o.result
    return "|".join([r.cigar, str(r.cost), str(r.text_consumed),
                     ",".join(map(str, r.window_distances)), str(r.rows_computed),
                     str(r.counters.entry_reads), str(r.counters.entry_writes),
                     str(r.counters.words_allocated)])


def digest(o) -> int:
    """64-bit digest of outcome_key (for full-config fixtures)."""
    return int.from_bytes(hashlib.sha1(outcome_key(o).encode()).digest()[:8], "little")
