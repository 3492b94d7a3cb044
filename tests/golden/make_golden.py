"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the reference checkout exists only here):
    python tests/golden/make_golden.py
Outputs (committed):
    known.json          outcome keys of the reference's known-answer vectors
    fuzz.json           digests of the randomized corpus (tests/corpus.py)
    sim.json            digests of reference-simulated sequences and recipe pairs
    configs.npz         per-pair digests of the BASELINE configs' recipe pairs
                        (cfg1 all 10,000; cfg2 all 100,000; cfg3 first 256;
                        cfg4 first 4; cfg5 first 64 per sweep point)
Everything is computed by `bitalign` (pkg/src/bitalign) -- its simulator,
its CLI recipe and its align_batch -- so the fixtures pin both the workload
generator port and the aligner to the reference's own outputs.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import random
import sys
import time
from multiprocessing import Pool

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
from bitalign import sim as rsim  # noqa: E402
from bitalign.window import WindowConfig, align_batch  # noqa: E402

import corpus  # noqa: E402

# BASELINE configs: ref_len, count, read_len, sub, ins, del, seed
CONFIGS = {
    1: (2_000_000, 10_000, 150, 0.01, 0.005, 0.005, 1501),
    2: (5_000_000, 100_000, 250, 0.04, 0.005, 0.005, 2502),
    3: (20_000_000, 138_929, 10_000, 0.01, 0.07, 0.07, 10003),
    4: (50_000_000, 20_000, 100_000, 0.04, 0.02, 0.04, 100004),
    5: (5_000_000, 8_192, 0, 0.04, 0.03, 0.03, 5005),
}
TAKE = {1: 10_000, 2: 100_000, 3: 256, 4: 4, 5: 64}
SWEEP5 = [(w, 3 * w // 8, k) for w in (32, 64, 128) for k in (w // 4, w // 2, w)]


def mixed_lengths(count, seed, lo=100, hi=50_000):
    rng = random.Random(seed)
    a, b = math.log(lo), math.log(hi)
    return [int(round(math.exp(rng.uniform(a, b)))) for _ in range(count)]


_REF = None


def _init(ref):
    global _REF
    _REF = ref


def _sim_one(args):
    index, pos, read_len, sub, ins, dele, seed = args
    prof = rsim.ErrorProfile(sub, ins, dele, rsim.derive_seed(seed, index + 1))
    rec = rsim.simulate_read(_REF, pos, read_len, prof)
    return rec.read, _REF[pos:pos + read_len]


def recipe(cfg_id, n, pool_size=8):
    ref_len, count, read_len, sub, ins, dele, seed = CONFIGS[cfg_id]
    ref = rsim.make_reference(ref_len, seed)
    lens = [read_len] * count if read_len else mixed_lengths(count, seed)
    prng = random.Random(rsim.derive_seed(seed, 0xB0B))
    jobs = []
    for i in range(n):
        pos = prng.randrange(0, ref_len - lens[i] + 1)
        jobs.append((i, pos, lens[i], sub, ins, dele, seed))
    with Pool(pool_size, initializer=_init, initargs=(ref,)) as pool:
        pairs = pool.map(_sim_one, jobs, chunksize=max(1, n // 64))
    return pairs


def sdig(s: str) -> str:
    return hashlib.sha1(s.encode()).hexdigest()[:16]


def main():
    t0 = time.time()
    known = []
    for p, t, w, o, k, prio in corpus.KNOWN:
        cfg = WindowConfig(window=w, overlap=o, k=k, priority=prio)
        known.append({"pattern": p, "text": t, "window": w, "overlap": o, "k": k,
                      "priority": prio,
                      "key": corpus.outcome_key(align_batch([(p, t)], cfg)[0])})
    with open(os.path.join(HERE, "known.json"), "w") as f:
        json.dump(known, f, indent=1)

    fuzz = []
    for (w, o, k, prio), pairs in corpus.fuzz_cases(2024, 80):
        cfg = WindowConfig(window=w, overlap=o, k=k, priority=prio)
        fuzz.append({"cfg": [w, o, k, prio],
                     "digests": [str(corpus.digest(x)) for x in align_batch(pairs, cfg)]})
    with open(os.path.join(HERE, "fuzz.json"), "w") as f:
        json.dump({"seed": 2024, "batches": 80, "cases": fuzz}, f)
    print("known/fuzz", time.time() - t0, flush=True)

    simg = {"reference": [], "reads": [], "recipes": {}}
    for seed in (0, 1, 7, 2**32 - 1, 2**32, 10003, 123456789012345):
        simg["reference"].append([5000, seed, sdig(rsim.make_reference(5000, seed))])
    ref = rsim.make_reference(20000, 42)
    rng = random.Random(99)
    for _ in range(60):
        pos, ln = rng.randrange(0, 10000), rng.randrange(1, 5000)
        sub, ins, dele = rng.random() * 0.3, rng.random() * 0.3, rng.random() * 0.3
        seed = rng.getrandbits(64)
        rd = rsim.simulate_read(ref, pos, ln, rsim.ErrorProfile(sub, ins, dele, seed)).read
        simg["reads"].append([pos, ln, sub, ins, dele, str(seed), sdig(rd)])

    digests = {}
    for cfg_id in (1, 2, 3, 4, 5):
        n = TAKE[cfg_id]
        pairs = recipe(cfg_id, n)
        simg["recipes"][str(cfg_id)] = [sdig(p + "|" + t) for p, t in pairs[:64]]
        print(f"cfg{cfg_id}: {n} pairs simulated", time.time() - t0, flush=True)
        if cfg_id == 5:
            for (w, o, k) in SWEEP5:
                cfg = WindowConfig(window=w, overlap=o, k=k)
                outs = align_batch(pairs, cfg, parallelism=8)
                digests[f"cfg5_w{w}_k{k}"] = np.array([corpus.digest(x) for x in outs],
                                                      dtype=np.uint64)
        else:
            outs = align_batch(pairs, WindowConfig(), parallelism=8)
            digests[f"cfg{cfg_id}"] = np.array([corpus.digest(x) for x in outs], dtype=np.uint64)
        print(f"cfg{cfg_id}: aligned", time.time() - t0, flush=True)
    with open(os.path.join(HERE, "sim.json"), "w") as f:
        json.dump(simg, f, indent=0)
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **digests)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
