"""N>1 path on CPU: world_size-2 gloo process group over 127.0.0.1.

The per-rank aligner is the oracle here (no GPU in the build container);
what is under test is the sharding and the ordered gather: the distributed
result must equal the single-process result slot for slot, like the
reference's parallelism-invariance tests (pkg/tests/test_window.py:161-169).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2203_15561_b200 import WindowConfig
from paper_2203_15561_b200.distributed import shard_indices


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pairs():
    import random

    import corpus
    rng = random.Random(91)
    pairs = []
    for _ in range(40):
        p = "".join(rng.choice("ACGT") for _ in range(rng.randrange(0, 500)))
        pairs.append((p, corpus.noisy_copy(rng, p, 0.1)))
    pairs.append(("AAAAAAAA", "TTTTTTTT"))
    return pairs


def _worker(rank, world, port, dst, out_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    import corpus
    from oracle import oracle
    from paper_2203_15561_b200.distributed import align_batch_distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = WindowConfig(window=32, overlap=8, k=8)
    got = align_batch_distributed(_pairs(), cfg, aligner=oracle.align_batch, dst=dst)
    if got is not None:
        with open(f"{out_path}.{rank}", "w") as f:
            f.write("\n".join(corpus.outcome_key(o) for o in got))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dst", [0, None])
def test_two_rank_gather_matches_single_process(tmp_path, oracle_mod, dst):
    import corpus
    out = str(tmp_path / "res")
    mp.start_processes(_worker, args=(2, _free_port(), dst, out), nprocs=2, join=True,
                       start_method="spawn")
    cfg = WindowConfig(window=32, overlap=8, k=8)
    expect = "\n".join(corpus.outcome_key(o) for o in oracle_mod.align_batch(_pairs(), cfg))
    ranks = [0] if dst == 0 else [0, 1]
    for r in ranks:
        assert open(f"{out}.{r}").read() == expect
    if dst == 0:
        assert not os.path.exists(f"{out}.1")


def test_shards_partition_and_balance():
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 60_000, size=777)
    for world in (1, 2, 3, 8):
        shards = [shard_indices(lens, 64, 24, world, r) for r in range(world)]
        assert np.array_equal(np.sort(np.concatenate(shards)), np.arange(777))
        from paper_2203_15561_b200._abi import num_windows
        cost = np.maximum(num_windows(lens, 64, 24), 1)
        loads = [int(cost[s].sum()) for s in shards]
        assert max(loads) - min(loads) <= int(cost.max())
    with pytest.raises(ValueError):
        shard_indices(lens, 64, 24, 2, 2)
