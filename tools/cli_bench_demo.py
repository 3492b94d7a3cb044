"""Write a BASELINE config's recipe pairs as a pair-list TSV and run the GPU
`bench` command on it (improved vs unimproved engine, reduction report, DP
cost overhead).  Usage: python tools/cli_bench_demo.py [config] [count] [extra CLI args]"""

from __future__ import annotations

import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2203_15561_b200 import sim  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    count = int(sys.argv[2]) if len(sys.argv) > 2 else None
    batch, _ = sim.config_pairs(cfg, count=count)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "pairs.tsv")
        with open(path, "w") as fh:
            for q in range(batch.n_pairs):
                p = sim.codes_to_str(batch.codes[batch.pat_off[q]:batch.pat_off[q] + batch.pat_len[q]])
                t = sim.codes_to_str(batch.codes[batch.txt_off[q]:batch.txt_off[q] + batch.txt_len[q]])
                fh.write(f"r{q + 1}\t{p}\t{t}\n")
        for _ in range(2):  # the first run pays context creation
            r = subprocess.run([sys.executable, "-m", "paper_2203_15561_b200.cli", "bench", "--pairs",
                                path, *sys.argv[3:]], cwd=ROOT, capture_output=True, text=True)
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)


if __name__ == "__main__":
    main()
