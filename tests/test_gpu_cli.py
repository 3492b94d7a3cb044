"""The `bitalign align` command line on the GPU: stdout, stderr and exit code
byte-identical to the reference CLI's (tests/golden/cli.json, made by
tests/golden/make_cli_golden.py from pkg/src/bitalign/cli.py) -- the parse,
the kernel and the native row writer end to end, as a user runs it."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "cli.json")))


@pytest.mark.gpu
@pytest.mark.parametrize("run", GOLD["runs"],
                         ids=[f"{r['file']}:{' '.join(r['argv']) or 'default'}" for r in GOLD["runs"]])
def test_cli_align_matches_reference(run, tmp_path):
    path = tmp_path / (run["file"] + ".tsv")
    path.write_bytes(GOLD["files"][run["file"]].encode("utf-8"))
    proc = subprocess.run([sys.executable, "-m", "paper_2203_15561_b200.cli", "align", "--pairs",
                           str(path), *run["argv"]], cwd=ROOT, capture_output=True, timeout=300)
    err = proc.stderr.decode("utf-8").replace(str(tmp_path), "<tmp>")
    assert (proc.returncode, proc.stdout.decode("utf-8"), err) == \
        (run["code"], run["out"], run["err"])


_TIMING = {"seconds_improved", "seconds_baseline", "throughput_improved", "throughput_baseline",
           "speedup"}


def _untimed(text: str) -> list:
    lines = text.splitlines()
    if not lines:
        return []
    head = lines[0].split("\t")
    return [lines[0]] + [{c: v for c, v in zip(head, row.split("\t")) if c not in _TIMING}
                         for row in lines[1:]]


@pytest.mark.gpu
@pytest.mark.parametrize("run", GOLD["bench_runs"],
                         ids=[f"{r['file']}:{' '.join(r['argv']) or 'default'}"
                              for r in GOLD["bench_runs"]])
def test_cli_bench_matches_reference(run, tmp_path):
    """`bench`: both engines on the GPU, the reduction report and the DP
    cost-overhead column equal to the reference's, timing columns aside."""
    path = tmp_path / (run["file"] + ".tsv")
    path.write_bytes(GOLD["files"][run["file"]].encode("utf-8"))
    proc = subprocess.run([sys.executable, "-m", "paper_2203_15561_b200.cli", "bench", "--pairs",
                           str(path), *run["argv"]], cwd=ROOT, capture_output=True, timeout=300)
    err = proc.stderr.decode("utf-8").replace(str(tmp_path), "<tmp>")
    assert (proc.returncode, _untimed(proc.stdout.decode("utf-8")), err) == \
        (run["code"], _untimed(run["out"]), run["err"])


@pytest.mark.gpu
def test_dp_distances_match_reference():
    """The GPU DP kernel against the reference's oracle.global_distance /
    semiglobal_distance (multi-block patterns, empty sides, non-ACGT and
    non-ASCII characters, which match themselves)."""
    from paper_2203_15561_b200 import groundtruth
    pairs = [(p, t) for p, t, _, _ in GOLD["dp"]]
    assert groundtruth.global_distances(pairs) == [g for _, _, g, _ in GOLD["dp"]]
    sg = [(p, t, s) for p, t, _, s in GOLD["dp"] if p]
    assert groundtruth.semiglobal_distances([(p, t) for p, t, _ in sg]) == [s for _, _, s in sg]
