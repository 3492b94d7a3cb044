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
