"""The GA_CHECK build: the kernel with its contract checks compiled in
(PrunedAccess-style tripwires on every band/wide/full-tier table read, bounds
on ops, window distances, ring entries and table stores) runs the bench
shapes and a fuzz corpus with zero violations and oracle-equal results.
Mirrors the reference's own tripwires: PrunedAccess (pkg/src/bitalign/
dptable.py:20-30, raised at :183-184) and StuckTraceback
(pkg/src/bitalign/backtrace.py:30-35)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_SO = os.path.join(ROOT, "paper_2203_15561_b200", "_genasm_check.so")


@pytest.mark.gpu
def test_check_build_clean():
    from paper_2203_15561_b200 import build
    if build.needs_build(CHECK_SO):
        build.build(check=True)
    env = dict(os.environ, GA_SO=CHECK_SO)
    proc = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "check_run.py")], env=env,
                          capture_output=True, text=True, timeout=1500)
    assert proc.returncode == 0, proc.stderr[-3000:]
    res = json.loads(proc.stdout.strip().splitlines()[-1])
    assert res["violations"] == 0, res
    assert res["mismatches"] == [], res
    assert res["cases"] > 40
