"""File formats and the CLI's host side against the reference's own outputs
(tests/golden/cli.json, made by tests/golden/make_cli_golden.py from
pkg/src/bitalign/{cli,io}.py).  CPU only: the native parser and row
formatter are host code in the same library (no CUDA call)."""

from __future__ import annotations

import io
import json
import os
import random

import numpy as np
import pytest

from paper_2203_15561_b200 import _abi
from paper_2203_15561_b200 import io as fmt
from paper_2203_15561_b200._abi import PackedResults

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cli.json")))
_CODE = {"A": 0, "C": 1, "G": 2, "T": 3}


def _codes(s: str) -> list[int]:
    return [_CODE.get(c, 4) for c in s]


@pytest.mark.parametrize("name", sorted(GOLD["files"]))
def test_read_pairs_python(name):
    text = GOLD["files"][name]
    exp = GOLD["pairs"][name]
    try:
        got = [[r.id, r.pattern, r.text] for r in fmt.read_pairs(io.StringIO(text, newline=None))]
    except fmt.PairParseError as exc:
        got = f"PairParseError: {exc}"
    assert got == exp


@pytest.mark.parametrize("name", sorted(GOLD["files"]))
@pytest.mark.parametrize("threads", [1, 3])
def test_parse_pairs_native(name, threads):
    """The native reader (any file; non-ASCII ones go through Python)."""
    data = GOLD["files"][name].encode("utf-8")
    exp = GOLD["pairs"][name]
    try:
        lp = fmt.parse_pairs_bytes(data, threads=threads)
    except fmt.PairParseError as exc:
        assert f"PairParseError: {exc}" == exp
        return
    assert isinstance(exp, list)
    b = lp.batch
    assert lp.n_pairs == len(exp)
    for q, (pid, pat, txt) in enumerate(exp):
        assert lp.id(q) == pid
        assert b.codes[b.pat_off[q]:b.pat_off[q] + b.pat_len[q]].tolist() == _codes(pat)
        assert b.codes[b.txt_off[q]:b.txt_off[q] + b.txt_len[q]].tolist() == _codes(txt)


def test_parse_pairs_native_multichunk():
    """A file large enough for several parser chunks, every newline style and
    skipped-line kind mixed in, against the Python reader line for line."""
    rng = random.Random(5)
    rows = []
    for q in range(40_000):
        kind = rng.random()
        if kind < 0.05:
            rows.append(rng.choice(["# c", "   #x\tA\tB", "", " \t ", "\x0b"]))
            continue
        p = "".join(rng.choice("ACGTacgtN") for _ in range(rng.randint(1, 90)))
        t = "".join(rng.choice("ACGTN") for _ in range(rng.randint(0, 90)))
        rows.append(f"id{q}\t{p}\t{t}")
    text = "".join(r + rng.choice(["\n", "\r\n", "\r"]) for r in rows)
    data = text.encode()
    assert len(data) > 3 << 20
    exp = fmt.read_pairs(io.StringIO(text, newline=None))
    lp = fmt.parse_pairs_bytes(data, threads=4)
    assert lp.n_pairs == len(exp)
    b = lp.batch
    for q in range(0, len(exp), 97):
        assert lp.id(q) == exp[q].id
        assert b.codes[b.pat_off[q]:b.pat_off[q] + b.pat_len[q]].tolist() == _codes(exp[q].pattern)
        assert b.codes[b.txt_off[q]:b.txt_off[q] + b.txt_len[q]].tolist() == _codes(exp[q].text)
    assert int(b.pat_len.sum() + b.txt_len.sum()) == sum(len(r.pattern) + len(r.text) for r in exp)
    # a malformed row deep in the file: the first one is reported, by line
    lines = (text.replace("\r\n", "\n").replace("\r", "\n")).split("\n")
    target = len(lines) * 3 // 4
    while not lines[target].startswith("id"):
        target += 1
    lines[target] = lines[target] + "\textra"
    lines[target + 5] = "x\t\ty" if lines[target + 5].startswith("id") else lines[target + 5]
    with pytest.raises(fmt.PairParseError) as ei:
        fmt.parse_pairs_bytes("\n".join(lines).encode(), threads=4)
    assert str(ei.value) == f"line {target + 1}: expected 3 tab-separated columns, got 4"


def test_cigar_helpers():
    for ops, exp, classic in GOLD["cigars"]:
        assert fmt.format_cigar(ops) == exp
        assert fmt.format_classic_cigar(ops) == classic
        assert fmt.parse_cigar(exp) == ops
    for text, exp in GOLD["parse"]:
        try:
            got = fmt.parse_cigar(text)
        except fmt.CigarError as exc:
            got = f"CigarError: {exc}"
        assert got == exp, text
    with pytest.raises(fmt.CigarError, match="unknown operator 'M'"):
        fmt.format_cigar("==M")


def test_fasta():
    for name, (text, exp, written) in GOLD["fasta"].items():
        try:
            recs = fmt.read_fasta(io.StringIO(text))
        except fmt.MalformedFasta as exc:
            assert f"MalformedFasta: {exc}" == exp, name
            continue
        assert [[r.id, r.sequence, sorted(r.nonstandard)] for r in recs] == exp, name
        buf = io.StringIO()
        fmt.write_fasta(recs, buf, line_width=7)
        assert buf.getvalue() == written, name


def _results_from_rows(lp: fmt.LoadedPairs, out_text: str, stats: bool, ops2: bool):
    """PackedResults reconstructed from the reference's rows (what the kernel
    returns for them), so the native formatter can be checked on CPU."""
    rows = out_text.splitlines()
    assert len(rows) == lp.n_pairs
    res = PackedResults.allocate(lp.batch, 64, 24, ops2=ops2)
    for q, row in enumerate(rows):
        cols = row.split("\t")
        r = res.results[q]
        if cols[1].startswith("ERROR WindowFailed"):
            r["status"] = _abi.GA_WINDOW_FAILED
            r["fail_window"] = int(cols[1].split("window ")[1].split()[0])
            continue
        r["status"] = _abi.GA_OK
        r["fail_window"] = -1
        r["cost"], r["text_consumed"] = int(cols[1]), int(cols[2])
        ops = fmt.parse_cigar(cols[3])
        r["ops_len"] = len(ops)
        a = int(res.ops_off[q])
        if ops2:
            for x, c in enumerate(ops):
                y = a + x
                res.ops[y >> 2] |= "=XID".index(c) << (2 * (y & 3))
        else:
            res.ops[a:a + len(ops)] = np.frombuffer(ops.encode(), np.uint8)
        if stats:
            (r["rows_computed"], r["entry_reads"], r["entry_writes"],
             r["words_allocated"]) = map(int, cols[4:8])
    return res


@pytest.mark.parametrize("ops2", [False, True])
def test_format_align_rows(ops2):
    """The native row writer reproduces the reference's stdout byte for byte
    (ASCII and 2-bit ops; --stats; --collapse-m through the equal rows)."""
    checked = 0
    for run in GOLD["runs"]:
        argv = run["argv"]
        if run["code"] == 2 or "--collapse-m" in argv:
            continue
        lp = fmt.parse_pairs_bytes(GOLD["files"][run["file"]].encode("utf-8"))
        stats = "--stats" in argv
        res = _results_from_rows(lp, run["out"], stats, ops2)
        k = int(argv[argv.index("--k") + 1]) if "--k" in argv else 64
        text, failed = fmt.format_align_rows(lp, res, k, stats=stats)
        assert text.decode("utf-8") == run["out"], (run["file"], argv)
        assert (failed > 0) == (run["code"] == 1)
        # collapse-m: '='/'X' runs fold into M
        text_m, _ = fmt.format_align_rows(lp, res, k, collapse_m=True, stats=stats)
        exp_m = []
        for row in run["out"].splitlines():
            cols = row.split("\t")
            if not cols[1].startswith("ERROR"):
                cols[3] = fmt.format_classic_cigar(fmt.parse_cigar(cols[3]))
            exp_m.append("\t".join(cols) + "\n")
        assert text_m.decode("utf-8") == "".join(exp_m)
        checked += 1
    assert checked >= 10


@pytest.mark.parametrize("run", GOLD["simulate"], ids=[" ".join(r["argv"]) for r in GOLD["simulate"]])
def test_simulate_matches_reference(run, tmp_path, capsys):
    """`simulate` (host code over the bit-exact simulator port): the four files,
    stderr and exit code equal to the reference CLI's."""
    from paper_2203_15561_b200 import cli
    prefix = str(tmp_path / "s")
    code = cli.main(["simulate", *run["argv"], "--out-prefix", prefix])
    err = capsys.readouterr().err
    files = {}
    for suffix in ("ref.fasta", "reads.fasta", "truth.tsv", "pairs.tsv"):
        path = f"{prefix}_{suffix}"
        if os.path.exists(path):
            files[suffix] = open(path, encoding="utf-8").read()
    assert (code, err, files) == (run["code"], run["err"], run["files"])


def test_groundtruth_symbol_ids():
    """The DP kernel's inputs: per-character ids in the batch layout, ACGT at
    0..3, every other character its own id (so 'N' matches 'N', 'N' != 'X')."""
    from paper_2203_15561_b200.groundtruth import _symbol_batch
    pairs = [("ACGTN", "NXAC"), ("é#", ""), ("", "TT")]
    b = _symbol_batch(pairs)
    assert b.pat_len.tolist() == [5, 2, 0] and b.txt_len.tolist() == [4, 0, 2]
    seq = "".join(p + t for p, t in pairs)
    ids = b.codes[:len(seq)].tolist()
    assert ids[:4] == [0, 1, 2, 3]
    for x, cx in zip(seq, ids):
        for y, cy in zip(seq, ids):
            assert (x == y) == (cx == cy)
    lp = fmt.parse_pairs_bytes(b"a\tACGTN\tNXac\n", symbols=True)
    assert lp.syms[:9].tolist()[:4] == [0, 1, 2, 3]
    s = lp.syms[:9].tolist()
    assert s[4] == s[5] and s[5] != s[6] and s[7:9] == [0, 1]  # N == N, N != X, 'ac' -> A, C
