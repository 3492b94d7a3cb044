"""Golden fixtures for the command-line front-end and the file formats, made
by running the REFERENCE (`bitalign.cli.main`, `bitalign.io`) in the build
container (the checkout exists only here):

    python tests/golden/make_cli_golden.py

Output (committed): tests/golden/cli.json with
    files   name -> TSV text fed to the CLI / the pair reader
    runs    [{file, argv, code, out, err}]      `align`: reference stdout/stderr/exit code
    bench_runs  the same for `bench` (timing columns differ by nature)
    pairs   name -> read_pairs result ([id, pattern, text] rows) or the error text
    cigars  [ops, format_cigar, format_classic_cigar]
    parse   [text, parse_cigar result or "CigarError: ..."]
    fasta   name -> [text, read_fasta records or error, write_fasta(records, width 7)]
    dp      [pattern, text, global_distance, semiglobal_distance or null]
    simulate  [{argv, code, err, files: suffix -> content}]  `simulate` runs
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import random
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from bitalign import cli as rcli  # noqa: E402
from bitalign import io as rio  # noqa: E402
from bitalign import oracle as roracle  # noqa: E402


def _random_pairs(seed: int, count: int, max_len: int, rate: float) -> str:
    rng = random.Random(seed)
    rows = ["# random pairs"]
    for q in range(count):
        n = rng.randint(1, max_len)
        p = "".join(rng.choice("ACGT") for _ in range(n))
        t = []
        for c in p:
            r = rng.random()
            if r < rate / 3:
                t.append(rng.choice("ACGT"))
            elif r < 2 * rate / 3:
                t.append(c + rng.choice("ACGT"))
            elif r < rate:
                continue
            else:
                t.append(c)
        if q % 7 == 3:  # some lowercase and N
            p = p[:3].lower() + p[3:]
            t = ["N"] + t
        rows.append(f"q{q}\t{p}\t{''.join(t)}")
    return "\n".join(rows) + "\n"


FILES = {
    "basic": "# test pairs\np1\tACGT\tACGT\np2\tACGT\tAGGT\np3\tACGTACGTACGT\tACGTACGTACGT\n",
    "fail": "bad\tAAAAAAAAAAAA\tTTTTTTTTTTTT\nok\tACGT\tACGT\n",
    "newlines": "a\tacgt\tACGT\r\n  # indented comment\r\n\x1c \t\n\rb\tACGTN\tACNT\rc\tGATTACA\t\n"
                "d\tTTTT\tTTAT",
    "badcols": "a\tACGT\tACGT\n\nb\tACGT\n",
    "emptypat": "# x\na\t\tACGT\n",
    "toomany": "a\tAC\tAC\tAC\n",
    "unicode": "réad\tACGTß\tACGTSS\nplain\tacgt\tACGT\n",
    "random": _random_pairs(7, 60, 400, 0.12),
    "random_hi": _random_pairs(11, 40, 300, 0.35),
}

RUNS = [
    ("basic", []), ("basic", ["--stats"]), ("basic", ["--collapse-m"]),
    ("basic", ["--mode", "baseline"]),
    ("basic", ["--mode", "baseline", "--stats"]),
    ("fail", ["--w", "8", "--o", "2", "--k", "2"]),
    ("fail", ["--w", "8", "--o", "2", "--k", "2", "--stats"]),
    ("newlines", ["--stats"]), ("badcols", []), ("emptypat", []), ("toomany", []),
    ("unicode", ["--stats"]),
    ("random", []), ("random", ["--stats", "--w", "32", "--o", "12", "--k", "8",
                                "--priority", "IDSM"]),
    ("random", ["--collapse-m", "--w", "48", "--o", "18", "--k", "30", "--priority", "SMDI"]),
    ("random", ["--mode", "baseline", "--stats", "--w", "32", "--o", "12", "--k", "16"]),
    ("random_hi", ["--stats", "--k", "16"]), ("random_hi", ["--w", "16", "--o", "4", "--k", "4"]),
    ("basic", ["--k", "0"]), ("basic", ["--o", "64"]), ("basic", ["--priority", "MSIX"]),
    ("basic", ["--w", "0"]),
]


BENCH_FILES = {
    "bench_two": "q1\t" + "ACGTTGCA" * 16 + "\t" + "ACGTTGCA" * 16 + "\nq2\t" + "ACGTTGCA" * 16
                 + "\t" + ("ACGTTGCA" * 16)[:64] + "T" + ("ACGTTGCA" * 16)[65:] + "\n",
    "bench_one": "q1\t" + "ACGTTGCA" * 8 + "\t" + "ACGTTGCA" * 8 + "\n",
    "bench_sweep": "q1\t" + "ACGT" * 32 + "\t" + "ACGT" * 32 + "\n",
    "bench_n": "a\tACGTNNACGTTAGC\tACGTNNACGATAGC\nb\tNNNN\tNNNN\nc\tACGTACGTAC\tTTTT\n",
}
BENCH_RUNS = [
    ("bench_two", []), ("bench_one", []), ("bench_sweep", ["--sweep-k", "16,32,64"]),
    ("bench_n", ["--w", "8", "--o", "2"]), ("bench_n", ["--w", "8", "--o", "2", "--k", "2"]),
    ("random", ["--w", "32", "--o", "12", "--sweep-k", "8,32", "--priority", "IDSM"]),
    ("random", ["--oracle-cap", "20000"]), ("random", ["--oracle-cap", "0"]),
    ("random_hi", ["--w", "48", "--o", "18", "--sweep-k", "12,48"]),
    ("bench_one", ["--sweep-k", "a,b"]), ("bench_one", ["--sweep-k", "0"]),
]


SIM_RUNS = [
    ["--ref-len", "2000", "--count", "5", "--read-len", "300", "--seed", "11", "--emit-pairs"],
    ["--ref-len", "100", "--count", "0", "--read-len", "50", "--seed", "1"],
    ["--ref-len", "5000", "--count", "40", "--read-len", "97", "--sub", "0.1", "--ins", "0.2",
     "--del", "0.3", "--seed", "77", "--emit-pairs"],
    ["--ref-len", "30000", "--count", "12", "--read-len", "2500", "--sub", "0.01", "--ins", "0.07",
     "--del", "0.07", "--seed", "10003"],
    ["--ref-len", "100", "--count", "1", "--read-len", "50", "--sub", "0.9", "--ins", "0.2"],
    ["--ref-len", "10", "--count", "1", "--read-len", "50"],
    ["--ref-len", "0", "--count", "1", "--read-len", "5"],
    ["--ref-len", "100", "--count", "1", "--read-len", "50", "--del", "-0.5"],
]


def _run(path: str, argv: list[str], cmd: str = "align") -> dict:
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = rcli.main([cmd, "--pairs", path, *argv])
    return {"code": code, "out": out.getvalue(), "err": err.getvalue()}


def main() -> None:
    res: dict = {"files": {**FILES, **BENCH_FILES}, "runs": [], "bench_runs": [], "pairs": {},
                 "cigars": [], "parse": [], "fasta": {}}
    with tempfile.TemporaryDirectory() as tmp:
        for name, text in res["files"].items():
            path = os.path.join(tmp, name + ".tsv")
            with open(path, "w", encoding="utf-8", newline="") as fh:
                fh.write(text)
            with open(path, encoding="utf-8") as fh:
                try:
                    res["pairs"][name] = [[r.id, r.pattern, r.text] for r in rio.read_pairs(fh)]
                except rio.PairParseError as exc:
                    res["pairs"][name] = f"PairParseError: {exc}"
        for name, argv in RUNS:
            r = _run(os.path.join(tmp, name + ".tsv"), argv)
            r["err"] = r["err"].replace(tmp, "<tmp>")
            res["runs"].append({"file": name, "argv": argv, **r})
        for name, argv in BENCH_RUNS:
            r = _run(os.path.join(tmp, name + ".tsv"), argv, "bench")
            r["err"] = r["err"].replace(tmp, "<tmp>")
            res["bench_runs"].append({"file": name, "argv": argv, **r})
    for ops in ["", "=", "====XX=", "IIDD=X=X", "X" * 12 + "=" * 3 + "D"]:
        res["cigars"].append([ops, rio.format_cigar(ops), rio.format_classic_cigar(ops)])
    for text in ["", "2=1I", "10=2X3D", "3=0X", "=3", "3=Q4X", "3=4", "12", "3M", "x1=", "1=x",
                 "1=ab2X", "٣=", "2=²1X"]:
        try:
            res["parse"].append([text, rio.parse_cigar(text)])
        except rio.CigarError as exc:
            res["parse"].append([text, f"CigarError: {exc}"])
    fastas = {
        "two": ">r1 desc\nacgt\nNNAC\n\n>r2\nGG\n",
        "empty_seq": ">r1\n>r2\nAC\n",
        "no_header": "ACGT\n>r1\nAC\n",
        "empty_id": ">\nAC\n",
        "long": ">x\n" + "ACGTTGCA" * 5 + "\n",
    }
    for name, text in fastas.items():
        try:
            recs = rio.read_fasta(io.StringIO(text))
            buf = io.StringIO()
            rio.write_fasta(recs, buf, line_width=7)
            res["fasta"][name] = [text, [[r.id, r.sequence, sorted(r.nonstandard)] for r in recs],
                                  buf.getvalue()]
        except rio.MalformedFasta as exc:
            res["fasta"][name] = [text, f"MalformedFasta: {exc}", None]
    res["simulate"] = []
    for argv in SIM_RUNS:
        with tempfile.TemporaryDirectory() as tmp:
            prefix = os.path.join(tmp, "s")
            out, err = io.StringIO(), io.StringIO()
            with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
                code = rcli.main(["simulate", *argv, "--out-prefix", prefix])
            files = {}
            for suffix in ("ref.fasta", "reads.fasta", "truth.tsv", "pairs.tsv"):
                if os.path.exists(f"{prefix}_{suffix}"):
                    with open(f"{prefix}_{suffix}", encoding="utf-8") as fh:
                        files[suffix] = fh.read()
            res["simulate"].append({"argv": argv, "code": code, "err": err.getvalue(),
                                    "files": files})
    rng = random.Random(99)
    res["dp"] = []
    for q in range(120):
        alpha = rng.choice(["ACGT", "ACGT", "ACGTN", "ACGTNX#", "ACé"])
        p = "".join(rng.choice(alpha) for _ in range(rng.choice([0, 1, 5, 63, 64, 65, 130, 700])
                                                        if q % 4 else rng.randint(0, 300)))
        if rng.random() < 0.6:
            t = list(p)
            for _ in range(rng.randint(0, max(1, len(p) // 5))):
                if t and rng.random() < 0.5:
                    del t[rng.randrange(len(t))]
                else:
                    t.insert(rng.randint(0, len(t)), rng.choice(alpha))
            t = "".join(t)
        else:
            t = "".join(rng.choice(alpha) for _ in range(rng.randint(0, 300)))
        res["dp"].append([p, t, roracle.global_distance(p, t),
                          roracle.semiglobal_distance(p, t) if p else None])
    with open(os.path.join(HERE, "cli.json"), "w") as fh:
        json.dump(res, fh, indent=0)
    print("wrote", os.path.join(HERE, "cli.json"), len(res["runs"]), "runs")


if __name__ == "__main__":
    main()
