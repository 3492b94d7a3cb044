"""Group SASS instructions of an ncu report into runs with equal execution count (basic blocks)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; ai, si, ei = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
data = [(int(r[ai], 16), int(r[ei] or 0), r[si].strip()) for r in rows[2:] if len(r) > ei]
tot = sum(d[1] for d in data)
blocks = []; cur = None
for a, e, s in data:
    if cur and e == cur[2] and e > 0:
        cur[1] = a; cur[3] += e; cur[4].append(s)
    else:
        cur = [a, a, e, e, [s]]; blocks.append(cur)
blocks.sort(key=lambda b: -b[3])
for b in blocks[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    ops = [x.split()[0] if not x.startswith("@") else x.split()[1] for x in b[4]]
    print(f"{hex(b[0])[-5:]}-{hex(b[1])[-5:]} n={len(b[4]):3d} x{b[2]:>11d} {100*b[3]/tot:5.1f}%  {' '.join(ops)[:150]}")
