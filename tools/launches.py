"""Print kernel durations (ms) from an `ncu --metrics gpu__time_duration.sum --csv` log."""
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    print(path, [(r[ki][:16], round(float(r[vi]) / 1e6, 2)) for r in rows[1:]])
