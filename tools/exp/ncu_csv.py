"""Print (launch, metric, value) rows of an `ncu --csv` log (mixed stdout)."""
import csv
import sys

for path in sys.argv[1:]:
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    print("==", path)
    for row in rows[1:]:
        d = dict(zip(h, row))
        print(d["ID"], d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"])
