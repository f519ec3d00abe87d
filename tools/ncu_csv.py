"""Print per-launch metrics from an `ncu --csv --metrics ...` log (other output lines are skipped).
    python tools/ncu_csv.py <file.csv> [...]"""
import csv
import sys
from collections import OrderedDict


def parse(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    if not rows:
        return OrderedDict()
    hdr = rows[0]
    iid, ik, im, iv = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    out = OrderedDict()
    for r in rows[1:]:
        d = out.setdefault(r[iid], {"kernel": r[ik][:60]})
        d[r[im]] = r[iv]
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        for i, d in parse(p).items():
            print(i, {k: v for k, v in d.items()})
