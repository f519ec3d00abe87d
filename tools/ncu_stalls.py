"""Stall breakdown and instruction counts of every kernel in an ncu --set full capture (plain text).

    python tools/ncu_stalls.py rep.ncu-rep [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys


def main(path, pat=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if pat and not re.search(pat, name):
            continue
        print("##", name[:100])
        for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
                  "dram__throughput.avg.pct_of_peak_sustained_elapsed"):
            if k in hdr:
                print(f"  {k:70s} {r[hdr.index(k)]}")
        st = []
        for i, k in enumerate(hdr):
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", k)
            if m:
                try:
                    st.append((float(r[i]), m.group(1)))
                except ValueError:
                    pass
        for v, n in sorted(st, reverse=True)[:10]:
            print(f"  stall {n:40s} {v:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
