"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*) into per-kernel
totals and shares of the captured steps (run here, no GPU needed).

    python tools/launch_summary.py gpurun_out/r01b_launches_c2.csv > profiles/r01b_launches_c2.txt

ncu serialises launches and replays each one cold (no L2 carry-over between kernels), so the
absolute times are not the bench's; the kernel SHARE of a step is what is compared with the
bench's live per-kernel event timing (kernels_ms_per_step).
"""
import collections
import csv
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9,
        "usecond": 1e-6, "msecond": 1e-3,
        "second": 1.0}


def main(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = collections.OrderedDict()
    for r in rows:
        lid = int(r["ID"])
        d = per.setdefault(lid, {"name": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
    agg = collections.OrderedDict()
    for d in per.values():
        base = re.sub(r"\(.*", "", d["name"]).replace("void ", "")
        a = agg.setdefault(base, {"n": 0, "t": 0.0, "rd": 0.0, "wr": 0.0, "grid": d["grid"], "block": d["block"]})
        a["n"] += 1
        a["t"] += d.get("gpu__time_duration.sum", 0.0)
        a["rd"] += d.get("dram__bytes_read.sum", 0.0)
        a["wr"] += d.get("dram__bytes_write.sum", 0.0)
    total = sum(a["t"] for a in agg.values())
    print(f"# ncu launch list {path.split('/')[-1]}: {len(per)} launches, cold-cache serialised replay")
    print(f"# {'kernel':60s} {'launches':>8s} {'mean ms':>9s} {'share':>7s} {'DRAM rd GB':>10s} {'DRAM wr GB':>10s}"
          f" {'GB/s':>8s}  grid x block")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        gbs = (a["rd"] + a["wr"]) / a["t"] / 1e9 if a["t"] else 0.0
        print(f"  {k[:60]:60s} {a['n']:8d} {a['t'] / a['n'] * 1e3:9.4f} {a['t'] / total:7.1%} "
              f"{a['rd'] / a['n'] / 1e9:10.4f} {a['wr'] / a['n'] / 1e9:10.4f} {gbs:8.0f}  {a['grid']} x {a['block']}")


if __name__ == "__main__":
    main(sys.argv[1])
