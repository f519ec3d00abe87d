"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the GEMM launches in an
ncu --set full capture -> profiles/ncu_traffic.json[config] (read by bench.py's roofline.traffic).

    python tools/ncu_traffic.py gpurun_out/r01_gemm_c2.ncu-rep c2
"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, cfg):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    per = []
    for r in rows[2:]:
        if "gemm" not in r[hdr.index("Kernel Name")]:
            continue
        per.append(float(r[ir]) * UNIT[units[ir]] + float(r[iw]) * UNIT[units[iw]])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "profiles", "ncu_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[cfg] = sum(per) / len(per)
    d[cfg + "_per_launch"] = per
    d[cfg + "_source"] = os.path.basename(rep)
    json.dump(d, open(path, "w"), indent=1)
    print(cfg, d[cfg])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
