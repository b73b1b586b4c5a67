"""Per-launch DRAM traffic of one kernel from an ncu metrics CSV
(dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum):

python tools/traffic.py gpurun_out/gemm_traffic.csv profiles/r01_gemm_traffic.json [kernel-regex]
"""
import re
import csv
import json
import sys


def main(src, dst, pattern=None):
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, d = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, names = {}, {}
    for r in d:
        per.setdefault(r[ii], {})[r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki].split("(")[0]
    launches = [{"id": k, "kernel": names[k], "dram_read": v["dram__bytes_read.sum"],
                 "dram_write": v["dram__bytes_write.sum"], "ns": v["gpu__time_duration.sum"]} for k, v in per.items()
                if pattern is None or re.search(pattern, names[k])]
    tot = sum(x["dram_read"] + x["dram_write"] for x in launches)
    out = {"source": src, "kernel_filter": pattern, "launches": len(launches), "traffic_bytes_per_launch": tot / max(1, len(launches)),
           "traffic_bytes_total": tot, "per_launch": launches,
           "note": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (cache-control all: cold L2 per launch)"}
    json.dump(out, open(dst, "w"), indent=1)
    print(f"{len(launches)} launches, {tot / 1e6:.1f} MB, {out['traffic_bytes_per_launch'] / 1e6:.2f} MB/launch")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
