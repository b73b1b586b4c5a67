"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys


def main(path, skip_frac=0.5):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    data = data[int(len(data) * skip_frac):]  # drop the warm-up step
    tot, cnt, allt = collections.defaultdict(float), collections.Counter(), 0.0
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")
        if "spin_kernel" in name:  # bench.py's GPU hold before the instrumented pass (torch.cuda._sleep)
            continue
        v = float(r[vi]) * scale.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
        allt += v
    print(f"launches {len(data)}  total {allt:.1f} us (cold-cache, serialised)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
        print(f"{k[:70]:70s} {cnt[k]:5d} {v:10.1f} us {100 * v / allt:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.5)
