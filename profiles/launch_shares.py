"""Per-kernel share of the timed region from an `ncu --metrics gpu__time_duration.sum --csv`
launch list (cold-cache, serialised: compare SHARES, not absolutes)."""
import collections
import csv
import re
import sys


def main(path, steps=1):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = None
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).split("::")[-1]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
        unit = r[ui]
    tot = sum(v[1] for v in agg.values())
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
    print(f"# {path}: {sum(v[0] for v in agg.values())} launches, total {tot * scale / 1e3:.3f} ms "
          f"over {steps} step(s) (ncu, serialised, cold caches)")
    print(f"{'kernel':40s} {'launches':>8s} {'ms/step':>9s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:40s} {n:8d} {t * scale / 1e3 / steps:9.3f} {100 * t / tot:6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
