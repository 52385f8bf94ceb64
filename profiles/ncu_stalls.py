"""Per-kernel warp-stall breakdown (warps stalled per issue-active cycle, by reason)
from an `ncu --set full` report exported with `ncu -i X --page raw --csv`."""
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    pre = "smsp__average_warps_issue_stalled_"
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        print("==", r[hdr.index("Kernel Name")][:60])
        items = []
        for i, h in enumerate(hdr):
            if h.startswith(pre):
                try:
                    items.append((float(r[i].replace(",", "")), h[len(pre):].replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        for v, h in sorted(items, reverse=True)[:8]:
            print(f"   {h:24s} {v:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
