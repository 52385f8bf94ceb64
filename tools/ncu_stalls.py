"""Per-kernel stall breakdown (warps stalled per issue-active cycle) from an ncu report:
python tools/ncu_stalls.py REP.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
pre = "smsp__average_warps_issue_stalled_"
for r in rows[2:]:
    print(r[h.index("Kernel Name")][:60])
    it = []
    for i, k in enumerate(h):
        if k.startswith(pre) and k.endswith("_per_issue_active.ratio"):
            try:
                it.append((float(r[i]), k[len(pre):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("   " + "  ".join(f"{n}={v:.2f}" for v, n in sorted(it, reverse=True)[:10]))
