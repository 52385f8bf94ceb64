"""Sum 'Instructions Executed' per CUDA source line from an ncu source-page CSV
(ncu -i REP --page source --csv --print-source cuda,sass --kernel-name regex:K > f.csv):
python tools/ncu_lines.py f.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, hdr, tot = None, None, 0.0
by, src = collections.Counter(), {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    try:
        ln, ie = int(r[0]), float(r[7])
    except ValueError:
        continue
    by[(cur, ln)] += ie
    src[(cur, ln)] = r[1].strip()[:100]
    tot += ie
print(f"total {tot / 1e6:.2f} M warp-instructions")
for k, v in by.most_common(top):
    print(f"{v / 1e6:8.2f}M {100 * v / tot:5.1f}% {k[0]}:{k[1]}  {src[k]}")
