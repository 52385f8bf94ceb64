"""Per-CUDA-line warp-stall samples and executed instructions from an ncu report
(--import-source on, -lineinfo): python ncu_lines.py REPORT KERNEL_REGEX [N]."""
import csv
import io
import subprocess
import sys


def main(rep, regex, n=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                          "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hi]
    ws, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    agg, cur = {}, None
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        if r[0]:
            cur = (int(r[0]), r[1].strip()) if r[0].isdigit() else None
            continue
        if cur is None or r[2] in ("", "..."):
            continue
        a = agg.setdefault(cur, [0, 0])
        a[0] += int(r[ws]) if r[ws].isdigit() else 0
        a[1] += int(r[ie]) if r[ie].isdigit() else 0
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"samples {ts}  warp-instructions {ti}")
    for (ln, src), (s, i) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
        print(f"{ln:5d} {100 * s / ts:5.1f}% {100 * i / ti:5.1f}%  {src[:88]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
