"""Per-kernel SASS hot spots from an ncu report: python ncu_source_top.py REPORT REGEX [N]."""
import collections
import csv
import io
import subprocess
import sys


def main(rep, regex, n=25, skip=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                          "--launch-count", "1", "--launch-skip", str(skip), "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break  # only the first kernel section
        if len(r) == len(hdr) and r[0] != "Address":
            data.append(r)
    si = hdr.index("Source")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    print("samples", sum(int(r[ws] or 0) for r in data), "warp-inst", sum(int(r[ie] or 0) for r in data))
    ops = collections.Counter()
    for r in data:
        t = r[si].split()
        if t:
            op = t[1] if t[0].startswith("@") else t[0]
            ops[op.split(".")[0]] += int(r[ie] or 0)
    print(ops.most_common(24))
    for r in sorted(data, key=lambda r: -int(r[ws] or 0))[:n]:
        print(f"{int(r[ws]):6d} {int(r[ie]):10d}  {r[si][:80]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25,
         int(sys.argv[4]) if len(sys.argv) > 4 else 0)
