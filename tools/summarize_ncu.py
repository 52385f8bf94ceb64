"""Summaries of an ncu round capture for profiles/ (run here, on the merged gpurun_out/):

python tools/summarize_ncu.py TAG
  gpurun_out/launches_timed_TAG.csv  -> profiles/r01/launch_shares_timed_TAG.txt
  gpurun_out/full_TAG.ncu-rep        -> profiles/r01/kernel_metrics_TAG.txt, stalls_TAG.txt
and prints the mean dram bytes per k_render_bwd launch (profiles/traffic.json)."""
import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r01")

METRICS = [("duration", "gpu__time_duration.sum", "us"),
           ("dram_read", "dram__bytes_read.sum", "Mbyte"),
           ("dram_write", "dram__bytes_write.sum", "Mbyte"),
           ("dram_%peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
           ("regs", "launch__registers_per_thread", "register/thread"),
           ("occupancy_%", "sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
           ("issue_active_%", "smsp__issue_active.avg.pct_of_peak_sustained_active", "%"),
           ("threads_per_inst", "smsp__thread_inst_executed_per_inst_executed.ratio", ""),
           ("fma_pipe_%", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "%"),
           ("alu_pipe_%", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "%"),
           ("sm_throughput_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
           ("inst_executed", "smsp__inst_executed.sum", "")]


def short(name):
    return name.replace("(anonymous namespace)::", "").replace("gsr::", "").split("(")[0]


def launch_shares(tag):
    path = os.path.join(ROOT, "gpurun_out", f"launches_timed_{tag}.csv")
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            v = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v  # -> us
            a = agg[short(d["Kernel Name"])]
            a[0] += 1
            a[1] += v
    steps = 2
    total = sum(v[1] for v in agg.values())
    out = [f"# gpurun_out/launches_timed_{tag}.csv: {sum(v[0] for v in agg.values())} launches, total "
           f"{total / 1e3:.3f} ms over {steps} step(s) (ncu, serialised, warm caches (--cache-control none))",
           f"{'kernel':40s} {'launches':>8s} {'ms/step':>9s} {'share':>7s}"]
    for n, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{n[:40]:40s} {c:8d} {v / 1e3 / steps:9.3f} {100 * v / total:6.2f}%")
    open(os.path.join(OUT, f"launch_shares_timed_{tag}.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out[:14]))


def full(tag):
    rep = os.path.join(ROOT, "gpurun_out", f"full_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    met, stalls, bwd = [], [], []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = short(d["Kernel Name"])
        met.append(f"== {name}")
        for lab, key, unit in METRICS:
            val = d.get(key, "n/a")
            try:
                x = float(val.replace(",", ""))
                if key in hdr and (key.startswith("dram__bytes") or key == "gpu__time_duration.sum"):
                    x *= scale.get(units[hdr.index(key)], 1.0)  # -> Mbyte / us
                val = f"{x:.6f}" if not key.startswith("launch__") else f"{x:.0f}"
            except ValueError:
                pass
            met.append(f"   {lab:26s} {val:>14s} {unit}")
        ks = [k for k in hdr if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
        vals = sorted(((k, float(d[k])) for k in ks if d[k] not in ("", "n/a")), key=lambda kv: -kv[1])
        stalls.append(f"== {name}")
        for k, v in vals[:8]:
            stalls.append(f"   {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:22s} {v:.3f}")
        if "k_render_bwd" in name:
            mb = [float(d[k].replace(",", "")) * scale.get(units[hdr.index(k)], 1.0)
                  for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
            bwd.append(1e6 * sum(mb))
    open(os.path.join(OUT, f"kernel_metrics_{tag}.txt"), "w").write("\n".join(met) + "\n")
    open(os.path.join(OUT, f"stalls_{tag}.txt"), "w").write("\n".join(stalls) + "\n")
    if bwd:
        print("k_render_bwd dram bytes per launch (mean of %d): %d" % (len(bwd), sum(bwd) / len(bwd)))


if __name__ == "__main__":
    tag = sys.argv[1]
    launch_shares(tag)
    full(tag)
