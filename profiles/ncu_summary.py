"""Summarise an ncu --set full report (raw page CSV) into per-kernel key metrics."""
import csv
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("sm__inst_executed.sum", "inst_executed"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("sm__inst_executed_pipe_xu.sum", "xu_inst"),
    ("lts__t_sectors_op_red.sum", "l2_red_sectors"),
    ("lts__t_requests_op_red.sum", "l2_red_requests"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_%"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kn = hdr.index("Kernel Name")
    for r in data:
        print("==", r[kn][:90])
        for m, short in WANT:
            if m in hdr:
                i = hdr.index(m)
                print(f"   {short:18s} {r[i]:>18s} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
