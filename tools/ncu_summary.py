"""Summarise an ncu report: key metrics, instruction mix, stall reasons (used for profiles/)."""
import collections
import csv
import io
import subprocess
import sys


def run(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    d = run(rep, "details")
    h = d[0]
    ni, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
            "Compute (SM) Throughput", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
            "Theoretical Occupancy", "Achieved Active Warps Per SM", "No Eligible", "Eligible Warps Per Scheduler",
            "Dynamic Shared Memory Per Block", "L2 Hit Rate", "Executed Instructions"]
    print("## key metrics")
    for row in d[1:]:
        if row[ni] in want:
            print("%-40s %12s %s" % (row[ni], row[vi], row[ui]))
    r = run(rep, "raw")
    h, v = r[0], r[2]
    print("## dram / fp64")
    for i, name in enumerate(h):
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__inst_executed_pipe_fp64.sum",
                    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                    "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"):
            print("%-70s %s %s" % (name, v[i], r[1][i]))
    print("## stall reasons (pc sampling, all samples)")
    st = [(name.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[i] or 0)) for i, name in enumerate(h)
          if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued")]
    tot = sum(x for _, x in st) or 1
    for name, x in sorted(st, key=lambda t: -t[1])[:12]:
        print("%-28s %6.2f%%" % (name, 100 * x / tot))
    s = run(rep, "source", ("--print-source=sass",))
    h = s[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    ops = collections.Counter()
    tot = 0
    for x in s[2:]:
        try:
            e = int(x[iE])
        except (ValueError, IndexError):
            continue
        t = x[iS].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        ops[op.split(".")[0]] += e
        tot += e
    print("## instruction mix (executed warp instructions)")
    for op, c in ops.most_common(16):
        print("%-10s %6.2f%%" % (op, 100 * c / tot))
    print("total", tot)


if __name__ == "__main__":
    main(sys.argv[1])
