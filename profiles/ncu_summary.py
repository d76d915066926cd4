"""Summarise an ncu report: headline metrics, stall reasons and hottest source lines.

    python profiles/ncu_summary.py <report.ncu-rep> [n_lines]
"""
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def details(rep):
    r = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = r[0]
    si, ni, ui, vi = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
            "Executed Ipc Active", "Registers Per Thread", "Achieved Occupancy",
            "Theoretical Occupancy", "Block Size", "Grid Size", "Warp Cycles Per Issued Instruction",
            "Dynamic Shared Memory Per Block", "L2 Hit Rate", "Issue Slots Busy")
    out = []
    for x in r[1:]:
        if x[ni] in keep:
            out.append(f"  {x[ni]}: {x[vi]} {x[ui]}")
    return out


def raw(rep):
    r = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, u, v = r[0], r[1], r[2]
    want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    return [f"  {k}: {v[h.index(k)]} {u[h.index(k)]}" for k in want if k in h]


def source(rep, n):
    r = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    cur, hdr, rows = None, None, []
    for x in r:
        if x and x[0] == "File Path":
            cur = x[1].split("/")[-1]
        elif x and x[0] == "Line No":
            hdr = x
        elif hdr and len(x) > 5 and x[2] == "-":
            d = dict(zip(hdr, x))
            rows.append((cur, x[0], x[1].strip()[:80], int(x[4] or 0), d))
    tot = sum(x[3] for x in rows) or 1
    stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: sum(int(x[4].get(c, 0) or 0) for x in rows) for c in stalls}
    out = ["  stall mix: " + ", ".join(f"{k[6:]} {100 * v / tot:.0f}%" for k, v in
                                     sorted(agg.items(), key=lambda kv: -kv[1])[:6])]
    for x in sorted(rows, key=lambda x: -x[3])[:n]:
        out.append(f"  {100 * x[3] / tot:5.1f}%  {x[0]}:{x[1]}  {x[2]}")
    return out


if __name__ == "__main__":
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    print(rep)
    print("\n".join(details(rep) + raw(rep) + source(rep, n)))
