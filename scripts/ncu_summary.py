"""Summarise an ncu report of k_eval: SOL, issue, occupancy, stalls, per-phase instruction
shares.  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep"""
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout


def main():
    det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
    h = det[0]
    want = ["Duration", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
            "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
            "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "Issued Instructions",
            "Avg. Active Threads Per Warp", "L2 Cache Throughput", "DRAM Throughput"]
    for row in det[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in want:
            print(f"{d['Metric Name']:34s} {d['Metric Value']} {d.get('Metric Unit','')}")
    raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    for vals in raw[2:]:
        row = dict(zip(hdr, vals))
        print(f"--- {row.get('Kernel Name', '?')[:70]}")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
                  for k, v in zip(hdr, vals)
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued")}
        tot = sum(stalls.values()) or 1
        print("stall samples:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in
                                           sorted(stalls.items(), key=lambda kv: -kv[1])[:8]))
        for k, v, u in zip(hdr, vals, units):
            if k in ("gpu__time_duration.sum",
                     "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                     "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                     "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"):
                print(f"{k:66s} {v} {u}")

if __name__ == "__main__":
    main()
