"""Summarise an ncu report: key SOL metrics and the top SASS lines by stall samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
h = det[0]
want = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread",
        "Executed Instructions", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "L2 Hit Rate", "Theoretical Occupancy", "Block Limit Registers", "Block Limit Shared Mem",
        "Grid Size", "Avg. Active Threads Per Warp", "Branch Efficiency")
for row in det[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:<40} {d['Metric Value']} {d['Metric Unit']}")
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
if raw:
    hh = raw[0]
    vals = raw[2] if len(raw) > 2 else raw[1]
    for k, v in zip(hh, vals):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                 "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                 "dram__throughput.avg.pct_of_peak_sustained_elapsed"):
            print(f"{k:<55} {v}")
sass = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
# the page holds one section per profiled kernel: take the first
h = sass[1]
data = []
for r in sass[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(h):
        data.append(r)
ix = {k: i for i, k in enumerate(h)}
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[S]] or 0) for r in data)
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = {}
for r in data:
    for k in stalls:
        agg[k] = agg.get(k, 0) + float(r[ix[k]] or 0)
print("stall totals:", sorted(((round(v / tot * 100, 1), k) for k, v in agg.items()), reverse=True)[:8])
for r in sorted(data, key=lambda r: -float(r[ix[S]] or 0))[:ntop]:
    sm = float(r[ix[S]] or 0)
    st = sorted(((float(r[ix[k]] or 0), k) for k in stalls), reverse=True)[:2]
    print(f"{r[ix['Address']][-5:]} {r[ix['Source']][:58]:<58} {100 * sm / tot:5.1f}% "
          f"ex={r[ix['Instructions Executed']]} {[(k[6:], int(v)) for v, k in st]}")
