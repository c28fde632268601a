"""Per-launch key metrics from an ncu report (one line per profiled kernel launch)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units, data = rows[0], rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
for r in data:
    name = r[ix["Kernel Name"]][:50]
    out = [name]
    for k in keys:
        if k in ix:
            out.append(f"{k.split('__')[1][:28]}={r[ix[k]]}{units[ix[k]]}")
    print(" | ".join(out))
