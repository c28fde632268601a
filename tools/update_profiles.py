"""Write the committed profiles of a measurement round from gpurun_out/ (tools/gpu_full.sh TAG
and tools/allcfg.sh TAG outputs): bench lines, ncu launch shares, full-capture summary, all-config
op table, and the per-kernel DRAM traffic / issue numbers in profiles/traffic.json.
usage: python tools/update_profiles.py TAG "build description" """
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

tag, desc = sys.argv[1], sys.argv[2]
G, P = "gpurun_out", "profiles"
py = sys.executable


def run(*a):
    return subprocess.run([py] + list(a), capture_output=True, text=True).stdout


shutil.copy(f"{G}/bench_full_{tag}.log", f"{P}/{tag}_bench_default.json")
shutil.copy(f"{G}/bench_ref_{tag}.log", f"{P}/{tag}_bench_reference.json")
with open(f"{P}/{tag}_ncu_launches.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 60, command:\n"
            "# python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline (8 GiB config 4, "
            f"1 GPU); build {tag} ({desc})\n# per-launch times are cold-cache and serialised: "
            "compare SHARES, not absolutes; step_share = avg launch / sum of the step's kernels\n\n")
    f.write(run("tools/launch_shares.py", f"{G}/launches_{tag}.csv"))
rep = f"{G}/full_{tag}.ncu-rep"
launches = run("tools/ncu_launches.py", rep)
summ = run("tools/ncu_summary.py", rep, "25")
rev = run("tools/ncu_pipes.py", rep, "0", "1409338390")
fwd = run("tools/ncu_pipes.py", rep, "2", "1073741824")
with open(f"{P}/{tag}_ncu_full_transcoders.txt", "w") as f:
    f.write("# ncu --set full --clock-control none --import-source on, bench.py --size-mib 1024 "
            "--steps 2 --warmup 1 (1 GiB of config-4 text), k_transcode launches 3-4 "
            "(k_transcode16 = utf16le_to_utf8, U8Pol = utf8_to_utf16le); B200, driver 580.159; "
            f"build {tag} ({desc})\n\n## per launch\n{launches}\n## sections, stalls, top SASS "
            f"(tools/ncu_summary.py; reverse first, then forward)\n{summ}\n## executed instruction "
            f"mix, reverse (tools/ncu_pipes.py, per UTF-16 input byte)\n"
            + "\n".join(rev.splitlines()[:32]) + "\n\n## executed instruction mix, forward (per "
            "UTF-8 input byte)\n" + "\n".join(fwd.splitlines()[:32]) + "\n")
# traffic / issue per kernel
busy = [float(x) / 100 for x in re.findall(r"Issue Slots Busy\s+([\d.]+) %", summ)]
lanes = [float(re.search(r"lane-instr/B ([\d.]+)", t).group(1)) for t in (rev, fwd)]
alu = [float(re.search(r"alu\s+([\d.]+) /B", t).group(1)) for t in (rev, fwd)]
rw = {}
for ln in launches.splitlines():
    k = "k_transcode16" if "k_transcode16" in ln else "k_transcode<U8Pol>"
    r = float(re.search(r"bytes_read.sum=([\d.]+)Gbyte", ln).group(1)) * 1e9
    w = float(re.search(r"bytes_write.sum=([\d.]+)Gbyte", ln).group(1)) * 1e9
    rw[k] = (r, w)
t = json.load(open(f"{P}/traffic.json"))
t["capture"] = f"{P}/{tag}_ncu_full_transcoders.txt"
for i, k in enumerate(("k_transcode16", "k_transcode<U8Pol>")):
    e = t[k]
    e["dram_read_bytes"], e["dram_write_bytes"] = rw[k]
    e["dram_bytes_per_input_byte"] = sum(rw[k]) / e["input_bytes"]
    e["lane_instr_per_input_byte"], e["alu_lane_instr_per_input_byte"] = lanes[i], alu[i]
    e["issue_slots_busy"] = busy[i]
json.dump(t, open(f"{P}/traffic.json", "w"), indent=1)
if os.path.exists(f"{G}/allcfg_{tag}.log"):
    rows = [json.loads(l) for l in open(f"{G}/allcfg_{tag}.log") if l.startswith("{")]
    json.dump(rows, open(f"{P}/{tag}_ops_allcfg.json", "w"), indent=1)
print(open(f"{P}/{tag}_ncu_launches.txt").read().splitlines()[-6:])
print({k: (round(t[k]["dram_bytes_per_input_byte"], 4), t[k]["lane_instr_per_input_byte"],
           t[k]["issue_slots_busy"]) for k in ("k_transcode16", "k_transcode<U8Pol>")})
