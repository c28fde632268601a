"""Write the committed profiles of a round-2 measurement (tools/r2_full.sh TAG outputs in
gpurun_out/): the bench lines (two-pass default, single-pass, reference arm), the ncu launch
list with per-kernel shares of the step, the DRAM traffic of the two planned transcoders
MEASURED at the bench size (8 GiB config 4, one ncu pass over the bench command), and the
full-set capture summary (sections, stall reasons, instruction mix, per-source-line
instructions and stalls) of the planned transcoders at 1 GiB.
usage: python tools/r2_profiles.py TAG "build description" """
import csv
import io
import json
import os
import shutil
import subprocess
import sys

tag, desc = sys.argv[1], sys.argv[2]
G, P = "gpurun_out", "profiles"
py = sys.executable


def run(*a, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([py] + list(a), capture_output=True, text=True, env=e).stdout


def last_json(path):
    lines = [ln for ln in open(path) if ln.startswith("{")]
    return lines[-1] if lines else "{}\n"


for src, dst in ((f"bench_{tag}.log", "bench_default"), (f"bench_chained_{tag}.log", "bench_chained"),
                 (f"bench_ref_{tag}.log", "bench_reference")):
    if os.path.exists(f"{G}/{src}"):
        with open(f"{P}/{tag}_{dst}.json", "w") as f:
            f.write(last_json(f"{G}/{src}"))

# ncu launch list -> per kernel launches, mean duration, share of the timed steps
rows = list(csv.reader(open(f"{G}/launches_{tag}.csv")))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = {}
order = []
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    per.setdefault(name, []).append(float(r[vi].replace(",", "")))
    order.append(name)
with open(f"{P}/{tag}_ncu_launches.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 40, command:\n"
            "# python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-per-op "
            "--no-per-config (8 GiB config 4, 1 GPU, two-pass step);\n"
            f"# build {tag} ({desc}).  Per-launch times are cold-cache and serialised: compare "
            "SHARES.\n# The first k_transcode<U8PolT> launch is bench.py's untimed setup pass (it "
            "learns the UTF-16 length); every step = k_plan8 + k_transcode_planned<U8PolT> + "
            "k_plan16 + k_transcode_planned<U16PolT>.\n\n")
    step = {k: v for k, v in per.items() if not k.startswith(("k_transcode<U8PolT", "ug::k_transcode<ug::U8PolT"))}
    tot = sum(sum(v) / len(v) for v in step.values())
    f.write(f"{'kernel':48s} {'launches':>8s} {'avg_us':>10s} {'step_share':>10s}\n")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
        avg = sum(v) / len(v) / 1e3
        share = (sum(v) / len(v) / tot) if k in step else float("nan")
        f.write(f"{k:48s} {len(v):8d} {avg:10.1f} {share:10.3f}\n")
    f.write("\nlaunch order: " + ", ".join(n.split("::")[-1] for n in order) + "\n")

# DRAM traffic at the bench size
rows = list(csv.reader(open(f"{G}/traffic8g_{tag}.csv")))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
m = {}
for r in rows[hdr + 1:]:
    if len(r) > vi:
        m.setdefault((r[ii], r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
bench = json.loads(last_json(f"{G}/bench_{tag}.log"))
n8, n16 = bench["config"]["bytes_utf8"], bench["config"]["units_utf16"]
tr = json.load(open(f"{P}/traffic.json")) if os.path.exists(f"{P}/traffic.json") else {}
tr = {k: v for k, v in tr.items() if not k.startswith("k_transcode_planned")}
for (i, k), d in m.items():
    fwd = "U8PolT" in k
    key = "k_transcode_planned<U8Pol>" if fwd else "k_transcode_planned<U16Pol>"
    inp = n8 if fwd else 2 * n16
    tr[key] = {"input_bytes": inp, "dram_read_bytes": d["dram__bytes_read.sum"],
               "dram_write_bytes": d["dram__bytes_write.sum"],
               "dram_bytes_per_input_byte": (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / inp,
               "algorithmic_bytes_per_input_byte": (n8 + 2 * n16) / inp,
               "lane_instr_per_input_byte": round(32 * d["smsp__inst_executed.sum"] / inp, 2),
               "capture": f"profiles/{tag}_ncu_traffic.txt",
               "config": "MEASURED at the bench size: ncu --metrics dram__bytes_read.sum,"
                         "dram__bytes_write.sum over bench.py --steps 2 --warmup 1 (8 GiB config 4)"}
tr["note_planned"] = ("k_transcode_planned<*>: traffic measured per launch at the bench size "
                      f"({tag}); the other entries are round-1 1 GiB captures")
json.dump(tr, open(f"{P}/traffic.json", "w"), indent=1)
shutil.copy(f"{G}/traffic8g_{tag}.csv", f"{P}/{tag}_ncu_traffic.txt")

# full capture summary
rep = f"{G}/full_{tag}.ncu-rep"
lib = f"{G}/lib_{tag}.so"
summ = run("tools/ncu_summary.py", rep, "20")
pipes_f = run("tools/ncu_pipes.py", rep, "planned<ug::U8PolT", "1073741824")
pipes_r = run("tools/ncu_pipes.py", rep, "planned<ug::U16PolT", "1409338390")
lines_f = run("tools/sass_lines.py", rep, "planned<ug::U8PolT", lib, "1073741824", "30",
              env={"STALLS": "25"})
lines_r = run("tools/sass_lines.py", rep, "planned<ug::U16PolT", lib, "1409338390", "30",
              env={"STALLS": "25"})
with open(f"{P}/{tag}_ncu_full_transcoders.txt", "w") as f:
    f.write("# ncu --set full --clock-control none --import-source on, tools/ncu_one.py c4 1024 "
            "(OPS=pfwd,prev: plan + planned forward, plan + planned reverse on 1 GiB of config-4 "
            f"text); B200, driver 580.159; build {tag} ({desc})\n\n## sections and stalls "
            "(forward first, then reverse)\n" + summ +
            "\n## executed instruction mix, forward (per UTF-8 input byte)\n" +
            "\n".join(pipes_f.splitlines()[:30]) +
            "\n\n## executed instruction mix, reverse (per UTF-16 input byte)\n" +
            "\n".join(pipes_r.splitlines()[:30]) +
            "\n\n## per source line (tools/sass_lines.py), forward\n" + lines_f +
            "\n## per source line, reverse\n" + lines_r)
print("written:", sorted(x for x in os.listdir(P) if x.startswith(tag)))
