"""Executed-instruction histogram by opcode (lane-ops per input byte) for one kernel of an ncu
report.  usage: ncu_ops.py report.ncu-rep input_bytes [kernel_index]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, nbytes = sys.argv[1], float(sys.argv[2])
kidx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
sec = sections[kidx]
h = sec["rows"][0]
ix = {k: i for i, k in enumerate(h)}
op = collections.Counter()
tot = 0
for r in sec["rows"][1:]:
    if len(r) != len(h):
        continue
    ex = float(r[ix["Instructions Executed"]] or 0)
    tot += ex
    src = re.sub(r"^@!?U?P\w+\s+", "", r[ix["Source"]].strip())
    op[src.split()[0] if src else "?"] += ex
print(sec["name"], f"total {tot:.0f} warp-instr = {tot * 32 / nbytes:.1f} lane-ops/byte")
for k, v in op.most_common(25):
    print(f"  {k:22s} {100 * v / tot:5.1f}%  {v * 32 / nbytes:6.2f}/byte")
