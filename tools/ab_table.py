"""Summarise tools/r2_ab.sh output: per (config, op) the best min_ms of each library."""
import collections
import json
import sys

best = collections.defaultdict(dict)
libs = []
for ln in open(sys.argv[1]):
    ln = ln.strip()
    if not ln.startswith("{"):
        continue
    d = json.loads(ln)
    lib = d["lib"]
    if lib not in libs:
        libs.append(lib)
    for k, v in d.items():
        if isinstance(v, dict) and "min_ms" in v:
            key = (d["cfg"], k)
            best[key][lib] = min(best[key].get(lib, 1e9), v["min_ms"])
print("cfg/op".ljust(28) + "".join(l[:18].rjust(20) for l in libs))
for key, m in best.items():
    b0 = m.get(libs[0])
    row = f"{key[0]}/{key[1]}".ljust(28)
    for l in libs:
        v = m.get(l)
        row += (f"{v:.4f} ({v / b0 - 1:+.1%})" if v and b0 else "-").rjust(20)
    print(row)
