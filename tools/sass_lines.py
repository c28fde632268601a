"""Per-source-line executed lane-instructions of one kernel from an ncu report (SASS page) joined
with nvdisasm line info of the SAME library build (checked instruction by instruction).

usage: sass_lines.py report.ncu-rep kernel_regex lib.so input_bytes [top]
Prints lane-instructions per input byte per source line, and per (file, function) region.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kre, lib, nbytes = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 60

raw = subprocess.run(["ncu", "-i", os.path.abspath(rep), "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, cwd=tempfile.gettempdir()).stdout
blocks, cur = [], None
for row in csv.reader(io.StringIO(raw)):
    if not row:
        continue
    if row[0] == "Kernel Name":
        cur = {"name": row[1], "rows": []}
        blocks.append(cur)
    elif row[0] == "Address":
        cur["hdr"] = row
    elif cur is not None and row[0].startswith("0x"):
        cur["rows"].append(row)
blk = [b for b in blocks if re.search(kre, b["name"])]
if not blk:
    sys.exit("no kernel matches: " + ", ".join(b["name"] for b in blocks))
b = blk[0]
hdr = b["hdr"]
ti = hdr.index("Thread Instructions Executed")
rows = [(int(r[0], 16), r[1].strip(), float(r[ti] or 0)) for r in b["rows"]]
base = rows[0][0]

# nvdisasm of the matching function
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
want = None
lineinfo = {}
texts = {}
for f in sorted(os.listdir(tmp)):
    if not f.endswith(".cubin"):
        continue
    dis = subprocess.run(["nvdisasm", "--print-line-info", "-c", os.path.join(tmp, f)],
                         capture_output=True, text=True).stdout
    fn, line = None, None
    for ln in dis.splitlines():
        m = re.match(r"^\s*\.text\.(\S+):", ln) or re.match(r"^\.text\.(\S+):", ln)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
        if m and fn:
            off = int(m.group(1), 16)
            lineinfo.setdefault(fn, {})[off] = line
            texts.setdefault(fn, {})[off] = m.group(2)
# pick the function whose instruction text matches the report's
best, score = None, -1
for fn, t in texts.items():
    s = sum(1 for a, txt, _ in rows[:400] if t.get(a - base, "").split()[:1] == txt.split()[:1])
    if s > score:
        best, score = fn, s
print(f"kernel {b['name']}\nfunction {best} (opcode match {score}/{min(400, len(rows))})")
li = lineinfo[best]
per_line = collections.Counter()
per_op = collections.Counter()
tot = 0.0
for a, txt, n in rows:
    ln = li.get(a - base, ("?", 0))
    per_line[ln] += n
    op = txt.split()[0] if not txt.startswith("@") else txt.split()[1]
    per_op[op.split(".")[0]] += n
    tot += n
print(f"total {tot / nbytes:.2f} lane-instr per input byte")
src_cache = {}


def src(fl):
    f, l = fl
    if f not in src_cache:
        p = None
        for d in ("paper_2111_08692_b200/csrc", "."):
            if os.path.exists(os.path.join(d, f)):
                p = os.path.join(d, f)
        src_cache[f] = open(p).read().splitlines() if p else []
    s = src_cache[f]
    return s[l - 1].strip()[:70] if 0 < l <= len(s) else ""


for fl, n in per_line.most_common(top):
    print(f"{n / nbytes:6.2f}/B {100 * n / tot:5.1f}%  {fl[0]}:{fl[1]:<5} {src(fl)}")
print("-- opcodes")
for op, n in per_op.most_common(25):
    print(f"{n / nbytes:6.2f}/B  {op}")

if os.environ.get("LISTING"):
    # the SASS listing with per-instruction lane-instructions per input byte (hot only)
    thr = float(os.environ.get("LISTING"))
    for a, txt, n in rows:
        if n / nbytes >= thr:
            ln = li.get(a - base, ("?", 0))
            print(f"{a - base:6x} {n / nbytes:6.3f} {ln[0]}:{ln[1]:<5} {txt}")

if os.environ.get("STALLS"):
    # warp-stall samples per source line, with the top reasons
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    idx = {c: hdr.index(c) for c in cols}
    si = hdr.index("Warp Stall Sampling (All Samples)")
    per = collections.defaultdict(lambda: collections.Counter())
    tot_s = 0.0
    for r in b["rows"]:
        a = int(r[0], 16)
        ln = li.get(a - base, ("?", 0))
        n = float(r[si] or 0)
        per[ln]["_all"] += n
        tot_s += n
        for c, i in idx.items():
            per[ln][c] += float(r[i] or 0)
    print(f"-- stall samples per line (total {tot_s:.0f})")
    for ln, cn in sorted(per.items(), key=lambda kv: -kv[1]["_all"])[:int(os.environ.get("STALLS"))]:
        reasons = sorted(((v, k[6:]) for k, v in cn.items() if k != "_all" and v), reverse=True)[:3]
        print(f"{100 * cn['_all'] / tot_s:5.1f}%  {ln[0]}:{ln[1]:<5} {src(ln)[:50]:50} " +
              " ".join(f"{k}={100 * v / cn['_all']:.0f}%" for v, k in reasons))
