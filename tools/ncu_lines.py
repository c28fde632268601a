"""Executed instructions per CUDA source line: joins an ncu report's SASS page (per-address
execution counts) with nvdisasm --print-line-info of the same build.
usage: ncu_lines.py report.ncu-rep kernel_substring section_index input_bytes [lib.so]"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, ksub, sidx, nbytes = sys.argv[1], sys.argv[2], int(sys.argv[3]), float(sys.argv[4])
COL = os.environ.get("COL", "Instructions Executed")  # e.g. COL=stall_barrier
FN = os.environ.get("FN", "")  # extra mangled-name filter for templates, e.g. FN=ILb0E (LE)
lib = sys.argv[5] if len(sys.argv) > 5 else "paper_2111_08692_b200/libunigpu.so"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines = {}
for cub in glob.glob(os.path.join(tmp, "kernels*.cubin")):
    dis = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True, text=True).stdout
    cur_fn, cur_line = None, None
    for ln in dis.splitlines():
        m = re.match(r"^\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+\S", ln)
        if m and cur_fn and ksub in cur_fn and FN in cur_fn:
            lines[int(m.group(1), 16)] = cur_line
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        secs.append(cur)
    elif cur is not None:
        cur.append(r)
sec = secs[sidx]
h = sec[0]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in sec[1:] if len(r) == len(h)]
base = int(data[0][ix["Address"]], 16)
agg = collections.Counter()
tot = 0
for r in data:
    ex = float(r[ix[COL]] or 0)
    tot += ex
    agg[lines.get(int(r[ix["Address"]], 16) - base, "?")] += ex
src_cache = {}
def src(key):
    f, l = key.rsplit(":", 1)
    for d in ("paper_2111_08692_b200/csrc",):
        p = os.path.join(d, f)
        if os.path.exists(p):
            if p not in src_cache:
                src_cache[p] = open(p).read().splitlines()
            return src_cache[p][int(l) - 1].strip()[:70]
    return ""
print(f"total {tot * 32 / nbytes:.1f} lane-ops/byte")
for k, v in agg.most_common(int(sys.argv[6]) if len(sys.argv) > 6 else 45):
    print(f"{v * 32 / nbytes:6.2f}/B {100 * v / tot:5.1f}%  {k:18s} {src(k) if k != '?' else ''}")
