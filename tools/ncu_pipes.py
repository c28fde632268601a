"""Executed SASS instructions of one kernel in an ncu report, grouped by opcode and by pipe.
usage: ncu_pipes.py report.ncu-rep section_index|kernel_regex input_bytes
(the source page lists each kernel more than once: prefer a kernel-name regex)"""
import collections, csv, io, re, subprocess, sys
rep, sel, nbytes = sys.argv[1], sys.argv[2], float(sys.argv[3])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
secs, names, cur = [], [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []; secs.append(cur); names.append(r[1] if len(r) > 1 else "")
    elif cur is not None:
        cur.append(r)
if sel.isdigit():
    sec = secs[int(sel)]
else:
    sec = secs[next(i for i, nm in enumerate(names) if re.search(sel, nm))]
h = sec[0]; ix = {k: i for i, k in enumerate(h)}
ops = collections.Counter()
for r in sec[1:]:
    if len(r) != len(h): continue
    src = r[ix["Source"]].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", src)
    if not m: continue
    ex = float(r[ix["Instructions Executed"]] or 0)
    ops[m.group(2) + (m.group(3) or "")] += ex
def pipe(op):
    b = op.split(".")[0]
    if b in ("IMAD", "FFMA", "FMUL", "FADD", "HFMA2", "IMUL"): return "fma"
    if b in ("LOP3", "SHF", "PRMT", "IADD3", "ISETP", "SEL", "LEA", "FSEL", "PLOP3", "MOV", "VIADD", "IABS", "BMSK", "SGXT", "P2R", "R2P", "FMNMX", "IMNMX", "VIMNMX", "FSETP", "LOP", "SHL", "SHR", "CS2R", "S2R") : return "alu"
    if b in ("LDS", "STS", "SHFL", "LDSM", "ATOMS", "LD", "ST", "LDG", "STG", "ATOMG", "RED", "SYNCS", "UBLKCP", "LDC", "S2UR", "MEMBAR", "ATOM", "REDUX"): return "mem"
    if b in ("POPC", "FLO", "BREV", "MUFU", "I2F", "F2I"): return "xu"
    if b.startswith("U"): return "uniform"
    return "ctrl"
byp = collections.Counter()
for op, v in ops.items(): byp[pipe(op)] += v
tot = sum(ops.values())
print("warp-instr %.3g, lane-instr/B %.2f" % (tot, tot * 32 / nbytes))
for p, v in byp.most_common(): print("  %-8s %6.2f /B  %5.1f%%" % (p, v * 32 / nbytes, 100 * v / tot))
for op, v in ops.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 25):
    print("  %-28s %-7s %6.2f /B" % (op, pipe(op), v * 32 / nbytes))
