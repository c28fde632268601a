"""Static SASS statistics per kernel of libunigpu.so (opcode histogram)."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2111_08692_b200/libunigpu.so"
pat = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f)
    c = collections.Counter(ops)
    print(f"{name[:70]:<70} {len(ops):6d} instr  " +
          " ".join(f"{k}:{v}" for k, v in c.most_common(12)))
