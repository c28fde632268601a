"""f2 file form throughput: write SIZE MiB of config-4 text to a file under DIR, then time
ug_utf8_to_utf16le_file and ug_utf16le_to_utf8_file (wall clock, input GB/s).  The input file
was just written, so it is read from the page cache, not the device: an upper bound for an
NVMe source.  usage: python tools/file_bench.py [SIZE_MIB] [DIR]"""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2111_08692_b200 as ug  # noqa: E402
import synth  # noqa: E402

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
d = sys.argv[2] if len(sys.argv) > 2 else tempfile.gettempdir()
a = synth.generate_range("c4", 0, mib << 20)
p8, p16, p8b = (os.path.join(d, f"ug_fb_{k}") for k in ("in8", "out16", "out8"))
with open(p8, "wb") as f:
    f.write(a.tobytes())
ug.utf8_to_utf16le_file(p8, p16)  # warm (CUDA context, staging)
t = time.perf_counter()
r = ug.utf8_to_utf16le_file(p8, p16)
t1 = time.perf_counter() - t
t = time.perf_counter()
r2 = ug.utf16le_to_utf8_file(p16, p8b)
t2 = time.perf_counter() - t
n16 = os.path.getsize(p16)
print({"size_mib": mib, "fwd": tuple(r), "rev": tuple(r2),
       "fwd_in_gbs": round(a.size / t1 / 1e9, 2), "rev_in_gbs": round(n16 / t2 / 1e9, 2),
       "fwd_s": round(t1, 3), "rev_s": round(t2, 3)})
assert r.error == 0 and r2.error == 0 and os.path.getsize(p8b) == a.size
for p in (p8, p16, p8b):
    os.unlink(p)
