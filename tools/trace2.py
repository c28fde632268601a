"""Per-iteration timeline of utf8_to_utf16le with a UG_TRACE build: usage trace2.py cfg mib"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2111_08692_b200 as ug  # noqa
import synth  # noqa
cfg = sys.argv[1]; mib = int(sys.argv[2])
x = synth.generate_range(cfg, 0, mib << 20)
t8 = torch.from_numpy(x).cuda()
o16 = torch.empty(t8.numel(), dtype=torch.int16, device="cuda")
for _ in range(3): ug.utf8_to_utf16le(t8, o16)
torch.cuda.synchronize()
L = ctypes.CDLL(os.environ["UG_LIB_OVERRIDE"])
buf = np.zeros((1024, 64, 12), dtype=np.uint64)
L.ug_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
L.ug_debug_trace(buf.ctypes.data, buf.nbytes)
b = buf.astype(np.int64)
nb = int((b[:, 0, 9] > 0).sum())
b = b[:nb]
t0 = b[:, 0, 8].min()
us = lambda v: (v - t0) / 1000.0
def stat(name, a):
    a = a[np.isfinite(a)]
    print("%-28s mean %6.2f p50 %6.2f p90 %6.2f" % (name, a.mean(), np.median(a), np.percentile(a, 90)))
it = slice(4, 40)
lw = (b[:, it, 9] - b[:, it, 8]) / 1000.0
an = (b[:, it, 10] - b[:, it, 9]) / 1000.0       # analyze + scan
em = (b[:, it, 11] - b[:, it, 10]) / 1000.0      # emit of i-2 (incl. prefix wait)
per = (b[:, 5:41, 8] - b[:, 4:40, 8]) / 1000.0   # iteration period
lbd = (b[:, it, 2] - b[:, it, 1]) / 1000.0       # look-back duration (from AGG)
pw = (b[:, it, 5] - b[:, it, 4]) / 1000.0
stat("iteration period", per.ravel()); stat("load wait", lw.ravel()); stat("analyze+scan", an.ravel())
stat("emit(i-2) incl wait", em.ravel()); stat("prefix wait (in emit)", pw.ravel()); stat("look-back from AGG", lbd.ravel())
print("rounds hist", np.bincount(b[:, it, 3].ravel().astype(int))[:8], "polls mean", b[:, it, 7].mean())
for i in range(3, 9):
    print("cta0 it%d t=%d load[%.2f,%.2f] agg %.2f end %.2f | lb[%.2f,%.2f] | pwait[%.2f,%.2f]" % (
        i, b[0, i, 0], us(b[0, i, 8]), us(b[0, i, 9]), us(b[0, i, 10]), us(b[0, i, 11]),
        us(b[0, i, 1]), us(b[0, i, 2]), us(b[0, i, 4]), us(b[0, i, 5])))
