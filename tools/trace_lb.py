"""Run utf8_to_utf16le once with a UG_TRACE build and summarise the look-back trace."""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2111_08692_b200 as ug  # noqa
import synth  # noqa
mib = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
x = synth.generate_range("c4", 0, mib << 20)
t8 = torch.from_numpy(x).cuda()
o16 = torch.empty(t8.numel(), dtype=torch.int16, device="cuda")
for _ in range(3):
    ug.utf8_to_utf16le(t8, o16)
torch.cuda.synchronize()
L = ctypes.CDLL(os.environ["UG_LIB_OVERRIDE"])
buf = np.zeros((1024, 64, 8), dtype=np.uint64)
L.ug_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
rc = L.ug_debug_trace(buf.ctypes.data, buf.nbytes)
nb = int((buf[:, 0, 1] > 0).sum())
b = buf[:nb].astype(np.int64)
t0 = b[:, 0, 1].min()
lb = (b[:, :, 2] - b[:, :, 1]) / 1000.0  # us
rounds = b[:, :, 3]
pw = (b[:, :, 5] - b[:, :, 4]) / 1000.0
valid = b[:, :, 1] > 0
print("ctas", nb, "rc", rc)
print("lookback us: mean %.2f p50 %.2f p90 %.2f max %.2f" % (lb[valid].mean(), np.median(lb[valid]), np.percentile(lb[valid], 90), lb[valid].max()))
ft = (b[:, :, 6] - b[:, :, 1]) / 1000.0
print("first poll done after us: mean %.2f p50 %.2f p90 %.2f" % (ft[valid].mean(), np.median(ft[valid]), np.percentile(ft[valid], 90)))
print("polls: mean %.1f p50 %.1f p90 %.1f" % (b[:, :, 7][valid].mean(), np.median(b[:, :, 7][valid]), np.percentile(b[:, :, 7][valid], 90)))
print("rounds: mean %.2f max %d hist %s" % (rounds[valid].mean(), rounds[valid].max(), np.bincount(rounds[valid].astype(int))[:10]))
v2 = b[:, :, 4] > 0
print("prefix wait us: mean %.2f p50 %.2f p90 %.2f" % (pw[v2].mean(), np.median(pw[v2]), np.percentile(pw[v2], 90)))
# iteration period
st = (b[:, 1:20, 1] - b[:, 0:19, 1]) / 1000.0
print("iteration period us (lookback start to start): mean %.2f" % st[st > 0].mean())
# a timeline for cta 0
for i in range(6):
    print("cta0 it%d tile %d lb_start %.2f lb_dur %.2f rounds %d pwait_start %.2f dur %.2f" % (
        i, b[0, i, 0], (b[0, i, 1] - t0) / 1000, lb[0, i], rounds[0, i], (b[0, i, 4] - t0) / 1000, pw[0, i]))
