"""Count rescans (flagged warps / tiles) on valid config-4 text with a UG_TRACE build."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2111_08692_b200 as ug  # noqa
import synth  # noqa
x = synth.generate_range("c4", 0, 64 << 20)
t8 = torch.from_numpy(x).cuda()
L = ctypes.CDLL(os.environ["UG_LIB_OVERRIDE"])
c = np.zeros(8, dtype=np.uint64)
print("validate", ug.utf8_validate(t8))
L.ug_debug_counters(ctypes.c_void_p(c.ctypes.data)); print("after validate", c)
o16 = torch.empty(t8.numel(), dtype=torch.int16, device="cuda")
print("transcode", ug.utf8_to_utf16le(t8, o16))
L.ug_debug_counters(ctypes.c_void_p(c.ctypes.data)); print("after transcode", c)
t, w = int(c[3]), int(c[4])
if c[2]:
    # bytes of the first flagged warp (tile t, warp w): 8 KiB tiles, 1 KiB per warp
    off = t * 8192 + w * 1024
    seg = x[off - 8: off + 1024 + 8]
    import oracle
    print("oracle on that region:", oracle.utf8_validate(seg))
