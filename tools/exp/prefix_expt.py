"""Reverse kernel with recorded true prefixes replayed (no look-back chain, real placement)
vs the real look-back.  UG_LIB_OVERRIDE=build_variants/libunigpu_pfx.so python ... [cfg]"""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2111_08692_b200 as ug  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
dev = torch.device("cuda:0")
x = synth.generate_range(cfg, 0, 1 << 30) if cfg != "c3" else None
if cfg == "c3":
    u16 = torch.from_numpy(synth.generate_range(cfg, 0, 1 << 30).view(np.int16)).to(dev)
else:
    t8 = torch.from_numpy(x).to(dev)
    u16 = torch.empty(t8.numel(), dtype=torch.int16, device=dev)
    r = ug.utf8_to_utf16le(t8, u16)
    u16 = u16[: r.written]
o8 = torch.empty(3 * u16.numel(), dtype=torch.uint8, device=dev)
L = ug.lib
L.ug_debug_prefix_mode.argtypes = [ctypes.c_int]


def timeit(reps=10):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = ug.utf16le_to_utf8(u16, o8); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), r


res = {"cfg": cfg}
L.ug_debug_prefix_mode(0); timeit(2)
res["lookback_ms"], r0 = timeit()
ref = o8[: r0.written].clone()
L.ug_debug_prefix_mode(1); ug.utf16le_to_utf8(u16, o8); torch.cuda.synchronize()
L.ug_debug_prefix_mode(2); timeit(2)
res["replayed_ms"], r2 = timeit()
res["same_output"] = bool(torch.equal(o8[: r2.written], ref)) and tuple(r2) == tuple(r0)
L.ug_debug_prefix_mode(0)
print(json.dumps(res))
