"""Per-op timing of one libunigpu build on a config's synthetic input (development tool).

usage: UG_LIB_OVERRIDE=path/lib.so python tools/opbench.py [config] [size_mib] [reps]
Prints one JSON line: per op min / mean ms, input GB/s and algorithmic HBM GB/s.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2111_08692_b200 as ug  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
dev = torch.device("cuda:0")
if cfg == "c3":
    u16h = synth.generate_range(cfg, 0, mib << 20)
    u16 = torch.from_numpy(u16h.view(np.int16)).to(dev)
    n8 = ug.utf8_length_from_utf16le(u16)
    t8 = torch.empty(n8, dtype=torch.uint8, device=dev)
    r = ug.utf16le_to_utf8(u16, t8)
    assert r.error == 0
else:
    x = synth.generate_range(cfg, 0, mib << 20)
    t8 = torch.from_numpy(x).to(dev)
    n16 = ug.utf16_length_from_utf8(t8)
    u16 = torch.empty(n16, dtype=torch.int16, device=dev)
    r = ug.utf8_to_utf16le(t8, u16)
    assert r.error == 0 or os.environ.get("UG_LIB_OVERRIDE", "").find("_no") >= 0 or os.environ.get("UG_LIB_OVERRIDE", "").find("_both") >= 0 or os.environ.get("UG_LIB_OVERRIDE", "").find("nolb") >= 0 or os.environ.get("UG_LIB_OVERRIDE", "").find("bothp") >= 0 or os.environ.get("UG_LIB_OVERRIDE", "").find("both") >= 0 or os.environ.get("UG_LIB_OVERRIDE", "").find("slong") >= 0 or os.environ.get("UG_LIB_OVERRIDE", "").find("sshort") >= 0, r
n8, n16 = t8.numel(), u16.numel()
# big-endian copies of the same text for the UTF-16BE ops
u16be = u16.view(torch.uint8).view(-1, 2).flip(1).contiguous().view(torch.int16).view(-1)
o16 = torch.empty(n8, dtype=torch.int16, device=dev)
o8 = torch.empty(3 * n16, dtype=torch.uint8, device=dev)
plan8, plan16 = ug.plan_buffer(dev), ug.plan_buffer(dev)
lens = torch.zeros(2, dtype=torch.int64, device=dev)
resb = ug.result_buffer(dev, 1)
ug.utf16_length_from_utf8_plan_async(t8, lens, plan8)
ug.utf8_length_from_utf16le_plan_async(u16, lens, plan16, len_off=8)
ops = {
    "utf8_to_utf16le_planned": (lambda: ug.utf8_to_utf16le_planned_async(t8, plan8, o16, resb),
                                n8, n8 + 2 * n16),
    "utf16le_to_utf8_planned": (lambda: ug.utf16le_to_utf8_planned_async(u16, plan16, o8, resb),
                                2 * n16, 2 * n16 + n8),
    "utf8_to_utf16le_keyed": (lambda: ug.utf8_to_utf16le_keyed_planned_async(t8, plan8, o16, resb),
                              n8, n8 + 2 * n16),
    "plan8": (lambda: ug.utf16_length_from_utf8_plan_async(t8, lens, plan8), n8, n8),
    "plan16": (lambda: ug.utf8_length_from_utf16le_plan_async(u16, lens, plan16, len_off=8),
               2 * n16, 2 * n16),
    "utf8_validate": (lambda: ug.utf8_validate(t8), n8, n8),
    "utf8_to_utf16le": (lambda: ug.utf8_to_utf16le(t8, o16), n8, n8 + 2 * n16),
    "utf16le_validate": (lambda: ug.utf16le_validate(u16), 2 * n16, 2 * n16),
    "utf16le_to_utf8": (lambda: ug.utf16le_to_utf8(u16, o8), 2 * n16, 2 * n16 + n8),
    "utf16_length_from_utf8": (lambda: ug.utf16_length_from_utf8(t8), n8, n8),
    "utf8_length_from_utf16le": (lambda: ug.utf8_length_from_utf16le(u16), 2 * n16, 2 * n16),
    "utf8_to_utf16be": (lambda: ug.utf8_to_utf16be(t8, o16), n8, n8 + 2 * n16),
    "utf16be_to_utf8": (lambda: ug.utf16be_to_utf8(u16be, o8), 2 * n16, 2 * n16 + n8),
    "utf16be_validate": (lambda: ug.utf16be_validate(u16be), 2 * n16, 2 * n16),
}
only = os.environ.get("OPS")
res = {"lib": os.path.basename(os.environ.get("UG_LIB_OVERRIDE", "libunigpu.so")), "cfg": cfg,
       "mib": mib}
peak = 6452.5
for name, (fn, nin, alg) in ops.items():
    if only and name not in only.split(","):
        continue
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    mn = min(ts)
    res[name] = {"min_ms": round(mn, 4), "mean_ms": round(sum(ts) / len(ts), 4),
                 "in_gbs": round(nin / mn / 1e6, 1), "hbm_gbs": round(alg / mn / 1e6, 1),
                 "frac": round(alg / mn / 1e6 / peak, 4)}
print(json.dumps(res))
