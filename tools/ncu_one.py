"""Minimal driver for ncu captures: one config, N launches of the chosen ops (default both
transcoders) with the library at UG_LIB_OVERRIDE.  usage: ncu ... python tools/ncu_one.py c4 1024"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2111_08692_b200 as ug  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ops = (os.environ.get("OPS") or "fwd,rev").split(",")
dev = torch.device("cuda:0")
x = synth.generate_range(cfg, 0, mib << 20)
if cfg == "c3":
    u16 = torch.from_numpy(x.view(np.int16)).to(dev)
    t8 = torch.empty(ug.utf8_length_from_utf16le(u16), dtype=torch.uint8, device=dev)
    ug.utf16le_to_utf8(u16, t8)
else:
    t8 = torch.from_numpy(x).to(dev)
    u16 = torch.empty(ug.utf16_length_from_utf8(t8), dtype=torch.int16, device=dev)
    ug.utf8_to_utf16le(t8, u16)
o16 = torch.empty(t8.numel(), dtype=torch.int16, device=dev)
o8 = torch.empty(3 * u16.numel(), dtype=torch.uint8, device=dev)
plan8, plan16 = ug.plan_buffer(dev), ug.plan_buffer(dev)
lens = torch.zeros(2, dtype=torch.int64, device=dev)
res = ug.result_buffer(dev, 1)
for _ in range(2):
    if "pfwd" in ops:
        ug.utf16_length_from_utf8_plan_async(t8, lens, plan8)
        ug.utf8_to_utf16le_planned_async(t8, plan8, o16, res)
    if "prev" in ops:
        ug.utf8_length_from_utf16le_plan_async(u16, lens, plan16, len_off=8)
        ug.utf16le_to_utf8_planned_async(u16, plan16, o8, res)
    if "fwd" in ops:
        assert ug.utf8_to_utf16le(t8, o16).error == 0
    if "rev" in ops:
        assert ug.utf16le_to_utf8(u16, o8).error == 0
    if "v8" in ops:
        ug.utf8_validate(t8)
    if "v16" in ops:
        ug.utf16le_validate(u16)
torch.cuda.synchronize()
print("bytes", t8.numel(), 2 * u16.numel())
