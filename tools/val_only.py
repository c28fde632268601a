"""Run each validator a few times on 256 MiB of config-4 text (for ncu captures)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2111_08692_b200 as ug  # noqa: E402
import synth  # noqa: E402
x = synth.generate_range("c4", 0, 256 << 20)
t = torch.from_numpy(x).cuda()
out = torch.empty(x.size, dtype=torch.int16, device="cuda")
r = ug.utf8_to_utf16le(t, out)
u = out[: r.written]
for _ in range(3):
    print(ug.utf8_validate(t), ug.utf16le_validate(u))
