"""Debug helper: run utf8_validate / utf8_to_utf16le on small cases at several offsets and
print GPU vs oracle (used while developing; not part of the test suite)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2111_08692_b200 as ug  # noqa: E402

dev = torch.device("cuda:0")
import os
cases = [bytes.fromhex("dca520b9"), bytes.fromhex("dca520"), bytes.fromhex("41b9"),
         bytes.fromhex("b9"), bytes.fromhex("dca5"), bytes.fromhex("dca52041")]
if os.environ.get("UG_LIB_OVERRIDE"):
    cases = cases[:1]
for c in cases:
    a = np.frombuffer(c, dtype=np.uint8)
    ref = oracle.utf8_validate(a)
    for pad_after in (0, 64):
        for off in ((0, 2, 3) if os.environ.get("UG_LIB_OVERRIDE") else range(16)):
            big = np.full(off + a.size + pad_after, 0xAA, np.uint8)
            big[off:off + a.size] = a
            t = torch.from_numpy(big).to(dev)[off:off + a.size]
            v1 = ug.utf8_validate(t)
            v2 = ug.utf8_validate(t)
            out = torch.zeros(a.size, dtype=torch.int16, device=dev)
            x = ug.utf8_to_utf16le(t, out)
            if os.environ.get("UG_LIB_OVERRIDE"):
                torch.cuda.synchronize()
                print("off", off, "pad", pad_after, "v1", v1, "v2", v2, "xc", x, flush=True)
            if tuple(v1) != tuple(ref) or tuple(v2) != tuple(ref) or x[:2] != ref[:2]:
                print("MISMATCH", c.hex(), "off", off, "pad_after", pad_after, "gpu", v1, v2,
                      "xc", x, "ref", ref)
print("debug done")
