"""e2e host-pipeline sweep: chunk size x staging slots on config 4 (both host calls, pinned).
usage: python tools/e2e_sweep.py [size_mib]"""
import itertools
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2111_08692_b200 as ug  # noqa: E402
import synth  # noqa: E402

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
x = synth.generate_range("c4", 0, mib << 20)
n8 = x.size
hin = torch.from_numpy(x).pin_memory()
h16 = torch.empty(n8, dtype=torch.int16).pin_memory()
h8 = torch.empty(n8, dtype=torch.uint8).pin_memory()
torch.cuda.set_device(0)
ug.utf8_to_utf16le_host(hin[:1 << 20], h16)
for chunk, slots in itertools.product([8 << 20, 16 << 20, 32 << 20, 64 << 20], [3, 4, 6, 8]):
    ug.set_host_chunk(chunk)
    ug.set_host_slots(slots)
    best = 1e9
    for _ in range(2):
        t = time.perf_counter()
        r1 = ug.utf8_to_utf16le_host(hin, h16)
        r2 = ug.utf16le_to_utf8_host(h16[: r1.written], h8)
        best = min(best, time.perf_counter() - t)
        assert r1.error == 0 and r2 == (0, r1.written, n8)
    print(f"chunk {chunk >> 20:3d} Mi slots {slots:2d}: {best:.4f} s  "
          f"{(n8 + 2 * r1.written) / best / 1e9:.2f} GB/s", flush=True)
