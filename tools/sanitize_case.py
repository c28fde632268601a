"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): both transcoders,
validators, length functions and the shard path on valid and invalid inputs, unaligned."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2111_08692_b200 as ug  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
valid_only = len(sys.argv) > 1 and sys.argv[1] == "valid"
a = np.frombuffer(synth.gen_chunk("mixed", "utf8", 100_003, 3, 0), dtype=np.uint8).copy()
cases = [a]
if not valid_only:
    b = a.copy()
    synth.inject_utf8_error(b, 40_000, 40_100, "surrogate", np.random.default_rng(1))
    c = a.copy()
    c[50_000:50_010] = 0x80
    cases += [b, c]
for x in cases:
    for off in (0, 5):
        big = torch.zeros(x.size + off + 64, dtype=torch.uint8, device=dev)
        t = big[off:off + x.size]
        t.copy_(torch.from_numpy(x))
        out16 = torch.zeros(x.size, dtype=torch.int16, device=dev)
        r = ug.utf8_to_utf16le(t, out16)
        ug.utf8_validate(t)
        ug.utf16_length_from_utf8(t)
        if r.error == 0:
            u = out16[: r.written]
            out8 = torch.zeros(3 * r.written, dtype=torch.uint8, device=dev)
            ug.utf16le_to_utf8(u, out8)
            ug.utf16le_validate(u)
            ug.utf8_length_from_utf16le(u)
        rec = ug.record_buffer(dev, 2)
        h = x.size // 2
        ug.utf8_to_utf16le_shard_async(t, 0, h, 0, 3, 0, out16, rec)
        ug.utf8_to_utf16le_shard_async(t, h, x.size - h, 3, 0, h, out16[h:], rec,
                                       rec_off=ug.RECORD_BYTES)
torch.cuda.synchronize()
print("sanitize case done", ug.launch_count())
