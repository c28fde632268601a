"""Race check by repetition: run each transcoder (single-pass and two-pass) many times on the
same inputs (several start alignments, one input with an injected error) and require
bit-identical outputs and results every time.  Development tool: python tools/stress_repeat.py [iterations]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2111_08692_b200 as ug  # noqa: E402
import synth  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
dev = torch.device("cuda:0")
x = synth.generate_range("c4", 0, 256 << 20)
bad = x.copy()
synth.inject_utf8_error(bad, 100 << 20, (100 << 20) + 999, "surrogate", np.random.default_rng(9))
fails = 0
for name, buf in (("clean", x), ("error", bad)):
    for off in (0, 3, 8):
        big = torch.zeros(buf.size + 16, dtype=torch.uint8, device=dev)
        big[off:off + buf.size] = torch.from_numpy(buf).to(dev)
        t8 = big[off:off + buf.size]
        o16 = torch.empty(buf.size, dtype=torch.int16, device=dev)
        r0 = ug.utf8_to_utf16le(t8, o16)
        ref16 = o16[: r0.written].clone()
        u16 = ref16.clone()
        o8 = torch.empty(3 * u16.numel(), dtype=torch.uint8, device=dev)
        q0 = ug.utf16le_to_utf8(u16, o8)
        ref8 = o8[: q0.written].clone()
        for k in range(iters):
            o16.fill_(0x5A5A if k % 2 else 0)
            r = ug.utf8_to_utf16le(t8, o16)
            if tuple(r) != tuple(r0) or not torch.equal(o16[: r.written], ref16):
                fails += 1
                print("FORWARD MISMATCH", name, off, k, r, r0)
            o8.fill_(0x5A if k % 2 else 0)
            q = ug.utf16le_to_utf8(u16, o8)
            if tuple(q) != tuple(q0) or not torch.equal(o8[: q.written], ref8):
                fails += 1
                print("REVERSE MISMATCH", name, off, k, q, q0)
            # the two-pass (planned) path, the bench's: the same results and units every time
            o16.fill_(0 if k % 2 else 0x5A5A)
            rp, _ = ug.utf8_to_utf16le_two_pass(t8, o16)
            if tuple(rp) != tuple(r0) or not torch.equal(o16[: rp.written], ref16):
                fails += 1
                print("PLANNED FORWARD MISMATCH", name, off, k, rp, r0)
            o8.fill_(0 if k % 2 else 0x5A)
            qp, _ = ug.utf16le_to_utf8_two_pass(u16, o8)
            if tuple(qp) != tuple(q0) or not torch.equal(o8[: qp.written], ref8):
                fails += 1
                print("PLANNED REVERSE MISMATCH", name, off, k, qp, q0)
        print(name, off, "forward", tuple(r0), "reverse", tuple(q0), "ok" if not fails else fails)
print("STRESS", "PASS" if fails == 0 else f"FAIL {fails}")
