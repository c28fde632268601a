"""Host<->device copy bandwidth on this box (pinned memory): H2D alone, D2H alone, both at once
on two streams.  The bound for the e2e (host-buffer) numbers.  Development tool."""
import json
import torch

N = 1 << 30
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_a = torch.empty(N, dtype=torch.uint8, device="cuda")
d_b = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


r = {"h2d_gbs": N / timed(lambda: d_a.copy_(h_in, non_blocking=True)) / 1e6,
     "d2h_gbs": N / timed(lambda: h_out.copy_(d_b, non_blocking=True)) / 1e6,
     "both_gbs_total": 2 * N / timed(both) / 1e6}
print(json.dumps({k: round(v, 1) for k, v in r.items()}))
