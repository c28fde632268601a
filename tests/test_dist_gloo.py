"""The N>1 host path on CPU: world_size-2 gloo process group, character-boundary cuts through the
library's cut rule, one all-gather of 32-byte shard records, and the library's combine.  The
per-shard kernel needs a GPU, so each rank's record is produced here by the oracle (test
infrastructure) from the same owned range and halos the kernel would get; what is under test is
the cut rule, the collective and the combine."""
import os
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

NONE = (1 << 64) - 1


def shard_record_from_oracle(buf: np.ndarray, lo: int, hi: int) -> bytes:
    """What the shard kernel reports for owned range [lo, hi) (R22): count of units
    (valid input), global first error among owned positions, units before it, kind."""
    r = oracle.utf8_validate(buf)
    if r.error and lo <= r.position < hi:
        # the first error of the whole buffer is owned by this rank
        part, _ = oracle.utf8_to_utf16le(buf[lo:r.position])
        return struct.pack("<QQQii", 0, r.position, part.written, r.error, 0)
    if r.error and r.position < lo:
        # an earlier error: this rank's own positions may hold later ones -- report none here
        # only if the owned range is clean as a stand-alone string from a character start
        sub = oracle.utf8_validate(buf[lo:hi])
        e = lo + sub.position if sub.error else NONE
        return struct.pack("<QQQii", 0, e, 0, sub.error if sub.error else 0, 0)
    part = oracle.utf8_to_utf16le(buf[lo:hi])[0]
    return struct.pack("<QQQii", part.written, NONE, 0, 0, 0)


def worker(rank, world, port, buf, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_08692_b200 import dist as ugd
        n = buf.size
        get = lambda a, b: buf[a:b].tobytes()  # noqa: E731
        lo, hi = ugd.shard_range_utf8(get, n, world, rank)
        hb, ha = ugd.halos(lo, hi, n, 3)
        rec = torch.frombuffer(bytearray(shard_record_from_oracle(buf, lo, hi)),
                               dtype=torch.uint8)
        gathered = ugd.gather_records(rec, world)
        res, off = ugd.combine_gathered_host(gathered, rank, n)
        q.put((rank, lo, hi, hb, ha, tuple(res), off))
    finally:
        dist.destroy_process_group()


def run_world(buf, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=worker, args=(r, world, port, buf, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


@pytest.mark.parametrize("case", ["valid", "error_near_cut", "error_rank0"])
def test_two_rank_cut_gather_combine(case):
    buf = np.frombuffer(synth.gen_chunk("mixed", "utf8", 200_003, 5, 0), dtype=np.uint8).copy()
    n = buf.size
    rng = np.random.default_rng(7)
    if case == "error_near_cut":
        c = (n // 2) & ~15
        synth.inject_utf8_error(buf, c - 3, c + 3, "surrogate", rng)
    elif case == "error_rank0":
        synth.inject_utf8_error(buf, 1000, 2000, "truncated", rng)
    out = run_world(buf)
    ref, _ = oracle.utf8_to_utf16le(buf)
    # the cuts tile the input and fall on character starts
    assert out[0][1] == 0 and out[-1][2] == n and out[0][2] == out[1][1]
    assert (buf[out[1][1]] & 0xC0) != 0x80
    assert out[0][3:5] == (0, 3) and out[1][3:5] == (3, 0)
    # every rank gets the unsharded result; offsets are the exclusive prefix of counts
    for r in out:
        assert r[5] == tuple(ref), (case, r, ref)
    if case == "valid":
        assert out[0][6] == 0
        assert out[1][6] == oracle.utf8_to_utf16le(buf[:out[1][1]])[0].written
