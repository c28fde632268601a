"""GPU parity at BASELINE.json's full sizes (tier T1, large).  Configs 1-3 are compared with the
oracle element by element.  Config 4 (8 GiB, > 2^32 output units):
  * the launch bench.py times (the shard call at G = 1) is compared with the oracle element by
    element over ALL 128 of its 64 MiB generator chunks (each is whole valid text, so chunk
    boundaries are character boundaries and the oracle's per-chunk outputs concatenate);
  * the sharded path at G = 2 / 4 / 8 (cuts at character starts, 3-byte halos, one shard
    launch per rank, records combined on the device by ug_combine_records_async) reproduces
    that output unit for unit, both directions, in its single-pass and two-pass (plan +
    planned kernel, the form bench.py times) forms;
  * BASELINE.json configs[4]'s 16 seeded error copies PER G, each an injected error of a random
    class within 3 bytes of a shard cut, patched in place on the device, through the SHARDED
    path: (error, position, written) against the oracle (written = the oracle's counts of the
    whole chunks before p plus the oracle on the partial chunk)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2111_08692_b200 as ug  # noqa: E402

DEV = torch.device("cuda:0")


def full_fwd_rev(x8: np.ndarray):
    t = torch.from_numpy(x8).to(DEV)
    out16 = torch.empty(x8.size, dtype=torch.int16, device=DEV)
    r = ug.utf8_to_utf16le(t, out16)
    back = torch.empty(x8.size, dtype=torch.uint8, device=DEV)
    r2 = ug.utf16le_to_utf8(out16[: r.written], back) if r.error == 0 else None
    return t, out16, r, back, r2


@pytest.mark.parametrize("key", ["c1", "c2a", "c2b"])
def test_full_size_utf8_configs(key):
    x = synth.generate(key)
    assert x.size == synth.CONFIGS[key].size
    ref_r, ref_o = oracle.utf8_to_utf16le(x)
    t, out16, r, back, r2 = full_fwd_rev(x)
    assert tuple(r) == tuple(ref_r)
    assert torch.equal(out16[: r.written], torch.from_numpy(ref_o.view(np.int16)).to(DEV))
    assert r2 == (0, r.written, x.size) and torch.equal(back, t)
    assert tuple(ug.utf8_validate(t)) == tuple(oracle.utf8_validate(x))
    assert ug.utf16_length_from_utf8(t) == r.written
    assert ug.utf8_length_from_utf16le(out16[: r.written]) == x.size
    # the two-pass path (the bench's): same result and the same units, both directions
    o2 = torch.empty(x.size, dtype=torch.int16, device=DEV)
    rp, ln = ug.utf8_to_utf16le_two_pass(t, o2)
    assert tuple(rp) == tuple(ref_r) and ln == r.written
    assert torch.equal(o2[: r.written], out16[: r.written])
    b2 = torch.empty(x.size, dtype=torch.uint8, device=DEV)
    rp2, ln2 = ug.utf16le_to_utf8_two_pass(out16[: r.written], b2)
    assert rp2 == (0, r.written, x.size) and ln2 == x.size and torch.equal(b2, t)


def test_full_size_config3_and_error_copy():
    u = synth.generate("c3")
    assert u.nbytes == synth.CONFIGS["c3"].size
    t = torch.from_numpy(u.view(np.int16)).to(DEV)
    ref_r, ref_o = oracle.utf16le_to_utf8(u)
    out8 = torch.empty(ref_r.written + 64, dtype=torch.uint8, device=DEV)
    r = ug.utf16le_to_utf8(t, out8)
    assert tuple(r) == tuple(ref_r)
    assert torch.equal(out8[: r.written], torch.from_numpy(ref_o).to(DEV))
    assert tuple(ug.utf16le_validate(t)) == tuple(oracle.utf16le_validate(u))
    assert ug.utf8_length_from_utf16le(t) == r.written
    o2 = torch.empty(ref_r.written + 64, dtype=torch.uint8, device=DEV)
    rp, ln = ug.utf16le_to_utf8_two_pass(t, o2)
    assert tuple(rp) == tuple(ref_r) and ln == r.written
    assert torch.equal(o2[: r.written], out8[: r.written])
    rng = np.random.default_rng(np.random.SeedSequence([4, 0xE, 1, 0]))
    for _ in range(2):
        v = u.copy()
        p, _ = synth.inject_utf16_error(v, 0, v.size - 1, rng)
        tv = torch.from_numpy(v.view(np.int16)).to(DEV)
        rv = ug.utf16le_to_utf8(tv, out8)
        assert tuple(rv) == tuple(oracle.utf16le_to_utf8(v)[0])
        assert (rv.error, rv.position) == (ug.SURROGATE, p)
        assert tuple(ug.utf16le_validate(tv)) == (ug.SURROGATE, p, 0)
        assert tuple(ug.utf16le_to_utf8_two_pass(tv, out8)[0]) == tuple(rv)


@pytest.fixture(scope="module")
def c4():
    return synth.generate("c4")


def _oracle_chunk(x):
    r, o = oracle.utf8_to_utf16le(x)
    assert r.error == 0
    return o


@pytest.fixture(scope="module")
def c4_ref(c4):
    """The bench launch at G = 1 and its element-by-element check against the oracle on every
    64 MiB chunk.  Returns (device input, device output, n16, oracle count per chunk)."""
    n = c4.size
    t = torch.from_numpy(c4).to(DEV)
    out16 = torch.empty(n, dtype=torch.int16, device=DEV)
    rec = ug.record_buffer(DEV, 1)
    ug.utf8_to_utf16le_shard_async(t, 0, n, 0, 0, 0, out16, rec)   # bench.py's launch, G = 1
    torch.cuda.synchronize()
    r = ug.decode_records(rec)[0]
    assert r.first_err == ug.NONE and r.too_small == 0
    n16 = r.count
    assert n16 > 2 ** 32                       # 64-bit offsets exercised
    C = synth.CHUNK
    nch = n // C
    workers = max(1, min(32, os.cpu_count() or 1))
    counts, off = [], 0
    with ThreadPoolExecutor(workers) as ex:    # the oracle releases the GIL (ctypes)
        for b0 in range(0, nch, workers):
            refs = list(ex.map(_oracle_chunk, [c4[c * C:(c + 1) * C]
                                                for c in range(b0, min(nch, b0 + workers))]))
            for c, ref in zip(range(b0, b0 + len(refs)), refs):
                got = out16[off:off + ref.size]
                assert torch.equal(got, torch.from_numpy(ref.view(np.int16)).to(DEV)), c
                counts.append(ref.size)
                off += ref.size
    assert off == n16
    return t, out16, n16, counts


def test_config4_full_size_bench_launch(c4_ref):
    t, out16, n16, counts = c4_ref
    n = t.numel()
    assert ug.utf16_length_from_utf8(t) == n16
    # the launch bench.py times (two-pass: the shard plan + the planned shard kernel at G = 1)
    # reproduces the oracle-verified output unit for unit, both directions
    plan = ug.plan_buffer(DEV)
    lens = torch.zeros(2, dtype=torch.int64, device=DEV)
    recp = ug.record_buffer(DEV, 1)
    o2 = torch.empty(n, dtype=torch.int16, device=DEV)
    ug.utf8_shard_plan_async(t, 0, n, 0, 0, lens, plan)
    ug.utf8_to_utf16le_shard_planned_async(t, 0, n, 0, 0, 0, plan, o2, recp)
    torch.cuda.synchronize()
    rp = ug.decode_records(recp)[0]
    assert rp.first_err == ug.NONE and rp.count == n16 and int(lens[0]) == n16
    assert torch.equal(o2[:n16], out16[:n16])
    del o2
    b2 = torch.empty(n, dtype=torch.uint8, device=DEV)
    ug.utf16le_shard_plan_async(out16[:n16], 0, n16, 0, 0, lens, plan, len_off=8)
    ug.utf16le_to_utf8_shard_planned_async(out16[:n16], 0, n16, 0, 0, 0, plan, b2, recp)
    torch.cuda.synchronize()
    rp2 = ug.decode_records(recp)[0]
    assert rp2.first_err == ug.NONE and rp2.count == n and int(lens[1]) == n
    assert torch.equal(b2, t)
    del b2
    # reverse through the shard call as well, then the round trip is the identity
    back = torch.empty(n, dtype=torch.uint8, device=DEV)
    rec = ug.record_buffer(DEV, 1)
    ug.utf16le_to_utf8_shard_async(out16[:n16], 0, n16, 0, 0, 0, back, rec)
    torch.cuda.synchronize()
    r2 = ug.decode_records(rec)[0]
    assert r2.first_err == ug.NONE and r2.count == n
    assert torch.equal(back, t)
    assert ug.utf8_length_from_utf16le(out16[:n16]) == n
    # the plain API agrees
    assert tuple(ug.utf8_to_utf16le(t, out16)) == (0, n, n16)
    # the streaming UTF-16 validator at the bench size (11.3 GB, word indices past 2^32 bytes),
    # clean and with a high surrogate followed by 'A' planted late in the buffer
    u = out16[:n16]
    assert tuple(ug.utf16le_validate(u)) == (0, n16, 0)
    for p in ((5 << 30) + 7, n16 - 1):
        keep = u[p - 2:p + 1].clone()
        prev2 = int(keep[0].item()) & 0xFFFF
        u[p - 1] = -0x2800  # 0xD800
        u[p] = 0x41
        want = p - 2 if (prev2 & 0xFC00) == 0xD800 else p - 1
        assert tuple(ug.utf16le_validate(u)) == (ug.SURROGATE, want, 0), p
        u[p - 2:p + 1] = keep
    assert tuple(ug.utf16le_validate(u)) == (0, n16, 0)


def shard_cuts_utf8(host: np.ndarray, G: int):
    """BASELINE north_star item 3 / DESIGN.md section 7: nominal cuts aligned down to 16 B,
    backed off to character starts by the library's cut rule."""
    from paper_2111_08692_b200 import dist as ugd
    n = host.size
    get = lambda a, b: host[a:b].tobytes()  # noqa: E731
    return [ugd.utf8_cut(get, c, n) for c in ugd.nominal_cuts(n, G)]


def run_sharded_fwd(t, cuts, out, validate=False, planned=False):
    """One shard launch per virtual rank over the device buffer t, then every rank's combine
    on the device.  Returns (global result, records, per-rank output offsets).  planned: the
    two-pass form (shard plan + planned shard kernel), as bench.py times it."""
    G = len(cuts) - 1
    n = t.numel()
    recs = ug.record_buffer(DEV, G)
    plan = ug.plan_buffer(DEV) if planned else None
    lens = torch.zeros(1, dtype=torch.int64, device=DEV)
    for k in range(G):
        lo, hi = cuts[k], cuts[k + 1]
        hb, ha = min(lo, 3), min(n - hi, 3)
        if planned:
            ug.utf8_shard_plan_async(t, lo, hi - lo, hb, ha, lens, plan)
            ug.utf8_to_utf16le_shard_planned_async(t, lo, hi - lo, hb, ha, lo, plan, out[lo:hi],
                                                   recs, rec_off=k * ug.RECORD_BYTES)
        elif validate:
            ug.utf8_validate_shard_async(t, lo, hi - lo, hb, ha, lo, recs,
                                         rec_off=k * ug.RECORD_BYTES)
        else:
            ug.utf8_to_utf16le_shard_async(t, lo, hi - lo, hb, ha, lo, out[lo:hi], recs,
                                           rec_off=k * ug.RECORD_BYTES)
    res = ug.result_buffer(DEV, G)
    offs = torch.zeros(G, dtype=torch.int64, device=DEV)
    for k in range(G):
        ug.combine_records_async(recs, G, k, n, res[k * ug.RESULT_BYTES:], offs[k:])
    torch.cuda.synchronize()
    results = ug.decode_results(res)
    assert all(r == results[0] for r in results)
    return results[0], ug.decode_records(recs), offs.cpu().tolist()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_config4_sharded_matches_oracle(c4, c4_ref, G):
    """The sharded forward at G ranks places every rank's output exactly where the oracle's
    (verified unsharded) output has it; the reverse per rank round-trips each rank's bytes."""
    t, out16, n16, _ = c4_ref
    n = c4.size
    cuts = shard_cuts_utf8(c4, G)
    outs = torch.empty(n, dtype=torch.int16, device=DEV)
    rp, recp, offp = run_sharded_fwd(t, cuts, outs, planned=True)   # the bench's two-pass form
    assert tuple(rp) == (0, n, n16)
    for k in range(G):
        assert torch.equal(outs[cuts[k]:cuts[k] + recp[k].count],
                           out16[offp[k]:offp[k] + recp[k].count]), k
    r, recs, offs = run_sharded_fwd(t, cuts, outs)
    assert tuple(r) == (0, n, n16)
    assert offs == list(np.cumsum([0] + [x.count for x in recs[:-1]]))
    back = torch.empty(max(cuts[k + 1] - cuts[k] for k in range(G)), dtype=torch.uint8,
                       device=DEV)
    rec = ug.record_buffer(DEV, 1)
    for k in range(G):
        lo, cnt, off = cuts[k], recs[k].count, offs[k]
        assert torch.equal(outs[lo:lo + cnt], out16[off:off + cnt]), k
        ug.utf16le_to_utf8_shard_async(outs[lo:lo + cnt], 0, cnt, 0, 0, off, back, rec)
        torch.cuda.synchronize()
        rr = ug.decode_records(rec)[0]
        assert rr.first_err == ug.NONE and rr.count == cuts[k + 1] - lo
        assert torch.equal(back[:rr.count], t[lo:cuts[k + 1]]), k


@pytest.mark.parametrize("G", [2, 4, 8])
def test_config4_error_copies_sharded(c4, c4_ref, G):
    """BASELINE.json configs[4]: 16 seeded copies per G, each with one injected error of a
    random class at a character start within 3 bytes of a uniformly chosen interior shard cut
    (SeedSequence([5, 0xE, G, j])), patched in place on the device and
    run through the SHARDED forward (cuts recomputed on the patched bytes) and the sharded
    validator.  Expected: kind = the injected class, position = p, written = the oracle's
    units before p."""
    t, _, _, counts = c4_ref
    n = c4.size
    C = synth.CHUNK
    prefix = np.concatenate([[0], np.cumsum(counts)])
    outs = torch.empty(n, dtype=torch.int16, device=DEV)
    for j in range(16):
        rng = np.random.default_rng(np.random.SeedSequence([5, 0xE, G, j]))
        k = int(rng.integers(1, G))
        c = (k * (n // G)) & ~15
        cls = synth.UTF8_ERROR_CLASSES[int(rng.integers(0, len(synth.UTF8_ERROR_CLASSES)))]
        p, saved = synth.inject_utf8_error(c4, c - 3, c + 3, cls, rng)
        assert abs(p - c) <= 3
        t[p:p + saved.size] = torch.from_numpy(c4[p:p + saved.size].copy()).to(DEV)
        try:
            cuts = shard_cuts_utf8(c4, G)
            ch = p // C
            want_wr = int(prefix[ch]) + oracle.utf8_to_utf16le(c4[ch * C:p])[0].written
            want = (synth.UTF8_EXPECTED_KIND[cls], p, want_wr)
            r, *_ = run_sharded_fwd(t, cuts, outs)
            assert tuple(r) == want, (G, j, cls, r, want)
            rp, *_ = run_sharded_fwd(t, cuts, outs, planned=True)
            assert tuple(rp) == want, (G, j, cls, "two-pass", rp, want)
            v, *_ = run_sharded_fwd(t, cuts, None, validate=True)
            assert (v.error, v.position, v.written) == (want[0], p, 0), (G, j, cls, v)
        finally:
            c4[p:p + saved.size] = saved
            t[p:p + saved.size] = torch.from_numpy(saved).to(DEV)
