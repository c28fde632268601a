"""GPU parity of the two-pass (planned) transcoders (DESIGN.md section 5 "planned"): the
plan pass (length-from + per-range output counts) followed by the planned transcoder, called
through the C-ABI binding, element by element against the oracle on the same seeded inputs as
the single-pass tests, at sizes spanning many CTA ranges (a plan has 2R sub-ranges of tiles,
R = the transcoder grid) with ragged tails, capacities, errors of every class at range and tile
edges, the shard forms, and a plan of another input (rejected with UG_ERR_ARG)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2111_08692_b200 as ug  # noqa: E402
from test_gpu_parity import DEV, LEADS, short_cases, to_dev  # noqa: E402

TILE = ug.planned_tile_bytes()  # the planned kernels' own tile


def planned_fwd(a: np.ndarray, cap=None, offset=0):
    _, t = to_dev(a, pad_before=offset, pad_after=64)
    cap = a.size if cap is None else cap
    big_out = torch.full((cap + 64,), 0x5A5A, dtype=torch.int16, device=DEV)
    r, ln = ug.utf8_to_utf16le_two_pass(t, big_out[:cap] if cap else big_out[:0], n=a.size,
                                        out_cap=cap)
    o = big_out.cpu().numpy().view(np.uint16)
    assert np.all(o[cap:] == 0x5A5A), "wrote past out_cap"
    assert ln == oracle.utf16_length_from_utf8(a)
    return r, o[: r.written if r.error >= 0 else 0]


def planned_rev(u: np.ndarray, cap=None, offset=0):
    _, t = to_dev(u.astype(np.uint16), pad_before=offset, pad_after=32)
    cap = 3 * u.size if cap is None else cap
    big_out = torch.full((cap + 64,), 0x5A, dtype=torch.uint8, device=DEV)
    r, ln = ug.utf16le_to_utf8_two_pass(t, big_out[:cap], n=u.size, out_cap=cap)
    o = big_out.cpu().numpy()
    assert np.all(o[cap:] == 0x5A), "wrote past out_cap"
    assert ln == oracle.utf8_length_from_utf16le(u)
    return r, o[: r.written if r.error >= 0 else 0]


def check8(a, offset=0, cap=None):
    ref_r, ref_o = oracle.utf8_to_utf16le(a, out_cap=cap)
    r, o = planned_fwd(a, cap=cap, offset=offset)
    assert tuple(r) == tuple(ref_r), (a[:48].tobytes().hex(), r, ref_r)
    if r.error >= 0:
        assert np.array_equal(o, ref_o)
    return r


def check16(u, offset=0, cap=None):
    ref_r, ref_o = oracle.utf16le_to_utf8(u, out_cap=cap)
    r, o = planned_rev(u, cap=cap, offset=offset)
    assert tuple(r) == tuple(ref_r), (r, ref_r)
    if r.error >= 0:
        assert np.array_equal(o, ref_o)
    return r


@pytest.mark.parametrize("n", [1, 2, 3, 17, 1023, TILE - 1, TILE, TILE + 5, 3 * TILE + 7])
def test_planned_small_sizes(n):
    a = np.frombuffer(synth.gen_chunk("mixed", "utf8", n, 11, n), dtype=np.uint8)
    for off in LEADS:
        check8(a, offset=off)
    u = oracle.utf8_to_utf16le(a)[1]
    for off in (0, 1, 7):
        check16(u, offset=off)


def test_planned_empty():
    t = torch.zeros(8, dtype=torch.uint8, device=DEV)
    o = torch.zeros(8, dtype=torch.int16, device=DEV)
    r, ln = ug.utf8_to_utf16le_two_pass(t, o, n=0)
    assert tuple(r) == (0, 0, 0) and ln == 0


@pytest.mark.parametrize("mib", [24, 41])
def test_planned_many_ranges(mib):
    """Inputs of several tiles per sub-range (R CTAs x 2 sub-ranges), ragged at the end:
    every CTA range boundary is crossed; both directions, element by element."""
    a = synth.generate("c4", size=(mib << 20) + 4099)
    check8(a, offset=3)
    u = oracle.utf8_to_utf16le(a)[1]
    check16(u, offset=1)
    # errors of every class at random places (the first error's kind / position / written)
    rng = np.random.default_rng(np.random.SeedSequence([0x2A, mib]))
    for cls in synth.UTF8_ERROR_CLASSES:
        b = a.copy()
        p, _ = synth.inject_utf8_error(b, 0, b.size - 8, cls, rng)
        r = check8(b)
        assert (r.error, r.position) == (synth.UTF8_EXPECTED_KIND[cls], p)
    v = u.copy()
    p, _ = synth.inject_utf16_error(v, 0, v.size - 1, rng)
    r = check16(v)
    assert (r.error, r.position) == (ug.SURROGATE, p)


def test_planned_phase_sweep_tile_edges():
    """Short strings straddling the first and second real tile edges at every phase and
    alignment, through the planned kernels (their per-tile count / decode split)."""
    cases = short_cases()[::3]
    for i, c in enumerate(cases):
        c = np.frombuffer(c, dtype=np.uint8)
        lead = LEADS[i % len(LEADS)]
        for edge in (TILE, 2 * TILE):
            for ph in range(-4, 2):
                pre = edge - lead + ph
                a = np.concatenate([np.full(pre, 0x41, np.uint8), c,
                                    np.full(40, 0x42, np.uint8)])
                check8(a, offset=lead)


def test_planned_capacity():
    a = np.frombuffer(synth.gen_chunk("mixed", "utf8", 300000, 3, 0), dtype=np.uint8)
    need = oracle.utf8_to_utf16le(a)[0].written
    for cap in (0, 1, 7, need // 2, need - 1, need):
        check8(a, cap=cap)
    u = oracle.utf8_to_utf16le(a)[1]
    need8 = oracle.utf16le_to_utf8(u)[0].written
    for cap in (0, 5, need8 - 1, need8):
        check16(u, cap=cap)


@pytest.mark.parametrize("key", ["c1", "c2a", "c2b", "c3"])
def test_planned_configs_reduced(key):
    x = synth.generate(key, size=16 << 20)
    if x.dtype == np.uint8:
        check8(x, offset=5)
        check16(oracle.utf8_to_utf16le(x)[1])
    else:
        check16(x)


def test_planned_rejects_a_plan_of_another_input():
    a = np.frombuffer(synth.gen_chunk("mixed", "utf8", 100000, 5, 0), dtype=np.uint8)
    t = torch.from_numpy(a.copy()).to(DEV)
    plan = ug.plan_buffer(DEV)
    lens = torch.zeros(1, dtype=torch.int64, device=DEV)
    res = ug.result_buffer(DEV, 1)
    out = torch.empty(a.size, dtype=torch.int16, device=DEV)
    ug.utf16_length_from_utf8_plan_async(t, lens, plan, n=a.size - 1)   # other n
    ug.utf8_to_utf16le_planned_async(t, plan, out, res)
    assert ug.decode_results(res)[0].error == ug.ERR_ARG
    ug.utf16_length_from_utf8_plan_async(t, lens, plan)                 # right plan: OK after
    ug.utf8_to_utf16le_planned_async(t, plan, out, res)
    assert tuple(ug.decode_results(res)[0]) == tuple(oracle.utf8_to_utf16le(a)[0])
    # the same pointer and n, but planned as a shard window with halos: a different window
    ug.utf8_shard_plan_async(t, 3, a.size - 6, 3, 3, lens, plan)
    ug.utf8_to_utf16le_planned_async(t[3:], plan, out, res, n=a.size - 6)
    assert ug.decode_results(res)[0].error == ug.ERR_ARG


@pytest.mark.parametrize("G", [2, 5])
def test_planned_shards(G):
    """The shard forms: per shard plan + planned kernel writing its 32-byte record, combined
    on the device, clean and with errors within 3 bytes of a cut."""
    c0 = synth.generate("c4", size=6 << 20)
    rng = np.random.default_rng(np.random.SeedSequence([0x5B, G]))
    for j in range(4):
        b = c0.copy()
        p = None
        if j:
            cut = (int(rng.integers(1, G)) * (b.size // G)) & ~15
            p, _ = synth.inject_utf8_error(b, cut - 3, cut + 3,
                                           synth.UTF8_ERROR_CLASSES[j % 5], rng)
        _, t = to_dev(b)
        n = b.size
        from test_gpu_parity import shard_plan
        cuts = shard_plan(b, G)
        recs = ug.record_buffer(DEV, G)
        lens = torch.zeros(G, dtype=torch.int64, device=DEV)
        outs = []
        for k in range(G):
            lo, hi = cuts[k], cuts[k + 1]
            plan = ug.plan_buffer(DEV)
            hb, ha = min(lo, 3), min(n - hi, 3)
            ug.utf8_shard_plan_async(t, lo, hi - lo, hb, ha, lens, plan, len_off=8 * k)
            out = torch.zeros(max(hi - lo, 1), dtype=torch.int16, device=DEV)
            ug.utf8_to_utf16le_shard_planned_async(t, lo, hi - lo, hb, ha, lo, plan, out, recs,
                                                   rec_off=k * ug.RECORD_BYTES)
            outs.append((out, plan))
        res = ug.result_buffer(DEV, 1)
        ug.combine_records_async(recs, G, 0, n, res)
        torch.cuda.synchronize()
        r = ug.decode_results(res)[0]
        ref_r, ref_o = oracle.utf8_to_utf16le(b)
        assert tuple(r) == tuple(ref_r), (j, r, ref_r)
        if p is not None:
            assert r.position == p
        else:
            recl = ug.decode_records(recs)
            got = np.concatenate([outs[k][0][: recl[k].count].cpu().numpy().view(np.uint16)
                                  for k in range(G)])
            assert np.array_equal(got, ref_o)


@pytest.mark.parametrize("key", ["c2a", "c2b"])
def test_planned_no_four_byte_text_with_errors(key):
    """Text without 4-byte characters takes the no-F forward (f1 for UTF-8, chosen by the plan):
    every error class that adds no >= F0 byte, at random places, and the truncated tail."""
    x = synth.generate(key, size=(6 << 20) + 333)
    assert not (x >= 0xF0).any()
    check8(x, offset=7)
    rng = np.random.default_rng(np.random.SeedSequence([0xF1, len(key)]))
    for cls in synth.UTF8_ERROR_CLASSES:
        b = x.copy()
        p, _ = synth.inject_utf8_error(b, 0, b.size - 8, cls, rng)
        r = check8(b)
        assert (r.error, r.position) == (synth.UTF8_EXPECTED_KIND[cls], p)
    check8(x[:-1])



def test_planned_ascii_tiles_output_phases():
    """All-ASCII tiles of the planned UTF-16 -> UTF-8 kernel (the warps' cooperative a2 path)
    at every output phase: ASCII runs of several tiles after mixed prefixes of different
    lengths, at three input address phases, with a mixed tail and an error after the run; an
    all-ASCII input at capacities around a tile's output."""
    rng = np.random.default_rng(2024)
    mixed = oracle.utf8_to_utf16le(
        np.frombuffer(synth.gen_chunk("mixed", "utf8", 4096, 5, 4096), dtype=np.uint8))[1]
    mixed = mixed[: np.nonzero((mixed & 0xFC00) != 0xDC00)[0][-1]]  # not ending inside a pair
    for pre in range(0, 8):
        run = rng.integers(0x20, 0x7F, 5 * TILE // 2 + int(rng.integers(0, 300))).astype(np.uint16)
        cut = int(np.nonzero((mixed[: 40 + pre] & 0xFC00) != 0xDC00)[0][-1])  # whole chars
        u = np.concatenate([mixed[:cut], run, mixed[:777]]).astype(np.uint16)
        for off in (0, 1, 7):
            check16(u, offset=off)
        v = u.copy()
        v[cut + run.size + 3] = 0xDC00  # a lone low after the run
        check16(v, offset=1)
    # all ASCII, every capacity edge around a tile's output
    a = rng.integers(0, 0x80, 4 * TILE).astype(np.uint16)
    check16(a)
    for cap in (TILE // 2 - 1, TILE // 2, TILE // 2 + 3, 3 * TILE // 2 + 1):
        check16(a, cap=cap)


@pytest.mark.parametrize("n", [1, 7, 8, 9, 100, 4097, 3 * TILE + 5, (1 << 20) + 3])
def test_planned_all_ascii_narrowing(n):
    """A window of ASCII words only is the narrowing copy's (k_narrow16, selected by the plan's
    total = word count): every input and output address phase, capacities below the need, and
    an input with one non-ASCII word (back on the tile kernel)."""
    rng = np.random.default_rng(n)
    u = rng.integers(0, 0x80, n).astype(np.uint16)
    ref_r, ref_o = oracle.utf16le_to_utf8(u)
    for off in (0, 1, 3, 7):
        _, t = to_dev(u, pad_before=off, pad_after=32)
        for oo in (0, 1, 5, 8):
            big = torch.full((n + oo + 64,), 0x5A, dtype=torch.uint8, device=DEV)
            r, ln = ug.utf16le_to_utf8_two_pass(t, big[oo:oo + n], n=n, out_cap=n)
            o = big.cpu().numpy()
            assert tuple(r) == tuple(ref_r) and ln == n
            assert np.array_equal(o[oo:oo + n], ref_o)
            assert np.all(o[:oo] == 0x5A) and np.all(o[oo + n:] == 0x5A)
    for cap in (0, n - 1, n // 2):
        if cap < 0:
            continue
        check16(u, cap=cap)
    v = u.copy()
    v[n // 2] = 0x00E9
    check16(v, offset=1)
    v[n // 2] = 0xDC00
    check16(v)


def test_planned_shards_ascii_and_mixed():
    """Shards of one buffer through the planned shard form, some all ASCII (narrowing copy),
    some mixed (tile kernel), records combined on the device: equal to the unsharded oracle."""
    rng = np.random.default_rng(99)
    a = rng.integers(0x20, 0x7F, 300000).astype(np.uint16)
    mixed = oracle.utf8_to_utf16le(
        np.frombuffer(synth.gen_chunk("mixed", "utf8", 60000, 3, 60000), dtype=np.uint8))[1]
    mixed = mixed[: np.nonzero((mixed & 0xFC00) != 0xDC00)[0][-1]]
    u = np.concatenate([a, mixed, a[:123457]]).astype(np.uint16)
    n = u.size
    cuts = [0, 150001, 300000, 300000 + mixed.size, 300000 + mixed.size + 60000, n]
    _, t = to_dev(u)
    G = len(cuts) - 1
    recs = ug.record_buffer(DEV, G)
    outs = []
    for k in range(G):
        lo, hi = cuts[k], cuts[k + 1]
        out = torch.zeros(3 * (hi - lo), dtype=torch.uint8, device=DEV)
        plan = ug.plan_buffer(DEV)
        lens = torch.zeros(1, dtype=torch.int64, device=DEV)
        ug.utf16le_shard_plan_async(t, lo, hi - lo, min(lo, 1), min(n - hi, 1), lens, plan)
        ug.utf16le_to_utf8_shard_planned_async(t, lo, hi - lo, min(lo, 1), min(n - hi, 1), lo,
                                               plan, out, recs, rec_off=k * ug.RECORD_BYTES)
        outs.append(out)
    res = ug.result_buffer(DEV, 1)
    ug.combine_records_async(recs, G, 0, n, res)
    torch.cuda.synchronize()
    (r,) = ug.decode_results(res)
    ref_r, ref_o = oracle.utf16le_to_utf8(u)
    assert tuple(r) == tuple(ref_r)
    records = ug.decode_records(recs)
    got = np.concatenate([outs[k][: records[k].count].cpu().numpy() for k in range(G)])
    assert np.array_equal(got, ref_o)


@pytest.mark.parametrize("n", [1, 7, 8, 9, 100, 4097, 3 * TILE + 5, (1 << 20) + 3])
def test_planned_all_ascii_widening(n):
    """A window of ASCII bytes only is the widening copy's (k_widen8, selected by the UTF-8
    plan's header word 9): every input and output address phase, capacities below the need,
    and inputs with one non-ASCII byte (valid, or invalid) back on the tile kernels."""
    rng = np.random.default_rng(n + 1)
    a = rng.integers(0, 0x80, n).astype(np.uint8)
    ref_r, ref_o = oracle.utf8_to_utf16le(a)
    for off in (0, 1, 7, 8):
        _, t = to_dev(a, pad_before=off, pad_after=64)
        for oo in (0, 1, 3, 8):
            big = torch.full((n + oo + 64,), 0x5A5A, dtype=torch.int16, device=DEV)
            r, ln = ug.utf8_to_utf16le_two_pass(t, big[oo:oo + n], n=n, out_cap=n)
            o = big.cpu().numpy().view(np.uint16)
            assert tuple(r) == tuple(ref_r) and ln == n
            assert np.array_equal(o[oo:oo + n], ref_o)
            assert np.all(o[:oo] == 0x5A5A) and np.all(o[oo + n:] == 0x5A5A)
    for cap in (0, n - 1, n // 2):
        check8(a, cap=cap)
    if n >= 2:
        v = a.copy()
        v[n // 2] = 0x80  # a lone continuation byte: an error, on the tile kernel
        check8(v, offset=1)
        v[n // 2 - 1:n // 2 + 1] = (0xC3, 0xA9)  # a valid 2-byte character
        check8(v)


def test_planned_fwd_shards_ascii_and_mixed():
    """UTF-8 shards of one buffer through the planned shard form, some all ASCII (widening
    copy), some mixed (tile kernels), records combined: equal to the unsharded oracle."""
    rng = np.random.default_rng(98)
    asc = rng.integers(0x20, 0x7F, 400000).astype(np.uint8)
    mixed = np.frombuffer(synth.gen_chunk("mixed", "utf8", 90000, 4, 90000), dtype=np.uint8)
    a = np.concatenate([asc, mixed, asc[:200001]])
    n = a.size
    cuts = [0, 200003, 400000, 400000 + mixed.size, 400000 + mixed.size + 100000, n]
    _, t = to_dev(a)
    G = len(cuts) - 1
    recs = ug.record_buffer(DEV, G)
    outs = []
    for k in range(G):
        lo, hi = cuts[k], cuts[k + 1]
        hb, ha = min(lo, 3), min(n - hi, 3)
        out = torch.zeros(hi - lo, dtype=torch.int16, device=DEV)
        plan = ug.plan_buffer(DEV)
        lens = torch.zeros(1, dtype=torch.int64, device=DEV)
        ug.utf8_shard_plan_async(t, lo, hi - lo, hb, ha, lens, plan)
        ug.utf8_to_utf16le_shard_planned_async(t, lo, hi - lo, hb, ha, lo, plan, out, recs,
                                               rec_off=k * ug.RECORD_BYTES)
        outs.append(out)
    res = ug.result_buffer(DEV, 1)
    ug.combine_records_async(recs, G, 0, n, res)
    torch.cuda.synchronize()
    (r,) = ug.decode_results(res)
    ref_r, ref_o = oracle.utf8_to_utf16le(a)
    assert tuple(r) == tuple(ref_r)
    records = ug.decode_records(recs)
    got = np.concatenate([outs[k][: records[k].count].cpu().numpy().view(np.uint16)
                          for k in range(G)])
    assert np.array_equal(got, ref_o)
