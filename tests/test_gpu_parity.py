"""GPU parity (tier T1): the CUDA path, called through the C-ABI binding, against the oracle,
element by element, on seeded inputs.  Bit-exact: output units, result struct (verdict, first
error offset, written count), length-from values.  Needs a B200 (sm_100a)."""
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
# the kernels' real tile (16 KiB: 512 threads x 32 bytes), queried from the library; tile t of
# a call covers input positions [t * TILE - lead, (t + 1) * TILE - lead), lead = address mod 16
TILE = ug.tile_bytes()
LEADS = (0, 1, 7, 15)


# ----------------------------------------------------------------------------- helpers
def to_dev(a: np.ndarray, pad_before=0, pad_after=0, fill=0xAA):
    """Upload with guard bytes around it (to catch reads/writes outside the range) and return
    (big tensor, view of the payload)."""
    a = np.ascontiguousarray(a)
    dt = {np.dtype(np.uint8): torch.uint8, np.dtype(np.uint16): torch.int16,
          np.dtype("<u2"): torch.int16}[a.dtype]
    big = np.full(pad_before + a.size + pad_after, fill, dtype=a.dtype)
    big[pad_before:pad_before + a.size] = a
    t = torch.from_numpy(big.view(np.int16) if a.dtype.itemsize == 2 else big).to(DEV)
    return t, t[pad_before:pad_before + a.size]


def gpu_fwd(a: np.ndarray, cap=None, offset=0):
    """utf8_to_utf16le on a device copy of `a` placed at byte `offset` of its buffer."""
    _, t = to_dev(a, pad_before=offset, pad_after=64)
    cap = a.size if cap is None else cap
    big_out = torch.full((cap + 64,), 0x5A5A, dtype=torch.int16, device=DEV)
    out = big_out[:cap] if cap else big_out[:0]
    r = ug.utf8_to_utf16le(t, out, n=a.size, out_cap=cap)
    o = big_out.cpu().numpy().view(np.uint16)
    assert np.all(o[cap:] == 0x5A5A), "wrote past out_cap"
    return r, o[: r.written if r.error >= 0 else 0]


def gpu_rev(u: np.ndarray, cap=None, offset=0):
    _, t = to_dev(u.astype(np.uint16), pad_before=offset, pad_after=32)
    cap = 3 * u.size if cap is None else cap
    big_out = torch.full((cap + 64,), 0x5A, dtype=torch.uint8, device=DEV)
    out = big_out[:cap]
    r = ug.utf16le_to_utf8(t, out, n=u.size, out_cap=cap)
    o = big_out.cpu().numpy()
    assert np.all(o[cap:] == 0x5A), "wrote past out_cap"
    return r, o[: r.written if r.error >= 0 else 0]


def check_utf8(a: np.ndarray, offset=0, cap=None):
    ref_r, ref_o = oracle.utf8_to_utf16le(a, out_cap=cap)
    r, o = gpu_fwd(a, cap=cap, offset=offset)
    assert tuple(r) == tuple(ref_r), (a[:64].tobytes().hex(), r, ref_r)
    if r.error >= 0:
        assert np.array_equal(o, ref_o)
    _, t = to_dev(a, pad_before=offset)
    v = ug.utf8_validate(t)
    rv = oracle.utf8_validate(a)
    assert tuple(v) == tuple(rv), (v, rv)
    assert ug.utf16_length_from_utf8(t) == oracle.utf16_length_from_utf8(a)
    return r


def check_utf16(u: np.ndarray, offset=0, cap=None):
    ref_r, ref_o = oracle.utf16le_to_utf8(u, out_cap=cap)
    r, o = gpu_rev(u, cap=cap, offset=offset)
    assert tuple(r) == tuple(ref_r), (r, ref_r)
    if r.error >= 0:
        assert np.array_equal(o, ref_o)
    _, t = to_dev(u.astype(np.uint16), pad_before=offset)
    v = ug.utf16le_validate(t)
    assert tuple(v) == tuple(oracle.utf16le_validate(u))
    assert ug.utf8_length_from_utf16le(t) == oracle.utf8_length_from_utf16le(u)
    return r


def h(s):
    return np.frombuffer(bytes.fromhex(s), dtype=np.uint8)


# ----------------------------------------------------------------------------- worked examples
def test_spec_examples(golden):
    for ex in golden["utf8_to_utf16le"]:
        a = h(ex["in"])
        r = check_utf8(a)
        assert r.position == ex["position"]
    ex = golden["utf8_surrogate_at_1000"]
    a = np.concatenate([np.full(ex["prefix_ascii"], 0x61, np.uint8), h(ex["bytes"])])
    r = check_utf8(a)
    assert (r.error, r.position) == (ug.SURROGATE, 1000)
    for ex in golden["utf16le_to_utf8"]:
        u = np.array([int(x, 16) for x in ex["in"]], dtype=np.uint16)
        r = check_utf16(u)
        assert r.position == ex["position"]


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5, 15, 16, 17, 31, 32, 33, 1023, 1024, 1025,
                               8191, 8192, 8193, TILE - 1, TILE, TILE + 1, TILE + 7,
                               2 * TILE + 3, 3 * TILE - 5])
def test_small_sizes(n):
    rng = np.random.default_rng(n)
    a = np.frombuffer(synth.gen_chunk("mixed", "utf8", n, 7, n), dtype=np.uint8) if n else \
        np.zeros(0, np.uint8)
    for off in (0, 1, 7, 15):
        check_utf8(a, offset=off)
    u = oracle.utf8_to_utf16le(a)[1]
    for off in (0, 1, 7):
        check_utf16(u, offset=2 * off)
    # a random single byte change
    if n:
        b = a.copy()
        b[rng.integers(0, n)] = rng.integers(0, 256)
        check_utf8(b, offset=3)


# ----------------------------------------------------------------------------- phase sweep
def short_cases():
    """Short strings: all 1-byte, a stride through 2-byte, class representatives of length 3-4
    (covering every rule), valid 4-byte characters."""
    cases = [bytes([b]) for b in range(256)]
    cases += [bytes([a, b]) for a in range(0x80, 0x100, 3) for b in range(0x00, 0x100, 7)]
    reps = [0x41, 0x80, 0x9F, 0xA0, 0xBF, 0xC0, 0xC2, 0xDF, 0xE0, 0xE4, 0xED, 0xEF, 0xF0, 0xF4,
            0xF5, 0xF8, 0xFF]
    rng = np.random.default_rng(0)
    for _ in range(600):
        L = int(rng.integers(3, 5))
        cases.append(bytes(int(x) for x in rng.choice(reps, L)))
    cases += ["\U0001F600".encode(), "\U0010FFFF".encode(), "￿".encode(), "߿".encode()]
    return cases


@pytest.mark.parametrize("boundary", [32, 1024, TILE, 2 * TILE])
def test_phase_sweep(boundary):
    """Each short string embedded in ASCII padding so that it straddles a thread (32 B), warp
    (1 KiB) or real tile edge (the first and the second tile edge: TMA halos, emit ownership
    split between two CTAs, the look-back between tiles) at every phase -4..+1, at input
    alignments (leads) 0 / 1 / 7 / 15.  The edge sits at position boundary - lead."""
    cases = short_cases()
    for i, c in enumerate(cases):
        c = np.frombuffer(c, dtype=np.uint8)
        lead = LEADS[i % len(LEADS)]
        for ph in range(-4, 2):
            pre = boundary - lead + ph
            a = np.concatenate([np.full(pre, 0x41, np.uint8), c, np.full(40, 0x42, np.uint8)])
            check_utf8(a, offset=lead)


def test_phase_sweep_at_input_end():
    """Errors and truncations in the last bytes of the input right at a real tile edge: the
    after-halo reads 0x00 (end of stream) and the classifier's look-ahead decides."""
    reps = [b"\xc3", b"\xe4\xbd", b"\xf0\x9f\x98", b"\xed\xa0\x80", b"\x80", b"\xc0\xaf",
            "\U0001F600".encode(), "你".encode()]
    for lead in LEADS:
        for c in reps:
            for ph in range(-4, 4):
                pre = TILE - lead + ph - len(c)
                if pre < 0:
                    continue
                a = np.frombuffer(b"A" * pre + c, dtype=np.uint8)
                check_utf8(a, offset=lead)


def test_valid_text_straddling_every_tile_phase():
    """Valid 4-byte / 3-byte / 2-byte characters across the first and second real tile edges
    at every byte phase and alignment: S:638 (round trip), both directions."""
    for ch in ("\U0001F600", "你", "é"):
        e = ch.encode()
        for edge in (TILE, 2 * TILE):
            for lead in LEADS:
                for ph in range(0, len(e) + 1):
                    pre = edge - lead - ph
                    a = np.frombuffer(b"a" * pre + e * 3 + b"z" * 5, dtype=np.uint8)
                    r = check_utf8(a, offset=lead)
                    assert r.error == 0
                    u = oracle.utf8_to_utf16le(a)[1]
                    check_utf16(u, offset=lead & ~1)


# ----------------------------------------------------------------------------- random fuzz
def test_fuzz_utf8():
    rng = np.random.default_rng(1234)
    reps = np.array([0x00, 0x41, 0x7F, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1, 0xC2,
                     0xDF, 0xE0, 0xE1, 0xEC, 0xED, 0xEE, 0xEF, 0xF0, 0xF1, 0xF3, 0xF4, 0xF5,
                     0xF7, 0xF8, 0xFF], dtype=np.uint8)
    for k in range(400):
        n = int(rng.integers(0, 300))
        if k % 3 == 0:
            a = reps[rng.integers(0, reps.size, n)]
        elif k % 3 == 1:
            a = rng.integers(0, 256, n, dtype=np.uint8)
        else:
            a = np.frombuffer(synth.gen_chunk("mixed", "utf8", n, 99, k), dtype=np.uint8).copy()
            if n:
                a[rng.integers(0, n)] = rng.integers(0x80, 0x100)
        check_utf8(a, offset=int(rng.integers(0, 16)))


def test_fuzz_utf16():
    rng = np.random.default_rng(4321)
    alpha = np.array([0x0041, 0x007F, 0x0080, 0x07FF, 0x0800, 0xD7FF, 0xD800, 0xDBFF, 0xDC00,
                      0xDFFF, 0xE000, 0xFFFF], dtype=np.uint16)
    for k in range(400):
        n = int(rng.integers(0, 200))
        u = alpha[rng.integers(0, alpha.size, n)] if k % 2 else \
            rng.integers(0, 65536, n).astype(np.uint16)
        check_utf16(u, offset=2 * int(rng.integers(0, 8)))


# ----------------------------------------------------------------------------- capacity
def test_capacity():
    a = np.frombuffer(synth.gen_chunk("mixed", "utf8", 50000, 3, 0), dtype=np.uint8)
    need = oracle.utf8_to_utf16le(a)[0].written
    for cap in (0, 1, 7, need // 2, need - 1, need, need + 1):
        check_utf8(a, cap=cap)
    u = oracle.utf8_to_utf16le(a)[1]
    need8 = oracle.utf16le_to_utf8(u)[0].written
    for cap in (0, 5, need8 - 1, need8):
        check_utf16(u, cap=cap)


# ----------------------------------------------------------------------------- configs
@pytest.fixture(scope="module")
def c0():
    return synth.generate("c0")


def test_config0_clean_and_error_copies(c0):
    r = check_utf8(c0)
    assert r.error == 0 and r.position == c0.size
    u = oracle.utf8_to_utf16le(c0)[1]
    check_utf16(u)
    rng = np.random.default_rng(np.random.SeedSequence([0, 0xE, 1, 0]))
    for cls in synth.UTF8_ERROR_CLASSES:
        for j in range(3):
            b = c0.copy()
            p, _ = synth.inject_utf8_error(b, 0, b.size - 8, cls, rng)
            r = check_utf8(b, offset=j)
            assert r.position == p and r.error == synth.UTF8_EXPECTED_KIND[cls], (cls, r, p)


def test_config3_error_copy():
    u = synth.generate("c3", size=4 << 20)
    check_utf16(u)
    rng = np.random.default_rng(np.random.SeedSequence([4, 0xE, 1, 0]))
    for j in range(6):
        v = u.copy()
        p, _ = synth.inject_utf16_error(v, 0, v.size - 1, rng)
        r = check_utf16(v)
        assert (r.error, r.position) == (ug.SURROGATE, p)


@pytest.mark.parametrize("key", ["c1", "c2a", "c2b", "c3"])
def test_configs_reduced(key):
    """Each config's generator at 8 MiB, both directions, element by element."""
    x = synth.generate(key, size=8 << 20)
    if x.dtype == np.uint8:
        check_utf8(x, offset=3)
        u = oracle.utf8_to_utf16le(x)[1]
        check_utf16(u)
    else:
        check_utf16(x)


# ----------------------------------------------------------------------------- async / host
def test_async_and_host_variants(c0):
    t, tin = to_dev(c0)
    out = torch.zeros(c0.size, dtype=torch.int16, device=DEV)
    res = ug.result_buffer(DEV, 2)
    ug.utf8_to_utf16le_async(tin, out, res)
    ug.utf8_validate_async(tin, res, result_off=ug.RESULT_BYTES)
    lens = torch.zeros(2, dtype=torch.int64, device=DEV)
    ug.utf16_length_from_utf8_async(tin, lens)
    torch.cuda.synchronize()
    r = ug.decode_results(res)
    ref = oracle.utf8_to_utf16le(c0)
    assert tuple(r[0]) == tuple(ref[0])
    assert tuple(r[1]) == tuple(oracle.utf8_validate(c0))
    assert int(lens[0]) == ref[0].written
    assert np.array_equal(out[: ref[0].written].cpu().numpy().view(np.uint16), ref[1])
    # host buffers (pinned)
    hin = torch.from_numpy(c0.copy()).pin_memory()
    hout = torch.zeros(c0.size, dtype=torch.int16).pin_memory()
    rh = ug.utf8_to_utf16le_host(hin, hout)
    assert tuple(rh) == tuple(ref[0])
    assert np.array_equal(hout[: rh.written].numpy().view(np.uint16), ref[1])
    h8 = torch.zeros(3 * rh.written, dtype=torch.uint8).pin_memory()
    rr = ug.utf16le_to_utf8_host(hout[: rh.written], h8)
    assert rr == (0, rh.written, c0.size) and bytes(h8[: rr.written].numpy()) == c0.tobytes()


# ----------------------------------------------------------------------------- virtual shards
def shard_plan(a: np.ndarray, G: int):
    """Nominal cuts k*floor(n/G) aligned down to 16, backed off to character starts."""
    n = a.size
    cuts = [0]
    for k in range(1, G):
        c = (k * (n // G)) & ~15
        cuts.append(c - ug.utf8_cut_backoff(a[max(0, c - 8):c + 8].tobytes(), c - max(0, c - 8)))
    cuts.append(n)
    return cuts


def run_shards_fwd(a: np.ndarray, G: int):
    """G logical shards of one device buffer, each through the shard kernel, records combined
    on the device."""
    _, t = to_dev(a)
    cuts = shard_plan(a, G)
    n = a.size
    recs = ug.record_buffer(DEV, G)
    outs = []
    for k in range(G):
        lo, hi = cuts[k], cuts[k + 1]
        out = torch.zeros(max(hi - lo, 1), dtype=torch.int16, device=DEV)
        ug.utf8_to_utf16le_shard_async(t, lo, hi - lo, min(lo, 3), min(n - hi, 3), lo, out, recs,
                                       rec_off=k * ug.RECORD_BYTES)
        outs.append(out)
    res = ug.result_buffer(DEV, G)
    offs = torch.zeros(G, dtype=torch.int64, device=DEV)
    for k in range(G):
        ug.combine_records_async(recs, G, k, n, res[k * ug.RESULT_BYTES:], offs[k:])
    torch.cuda.synchronize()
    results = ug.decode_results(res)
    assert all(r == results[0] for r in results)
    records = ug.decode_records(recs)
    return results[0], records, outs, offs.cpu().tolist(), cuts


@pytest.mark.parametrize("G", [2, 3, 8])
def test_virtual_shards_match_unsharded(c0, G):
    r, records, outs, offs, cuts = run_shards_fwd(c0, G)
    ref_r, ref_o = oracle.utf8_to_utf16le(c0)
    assert tuple(r) == tuple(ref_r)
    got = np.concatenate([outs[k][: records[k].count].cpu().numpy().view(np.uint16)
                          for k in range(G)])
    assert np.array_equal(got, ref_o)
    assert offs == list(np.cumsum([0] + [rec.count for rec in records[:-1]]))
    # the reverse direction on each rank's whole-character output, no new cuts
    for k in range(G):
        u = outs[k][: records[k].count]
        out8 = torch.zeros(3 * max(u.numel(), 1), dtype=torch.uint8, device=DEV)
        rr = ug.utf16le_to_utf8(u, out8)
        assert rr.error == 0 and bytes(out8[: rr.written].cpu().numpy()) == \
            c0[cuts[k]:cuts[k + 1]].tobytes()


def test_virtual_shards_error_near_cut(c0):
    """Errors placed within 3 bytes of a shard cut: the global first error, kind and written
    count are exact (BASELINE config 4's error copies, at 1 MiB)."""
    G = 4
    rng = np.random.default_rng(np.random.SeedSequence([5, 0xE, G, 0]))
    for j in range(16):
        b = c0.copy()
        k = int(rng.integers(1, G))
        c = (k * (b.size // G)) & ~15
        cls = synth.UTF8_ERROR_CLASSES[j % 5]
        p, _ = synth.inject_utf8_error(b, c - 3, c + 3, cls, rng)
        r, *_ = run_shards_fwd(b, G)
        ref = oracle.utf8_to_utf16le(b)[0]
        assert tuple(r) == tuple(ref) and r.position == p, (cls, r, ref, p)


# ----------------------------------------------------------------------------- host pipeline
def host_run(x: np.ndarray, chunk: int, cap=None):
    """*_host on pinned copies of `x` with the pipeline's chunk size set to `chunk` units;
    guards after out_host[cap] catch writes past the capacity."""
    fwd = x.dtype == np.uint8
    cap = (x.size if fwd else 3 * x.size) if cap is None else cap
    prev = ug.set_host_chunk(chunk)
    try:
        hin = torch.from_numpy(x.copy() if fwd else x.astype(np.uint16).view(np.int16)).pin_memory()
        if fwd:
            hout = torch.full((cap + 16,), 0x5A5A, dtype=torch.int16).pin_memory()
            r = ug.utf8_to_utf16le_host(hin, hout[:cap])
            o = hout.numpy().view(np.uint16)
            guard = 0x5A5A
        else:
            hout = torch.full((cap + 16,), 0x5A, dtype=torch.uint8).pin_memory()
            r = ug.utf16le_to_utf8_host(hin, hout[:cap])
            o = hout.numpy()
            guard = 0x5A
    finally:
        ug.set_host_chunk(prev)
    assert np.all(o[cap:] == guard), "wrote past out_cap"
    return r, o[: r.written if r.error >= 0 else 0]


def check_host(x: np.ndarray, chunk: int, cap=None):
    fwd = x.dtype == np.uint8
    ref_r, ref_o = (oracle.utf8_to_utf16le(x, out_cap=cap) if fwd
                    else oracle.utf16le_to_utf8(x, out_cap=cap))
    r, o = host_run(x, chunk, cap)
    assert tuple(r) == tuple(ref_r), (chunk, cap, r, ref_r)
    if r.error >= 0:
        assert np.array_equal(o, ref_o)
    return r


@pytest.mark.parametrize("chunk", [1, 7, 1000, 4099, 65536, 0])
def test_host_pipeline_chunks(c0, chunk):
    """The pipelined host path (chunks cut at character starts, one shard kernel each, outputs
    placed by the records' prefix) equals the oracle at any chunk size, both directions."""
    a = c0[: 3000] if chunk < 1000 else c0
    r = check_host(a, chunk)
    assert r.error == 0
    u = oracle.utf8_to_utf16le(a)[1]
    check_host(u, chunk)


def test_host_pipeline_errors_at_chunk_cuts(c0):
    """First errors injected within a few units of chunk cuts; data verdicts, positions and
    written counts match the oracle, and only the prefix before the error is delivered."""
    chunk = 4099
    rng = np.random.default_rng(np.random.SeedSequence([0, 0xF2, 1, 0]))
    for k, cls in enumerate(synth.UTF8_ERROR_CLASSES):
        for cut in (chunk * (3 + k), chunk * (40 + 7 * k)):
            b = c0.copy()
            p, _ = synth.inject_utf8_error(b, cut - 4, cut + 4, cls, rng)
            r = check_host(b, chunk)
            assert (r.error, r.position) == (synth.UTF8_EXPECTED_KIND[cls], p), (cls, r, p)
    u = synth.generate("c3", size=1 << 20)
    for cut in (3001 * 5, 3001 * 77):
        v = u.copy()
        p, _ = synth.inject_utf16_error(v, cut - 2, cut + 2, rng)
        r = check_host(v, 3001)
        assert (r.error, r.position) == (ug.SURROGATE, p)


def test_host_pipeline_capacity(c0):
    a = c0[: 300000]
    need = oracle.utf8_to_utf16le(a)[0].written
    for cap in (0, 1, need // 2, need - 1, need):
        check_host(a, 5000, cap=cap)
    b = a.copy()
    rng = np.random.default_rng(7)
    synth.inject_utf8_error(b, 150000, 160000, "stray_continuation", rng)
    wr = oracle.utf8_to_utf16le(b)[0].written
    for cap in (wr - 1, wr, wr + 1):
        check_host(b, 5000, cap=cap)
    u = oracle.utf8_to_utf16le(a)[1]
    need8 = oracle.utf16le_to_utf8(u)[0].written
    for cap in (0, need8 - 1, need8):
        check_host(u, 3333, cap=cap)


# ----------------------------------------------------------------------------- length reductions
@pytest.mark.parametrize("kind", ["uniform", "alphabet"])
def test_length_from_large_random(kind):
    """Both length reductions on inputs large enough for their unrolled grid-stride loops
    (> 3 x grid x 512 vectors), against the oracle, at an odd offset."""
    rng = np.random.default_rng(np.random.SeedSequence([0x1E, 16, len(kind)]))
    n = (64 << 20) + 13
    alpha = np.array([0x41, 0x7F, 0x80, 0x7FF, 0x800, 0xD7FF, 0xD800, 0xDBFF, 0xDC00, 0xDFFF,
                      0xE000, 0xFFFF], dtype=np.uint16)
    u = (rng.integers(0, 65536, n).astype(np.uint16) if kind == "uniform"
         else alpha[rng.integers(0, alpha.size, n)])
    _, t = to_dev(u, pad_before=3)
    assert ug.utf8_length_from_utf16le(t) == oracle.utf8_length_from_utf16le(u)
    b = u.view(np.uint8)
    _, t8 = to_dev(b, pad_before=5)
    assert ug.utf16_length_from_utf8(t8) == oracle.utf16_length_from_utf8(b)


# ----------------------------------------------------------------------------- UTF-16BE (f3)
def be_raw(u_native: np.ndarray) -> np.ndarray:
    """Memory words of the big-endian encoding of the code units u_native."""
    return np.frombuffer(u_native.astype(">u2").tobytes(), dtype="<u2").copy()


def check_utf16be(w: np.ndarray, offset=0, cap=None):
    """w: raw big-endian words as stored in memory."""
    ref_r, ref_o = oracle.utf16be_to_utf8(w, out_cap=cap)
    _, t = to_dev(w.astype(np.uint16), pad_before=offset, pad_after=32)
    cap_ = 3 * w.size if cap is None else cap
    big_out = torch.full((cap_ + 64,), 0x5A, dtype=torch.uint8, device=DEV)
    r = ug.utf16be_to_utf8(t, big_out[:cap_], out_cap=cap_)
    o = big_out.cpu().numpy()
    assert np.all(o[cap_:] == 0x5A), "wrote past out_cap"
    assert tuple(r) == tuple(ref_r), (r, ref_r)
    if r.error >= 0:
        assert np.array_equal(o[: r.written], ref_o)
    assert tuple(ug.utf16be_validate(t)) == tuple(oracle.utf16be_validate(w))
    assert ug.utf8_length_from_utf16be(t) == oracle.utf8_length_from_utf16be(w)
    return r


def check_utf8_be(a: np.ndarray, offset=0, cap=None):
    ref_r, ref_o = oracle.utf8_to_utf16be(a, out_cap=cap)
    _, t = to_dev(a, pad_before=offset, pad_after=64)
    cap_ = a.size if cap is None else cap
    big_out = torch.full((cap_ + 64,), 0x5A5A, dtype=torch.int16, device=DEV)
    r = ug.utf8_to_utf16be(t, big_out[:cap_], out_cap=cap_)
    o = big_out.cpu().numpy().view(np.uint16)
    assert np.all(o[cap_:] == 0x5A5A), "wrote past out_cap"
    assert tuple(r) == tuple(ref_r), (r, ref_r)
    if r.error >= 0:
        assert np.array_equal(o[: r.written], ref_o)
    return r


def test_utf16be_fuzz():
    rng = np.random.default_rng(0xBE)
    alpha = np.array([0x0041, 0x007F, 0x0080, 0x07FF, 0x0800, 0xD7FF, 0xD800, 0xDBFF, 0xDC00,
                      0xDFFF, 0xE000, 0xFFFF, 0x0100, 0x1234], dtype=np.uint16)
    for k in range(300):
        n = int(rng.integers(0, 200))
        cu = alpha[rng.integers(0, alpha.size, n)] if k % 2 else \
            rng.integers(0, 65536, n).astype(np.uint16)
        check_utf16be(be_raw(cu), offset=2 * int(rng.integers(0, 8)))


def test_utf8_to_utf16be_fuzz():
    rng = np.random.default_rng(0xBE8)
    for k in range(300):
        n = int(rng.integers(0, 300))
        a = np.frombuffer(synth.gen_chunk("mixed", "utf8", n, 98, k), dtype=np.uint8).copy()
        if n and k % 3 == 0:
            a[rng.integers(0, n)] = rng.integers(0x80, 0x100)
        check_utf8_be(a, offset=int(rng.integers(0, 16)))


@pytest.mark.parametrize("key", ["c0", "c1", "c3"])
def test_utf16be_configs(key):
    """Config text (several tiles, ragged tail) both ways in BE, element by element, plus an
    error copy, the ASCII warp paths (c1) and capacity clipping."""
    x = synth.generate(key, size=None if key == "c0" else (4 << 20) + (5 if key == "c1" else 6))
    if x.dtype == np.uint8:
        r = check_utf8_be(x, offset=3)
        assert r.error == 0
        u = oracle.utf8_to_utf16le(x)[1]
    else:
        u = x
    w = be_raw(u)
    assert check_utf16be(w, offset=2).error == 0
    v = u.copy()
    p, _ = synth.inject_utf16_error(v, v.size // 3, v.size // 3 + 999, np.random.default_rng(5))
    r = check_utf16be(be_raw(v))
    assert (r.error, r.position) == (ug.SURROGATE, p)
    need = oracle.utf16le_to_utf8(u)[0].written
    check_utf16be(w, cap=need - 1)
    if x.dtype == np.uint8:
        check_utf8_be(x, cap=u.size // 2)


def test_utf16be_async():
    x = synth.generate("c0")
    u = oracle.utf8_to_utf16le(x)[1]
    w = be_raw(u)
    _, tw = to_dev(w)
    _, t8 = to_dev(x)
    res = ug.result_buffer(DEV, 3)
    out8 = torch.zeros(3 * w.size, dtype=torch.uint8, device=DEV)
    out16 = torch.zeros(x.size, dtype=torch.int16, device=DEV)
    lens = torch.zeros(1, dtype=torch.int64, device=DEV)
    ug.utf16be_to_utf8_async(tw, out8, res)
    ug.utf16be_validate_async(tw, res, result_off=ug.RESULT_BYTES)
    ug.utf8_to_utf16be_async(t8, out16, res, result_off=2 * ug.RESULT_BYTES)
    ug.utf8_length_from_utf16be_async(tw, lens)
    torch.cuda.synchronize()
    r = ug.decode_results(res)
    assert tuple(r[0]) == (0, w.size, x.size) and tuple(r[1])[:2] == (0, w.size)
    assert tuple(r[2]) == (0, x.size, u.size) and int(lens[0]) == x.size
    assert bytes(out8[: x.size].cpu().numpy()) == x.tobytes()
    assert np.array_equal(out16[: u.size].cpu().numpy().view(np.uint16), w)


def test_utf16be_host_pipeline(c0):
    """UTF-16BE through the chunked host pipeline, both directions, small chunks (cuts inside
    surrogate pairs are backed off with the BE rule)."""
    u = oracle.utf8_to_utf16le(c0)[1]
    w = be_raw(u)
    prev = ug.set_host_chunk(4097)
    try:
        hin = torch.from_numpy(c0.copy()).pin_memory()
        h16 = torch.zeros(c0.size, dtype=torch.int16).pin_memory()
        r = ug.utf8_to_utf16be_host(hin, h16)
        assert tuple(r) == (0, c0.size, u.size)
        assert np.array_equal(h16[: u.size].numpy().view(np.uint16), w)
        hw = torch.from_numpy(w.view(np.int16).copy()).pin_memory()
        h8 = torch.zeros(3 * w.size, dtype=torch.uint8).pin_memory()
        r = ug.utf16be_to_utf8_host(hw, h8)
        assert tuple(r) == (0, w.size, c0.size) and bytes(h8[: c0.size].numpy()) == c0.tobytes()
        v = u.copy()
        p, _ = synth.inject_utf16_error(v, 4097 * 7 - 2, 4097 * 7 + 2, np.random.default_rng(3))
        hv = torch.from_numpy(be_raw(v).view(np.int16).copy()).pin_memory()
        r = ug.utf16be_to_utf8_host(hv, h8)
        assert tuple(r) == tuple(oracle.utf16be_to_utf8(be_raw(v))[0]) and r.position == p
    finally:
        ug.set_host_chunk(prev)


@pytest.mark.parametrize("G", [2, 5])
def test_utf16be_virtual_shards(c0, G):
    """BE reverse and BE validation as G shards of one buffer (cuts by the BE rule), records
    combined on the device: equal to the unsharded oracle, including an error near a cut."""
    u = oracle.utf8_to_utf16le(c0)[1]
    for inject in (False, True):
        v = u.copy()
        n = v.size
        if inject:
            c = (n // G) & ~15
            synth.inject_utf16_error(v, c - 2, c + 2, np.random.default_rng(G))
        w = be_raw(v)
        _, t = to_dev(w)
        cuts = [0] + [((k * (n // G)) & ~15) - ug.utf16be_cut_backoff(w, (k * (n // G)) & ~15)
                      for k in range(1, G)] + [n]
        recs = ug.record_buffer(DEV, 2 * G)
        outs = []
        for k in range(G):
            lo, hi = cuts[k], cuts[k + 1]
            out = torch.zeros(3 * max(hi - lo, 1), dtype=torch.uint8, device=DEV)
            ug.utf16be_to_utf8_shard_async(t, lo, hi - lo, min(lo, 1), min(n - hi, 1), lo, out,
                                           recs, rec_off=k * ug.RECORD_BYTES)
            ug.utf16be_validate_shard_async(t, lo, hi - lo, min(lo, 1), min(n - hi, 1), lo, recs,
                                            rec_off=(G + k) * ug.RECORD_BYTES)
            outs.append(out)
        res = ug.result_buffer(DEV, 2)
        ug.combine_records_async(recs, G, 0, n, res)
        ug.combine_records_async(recs[G * ug.RECORD_BYTES:], G, 0, n, res[ug.RESULT_BYTES:])
        torch.cuda.synchronize()
        r, rv = ug.decode_results(res)
        ref_r, ref_o = oracle.utf16be_to_utf8(w)
        assert tuple(r) == tuple(ref_r)
        assert tuple(rv)[:2] == tuple(oracle.utf16be_validate(w))[:2]
        if not inject:
            records = ug.decode_records(recs)
            got = np.concatenate([outs[k][: records[k].count].cpu().numpy() for k in range(G)])
            assert np.array_equal(got, ref_o)


# ----------------------------------------------------------------------------- randomized mix
def test_randomized_mix_all_entry_points():
    """60 random cases over every entry point: sizes spanning 0..~3 MiB (many tiles and a
    ragged tail), random start alignment, 0-3 injected errors of random classes, random output
    capacity (ample, exact, one short), LE and BE; each result and output prefix against the
    oracle."""
    rng = np.random.default_rng(np.random.SeedSequence([0x5EED, 60]))
    for case in range(60):
        n = int(rng.choice([0, 1, 7, 33, 1000, 16384, 16385, 70000, 1 << 20, 3 << 20]))
        n += int(rng.integers(0, 64)) if n > 64 else 0
        a = np.frombuffer(synth.gen_chunk("mixed", "utf8", n, 77, case), dtype=np.uint8).copy()
        nerr = int(rng.integers(0, 4)) if n > 200 else 0
        for _ in range(nerr):
            cls = synth.UTF8_ERROR_CLASSES[int(rng.integers(0, 5))]
            synth.inject_utf8_error(a, 0, max(0, a.size - 8), cls, rng)
        off = int(rng.integers(0, 16))
        need = oracle.utf8_to_utf16le(a)[0]
        cap_choice = int(rng.integers(0, 3))
        written = need.written if need.error >= 0 else 0
        cap = [None, written, max(0, written - 1)][cap_choice]
        be = bool(rng.integers(0, 2))
        if be:
            check_utf8_be(a, offset=off, cap=cap)
        else:
            check_utf8(a, offset=off, cap=cap)
        # the reverse direction on the valid prefix's units, with a lone surrogate sometimes
        u = oracle.utf8_to_utf16le(a)[1].copy()
        if u.size > 10 and rng.integers(0, 2):
            synth.inject_utf16_error(u, 0, u.size - 1, rng)
        offw = 2 * int(rng.integers(0, 8))
        if be:
            check_utf16be(be_raw(u), offset=offw)
        else:
            check_utf16(u, offset=offw)


def test_reverse_dense_3byte_text():
    """CJK text as UTF-16 (3 output bytes per word: a tile emits ~1.4x its size, near the
    stage's worst case).  Clean, with lone surrogates in the middle of a tile and at tile
    edges, and with the output capacity cut inside a tile; LE and BE."""
    x = synth.generate("c2b", size=(2 << 20) + 7)
    u = oracle.utf8_to_utf16le(x)[1]
    assert check_utf16(u).error == 0
    assert check_utf16be(be_raw(u), offset=2).error == 0
    rng = np.random.default_rng(0x2B)
    TILE_W = TILE // 2  # words per tile
    for centre in (TILE_W * 3 + TILE_W // 2, TILE_W * 7, TILE_W * 11 + TILE_W // 2 + 40):
        v = u.copy()
        p, _ = synth.inject_utf16_error(v, centre - 24, centre + 24, rng)
        r = check_utf16(v)
        assert (r.error, r.position) == (ug.SURROGATE, p)
        r = check_utf16be(be_raw(v))
        assert (r.error, r.position) == (ug.SURROGATE, p)
    need = oracle.utf16le_to_utf8(u)[0].written
    for cap in (3 * TILE_W * 5 // 2 + 1000, need - 1):
        check_utf16(u, cap=cap)


# ----------------------------------------------------------------------------- API hardening
def test_binding_bounds_and_slots():
    """The binding rejects n / out_cap beyond the tensors, shard halos outside the input and
    result / record slots outside their buffers, before any C call."""
    t = torch.zeros(64, dtype=torch.uint8, device=DEV)
    o = torch.zeros(64, dtype=torch.int16, device=DEV)
    with pytest.raises(ValueError, match="exceeds the input"):
        ug.utf8_to_utf16le(t, o, n=65)
    with pytest.raises(ValueError, match="out_cap"):
        ug.utf8_to_utf16le(t, o, out_cap=65)
    with pytest.raises(ValueError, match="exceeds the input"):
        ug.utf8_to_utf16le_shard_async(t, 10, 60, 0, 0, 0, o, ug.record_buffer(DEV, 1))
    with pytest.raises(ValueError, match="halos"):
        ug.utf8_to_utf16le_shard_async(t, 1, 10, 3, 0, 0, o, ug.record_buffer(DEV, 1))
    with pytest.raises(ValueError, match="slot"):
        ug.utf8_validate_async(t, ug.result_buffer(DEV, 1), result_off=8)
    with pytest.raises(ValueError, match="CUDA tensor"):
        ug.utf8_validate_async(t, torch.zeros(24, dtype=torch.uint8))
    r = ug.utf8_to_utf16le(t, o, n=10, out_cap=10)
    assert tuple(r) == (0, 10, 10)


def test_length_ex_on_device():
    import ctypes
    t = torch.zeros(7, dtype=torch.uint8, device=DEV)
    assert ug.utf16_length_from_utf8(t) == 7
    out = ctypes.c_uint64(9)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert ug.lib.ug_utf16_length_from_utf8_ex(ctypes.c_void_p(t.data_ptr()), 7,
                                               ctypes.byref(out), s) == ug.OK
    assert out.value == 7
    assert ug.lib.ug_utf16_length_from_utf8_ex(ctypes.c_void_p(0), 3, ctypes.byref(out),
                                               s) == ug.ERR_ARG and out.value == 0


def test_same_stream_threads_get_their_own_results():
    """Synchronous calls from several host threads on ONE stream (torch's default): each gets
    its own input's result (the workspace mutex spans launch -> read-back)."""
    import threading
    rng = np.random.default_rng(77)
    inputs = []
    for k in range(8):
        a = np.frombuffer(synth.gen_chunk("mixed", "utf8", 200000 + 1000 * k, 31, k),
                          dtype=np.uint8).copy()
        if k % 2:
            synth.inject_utf8_error(a, 1000, a.size - 8, "surrogate", rng)
        inputs.append(a)
    dev_in = [torch.from_numpy(a).to(DEV) for a in inputs]
    dev_out = [torch.empty(a.size, dtype=torch.int16, device=DEV) for a in inputs]
    want = [tuple(oracle.utf8_to_utf16le(a)[0]) for a in inputs]
    want_len = [oracle.utf16_length_from_utf8(a) for a in inputs]
    torch.cuda.synchronize()
    errs = []

    def worker(k):
        try:
            for _ in range(25):
                r = ug.utf8_to_utf16le(dev_in[k], dev_out[k], stream=0)
                if tuple(r) != want[k]:
                    errs.append((k, r, want[k]))
                v = ug.utf16_length_from_utf8(dev_in[k], stream=0)
                if v != want_len[k]:
                    errs.append((k, "len", v, want_len[k]))
        except Exception as e:  # noqa: BLE001
            errs.append((k, repr(e)))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs[:5]


def test_host_pipeline_streams_many_chunks_in_bounded_memory(c0):
    """f2 streaming: ~660 chunks (165x the 4 staging slots) through the bounded ring; the
    workspace stays O(chunk) and the result equals the oracle, with capacity guards, both
    directions."""
    a = np.concatenate([c0, c0[: 400000]])
    chunk = 2203
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()
    ug.lib.ug_release_workspaces()   # measure this call's allocations only
    r = check_host(a, chunk)
    assert r.error == 0
    held = ug.workspace_bytes(s)
    slot = (chunk + 3 + 6 + 15) + 2 * (chunk + 3) + 15
    nch = a.size // chunk + 2
    assert held <= 4 * slot + nch * 32 + (1 << 20), (held, slot)   # + status words / records
    u = oracle.utf8_to_utf16le(a)[1]
    check_host(u, chunk)
    need8 = oracle.utf16le_to_utf8(u)[0].written
    check_host(u, chunk, cap=need8 - 1)
    check_host(a, chunk, cap=r.written // 2)


# ----------------------------------------------------------------------------- C multi-GPU entry
@pytest.mark.parametrize("G", [1, 2, 5])
def test_sharded_c_entry_virtual_shards(c0, G):
    """ug_sharded_* (one process, record all-gather by device copies + a combine per shard):
    G shards on this device, clean and with errors injected near the cuts, both directions,
    against the oracle."""
    _, t = to_dev(c0)
    n = c0.size
    cuts = shard_plan(c0, G)

    def descs(tin, cuts, outs, halo):
        N = tin.numel()
        return [dict(t_in=tin, offset=cuts[k], n=cuts[k + 1] - cuts[k],
                     halo_before=min(cuts[k], halo), halo_after=min(N - cuts[k + 1], halo),
                     global_off=cuts[k], t_out=outs[k] if outs else None)
                for k in range(len(cuts) - 1)]
    outs = [torch.zeros(max(cuts[k + 1] - cuts[k], 1), dtype=torch.int16, device=DEV)
            for k in range(G)]
    r, offs = ug.sharded_utf8_to_utf16le(descs(t, cuts, outs, 3))
    ref_r, ref_o = oracle.utf8_to_utf16le(c0)
    assert tuple(r) == tuple(ref_r)
    got = np.concatenate([outs[k][: (offs[k + 1] if k + 1 < G else r.written) - offs[k]]
                          .cpu().numpy().view(np.uint16) for k in range(G)])
    assert np.array_equal(got, ref_o)
    v = ug.sharded_utf8_validate(descs(t, cuts, None, 3))
    assert tuple(v) == tuple(oracle.utf8_validate(c0))
    # reverse: shard the UTF-16 output at word cuts backed off a low surrogate
    u = ref_o
    tu = torch.from_numpy(u.view(np.int16).copy()).to(DEV)
    m = u.size
    wc = [0] + [((k * (m // G)) & ~15) - ug.utf16_cut_backoff(u, (k * (m // G)) & ~15)
                for k in range(1, G)] + [m]
    outs8 = [torch.zeros(3 * max(wc[k + 1] - wc[k], 1), dtype=torch.uint8, device=DEV)
             for k in range(G)]
    r2, offs2 = ug.sharded_utf16le_to_utf8(descs(tu, wc, outs8, 1))
    assert tuple(r2) == (0, m, n)
    back = b"".join(bytes(outs8[k][: (offs2[k + 1] if k + 1 < G else n) - offs2[k]]
                          .cpu().numpy()) for k in range(G))
    assert back == c0.tobytes()
    assert tuple(ug.sharded_utf16le_validate(descs(tu, wc, None, 1))) == (0, m, 0)
    # errors within 3 bytes of a cut
    rng = np.random.default_rng(np.random.SeedSequence([0, 0xC, G, 0]))
    for j in range(6):
        b = c0.copy()
        k = int(rng.integers(1, G)) if G > 1 else 0
        c = cuts[k] if G > 1 else int(rng.integers(8, n - 8))
        cls = synth.UTF8_ERROR_CLASSES[j % 5]
        p, _ = synth.inject_utf8_error(b, max(0, c - 3), c + 3, cls, rng)
        _, tb = to_dev(b)
        bc = shard_plan(b, G)
        outs = [torch.zeros(max(bc[k + 1] - bc[k], 1), dtype=torch.int16, device=DEV)
                for k in range(G)]
        rb, _ = ug.sharded_utf8_to_utf16le(descs(tb, bc, outs, 3))
        assert tuple(rb) == tuple(oracle.utf8_to_utf16le(b)[0]) and rb.position == p, (cls, rb)
        vb = ug.sharded_utf8_validate(descs(tb, bc, None, 3))
        assert (vb.error, vb.position) == (rb.error, p)
