"""GPU parity at BASELINE.json's full sizes (tier T1, large).  Configs 1-3 are compared with the
oracle element by element; config 4 (8 GiB, > 2^32 output units) is checked in the launch
configuration bench.py times (the shard call at G = 1) on sampled 64 MiB generator chunks against
the oracle, plus properties that hold at any size (round trip = identity, written = length
function, injected errors exact).  Each 64 MiB generator chunk is whole valid text, so chunk
boundaries are character boundaries."""
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
    rng = np.random.default_rng(np.random.SeedSequence([4, 0xE, 1, 0]))
    for _ in range(2):
        v = u.copy()
        p, _ = synth.inject_utf16_error(v, 0, v.size - 1, rng)
        tv = torch.from_numpy(v.view(np.int16)).to(DEV)
        rv = ug.utf16le_to_utf8(tv, out8)
        assert tuple(rv) == tuple(oracle.utf16le_to_utf8(v)[0])
        assert (rv.error, rv.position) == (ug.SURROGATE, p)
        assert tuple(ug.utf16le_validate(tv)) == (ug.SURROGATE, p, 0)


@pytest.fixture(scope="module")
def c4():
    return synth.generate("c4")


def chunk_units_gpu(t, nchunks):
    """UTF-16 length of each 64 MiB chunk (product length kernel on character-aligned
    sub-ranges)."""
    C = synth.CHUNK
    return [ug.utf16_length_from_utf8(t[c * C:(c + 1) * C]) for c in range(nchunks)]


def test_config4_full_size_bench_launch(c4):
    n = c4.size
    t = torch.from_numpy(c4).to(DEV)
    out16 = torch.empty(n, dtype=torch.int16, device=DEV)
    rec = ug.record_buffer(DEV, 1)
    # bench.py's launch at G = 1: the shard call over the whole buffer, no halos
    ug.utf8_to_utf16le_shard_async(t, 0, n, 0, 0, 0, out16, rec)
    torch.cuda.synchronize()
    r = ug.decode_records(rec)[0]
    assert r.first_err == ug.NONE and r.too_small == 0
    n16 = r.count
    assert n16 > 2 ** 32                       # 64-bit offsets exercised
    assert ug.utf16_length_from_utf8(t) == n16
    lens = chunk_units_gpu(t, n // synth.CHUNK)
    assert sum(lens) == n16
    offs = np.concatenate([[0], np.cumsum(lens)])
    rng = np.random.default_rng(45)
    picks = sorted(set([0, len(lens) - 1] + rng.integers(1, len(lens) - 1, 3).tolist()))
    for c in picks:
        x = c4[c * synth.CHUNK:(c + 1) * synth.CHUNK]
        ref = oracle.utf8_to_utf16le(x)[1]
        got = out16[int(offs[c]):int(offs[c + 1])]
        assert torch.equal(got, torch.from_numpy(ref.view(np.int16)).to(DEV)), c
    # reverse through the shard call as well, then the round trip is the identity
    back = torch.empty(n, dtype=torch.uint8, device=DEV)
    ug.utf16le_to_utf8_shard_async(out16[:n16], 0, n16, 0, 0, 0, back, rec)
    torch.cuda.synchronize()
    r2 = ug.decode_records(rec)[0]
    assert r2.first_err == ug.NONE and r2.count == n
    assert torch.equal(back, t)
    # the plain API agrees
    assert tuple(ug.utf8_to_utf16le(t, out16)) == (0, n, n16)


def test_config4_error_copies_near_shard_cuts(c4):
    """BASELINE config 4's error copies: one injected error within 3 bytes of an 8-way shard
    cut; unsharded call on the full 8 GiB gives e = p, the injected kind, and written = units
    before p (GPU lengths of whole chunks + the oracle on the partial chunk)."""
    n = c4.size
    t = torch.from_numpy(c4).to(DEV)
    out16 = torch.empty(n, dtype=torch.int16, device=DEV)
    G = 8
    rng = np.random.default_rng(np.random.SeedSequence([5, 0xE, G, 0]))
    for j in range(3):
        k = int(rng.integers(1, G))
        c = (k * (n // G)) & ~15
        cls = synth.UTF8_ERROR_CLASSES[int(rng.integers(0, 5))]
        p, saved = synth.inject_utf8_error(c4, c - 3, c + 3, cls, rng)
        t[p:p + saved.size] = torch.from_numpy(c4[p:p + saved.size].copy()).to(DEV)
        try:
            r = ug.utf8_to_utf16le(t, out16)
            C = synth.CHUNK
            ch = p // C
            before = ug.utf16_length_from_utf8(t[:ch * C])
            part = oracle.utf8_to_utf16le(c4[ch * C:p])[0].written
            assert (r.error, r.position, r.written) == \
                (synth.UTF8_EXPECTED_KIND[cls], p, before + part), (cls, r, p)
            v = ug.utf8_validate(t)
            assert (v.error, v.position) == (synth.UTF8_EXPECTED_KIND[cls], p)
        finally:
            c4[p:p + saved.size] = saved
            t[p:p + saved.size] = torch.from_numpy(saved).to(DEV)
