"""GPU parity of the streaming UTF-16 validator (k_validate16: 16-byte chunks per lane, four per
lane in flight, 2 KiB warp rounds, the pairing rule) against the oracle: every
error class (lone high, lone low, high at the end, low at the start) at every word phase around
chunk, warp-round and CTA-round boundaries, at every even address phase, LE and BE, and
through the shard form with halos (a pair split by the cut).  Needs a B200."""
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
CHUNK_W = 8          # words per 16-byte chunk
ROUND_W = 32 * 4 * CHUNK_W   # words per warp round (32 lanes x 4 chunks)


def valid_text(n_words, seed):
    """Valid mixed UTF-16 (the config-4 recipe of synth, converted by the oracle)."""
    lo = seed * 4096
    a = synth.generate_range("c4", lo, lo + 4 * n_words + 64)
    # whole characters only: from the first lead byte to the last one (exclusive)
    lead = np.nonzero((a & 0xC0) != 0x80)[0]
    a = a[lead[0]:lead[-1]]
    r, u = oracle.utf8_to_utf16le(a)
    assert r.error == 0 and len(u) >= n_words
    u = np.asarray(u[:n_words], dtype=np.uint16).copy()
    if n_words and (u[-1] & 0xFC00) == 0xD800:  # do not end on half a pair
        u[-1] = 0x0041
    return u


def run(u, off_words, be=False):
    big = np.full(off_words + u.size + 16, 0xD800, dtype=np.uint16)  # guards: lone highs
    big[off_words:off_words + u.size] = u
    if be:
        big = big.byteswap()
    t = torch.from_numpy(big.view(np.int16)).to(DEV)[off_words:off_words + u.size]
    return tuple(ug.utf16be_validate(t) if be else ug.utf16le_validate(t))


def ref(u):
    return tuple(oracle.utf16le_validate(u))


@pytest.mark.parametrize("off", [0, 1, 3, 7])
def test_lone_surrogates_at_boundaries(off):
    base = valid_text(3 * ROUND_W + 77, 11)
    # strip pairs so that insertions below are the only surrogates near the probe
    base[(base & 0xF800) == 0xD800] = 0x20AC
    cuts = []
    for b in (CHUNK_W, 2 * CHUNK_W, ROUND_W, 2 * ROUND_W):
        for d in range(-3, 4):
            cuts.append(b - off + d)
    for p in sorted(set(c for c in cuts if 0 <= c < base.size)):
        for kind in ("high", "low", "pair_ok", "high_high"):
            u = base.copy()
            if kind == "high":
                u[p] = 0xD83D
            elif kind == "low":
                u[p] = 0xDE00
            elif kind == "pair_ok":
                if p + 1 >= u.size:
                    continue
                u[p], u[p + 1] = 0xD83D, 0xDE00
            else:
                if p + 1 >= u.size:
                    continue
                u[p], u[p + 1] = 0xD83D, 0xD83D
            want = ref(u)
            assert run(u, off) == want, (p, kind, off)


@pytest.mark.parametrize("n", [0, 1, 2, 7, 8, 9, 15, 16, 17, 1023, 1024, 1025, 4097, 70000])
def test_sizes_and_ends(n):
    u = valid_text(max(n, 1), 5)[:n].copy()
    for off in (0, 5):
        assert run(u, off) == ref(u)
        if n:
            v = u.copy()
            v[-1] = 0xD801  # high at the end: the word at n reads as 0 (no halo)
            assert run(v, off) == ref(v)
            v = u.copy()
            v[0] = 0xDC01  # low at the start: the word before reads as 0
            assert run(v, off) == ref(v)


def test_random_dense_surrogates_le_be():
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(1, 9000))
        pool = np.array([0x41, 0x20AC, 0xD83D, 0xDE00, 0xDBFF, 0xDC00, 0xFFFF], np.uint16)
        u = pool[rng.integers(0, pool.size, n)]
        # mostly valid: pair up where possible, then sprinkle one error
        u = valid_text(n, trial + 100) if trial % 2 else u
        if trial % 2:
            u[int(rng.integers(0, n))] = pool[int(rng.integers(2, 6))]
        off = int(rng.integers(0, 8))
        want = ref(u)
        assert run(u, off) == want
        assert run(u, off, be=True) == want


def test_large_valid_and_late_error():
    u = valid_text(3_000_000, 3)
    assert run(u, 0) == ref(u)
    for p in (u.size - 1, u.size // 2 + 3, 123457):
        v = u.copy()
        v[p] = 0xDFFF if v[p - 1] & 0xFC00 != 0xD800 else 0x0041
        if v[p] == 0x0041:  # broke a pair: the high before p is now lone
            pass
        assert run(v, 3) == ref(v)


def test_shard_halos_split_pair():
    """The shard form: a pair split by a cut is valid through the halos; a lone high at the
    shard's last word is an error only when the next shard does not start with a low."""
    u = valid_text(20000, 9)
    t = torch.from_numpy(u.view(np.int16)).to(DEV)
    pairs = np.nonzero((u[:-1] & 0xFC00) == 0xD800)[0]
    cut = int(pairs[len(pairs) // 2]) + 1  # between the high and its low
    n = u.size
    for v in (u, u.copy()):
        if v is not u:
            v[cut] = 0x0041  # the high before the cut is now lone: error at cut - 1
            t = torch.from_numpy(v.view(np.int16)).to(DEV)
        recs = ug.record_buffer(DEV, 2)
        for r, (lo, hi) in enumerate(((0, cut), (cut, n))):
            ug.utf16le_validate_shard_async(t, lo, hi - lo, min(lo, 1), min(n - hi, 1), lo,
                                            recs, rec_off=r * ug.RECORD_BYTES)
        res = ug.result_buffer(DEV, 1)
        ug.combine_records_async(recs, 2, 0, n, res)
        torch.cuda.synchronize()
        (rv,) = ug.decode_results(res)
        assert tuple(rv)[:2] == ref(v)[:2]
