"""GPU parity of f4: the planned UTF-8 -> UTF-16LE transcoder
with the keyed 12-byte decoder (`ug_utf8_to_utf16le_keyed_planned_async`), called through the
C-ABI binding after the ordinary plan pass, element by element against the oracle: sizes
around the planned tile, every input alignment, short strings straddling tile edges at every
phase, width-dense text of every width mix (all three key paths and the thread-edge
straddles), errors of every class, capacities, the BASELINE configs at reduced size and
config 4 at 256 MiB."""
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

TILE = ug.planned_tile_bytes()


def keyed_fwd(a: np.ndarray, cap=None, offset=0):
    _, t = to_dev(a, pad_before=offset, pad_after=64)
    cap = a.size if cap is None else cap
    big_out = torch.full((cap + 64,), 0x5A5A, dtype=torch.int16, device=DEV)
    r, ln = ug.utf8_to_utf16le_keyed_two_pass(t, big_out[:cap], n=a.size, out_cap=cap)
    o = big_out.cpu().numpy().view(np.uint16)
    assert np.all(o[cap:] == 0x5A5A), "wrote past out_cap"
    return r, o[: r.written if r.error >= 0 else 0]


def check(a, offset=0, cap=None):
    ref_r, ref_o = oracle.utf8_to_utf16le(a, out_cap=cap)
    r, o = keyed_fwd(a, cap=cap, offset=offset)
    assert tuple(r) == tuple(ref_r), (a[:48].tobytes().hex(), r, ref_r)
    if r.error >= 0:
        assert np.array_equal(o, ref_o)
    return r


def dense(widths, nbytes, seed):
    """Text of characters whose UTF-8 widths are drawn from `widths` (seeded)."""
    rng = np.random.default_rng(seed)
    lo = {1: 0x20, 2: 0x80, 3: 0x800, 4: 0x10000}
    hi = {1: 0x7F, 2: 0x7FF, 3: 0xFFFF, 4: 0x10FFFF}
    w = rng.choice(widths, size=nbytes)
    cps = [int(rng.integers(lo[x], hi[x] + 1)) for x in w]
    cps = [c if not 0xD800 <= c <= 0xDFFF else 0xE000 for c in cps]
    b = "".join(map(chr, cps)).encode("utf-8")[:nbytes]
    return np.frombuffer(b, dtype=np.uint8).copy()


@pytest.mark.parametrize("n", [1, 2, 3, 17, 1023, TILE - 1, TILE, TILE + 5, 3 * TILE + 7])
def test_keyed_small_sizes(n):
    a = np.frombuffer(synth.gen_chunk("mixed", "utf8", n, 11, n), dtype=np.uint8)
    for off in LEADS:
        check(a, offset=off)


@pytest.mark.parametrize("widths", [(1,), (2,), (3,), (4,), (1, 2), (1, 3), (1, 4), (2, 3),
                                    (2, 4), (3, 4), (1, 2, 3), (2, 3, 4), (1, 2, 3, 4)])
def test_keyed_width_mixes(widths):
    """Every key path, thread-edge straddles at every phase (a truncated tail, too)."""
    a = dense(widths, 3 * TILE + 77, seed=sum(10 ** i * w for i, w in enumerate(widths)))
    for off in (0, 1, 7):
        check(a, offset=off)
    check(a[: a.size - 1])  # a truncated last character (when it is multi-byte)


def test_keyed_phase_sweep_tile_edges():
    cases = short_cases()[::3]
    for i, c in enumerate(cases):
        c = np.frombuffer(c, dtype=np.uint8)
        lead = LEADS[i % len(LEADS)]
        for edge in (TILE, 2 * TILE):
            for ph in range(-4, 2):
                pre = edge - lead + ph
                a = np.concatenate([np.full(pre, 0x41, np.uint8), c,
                                    np.full(40, 0x42, np.uint8)])
                check(a, offset=lead)


def test_keyed_errors_every_class():
    a = synth.generate("c4", size=(8 << 20) + 4099)
    rng = np.random.default_rng(np.random.SeedSequence([0xF4]))
    for cls in synth.UTF8_ERROR_CLASSES:
        for _ in range(3):
            b = a.copy()
            p, _ = synth.inject_utf8_error(b, 0, b.size - 8, cls, rng)
            r = check(b)
            assert (r.error, r.position) == (synth.UTF8_EXPECTED_KIND[cls], p)


def test_keyed_capacity():
    a = np.frombuffer(synth.gen_chunk("mixed", "utf8", 300000, 3, 0), dtype=np.uint8)
    need = oracle.utf8_to_utf16le(a)[0].written
    for cap in (0, 1, 7, need // 2, need - 1, need):
        check(a, cap=cap)


@pytest.mark.parametrize("key", ["c1", "c2a", "c2b", "c3", "c4"])
def test_keyed_configs(key):
    size = (256 << 20) if key == "c4" else (16 << 20)
    x = synth.generate(key, size=size)
    if x.dtype != np.uint8:  # config 3 is UTF-16 input: its UTF-8 form
        x = oracle.utf16le_to_utf8(x)[1]
    check(x, offset=5)
