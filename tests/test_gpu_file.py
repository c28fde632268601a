"""GPU parity of the f2 file form ("input ... on NVMe"):
`ug_utf8_to_utf16le_file` / `ug_utf16le_to_utf8_file` stream a file through bounded memory in
segments cut at character starts.  Small segments and host chunks force many segments and many
chunks per segment; results and output files are compared with the oracle: valid text both
ways (a round trip), every UTF-8 error class within 3 bytes of a segment cut, a truncated
character at the end of the file, a lone surrogate at a cut, an empty file, and the argument
errors (missing file, odd-sized UTF-16 file)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2111_08692_b200 as ug  # noqa: E402

SEG = 1 << 20      # file segment (input units)
CHUNK = 256 << 10  # host pipeline chunk (input units)


@pytest.fixture(autouse=True)
def small_segments():
    p_seg, p_ch = ug.set_file_segment(SEG), ug.set_host_chunk(CHUNK)
    yield
    ug.set_file_segment(p_seg)
    ug.set_host_chunk(p_ch)


def fwd_file(tmp_path, a: np.ndarray):
    src, dst = tmp_path / "in8", tmp_path / "out16"
    src.write_bytes(a.tobytes())
    r = ug.utf8_to_utf16le_file(src, dst)
    return r, np.frombuffer(dst.read_bytes(), dtype=np.uint16)


def rev_file(tmp_path, u: np.ndarray):
    src, dst = tmp_path / "in16", tmp_path / "out8"
    src.write_bytes(u.astype(np.uint16).tobytes())
    r = ug.utf16le_to_utf8_file(src, dst)
    return r, np.frombuffer(dst.read_bytes(), dtype=np.uint8)


def test_file_round_trip(tmp_path):
    a = synth.generate("c4", size=(5 << 20) + 12345)
    ref_r, ref_o = oracle.utf8_to_utf16le(a)
    r, o = fwd_file(tmp_path, a)
    assert tuple(r) == tuple(ref_r) and np.array_equal(o, ref_o)
    r2, o2 = rev_file(tmp_path, o)
    assert tuple(r2) == tuple(oracle.utf16le_to_utf8(o)[0]) and np.array_equal(o2, a)


@pytest.mark.parametrize("cls", synth.UTF8_ERROR_CLASSES)
def test_file_errors_at_segment_cuts(tmp_path, cls):
    base = synth.generate("c4", size=(3 << 20) + 777)
    rng = np.random.default_rng(np.random.SeedSequence([0xF2, len(cls)]))
    for cut in (SEG, 2 * SEG):
        a = base.copy()
        p, _ = synth.inject_utf8_error(a, cut - 3, cut + 3, cls, rng)
        ref_r, ref_o = oracle.utf8_to_utf16le(a)
        r, o = fwd_file(tmp_path, a)
        assert tuple(r) == tuple(ref_r), (cls, cut, p, r, ref_r)
        assert (r.error, r.position) == (synth.UTF8_EXPECTED_KIND[cls], p)
        assert np.array_equal(o, ref_o[: r.written])


def test_file_large_segments(tmp_path):
    """Segments of 9 Mi units (reads / writes split over the I/O threads, >= 8 MiB each) and a
    file that is not a multiple of them, both directions, exact to the last byte."""
    p = ug.set_file_segment(9 << 20)
    try:
        a = synth.generate("c4", size=(29 << 20) + 4097)
        ref_r, ref_o = oracle.utf8_to_utf16le(a)
        r, o = fwd_file(tmp_path, a)
        assert tuple(r) == tuple(ref_r) and np.array_equal(o, ref_o)
        r2, o2 = rev_file(tmp_path, o)
        assert tuple(r2) == tuple(oracle.utf16le_to_utf8(o)[0]) and np.array_equal(o2, a)
    finally:
        ug.set_file_segment(p)


def test_file_truncated_at_end(tmp_path):
    a = np.concatenate([synth.generate("c0"), np.frombuffer("€".encode()[:2], np.uint8)])
    ref_r, ref_o = oracle.utf8_to_utf16le(a)
    r, o = fwd_file(tmp_path, a)
    assert tuple(r) == tuple(ref_r) and r.error == ug.TOO_SHORT
    assert np.array_equal(o, ref_o[: r.written])


def test_file_lone_surrogate_at_cut(tmp_path):
    a = synth.generate("c4", size=(2 << 20) + 99)
    u = oracle.utf8_to_utf16le(a)[1].copy()
    rng = np.random.default_rng(7)
    p, _ = synth.inject_utf16_error(u, SEG - 1, SEG + 1, rng)
    ref_r, ref_o = oracle.utf16le_to_utf8(u)
    r, o = rev_file(tmp_path, u)
    assert tuple(r) == tuple(ref_r) and (r.error, r.position) == (ug.SURROGATE, p)
    assert np.array_equal(o, ref_o[: r.written])


def test_file_empty_and_errors(tmp_path):
    r, o = fwd_file(tmp_path, np.zeros(0, np.uint8))
    assert tuple(r) == (0, 0, 0) and o.size == 0
    missing = tmp_path / "does-not-exist"
    assert ug.utf8_to_utf16le_file(missing, tmp_path / "x").error == ug.ERR_ARG
    odd = tmp_path / "odd16"
    odd.write_bytes(b"abc")
    assert ug.utf16le_to_utf8_file(odd, tmp_path / "y").error == ug.ERR_ARG
