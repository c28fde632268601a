"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/unigpu.h
declares, and its host-side logic (cut back-off, record combine, argument checks that return
before touching the GPU) behaves as specified.  No compute calls need a GPU here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ug():
    import __graft_entry__
    __graft_entry__.build_library()
    import paper_2111_08692_b200 as ug
    return ug


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "unigpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([A-Za-z_][A-Za-z0-9_]*)\s*\(",
                       src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_north_star_names():
    names = declared_symbols()
    for n in ("utf8_validate", "utf16le_validate", "utf8_to_utf16le", "utf16le_to_utf8",
              "utf16_length_from_utf8", "utf8_length_from_utf16le"):
        assert n in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol(ug):
    lib = ctypes.CDLL(ug.LIB_PATH)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_and_names(ug):
    assert ug.lib.ug_abi_version() == 1
    assert ug.tile_bytes() == 16384  # NT (512 threads) x 32 bytes, csrc/device.cuh
    assert ug.planned_tile_bytes() == 8192  # NTP (256 threads) x 32 bytes
    assert ug.error_name(0) == "OK" and ug.error_name(6) == "Surrogate"
    assert ug.error_name(-3) == "OutputTooSmall"


def test_sass_is_sm100a_with_tma(ug):
    """The kernels are compiled for sm_100a and use TMA bulk copies (UBLKCP)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", ug.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "UBLKCP" in out and "PRMT" in out


def test_utf8_cut_backoff(ug):
    """back off over at most 3 continuation bytes."""
    s = "aé你\U0001F600".encode()  # 61 C3A9 E4BDA0 F09F9880
    starts = {0, 1, 3, 6}
    for at in range(len(s)):
        k = ug.utf8_cut_backoff(s, at)
        assert at - k in starts and 0 <= k <= 3, (at, k)
    # never further than 3, even over a run of continuation bytes
    run = bytes([0x41] + [0x80] * 6)
    assert ug.utf8_cut_backoff(run, 6) == 3
    # at the start of the buffer nothing is readable before the cut
    assert ug.utf8_cut_backoff(bytes([0x80, 0x80]), 0) == 0


def test_utf16_cut_backoff(ug):
    w = [0x41, 0xD83D, 0xDE00, 0x42]
    assert [ug.utf16_cut_backoff(w, i) for i in range(4)] == [0, 0, 1, 0]
    # the same text stored big-endian: memory words are the byte-swapped units
    be = [((x >> 8) | (x << 8)) & 0xFFFF for x in w]
    assert [ug.utf16be_cut_backoff(be, i) for i in range(4)] == [0, 0, 1, 0]
    assert ug.utf16be_cut_backoff(w, 2) == 0  # LE words read as BE are not low surrogates


def test_combine_records_host(ug):
    N = ug.NONE
    # three valid shards: offsets are exclusive prefixes of the counts
    recs = [(10, N, 0, 0, 0), (7, N, 0, 0, 0), (5, N, 0, 0, 0)]
    for rank, off in enumerate([0, 10, 17]):
        r, o = ug.combine_records_host(recs, rank, 100)
        assert r == (0, 100, 22) and o == off
    # errors on ranks 1 and 2: the smaller global offset wins; written adds the rank offset
    recs = [(10, N, 0, 0, 0), (7, 55, 3, 4, 0), (5, 60, 1, 2, 0)]
    r, o = ug.combine_records_host(recs, 2, 100)
    assert r == (4, 55, 13) and o == 17
    # a too-small buffer before the error owner makes the call OutputTooSmall
    recs = [(10, N, 0, 0, 1), (7, 55, 3, 4, 0)]
    r, _ = ug.combine_records_host(recs, 0, 100)
    assert r == (-3, 13, 0)
    # ... but not after it
    recs = [(10, 5, 2, 3, 0), (7, N, 0, 0, 1)]
    r, _ = ug.combine_records_host(recs, 0, 100)
    assert r == (3, 5, 2)


def test_argument_errors_need_no_gpu(ug):
    """API misuse is rejected on the host before any CUDA call."""
    null = None
    r = ug.lib.utf8_validate(ctypes.c_void_p(0), 5, ctypes.c_void_p(0))
    assert r.error == ug.ERR_ARG
    r = ug.lib.utf8_to_utf16le(ctypes.c_void_p(0), 5, ctypes.c_void_p(0), 0, ctypes.c_void_p(0))
    assert r.error == ug.ERR_ARG
    assert ug.lib.ug_utf8_validate_async(ctypes.c_void_p(16), 4, ctypes.c_void_p(0),
                                         ctypes.c_void_p(0)) == ug.ERR_ARG
    # empty input is OK without launching anything
    r = ug.lib.utf16le_to_utf8(ctypes.c_void_p(0), 0, ctypes.c_void_p(0), 0, ctypes.c_void_p(0))
    assert (r.error, r.position, r.written) == (0, 0, 0)
    assert null is None


def test_product_does_not_import_oracle():
    """The product package and the oracle share no code: neither imports / includes the
    other."""
    pkg = os.path.join(ROOT, "paper_2111_08692_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert not re.search(r'#include\s+".*oracle', txt), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".c", ".h", ".py")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2111_08692_b200", txt, re.M), f
            assert not re.search(r'#include\s+".*(unigpu|csrc)', txt), f


def test_argument_errors_exhaustive_need_no_gpu(ug):
    """Every documented API-misuse case of include/unigpu.h returns UG_ERR_ARG from the host
    checks, before any CUDA call (so also on a machine without a GPU)."""
    V, L = ctypes.c_void_p, ug.lib
    big = (1 << 38)  # one past the largest n
    odd = V(0x1001)
    for fn in (L.utf16le_validate, L.utf16be_validate):
        assert fn(odd, 4, V(0)).error == ug.ERR_ARG            # odd UTF-16 pointer
        assert fn(V(0), 4, V(0)).error == ug.ERR_ARG           # NULL with n > 0
        assert fn(V(0x1000), big, V(0)).error == ug.ERR_ARG    # n too large
    assert L.utf8_validate(V(0x1000), big, V(0)).error == ug.ERR_ARG
    for fn in (L.utf8_to_utf16le, L.utf8_to_utf16be):
        assert fn(V(0x1000), 4, odd, 4, V(0)).error == ug.ERR_ARG   # odd UTF-16 output
        assert fn(V(0x1000), 4, V(0), 4, V(0)).error == ug.ERR_ARG  # NULL output, cap > 0
        assert fn(V(0x1000), big, V(0x2000), 4, V(0)).error == ug.ERR_ARG
    for fn in (L.utf16le_to_utf8, L.utf16be_to_utf8):
        assert fn(odd, 4, V(0x2000), 12, V(0)).error == ug.ERR_ARG
        assert fn(V(0x1000), 4, V(0), 12, V(0)).error == ug.ERR_ARG
    for fn in (L.ug_utf8_to_utf16le_async, L.ug_utf8_to_utf16be_async):
        assert fn(V(0x1000), 4, odd, 4, V(0x3000), V(0)) == ug.ERR_ARG
        assert fn(V(0x1000), 4, V(0x2000), 4, V(0), V(0)) == ug.ERR_ARG   # no result slot
    for fn in (L.ug_utf16le_validate_async, L.ug_utf16be_validate_async):
        assert fn(odd, 4, V(0x3000), V(0)) == ug.ERR_ARG
    assert L.ug_utf16_length_from_utf8_async(V(0x1000), 4, V(0), V(0)) == ug.ERR_ARG
    assert L.ug_utf8_length_from_utf16be_async(odd, 4, V(0x3000), V(0)) == ug.ERR_ARG
    assert L.ug_utf8_to_utf16le_shard_async(V(0x1000), 4, 0, 0, 0, V(0x2000), 4, V(0),
                                            V(0)) == ug.ERR_ARG  # no record slot
    # host-buffer variants
    assert L.utf8_to_utf16le_host(V(0), 4, V(0x2000), 4, V(0)).error == ug.ERR_ARG
    assert L.utf8_to_utf16le_host(V(0x1000), 4, odd, 4, V(0)).error == ug.ERR_ARG
    assert L.utf16le_to_utf8_host(odd, 4, V(0x2000), 12, V(0)).error == ug.ERR_ARG
    assert L.utf16le_to_utf8_host(V(0x1000), big, V(0x2000), 12, V(0)).error == ug.ERR_ARG
    # n = 0 succeeds without touching memory or the GPU, whatever the pointers
    for fn in (L.utf8_to_utf16be, L.utf16be_to_utf8):
        r = fn(V(0), 0, V(0), 0, V(0))
        assert (r.error, r.position, r.written) == (0, 0, 0)


def test_binding_rejects_wrong_tensors(ug):
    """The Python binding refuses, before any C call, what the raw-pointer ABI cannot check: a
    CPU tensor for a device function (no CPU fallback), a host function given a CUDA tensor, a
    wrong element size (units would be miscounted) and non-contiguous views."""
    torch = pytest.importorskip("torch")
    b8, w16 = torch.zeros(8, dtype=torch.uint8), torch.zeros(8, dtype=torch.int16)
    with pytest.raises(ValueError, match="CUDA tensor"):
        ug.utf8_validate(b8)
    with pytest.raises(ValueError, match="CUDA tensor"):
        ug.utf16be_to_utf8(w16, b8)
    with pytest.raises(ValueError, match="1-byte"):
        ug.utf8_validate(w16)
    with pytest.raises(ValueError, match="2-byte"):
        ug.utf8_length_from_utf16le(b8)
    with pytest.raises(ValueError, match="2-byte"):
        ug.utf8_to_utf16le_host(b8, b8)
    with pytest.raises(ValueError, match="contiguous"):
        ug.utf8_to_utf16le_host(b8[::2], w16)
    with pytest.raises(TypeError):
        ug.utf8_validate(b"\x41")
    assert ug._expect("utf8_length_from_utf16be") == (2, None, False)
    assert ug._expect("utf8_to_utf16le_shard_async") == (1, 2, False)
    assert ug._expect("utf16le_to_utf8_host") == (2, 1, True)


def test_length_ex_error_channel_needs_no_gpu(ug):
    """ug_*_length_*_ex report API misuse as UG_ERR_ARG (the plain forms return 0, which is
    indistinguishable from an empty count) and leave *len = 0."""
    V, L = ctypes.c_void_p, ug.lib
    out = ctypes.c_uint64(77)
    assert L.ug_utf16_length_from_utf8_ex(V(0), 5, ctypes.byref(out), V(0)) == ug.ERR_ARG
    assert out.value == 0
    assert L.ug_utf8_length_from_utf16le_ex(V(0x1001), 4, ctypes.byref(out), V(0)) == ug.ERR_ARG
    assert L.ug_utf8_length_from_utf16be_ex(V(0x1000), 4, V(0), V(0)) == ug.ERR_ARG  # no len
    assert L.ug_utf16_length_from_utf8_ex(V(0x1000), (1 << 62) + 1, ctypes.byref(out),
                                          V(0)) == ug.ERR_ARG
    out.value = 5
    assert L.ug_utf16_length_from_utf8_ex(V(0), 0, ctypes.byref(out), V(0)) == ug.OK
    assert out.value == 0


def test_sharded_c_entry_argument_errors_need_no_gpu(ug):
    """ug_sharded_*: no shards / too many / shards out of order are UG_ERR_ARG on the host."""
    import ctypes as C
    assert ug.lib.ug_sharded_utf8_validate(C.c_void_p(0), 1).error == ug.ERR_ARG
    arr = (ug._CShardDesc * 2)()
    arr[0].in_, arr[0].n, arr[0].in_global_offset = 0x1000, 10, 0
    arr[1].in_, arr[1].n, arr[1].in_global_offset = 0x2000, 10, 11   # gap: not in order
    assert ug.lib.ug_sharded_utf8_validate(C.cast(arr, C.c_void_p), 2).error == ug.ERR_ARG
    assert ug.lib.ug_sharded_utf8_validate(C.cast(arr, C.c_void_p), 0).error == ug.ERR_ARG
    assert ug.lib.ug_sharded_utf16le_to_utf8(C.cast(arr, C.c_void_p), 2000,
                                             C.c_void_p(0)).error == ug.ERR_ARG
