"""Pins for the oracle (tier T0, CPU only).

Each test ties oracle/oracle.c to something OTHER than itself:
  * the worked examples printed in SPEC.md (tests/golden/spec_examples.json, each cited);
  * CPython's strict codecs (bytes.decode / str.encode), an independent library routine;
  * closed forms: the valid-string recurrence V(n), partition counts, composition of the
    first-error histograms, the two-word UTF-16 counts;
  * invariants: round trips, output-length laws, capacity behaviour.
A plausible slip anywhere in the oracle (a dropped rule, a wrong mask or shift, an off-by-one
at the end of the buffer, a transposed pair) fails at least one of these.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from oracle import (HEADER_BITS, OK, OUTPUT_TOO_SMALL, OVERLONG, SURROGATE, TOO_LARGE,
                    TOO_LONG, TOO_SHORT)

KIND = {"OK": OK, "HeaderBits": HEADER_BITS, "TooShort": TOO_SHORT, "TooLong": TOO_LONG,
        "Overlong": OVERLONG, "TooLarge": TOO_LARGE, "Surrogate": SURROGATE}

# per-character counts of valid UTF-8 sequences by length:
# 128 one-byte, 0x800-0x80 two-byte, 0x10000-0x800-0x800 (surrogates) three-byte,
# 0x110000-0x10000 four-byte.
CHAR_COUNTS = (128, 1920, 61440, 1048576)


def V(n):
    """Number of valid UTF-8 strings of n bytes: concatenations of valid characters."""
    v = [1]
    for k in range(1, n + 1):
        v.append(sum(c * v[k - j - 1] for j, c in enumerate(CHAR_COUNTS) if k - j - 1 >= 0))
    return v[n]


def h(s):
    return bytes.fromhex(s)


def w16(ws):
    return np.array([int(x, 16) for x in ws], dtype=np.uint16)


# ------------------------------------------------------------------ worked examples
def test_spec_decode_encode_examples(golden):
    for ex in golden["decode_utf8_at"]:
        k, cp, ln = oracle.decode_utf8_at(h(ex["bytes"]), 0)
        if "kind" in ex:
            assert k == KIND[ex["kind"]], ex
        else:
            assert (k, cp, ln) == (0, int(ex["cp"], 16), ex["len"]), ex
    for ex in golden["encode_utf8"]:
        assert oracle.encode_utf8(int(ex["cp"], 16)) == h(ex["bytes"]), ex
    for ex in golden["decode_utf16_at"]:
        k, cp, ln = oracle.decode_utf16_at(w16(ex["words"]), 0)
        if "kind" in ex:
            assert k == KIND[ex["kind"]], ex
        else:
            assert (k, cp, ln) == (0, int(ex["cp"], 16), ex["len"]), ex
    for ex in golden["encode_utf16"]:
        assert oracle.encode_utf16(int(ex["cp"], 16)) == [int(x, 16) for x in ex["words"]], ex


def test_spec_lead_examples(golden):
    for ex in golden["utf8_sequence_length"]:
        b = int(ex["byte"], 16)
        if "kind" in ex:
            k, _, _ = oracle.decode_utf8_at(bytes([b, 0x80, 0x80, 0x80]), 0)
            assert k == KIND[ex["kind"]]
        else:
            # the decoder asks for exactly len-1 continuation bytes: valid with them
            assert lead_length(b) == ex["len"]


def lead_length(b):
    """Sequence length the oracle assigns to lead byte b: 1 + the number of continuation
    bytes after which it stops reporting TooShort."""
    k, _, _ = oracle.decode_utf8_at(bytes([b]), 0)
    if k == 0:
        return 1
    if k in (TOO_LONG, HEADER_BITS):
        return k and -k
    for m in range(1, 4):
        k, _, _ = oracle.decode_utf8_at(bytes([b] + [0xBF] * m), 0)
        if k != TOO_SHORT:
            return m + 1
    raise AssertionError(b)


def test_lead_partition(golden):
    """256 lead bytes split 128/32/16/8 and 64 TooLong, 8 HeaderBits."""
    part = golden["partitions"]["utf8_lead_classes"]
    counts = {}
    for b in range(256):
        L = lead_length(b)
        key = {-TOO_LONG: "TooLong", -HEADER_BITS: "HeaderBits"}.get(L, str(L))
        counts[key] = counts.get(key, 0) + 1
    assert counts == {k: v for k, v in part.items() if k != "cite"}


def test_utf16_partition(golden):
    """63488 BMP words, 1024 high and 1024 low surrogates."""
    part = golden["partitions"]["utf16_words"]
    lone = sum(1 for w in range(65536)
               if oracle.decode_utf16_at(np.array([w], np.uint16), 0)[0] == SURROGATE)
    highs = sum(1 for w in range(65536)
                if oracle.decode_utf16_at(np.array([w, 0xDC00], np.uint16), 0)[2] == 2)
    assert lone == part["high"] + part["low"]
    assert highs == part["high"]
    assert 65536 - lone == part["bmp"]


def test_spec_transcode_examples(golden):
    for ex in golden["utf8_to_utf16le"]:
        r, out = oracle.utf8_to_utf16le(h(ex["in"]))
        assert r.error == KIND[ex["kind"]] and r.position == ex["position"], ex
        assert out.tolist() == [int(x, 16) for x in ex["out"]], ex
        assert oracle.utf8_validate(h(ex["in"]))[:2] == (r.error, r.position)
    ex = golden["utf8_surrogate_at_1000"]
    s = b"a" * ex["prefix_ascii"] + h(ex["bytes"])
    r = oracle.utf8_validate(s)
    assert (r.error, r.position) == (KIND[ex["kind"]], ex["position"])
    for ex in golden["utf16le_to_utf8"]:
        r, out = oracle.utf16le_to_utf8(w16(ex["in"]))
        assert r.error == KIND[ex["kind"]] and r.position == ex["position"], ex
        assert out.tobytes() == h(ex["out"]), ex
        assert oracle.utf16le_validate(w16(ex["in"]))[:2] == (r.error, r.position)


# ------------------------------------------------------------------ exhaustive vs CPython
def cpython_offset8(b: bytes) -> int:
    try:
        b.decode("utf-8")
        return -1
    except UnicodeDecodeError as e:
        return e.start


@pytest.mark.parametrize("length", [1, 2, 3])
def test_exhaustive_offsets_vs_cpython(length):
    """Every 1-, 2- and 3-byte string: verdict and first-error offset equal CPython's strict
    UTF-8 decoder (UnicodeDecodeError.start), string by string."""
    off, kind = oracle.sweep_utf8_offsets(length)
    ref = np.empty(256 ** length, dtype=np.int8)
    for x in range(256 ** length):
        ref[x] = cpython_offset8(x.to_bytes(length, "big"))
    bad = np.nonzero(off != ref)[0]
    assert bad.size == 0, [(hex(int(x)), int(off[x]), int(ref[x])) for x in bad[:10]]
    assert int((off == -1).sum()) == V(length)
    assert np.all((kind == 0) == (off == -1))


def test_kind_histograms_small():
    """Kind histograms under the precedence reading R2.  These pin the
    precedence proposal, and the per-rule counts below are closed forms."""
    exp = {1: {OK: 128, TOO_LONG: 64, TOO_SHORT: 56, HEADER_BITS: 8},
           2: {OK: 18304, TOO_LONG: 24576, TOO_SHORT: 19456, HEADER_BITS: 3072, OVERLONG: 128},
           3: {OK: 2650112, TOO_LONG: 7462912, TOO_SHORT: 5678080, HEADER_BITS: 932864,
               OVERLONG: 51200, SURROGATE: 2048}}
    for length, e in exp.items():
        hk, ho = oracle.sweep_utf8(length)
        got = {k: int(v) for k, v in enumerate(hk) if v}
        assert got == e, (length, got)
    # closed forms: a lone 2-byte string C0/C1 + continuation is the only overlong (2*64)
    assert exp[2][OVERLONG] == 2 * 64
    # 3-byte surrogates: ED A0..BF 80..BF = 32*64
    assert exp[3][SURROGATE] == 32 * 64
    # 3-byte overlongs: C0/C1 cont, any (2*64*256) + E0 80..9F 80..BF (32*64)
    #                  + ASCII then C0/C1 cont (128*2*64)
    assert exp[3][OVERLONG] == 2 * 64 * 256 + 32 * 64 + 128 * 2 * 64


@pytest.mark.slow
def test_four_byte_sweep_closed_form():
    """All 2^32 four-byte strings.  Valid = V(4); first-error offsets compose from the shorter
    pinned histograms: offset k errors = V(k) * (#(4-k)-byte strings failing at 0)."""
    nparts = 64
    with ThreadPoolExecutor(8) as ex:
        parts = list(ex.map(lambda p: oracle.sweep_utf8(4, p, nparts), range(nparts)))
    hk = sum(p[0] for p in parts)
    ho = sum(p[1] for p in parts)
    assert int(hk[OK]) == V(4) == 383270912
    fail0 = {1: 128, 2: 30848, 3: 7835648}  # pinned against CPython above
    assert int(ho[3]) == V(3) * fail0[1]
    assert int(ho[2]) == V(2) * fail0[2]
    assert int(ho[1]) == V(1) * fail0[3]
    assert int(ho.sum()) + V(4) == 2 ** 32
    # rule 5 and rule 6 counts among 4-byte strings (closed forms)
    assert int(hk[TOO_LARGE]) == 48 * 64 ** 2 + 3 * 64 ** 3
    assert int(hk[SURROGATE]) == 32 * 64 * 256 + 128 * 32 * 64


def test_two_byte_offsets_hist():
    hk, ho = oracle.sweep_utf8(2)
    assert (int(ho[0]), int(ho[1])) == (30848, 16384)


# ------------------------------------------------------------------ all scalar values
def all_scalars():
    cps = np.arange(0x110000, dtype=np.uint32)
    return cps[(cps < 0xD800) | (cps > 0xDFFF)]


def test_all_scalars_round_trip_vs_cpython():
    """All 1,112,064 scalar values: the oracle's transcoders equal CPython's encoders in both
    directions, and decode(encode(cp)) = cp."""
    cps = all_scalars()
    assert cps.size == 1112064 == sum(CHAR_COUNTS)
    text = cps.astype("<u4").tobytes().decode("utf-32-le")
    u8 = text.encode("utf-8")
    u16 = np.frombuffer(text.encode("utf-16-le"), dtype="<u2")
    r, out16 = oracle.utf8_to_utf16le(u8)
    assert r == (OK, len(u8), u16.size)
    assert np.array_equal(out16, u16)
    r, out8 = oracle.utf16le_to_utf8(u16)
    assert r == (OK, u16.size, len(u8))
    assert out8.tobytes() == u8
    assert oracle.utf16_length_from_utf8(u8) == u16.size
    assert oracle.utf8_length_from_utf16le(u16) == len(u8)
    # per-character primitives on a stride through every range (incl. all boundaries)
    picks = np.unique(np.concatenate([cps[::997], [0, 0x7F, 0x80, 0x7FF, 0x800, 0xD7FF, 0xE000,
                                                   0xFFFF, 0x10000, 0x10FFFF]]))
    for cp in picks.tolist():
        b = chr(cp).encode("utf-8")
        assert oracle.encode_utf8(cp) == b
        assert oracle.decode_utf8_at(b, 0) == (0, cp, len(b))
        w = np.frombuffer(chr(cp).encode("utf-16-le"), dtype="<u2")
        assert oracle.encode_utf16(cp) == w.tolist()
        assert oracle.decode_utf16_at(w, 0) == (0, cp, w.size)
    for cp in (0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0x110000, 0xFFFFFFFF):
        assert oracle.encode_utf8(cp) is None and oracle.encode_utf16(cp) is None


# ------------------------------------------------------------------ UTF-16 closed forms
@pytest.mark.slow
def test_utf16_all_pairs_closed_form():
    """All 2^32 two-word strings: valid = 63488^2 + 1024^2; first error at 0
    when w0 is a low, or a high not followed by a low; at 1 when w0 is BMP and w1 is any
    surrogate (a lone low, or a high at the end)."""
    nparts = 64
    with ThreadPoolExecutor(8) as ex:
        parts = list(ex.map(lambda p: oracle.sweep_utf16_pairs(p, nparts), range(nparts)))
    valid = sum(p[0] for p in parts)
    ho = sum(p[1] for p in parts)
    assert valid == 63488 ** 2 + 1024 ** 2
    assert int(ho[0]) == 1024 * 65536 + 1024 * (65536 - 1024)
    assert int(ho[1]) == 63488 * 2048


# ------------------------------------------------------------------ random fuzz vs CPython
LEADISH = np.array([0x00, 0x41, 0x7F, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1, 0xC2,
                    0xDF, 0xE0, 0xE1, 0xEC, 0xED, 0xEE, 0xEF, 0xF0, 0xF1, 0xF3, 0xF4, 0xF5,
                    0xF7, 0xF8, 0xFF], dtype=np.uint8)


def fuzz_strings(rng, count, maxlen):
    for _ in range(count):
        n = int(rng.integers(0, maxlen + 1))
        mode = rng.integers(0, 3)
        if mode == 0:  # class representatives (SURVEY.md C.4 alphabet)
            yield LEADISH[rng.integers(0, LEADISH.size, n)].tobytes()
        elif mode == 1:  # raw random bytes
            yield rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        else:  # valid text with one random byte overwritten
            cps = rng.integers(0, 0x110000, max(n // 2, 1))
            cps = cps[(cps < 0xD800) | (cps > 0xDFFF)]
            b = bytearray("".join(map(chr, cps.tolist())).encode("utf-8"))
            if b:
                b[int(rng.integers(0, len(b)))] = int(rng.integers(0, 256))
            yield bytes(b)


def test_fuzz_utf8_vs_cpython():
    """Verdict, first-error offset, written count and output prefix equal CPython on
    60,000 seeded random strings."""
    rng = np.random.default_rng(20211117)
    for s in fuzz_strings(rng, 60000, 48):
        e = cpython_offset8(s)
        r, out = oracle.utf8_to_utf16le(s)
        pre = s if e < 0 else s[:e]
        ref = np.frombuffer(pre.decode("utf-8").encode("utf-16-le"), dtype="<u2")
        assert (r.error == OK) == (e < 0), s.hex()
        assert r.position == (len(s) if e < 0 else e), s.hex()
        assert r.written == ref.size and np.array_equal(out, ref), s.hex()
        assert oracle.utf8_validate(s)[:2] == r[:2]
        if e < 0:
            assert oracle.utf16_length_from_utf8(s) == ref.size


def cpython_offset16(u: np.ndarray) -> int:
    try:
        u.astype("<u2").tobytes().decode("utf-16-le")
        return -1
    except UnicodeDecodeError as e:
        return e.start // 2


def test_fuzz_utf16_vs_cpython():
    rng = np.random.default_rng(2781)
    alphabet = np.array([0x0041, 0x007F, 0x0080, 0x07FF, 0x0800, 0xD7FF, 0xD800, 0xDBFF,
                         0xDC00, 0xDFFF, 0xE000, 0xFFFF], dtype=np.uint16)
    for _ in range(60000):
        n = int(rng.integers(0, 24))
        u = alphabet[rng.integers(0, alphabet.size, n)] if rng.integers(0, 2) else \
            rng.integers(0, 65536, n).astype(np.uint16)
        e = cpython_offset16(u)
        r, out = oracle.utf16le_to_utf8(u)
        pre = u if e < 0 else u[:e]
        ref = pre.astype("<u2").tobytes().decode("utf-16-le").encode("utf-8")
        assert (r.error == OK) == (e < 0), u
        assert r.error in (OK, SURROGATE)
        assert r.position == (n if e < 0 else e), u
        assert out.tobytes() == ref and r.written == len(ref), u
        assert oracle.utf16le_validate(u)[:2] == r[:2]
        if e < 0:
            assert oracle.utf8_length_from_utf16le(u) == len(ref)


def test_length_functions_closed_form():
    """Length-from formulas over all single bytes / words (partition S:85-86): UTF-16 units =
    192 non-continuation bytes + 16 bytes >= F0; UTF-8 bytes = 128*1 + 1920*2 + 2048*2 +
    (65536-128-1920-2048)*3."""
    assert oracle.utf16_length_from_utf8(np.arange(256, dtype=np.uint8)) == 192 + 16
    assert oracle.utf8_length_from_utf16le(np.arange(65536, dtype=np.uint16)) == \
        128 + 1920 * 2 + 2048 * 2 + (65536 - 128 - 1920 - 2048) * 3
    assert oracle.utf16_length_from_utf8(b"") == 0 == oracle.utf8_length_from_utf16le(b"")


def test_capacity_contract():
    """A too-small output buffer: {OUTPUT_TOO_SMALL, required, 0} and nothing written past
    out_cap (R5); exact capacity succeeds."""
    s = "aé你\U0001F600".encode("utf-8") * 5
    ref = np.frombuffer(s.decode("utf-8").encode("utf-16-le"), dtype="<u2")
    r, out = oracle.utf8_to_utf16le(s, out_cap=ref.size)
    assert r == (OK, len(s), ref.size) and np.array_equal(out, ref)
    for cap in range(ref.size):
        r, _ = oracle.utf8_to_utf16le(s, out_cap=cap)
        assert r == (OUTPUT_TOO_SMALL, ref.size, 0)
    u = ref
    r, out = oracle.utf16le_to_utf8(u, out_cap=len(s))
    assert r == (OK, u.size, len(s)) and out.tobytes() == s
    r, _ = oracle.utf16le_to_utf8(u, out_cap=len(s) - 1)
    assert r == (OUTPUT_TOO_SMALL, len(s), 0)
    # capacity check applies to the prefix before the first error only
    bad = s[:6] + b"\xff" + s
    need = oracle.utf8_to_utf16le(bad)[0].written
    assert need == 3
    r, _ = oracle.utf8_to_utf16le(bad, out_cap=need)
    assert r == (HEADER_BITS, 6, need)
    r, _ = oracle.utf8_to_utf16le(bad, out_cap=need - 1)
    assert r == (OUTPUT_TOO_SMALL, need, 0)


# ------------------------------------------------------------------ UTF-16BE
def be_words(b: bytes) -> np.ndarray:
    """The words of a big-endian UTF-16 byte string as they sit in (little-endian) memory."""
    return np.frombuffer(b, dtype="<u2").copy()


def test_utf16be_spec_example():
    """utf16be file [0x00,0x41] -> words [0x0041]."""
    u = be_words(bytes([0x00, 0x41]))
    assert list(oracle.byteswap16(u)) == [0x0041]
    r, out = oracle.utf16be_to_utf8(u)
    assert tuple(r) == (OK, 1, 1) and out.tobytes() == b"A"
    r, out = oracle.utf8_to_utf16be(b"A")
    assert tuple(r) == (OK, 1, 1) and out.astype("<u2").tobytes() == bytes([0x00, 0x41])


def test_fuzz_utf16be_vs_cpython():
    """BE against CPython's own utf-16-be codec (independent of the oracle's byte swap):
    decode of valid and invalid word strings, encode of valid text, lengths."""
    rng = np.random.default_rng(0xBE16)
    alphabet = np.array([0x0041, 0x007F, 0x0080, 0x07FF, 0x0800, 0xD7FF, 0xD800, 0xDBFF,
                         0xDC00, 0xDFFF, 0xE000, 0xFFFF, 0x0100, 0x1234], dtype=np.uint16)
    for _ in range(20000):
        n = int(rng.integers(0, 24))
        cu = alphabet[rng.integers(0, alphabet.size, n)] if rng.integers(0, 2) else \
            rng.integers(0, 65536, n).astype(np.uint16)
        raw = cu.astype(">u2").tobytes()          # big-endian bytes of the code units
        u = be_words(raw)
        try:
            ref = raw.decode("utf-16-be").encode("utf-8")
            e = -1
        except UnicodeDecodeError as x:
            e = x.start // 2
            ref = raw[: 2 * e].decode("utf-16-be").encode("utf-8")
        r, out = oracle.utf16be_to_utf8(u)
        assert (r.error == OK) == (e < 0), cu
        assert r.position == (n if e < 0 else e), cu
        assert out.tobytes() == ref and r.written == len(ref), cu
        assert oracle.utf16be_validate(u)[:2] == r[:2]
        if e < 0:
            assert oracle.utf8_length_from_utf16be(u) == len(ref)
            r2, back = oracle.utf8_to_utf16be(ref)
            assert r2.error == OK and back.astype("<u2").tobytes() == raw
