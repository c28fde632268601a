"""The derived facts the GPU design rests on, re-verified against the
oracle on CPU.  The models here are written in the tests, independently of both the oracle and
the CUDA kernels (which implement the same mathematics in their own code):

(i)  local first-error predicate: e = min{i : A(i) or B(i)}, each term reading only bytes
     [i-3, i+3] -- what makes the first error exact across tiles and shards;
(ii) HISTORICAL -- the paper's (Keiser-Lemire) nibble-table classifier that the first GPU
     kernels ran (round 1; replaced by the bit-plane classifier, D3): classes for
     the six value rules (PAPER.md:80-82 and the C0/C1 and F5..FF leads) AND-ed from three
     16-entry tables keyed by hi(prev1), lo(prev1), hi(cur), plus bit logic for the structural
     rules and the continuation-count check.  It flags iff the input is invalid, and the first
     flagged position r obeys e <= r <= e + 3 when positions n, n+1, n+2 are classified
     against 0x00 padding.  Kept as the derivation of the flag-window argument; the classifier
     the kernels RUN is pinned by tests/test_kernel_math_cpu.py (the product's own utf8.cuh
     compiled for the host, in the kernels' warp layout);
(iii) the UTF-16 pairing predicate.
"""
import itertools

import numpy as np

import oracle

ALPHABET = [0x00, 0x41, 0x7F, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1, 0xC2, 0xDF,
            0xE0, 0xE1, 0xEC, 0xED, 0xEE, 0xEF, 0xF0, 0xF1, 0xF3, 0xF4, 0xF5, 0xF7, 0xF8, 0xFF]


def cont(b):
    return (b & 0xC0) == 0x80


def decl(b):
    if b < 0x80:
        return 1
    if b < 0xC0:
        return 0
    if b < 0xE0:
        return 2
    if b < 0xF0:
        return 3
    if b < 0xF8:
        return 4
    return 0


def local_first_error(s: bytes):
    n = len(s)
    for i in range(n):
        if not cont(s[i]):
            if oracle.decode_utf8_at(s, i)[0] != 0:
                return i
        else:
            ok = False
            for d in (1, 2, 3):
                j = i - d
                if j < 0:
                    break
                if not cont(s[j]):
                    ok = decl(s[j]) > d
                    break
            if not ok:
                return i
    return -1


# ---- (ii) classifier model -------------------------------------------------------------
# six value classes as nibble rectangles (hi(prev1), lo(prev1), hi(cur)), derived from the
# rules: 2-byte overlong C0/C1; 3-byte overlong E0 80..9F; surrogate ED A0..BF;
# 4-byte overlong F0 80..8F; too large F4 90..BF and F5..FF leads.
CLASSES = [
    ({0xC}, {0, 1}, set(range(8, 12))),        # overlong-2
    ({0xE}, {0}, {8, 9}),                      # overlong-3
    ({0xE}, {0xD}, {0xA, 0xB}),                # surrogate
    ({0xF}, {0}, {8}),                         # overlong-4
    ({0xF}, {4}, {9, 0xA, 0xB}),               # too-large (F4 90..)
    ({0xF}, set(range(5, 16)), set(range(8, 12))),  # too-large (F5..FF leads)
]
T1 = [sum(1 << k for k, c in enumerate(CLASSES) if v in c[0]) for v in range(16)]
T2 = [sum(1 << k for k, c in enumerate(CLASSES) if v in c[1]) for v in range(16)]
T3 = [sum(1 << k for k, c in enumerate(CLASSES) if v in c[2]) for v in range(16)]


def special(p1, c):
    return T1[p1 >> 4] & T2[p1 & 15] & T3[c >> 4]


def flags(s: bytes):
    """Flag per position 0 .. n+2 (bytes outside [0, n) read as 0x00)."""
    n = len(s)
    b = lambda i: s[i] if 0 <= i < n else 0  # noqa: E731
    out = []
    for i in range(n + 3):
        c, p1, p2, p3 = b(i), b(i - 1), b(i - 2), b(i - 3)
        too_short = p1 >= 0xC0 and not cont(c)
        too_long = p1 < 0x80 and cont(c)
        must23 = p2 >= 0xE0 or p3 >= 0xF0
        two = cont(p1) and cont(c)
        out.append(bool(too_short or too_long or (two != must23) or special(p1, c)))
    return out


def test_tables_equal_direct_predicate_on_all_pairs():
    """AND of the three lookups equals the rectangle membership on all 65,536 (prev1, cur)."""
    for p1 in range(256):
        for c in range(256):
            direct = 0
            for k, (s1, s2, s3) in enumerate(CLASSES):
                if (p1 >> 4) in s1 and (p1 & 15) in s2 and (c >> 4) in s3:
                    direct |= 1 << k
            assert special(p1, c) == direct


def strings_upto(maxlen):
    for n in range(0, maxlen + 1):
        yield from (bytes(t) for t in itertools.product(ALPHABET, repeat=n))


def check(s):
    r = oracle.utf8_validate(s)
    e = -1 if r.error == 0 else r.position
    assert local_first_error(s) == e, s.hex()
    f = flags(s)
    if e < 0:
        assert not any(f), s.hex()
    else:
        first = f.index(True)
        assert e <= first <= e + 3, (s.hex(), e, first)


def test_local_predicate_and_classifier_exhaustive_alphabet():
    """Every string of length <= 4 over 27 class representatives (551,881 strings)."""
    for s in strings_upto(4):
        check(s)


def test_local_predicate_and_classifier_random():
    rng = np.random.default_rng(8692)
    alpha = np.array(ALPHABET, dtype=np.uint8)
    for _ in range(30000):
        n = int(rng.integers(5, 13))
        s = alpha[rng.integers(0, alpha.size, n)].tobytes()
        check(s)
    for _ in range(10000):
        s = rng.integers(0, 256, int(rng.integers(1, 16)), dtype=np.uint8).tobytes()
        check(s)


def test_utf16_pairing_predicate():
    """err(i) = (H(u_i) and not L(u_{i+1})) or (L(u_i) and not H(u_{i-1})); e = min over i
    (PAPER.md:87), against the oracle on all strings of length <= 6 over 6 words."""
    words = [0x0041, 0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0xE000]
    H = lambda w: 0xD800 <= w <= 0xDBFF  # noqa: E731
    L = lambda w: 0xDC00 <= w <= 0xDFFF  # noqa: E731
    for n in range(7):
        for t in itertools.product(words, repeat=n):
            errs = [i for i in range(n)
                    if (H(t[i]) and not (i + 1 < n and L(t[i + 1])))
                    or (L(t[i]) and not (i >= 1 and H(t[i - 1])))]
            r = oracle.utf16le_validate(np.array(t, dtype=np.uint16))
            assert (errs[0] if errs else -1) == (r.position if r.error else -1), t


def test_utf16_xor_pairing_form():
    """The streaming validator's form (kernels.cu k_validate16): with H(-1) = L(n) = 0, a
    string is valid iff H(u_{i-1}) == L(u_i) for every i in [0, n]; the first i where they
    differ, f, lies at e or e + 1 for the first error e (a lone low flags at itself, a lone high
    at the next word), so rescanning words f - 1 .. f finds e.  Against the oracle on all
    strings of length <= 6 over 6 words (every neighbour combination of the two classes)."""
    words = [0x0041, 0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0xE000]
    H = lambda w: 0xD800 <= w <= 0xDBFF  # noqa: E731
    L = lambda w: 0xDC00 <= w <= 0xDFFF  # noqa: E731
    for n in range(7):
        for t in itertools.product(words, repeat=n):
            hp = [False] + [H(w) for w in t]          # H(u_{i-1}), i = 0 .. n
            lw = [L(w) for w in t] + [False]          # L(u_i),     i = 0 .. n
            flags = [i for i in range(n + 1) if hp[i] != lw[i]]
            r = oracle.utf16le_validate(np.array(t, dtype=np.uint16))
            assert bool(flags) == bool(r.error), t
            if flags:
                assert r.position in (flags[0], flags[0] - 1), (t, flags, r)


def test_utf16_ascii_window_iff_width_sum_equals_count():
    """k_narrow16's selection (kernels.cu): the UTF-8 width sum of a UTF-16 window equals its
    word count iff every word is below 0x80 (every width is >= 1; a surrogate counts 2, so no
    invalid window qualifies) -- on every single word and on random mixes, against the oracle's
    utf8_length_from_utf16le."""
    for w in range(0x10000):
        u = np.array([w], dtype=np.uint16)
        assert (oracle.utf8_length_from_utf16le(u) == 1) == (w < 0x80), hex(w)
    rng = np.random.default_rng(5)
    for _ in range(2000):
        n = int(rng.integers(1, 40))
        u = rng.integers(0, 0x80, n).astype(np.uint16)
        if rng.integers(0, 2):
            u[int(rng.integers(0, n))] = int(rng.integers(0x80, 0x10000))
        assert (oracle.utf8_length_from_utf16le(u) == n) == bool(np.all(u < 0x80))
