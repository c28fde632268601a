"""The f4 tables (section 4), as the library
builds them on the host (`ug_utf8_keyed_tables`, no GPU), pinned by brute force and by
Python's own UTF-8 codec -- not by re-running the builder's rule:

* the shape: 64 + 81 + 64 = 209 shuffle entries (PAPER.md:95's index ranges);
* the SPEC examples: keys 0xFFF / 0xAAA / 0x924;
* maximality: for every one of the 4096 keys, the bytes consumed equal the
  best over ALL 209 length tuples (each tuple scored by how many of its leading characters
  end exactly at the key's ends), and the path is the earliest that reaches it;
* shuffle soundness: every entry, applied to 12 distinct marker bytes the way
  the kernel applies it (mux(M, prmt(w0, w1, A), prmt(w2, 0, B)), PRMT as PTX defines it),
  puts each character's bytes in its lane, last byte lowest, zeros elsewhere;
* end-to-end: random valid 12-byte windows of every width mix, keyed and shuffled, give back
  the characters Python decodes from the same bytes.
"""
import random

import numpy as np
import pytest

NCH = {0: 6, 1: 4, 2: 3}
MAXL = {0: 2, 1: 3, 2: 4}
BASE = {0: 0, 1: 64, 2: 145}


@pytest.fixture(scope="module")
def tables():
    import paper_2111_08692_b200 as ug
    return ug.keyed_tables()


def path_of(idx):
    return 0 if idx < 64 else (1 if idx < 145 else 2)


def tuples():
    """All 209 (path, lengths) in index order, enumerated here independently."""
    import itertools
    out = []
    for path in (0, 1, 2):
        for t in itertools.product(range(1, MAXL[path] + 1), repeat=NCH[path]):
            out.append((path, t))
    return out


def prmt(a, b, sel):
    """PTX prmt.b32 default mode: byte i = byte (sel >> 4i) & 7 of {b, a}, msb-replicated if
    bit 3 of that nibble is set."""
    v = (b << 32) | a
    d = 0
    for i in range(4):
        s = (sel >> (4 * i)) & 0xF
        byte = (v >> (8 * (s & 7))) & 0xFF
        if s & 8:
            byte = 0xFF if byte & 0x80 else 0
        d |= byte << (8 * i)
    return d


def lanes(entry, window):
    w = [int.from_bytes(bytes(window[4 * k:4 * k + 4]), "little") for k in range(3)]
    out = []
    for r in range(4):
        sel, m = int(entry[r]), int(entry[4 + r])
        a = prmt(w[0], w[1], sel & 0xFFFF)
        b = prmt(w[2], 0, sel >> 16)
        out.append((a & m) | (b & ~m & 0xFFFFFFFF))
    return out


def char_lanes(path, v, nch):
    """The per-character lane values: 16-bit halves (path a) or whole registers."""
    if path == 0:
        return [(v[j // 2] >> (16 * (j % 2))) & 0xFFFF for j in range(nch)]
    return [v[j] for j in range(nch)]


def test_shape(tables):
    key, shuf = tables
    assert key.shape == (4096,) and shuf.shape == (209, 8)
    idx = key >> 8
    assert int(idx.max()) < 209
    assert int((key & 15).max()) <= 12


@pytest.mark.parametrize("k,consumed,path,nch", [
    (0xFFF, 6, 0, 6),    # 12 ASCII bytes -> six 1-byte characters, path (a)
    (0xAAA, 12, 0, 6),   # six 2-byte characters, path (a)
    (0x924, 12, 1, 4),   # four 3-byte characters, path (b)
])
def test_spec_examples(tables, k, consumed, path, nch):
    key, _ = tables
    e = int(key[k])
    assert (e & 15, path_of(e >> 8), (e >> 4) & 7) == (consumed, path, nch)


def test_maximality_all_keys(tables):
    key, _ = tables
    all_t = tuples()
    assert len(all_t) == 209 and [t for t in all_t[:1]] == [(0, (1,) * 6)]
    for k in range(4096):
        ends = [i for i in range(12) if k >> i & 1]
        best, best_path = 0, None
        for path, t in all_t:   # score every tuple: leading characters ending at the key's ends
            s, c = -1, 0
            for ln in t:
                e = s + ln
                if e > 11 or not (k >> e & 1) or any(s < x < e for x in ends):
                    break
                c, s = c + ln, e
            if c > best or (c == best and c > 0 and best_path is not None and path < best_path):
                best, best_path = c, path
        e = int(key[k])
        assert e & 15 == best, (hex(k), e & 15, best)
        if best:
            assert path_of(e >> 8) == best_path, hex(k)
            # the entry's tuple prefix = the key's first characters
            path, t = all_t[e >> 8]
            nch = (e >> 4) & 7
            starts = [-1] + ends
            assert list(t[:nch]) == [ends[j] - starts[j] for j in range(nch)], hex(k)
            assert sum(t[:nch]) == best
        else:
            assert e == 0


def test_shuffle_soundness(tables):
    _, shuf = tables
    window = [0x10 + i for i in range(12)]  # distinct markers, all < 0x80
    for i, (path, t) in enumerate(tuples()):
        v = lanes(shuf[i], window)
        got = char_lanes(path, v, NCH[path])
        s = 0
        width = 2 if path == 0 else 4
        for j, ln in enumerate(t):
            want = [window[s + ln - 1 - k] for k in range(ln)] + [0] * (width - ln)
            have = [(got[j] >> (8 * k)) & 0xFF for k in range(width)]
            assert have == want, (i, path, t, j)
            s += ln
        if path == 0:
            assert v[3] == 0
        elif path == 2:
            assert v[3] == 0


@pytest.mark.parametrize("mix", [(1,), (2,), (3,), (4,), (1, 2), (1, 3), (2, 3, 4), (1, 2, 3, 4)])
def test_windows_decode_like_python(tables, mix):
    key, shuf = tables
    rng = random.Random(hash(mix) & 0xFFFF)
    lo = {1: 0x20, 2: 0x80, 3: 0x800, 4: 0x10000}
    hi = {1: 0x7F, 2: 0x7FF, 3: 0xFFFF, 4: 0x10FFFF}
    for _ in range(400):
        chars = []
        while sum(len(c.encode()) for c in chars) < 16:
            w = rng.choice(mix)
            cp = rng.randint(lo[w], hi[w])
            if 0xD800 <= cp <= 0xDFFF:
                continue
            chars.append(chr(cp))
        data = "".join(chars).encode("utf-8")
        window = list(data[:12])
        # key: bit i = byte i is the last byte of its character (by Python's boundaries)
        k, pos = 0, 0
        for c in chars:
            pos += len(c.encode())
            if pos - 1 < 12:
                k |= 1 << (pos - 1)
        e = int(key[k])
        consumed, nch, idx = e & 15, (e >> 4) & 7, e >> 8
        assert consumed > 0
        got = char_lanes(path_of(idx), lanes(shuf[idx], window), nch)
        for j in range(nch):
            ln = len(chars[j].encode())
            bs = bytes((got[j] >> (8 * (ln - 1 - q))) & 0xFF for q in range(ln))
            assert bs.decode("utf-8") == chars[j]
            assert got[j] >> (8 * ln) == 0  # zero above the character
        assert consumed == sum(len(c.encode()) for c in chars[:nch])
