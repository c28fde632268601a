"""Seeded synthetic inputs for BASELINE.json's five configs.

This module serves both the oracle tests and the CUDA parity tests / bench, and holds NONE of
the method's arithmetic: code points are drawn with numpy's PCG64 and turned into UTF-8 /
UTF-16LE bytes by CPython's own codecs (``str.encode``), a library routine.  The only
per-character facts used here are the byte lengths of the ranges the generator itself draws
from (ASCII 1 byte, U+0080..07FF 2, U+0800..FFFF 3, supplementary 4), needed to
fill each buffer to an exact size.

Stand-ins: the paper measures on lipsum text in several languages, which is not
in this container; configs 2 and 3 reproduce the byte-class profile of those corpora
(2-byte scripts, CJK, emoji), config 0/4 a mixed profile, config 1 pure ASCII.

Big buffers are produced in 64 MiB chunks; chunk c draws from
``SeedSequence(seed, spawn_key=(c,))`` and is filled exactly (at most 3 bytes / 1 word of
U+0020 padding), so the concatenation is valid, exact-size and deterministic.
"""
from __future__ import annotations

import hashlib
import os
from concurrent.futures import ProcessPoolExecutor
from dataclasses import dataclass
from multiprocessing import get_context, shared_memory

import numpy as np

RNG_ID = "numpy.PCG64 via SeedSequence(seed, spawn_key=(chunk,))"
MiB = 1 << 20
GiB = 1 << 30
CHUNK = 64 * MiB

# ASCII punctuation used inside config-2A words (0x21-2F, 3A-40, 5B-60, 7B-7E)
PUNCT = np.array(list(range(0x21, 0x30)) + list(range(0x3A, 0x41)) + list(range(0x5B, 0x61))
                 + list(range(0x7B, 0x7F)), dtype=np.uint32)


@dataclass(frozen=True)
class Config:
    key: str
    encoding: str   # "utf8" or "utf16le": the encoding of the generated buffer
    size: int       # bytes
    seed: int
    mix: str        # generator name
    desc: str


CONFIGS = {
    "c0": Config("c0", "utf8", 1 * MiB, 0, "mixed",
                 "1 MiB mixed UTF-8 (60% ASCII, 25% 2-byte, 10% 3-byte, 5% 4-byte), seed 0"),
    "c1": Config("c1", "utf8", 1 * GiB, 1, "ascii", "1 GiB ASCII (0x20-0x7E, 2% LF)"),
    "c2a": Config("c2a", "utf8", 256 * MiB, 2, "words2",
                  "256 MiB text A: words of U+0400-06FF (80%) and ASCII (20%)"),
    "c2b": Config("c2b", "utf8", 256 * MiB, 3, "words3",
                  "256 MiB text B: words of U+4E00-9FFF (90%) and spaces (10%)"),
    "c3": Config("c3", "utf16le", 512 * MiB, 4, "emoji",
                 "512 MiB UTF-16LE: 70% U+1F300-1FAFF pairs, 30% ASCII"),
    "c4": Config("c4", "utf8", 8 * GiB, 5, "mixed", "8 GiB mixed UTF-8 (config-0 mix)"),
}


def chunk_rng(seed: int, chunk: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(chunk,)))


# ----------------------------------------------------------------------------- draws
def _draw_mixed(rng, m):
    """Config-0 mixture: 60% ASCII U+0020-007E (10% of those -> LF), 25% U+0080-07FF, 10%
    U+0800-FFFF minus D800-DFFF, 5% U+10000-10FFFF.  Returns (code points, byte lengths)."""
    u = rng.random(m, dtype=np.float32)
    cls = (u >= 0.60).view(np.uint8) + (u >= 0.85).view(np.uint8) + (u >= 0.95).view(np.uint8)
    del u
    lo = np.array([0x20, 0x80, 0x800, 0x10000], dtype=np.uint32)
    span = np.array([0x7F - 0x20, 0x800 - 0x80, 0x10000 - 0x800 - 0x800, 0x110000 - 0x10000],
                    dtype=np.float32)
    r = rng.random(m, dtype=np.float32)
    r *= span[cls]
    cp = r.astype(np.uint32)
    del r
    cp += lo[cls]
    cp[(cls == 2) & (cp >= 0xD800)] += 0x800                   # skip the surrogate block
    cp[(cls == 0) & (rng.random(m, dtype=np.float32) < 0.10)] = 0x0A
    return cp, cls + np.uint8(1)


def _draw_words(rng, m, mean_len, script_lo, script_hi, script_bytes, punct_frac):
    """Words of geometric length (mean `mean_len`) each followed by U+0020."""
    nw = m // (mean_len + 1) + 16
    lens = rng.geometric(1.0 / mean_len, nw)
    total = int(lens.sum() + nw)
    cp = rng.integers(script_lo, script_hi + 1, total, dtype=np.uint32)
    nb = np.full(total, script_bytes, dtype=np.int64)
    if punct_frac:
        k = rng.random(total) < punct_frac
        cp[k] = PUNCT[rng.integers(0, PUNCT.size, int(k.sum()))]
        nb[k] = 1
    ends = np.cumsum(lens + 1) - 1
    cp[ends] = 0x20
    nb[ends] = 1
    return cp, nb


def _draw_emoji(rng, m):
    """Config 3: 70% U+1F300-1FAFF, 30% ASCII as in config 0.  Lengths in UTF-16 words."""
    u = rng.random(m) < 0.70
    r = rng.random(m)
    cp = np.where(u, 0x1F300 + np.floor(r * (0x1FB00 - 0x1F300)),
                  0x20 + np.floor(r * (0x7F - 0x20))).astype(np.uint32)
    cp[~u & (rng.random(m) < 0.10)] = 0x0A
    return cp, np.where(u, 2, 1).astype(np.int64)


def _draw_ascii(rng, m):
    """Config 1: bytes uniform in 0x20-0x7E, 2% of them replaced by LF."""
    cp = rng.integers(0x20, 0x7F, m, dtype=np.uint32)
    cp[rng.random(m, dtype=np.float32) < 0.02] = 0x0A
    return cp, np.ones(m, dtype=np.uint8)


def _draw(mix, rng, m):
    if mix == "ascii":
        return _draw_ascii(rng, m)
    if mix == "mixed":
        return _draw_mixed(rng, m)
    if mix == "words2":  # mean 6, 1/15 punctuation in words -> 80% script / 20% ASCII
        return _draw_words(rng, m, 6, 0x0400, 0x06FF, 2, 1.0 / 15)
    if mix == "words3":  # mean 9 (R17) -> 90% CJK / 10% spaces
        return _draw_words(rng, m, 9, 0x4E00, 0x9FFF, 3, 0.0)
    if mix == "emoji":
        return _draw_emoji(rng, m)
    raise ValueError(mix)


_MEAN_UNITS = {"ascii": 1.0, "mixed": 1.6, "words2": 1.8, "words3": 2.8, "emoji": 1.7}


def _encode(cp: np.ndarray, encoding: str) -> bytes:
    text = cp.astype("<u4").tobytes().decode("utf-32-le")
    return text.encode("utf-8" if encoding == "utf8" else "utf-16-le")


def gen_chunk(mix: str, encoding: str, nbytes: int, seed: int, chunk: int) -> bytes:
    """Exactly `nbytes` of valid text: draw characters until the next one would overflow, then
    pad with U+0020 (<= 3 bytes / 1 word)."""
    rng = chunk_rng(seed, chunk)
    unit = 1 if encoding == "utf8" else 2
    target = nbytes // unit
    cps, lens = [], []
    have = 0
    while True:
        m = int((target - have) / _MEAN_UNITS[mix] * 1.05) + 64
        cp, ln = _draw(mix, rng, m)
        cs = np.cumsum(ln, dtype=np.int64)
        fit = int(np.searchsorted(cs, target - have, side="right"))
        cps.append(cp[:fit])
        have += int(cs[fit - 1]) if fit else 0
        if fit < cp.size:
            break
    cp = np.concatenate(cps) if cps else np.zeros(0, np.uint32)
    pad = target - have
    cp = np.concatenate([cp, np.full(pad, 0x20, np.uint32)])
    out = _encode(cp, encoding)
    assert len(out) == nbytes, (len(out), nbytes)
    return out


def _worker(args):
    name, mix, encoding, total, seed, c = args
    shm = shared_memory.SharedMemory(name=name)
    try:
        lo = c * CHUNK
        nb = min(CHUNK, total - lo)
        shm.buf[lo:lo + nb] = gen_chunk(mix, encoding, nb, seed, c)
    finally:
        shm.close()
    return c


def generate(cfg: Config | str, size: int | None = None, chunks: range | None = None,
             workers: int | None = None) -> np.ndarray:
    """Generate config `cfg` (optionally truncated to `size` bytes, a multiple of the chunk
    structure is kept: chunk c always covers bytes [c*CHUNK, (c+1)*CHUNK)).  `chunks` selects a
    subset of chunks (the others are left zero) -- used by ranks that need only their shard.
    Returns uint8 (UTF-8) or uint16 (UTF-16LE) array."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    total = cfg.size if size is None else size
    nch = (total + CHUNK - 1) // CHUNK
    sel = list(range(nch)) if chunks is None else [c for c in chunks if 0 <= c < nch]
    dt = np.uint8 if cfg.encoding == "utf8" else np.dtype("<u2")
    if nch <= 1 or len(sel) <= 1:
        buf = bytearray(total)
        for c in sel:
            lo = c * CHUNK
            nb = min(CHUNK, total - lo)
            buf[lo:lo + nb] = gen_chunk(cfg.mix, cfg.encoding, nb, cfg.seed, c)
        return np.frombuffer(bytes(buf), dtype=dt).copy()
    shm = shared_memory.SharedMemory(create=True, size=total)
    try:
        nw = workers or min(len(sel), max(1, (os.cpu_count() or 2) - 1), 32)
        with ProcessPoolExecutor(nw, mp_context=get_context("fork")) as ex:
            list(ex.map(_worker, [(shm.name, cfg.mix, cfg.encoding, total, cfg.seed, c)
                                  for c in sel]))
        arr = np.empty(total // np.dtype(dt).itemsize, dtype=dt)
        arr.view(np.uint8)[:] = np.frombuffer(shm.buf, dtype=np.uint8, count=total)
        return arr
    finally:
        shm.close()
        shm.unlink()


def generate_range(cfg: Config | str, lo: int, hi: int, workers: int | None = None) -> np.ndarray:
    """Bytes [lo, hi) of config `cfg` (byte offsets, clipped to the config size), generating
    only the chunks that cover them.  Identical to generate(cfg)[lo:hi] (as bytes)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    lo, hi = max(0, lo), min(cfg.size, hi)
    if hi <= lo:
        return np.zeros(0, dtype=np.uint8)
    c0, c1 = lo // CHUNK, (hi - 1) // CHUNK
    span = (c1 - c0 + 1) * CHUNK
    sub = Config(cfg.key, cfg.encoding, cfg.size, cfg.seed, cfg.mix, cfg.desc)
    total = min(cfg.size - c0 * CHUNK, span)
    shm = shared_memory.SharedMemory(create=True, size=total)
    try:
        sel = list(range(c0, c1 + 1))
        nw = workers or min(len(sel), max(1, (os.cpu_count() or 2) - 1), 32)
        args = [(shm.name, sub.mix, sub.encoding, cfg.size, cfg.seed, c, c0 * CHUNK) for c in sel]
        if len(sel) == 1:
            _worker_off(args[0])
        else:
            with ProcessPoolExecutor(nw, mp_context=get_context("fork")) as ex:
                list(ex.map(_worker_off, args))
        out = np.empty(hi - lo, dtype=np.uint8)
        out[:] = np.frombuffer(shm.buf, dtype=np.uint8, count=total)[lo - c0 * CHUNK:hi - c0 * CHUNK]
        return out
    finally:
        shm.close()
        shm.unlink()


def _worker_off(args):
    name, mix, encoding, total, seed, c, base = args
    shm = shared_memory.SharedMemory(name=name)
    try:
        lo = c * CHUNK
        nb = min(CHUNK, total - lo)
        shm.buf[lo - base:lo - base + nb] = gen_chunk(mix, encoding, nb, seed, c)
    finally:
        shm.close()
    return c


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(a.view(np.uint8).tobytes()).hexdigest()


# ----------------------------------------------------------------------------- errors
UTF8_ERROR_CLASSES = ("overlong", "surrogate", "too_large", "truncated", "stray_continuation")
# the oracle kind each injected class must produce
UTF8_EXPECTED_KIND = {"overlong": 4, "surrogate": 6, "too_large": 5, "truncated": 2,
                      "stray_continuation": 3}


def _char_start_at_or_after(buf: np.ndarray, r: int) -> int:
    p = r
    while p < buf.size and (int(buf[p]) & 0xC0) == 0x80:
        p += 1
    return p


def utf8_error_bytes(cls: str, rng) -> bytes:
    """Byte pattern written at a character start for each injected class."""
    r = lambda lo, hi: int(rng.integers(lo, hi + 1))  # noqa: E731
    if cls == "overlong":
        v = r(0, 2)
        if v == 0:
            return bytes([r(0xC0, 0xC1), r(0x80, 0xBF)])
        if v == 1:
            return bytes([0xE0, r(0x80, 0x9F), r(0x80, 0xBF)])
        return bytes([0xF0, r(0x80, 0x8F), r(0x80, 0xBF), r(0x80, 0xBF)])
    if cls == "surrogate":
        return bytes([0xED, r(0xA0, 0xBF), r(0x80, 0xBF)])
    if cls == "too_large":
        if r(0, 1):
            return bytes([0xF4, r(0x90, 0xBF), r(0x80, 0xBF), r(0x80, 0xBF)])
        return bytes([r(0xF5, 0xF7), r(0x80, 0xBF), r(0x80, 0xBF), r(0x80, 0xBF)])
    if cls == "truncated":
        L = r(2, 4)
        lead = {2: r(0xC2, 0xDF), 3: r(0xE1, 0xEC), 4: r(0xF1, 0xF3)}[L]
        k = r(0, L - 2)
        return bytes([lead] + [r(0x80, 0xBF) for _ in range(k)] + [0x20])
    if cls == "stray_continuation":
        return bytes([r(0x80, 0xBF)])
    raise ValueError(cls)


def inject_utf8_error(buf: np.ndarray, lo: int, hi: int, cls: str, rng):
    """Overwrite, in place, bytes at a character start p in [lo, hi] (first char start at or
    after a uniform draw in [lo, hi]) with class `cls`.  Returns (p, saved original bytes) so
    the caller can undo it.  The first error of the result is at p, by construction: all bytes
    before p are untouched valid text."""
    pat = utf8_error_bytes(cls, rng)
    for _ in range(64):
        p = _char_start_at_or_after(buf, int(rng.integers(lo, hi + 1)))
        if p + len(pat) <= buf.size and p <= hi:
            break
    else:
        raise RuntimeError("no character start in range")
    saved = buf[p:p + len(pat)].copy()
    buf[p:p + len(pat)] = np.frombuffer(pat, dtype=np.uint8)
    return p, saved


def inject_utf16_error(u: np.ndarray, lo: int, hi: int, rng):
    """Config 3's error copy: replace a single-unit BMP character u[p] (p in [lo, hi]) by a
    random high or low surrogate.  The next unit starts a character (never a low) and the
    previous one ends a character (never a high), so the first error is at p."""
    for _ in range(10000):
        p = int(rng.integers(lo, hi + 1))
        w = int(u[p])
        if not (0xD800 <= w <= 0xDFFF):
            break
    else:
        raise RuntimeError("no BMP unit in range")
    saved = int(u[p])
    u[p] = int(rng.integers(0xD800, 0xDC00)) if rng.integers(0, 2) else \
        int(rng.integers(0xDC00, 0xE000))
    return p, saved
