// utf8_keyed.cuh -- SURVEY 8(f) f4: the paper's keyed 12-byte UTF-8 -> UTF-16 routine
// (section 4 "Algorithms"; table shapes), re-expressed for
// one GPU thread over its own 32 bytes, as a research comparison with the end-position SWAR
// decoder of a7 (utf8.cuh units4).  Host-compilable: tests/emu/kernel_math_emu.cpp runs it on
// every fuzz8 chunk beside units4 and checks both against the oracle.
//
//  * KEY: bit i of a 12-bit word = "byte i of the window is the LAST byte of its
//    character" (the end-of-character convention of SPEC.md S:289-292; the paper's leading-byte
//    mask carries the same information).  The key table maps each of the 4096 keys to the
//    number of bytes consumed, the number of characters decoded and a shuffle index.  The
//    paper's "1024-entry table" cannot be indexed by 12 bits (R23): 4096 entries here.
//  * THREE PATHS: index [0, 64) = six characters of 1-2 bytes, [64, 145) = four
//    of 1-3 bytes, [145, 209) = three of 1-4 bytes.  For a key the path consuming the most
//    bytes wins, ties to the earlier path; a path takes the longest prefix of
//    the window's whole characters that fits its length bound and character count.
//  * SHUFFLE ("the shuffle mask can then be applied to the 12 input bytes"): on
//    the GPU a byte shuffle of a 12-byte window held in three registers w0..w2 is, per output
//    register, mux(M, prmt(w0, w1, A), prmt(w2, 0, B)) -- two PRMT and one LOP3; an entry holds
//    the four (A | B << 16) selector pairs and the four byte masks M.  Path (a) places each
//    character in a 16-bit lane (last byte low, lead byte high, zero for ASCII); paths (b) and
//    (c) in a 32-bit lane, last byte lowest, zero above the character's length.
//  * FAST PATHS (-DUG_KEYED_FASTPATHS, off by default: 11-16 % slower on the GPU):
//    before the lookup, 16 ASCII bytes, 16 bytes of two-byte characters or 12 bytes of
//    three-byte characters (R23) are decoded directly.
//  * Emission follows a7 exactly, so the planned kernel's per-thread counts and offsets hold:
//    a thread emits the units of the positions it owns, a character's unit at its last byte
//    and a 4-byte character's high surrogate at its third byte.  Characters straddling the
//    thread's first or last byte are decoded one at a time outside the keyed loop.
#pragma once
#include <cstdint>

#include "swar.cuh"

namespace ug {
namespace keyed {

constexpr int KEYS = 4096;
constexpr int SHUFFLES = 64 + 81 + 64;  // PAPER.md:95 index ranges
constexpr int SHUF_WORDS = 8;           // per shuffle entry: 4 selector pairs, 4 byte masks

// ---------------------------------------------------------------- tables (host)
// Key entry: bits 0-3 bytes consumed (0: no whole character in the window), bits 4-6
// characters decoded, bits 8-15 shuffle index.
inline uint16_t key_entry(int consumed, int nch, int idx) {
  return (uint16_t)(consumed | (nch << 4) | (idx << 8));
}

// Shuffle entry for a path (0 = a, 1 = b, 2 = c) and its tuple of character lengths.
inline void shuffle_entry(int path, const int *len, uint32_t *e) {
  const int nch = path == 0 ? 6 : (path == 1 ? 4 : 3);
  uint8_t src[4][4];  // window byte feeding each output byte, 0xFF = zero
  for (int r = 0; r < 4; r++)
    for (int k = 0; k < 4; k++) src[r][k] = 0xFF;
  int s = 0;
  for (int j = 0; j < nch; j++) {
    const int l = len[j];
    if (path == 0) {  // 16-bit lane j % 2 of register j / 2: low = last byte, high = lead
      src[j / 2][2 * (j % 2)] = (uint8_t)(s + l - 1);
      if (l == 2) src[j / 2][2 * (j % 2) + 1] = (uint8_t)s;
    } else {          // 32-bit lane j: byte k = the k-th byte from the character's end
      for (int k = 0; k < l; k++) src[j][k] = (uint8_t)(s + l - 1 - k);
    }
    s += l;
  }
  for (int r = 0; r < 4; r++) {
    uint32_t a = 0, b = 0, m = 0;
    for (int k = 0; k < 4; k++) {
      const int w = src[r][k];
      if (w < 8) {
        a |= (uint32_t)w << (4 * k);
        m |= 0xFFu << (8 * k);
      } else {
        b |= (uint32_t)(w < 12 ? w - 8 : 4) << (4 * k);  // byte 0 of the zero register
      }
    }
    e[r] = a | (b << 16);
    e[4 + r] = m;
  }
}

// key[KEYS], shuf[SHUFFLES * SHUF_WORDS]
inline void build_tables(uint16_t *key, uint32_t *shuf) {
  static const int NCH[3] = {6, 4, 3}, MAXL[3] = {2, 3, 4}, BASE[3] = {0, 64, 145};
  for (int path = 0; path < 3; path++) {
    const int count = path == 0 ? 64 : (path == 1 ? 81 : 64);
    for (int i = 0; i < count; i++) {
      int len[6], v = i;
      for (int j = NCH[path] - 1; j >= 0; j--) {  // mixed radix, character 0 most significant
        len[j] = 1 + v % MAXL[path];
        v /= MAXL[path];
      }
      shuffle_entry(path, len, shuf + (size_t)(BASE[path] + i) * SHUF_WORDS);
    }
  }
  for (int k = 0; k < KEYS; k++) {
    int len[12], nc = 0, prev = -1;
    for (int i = 0; i < 12; i++)
      if (k >> i & 1) {
        len[nc++] = i - prev;
        prev = i;
      }
    int best = 0, bpath = -1, bn = 0;
    for (int path = 0; path < 3; path++) {
      int c = 0, n = 0;
      while (n < nc && n < NCH[path] && len[n] <= MAXL[path]) c += len[n++];
      if (c > best) best = c, bpath = path, bn = n;
    }
    if (bpath < 0) {
      key[k] = 0;
      continue;
    }
    int idx = 0;
    for (int j = 0; j < NCH[bpath]; j++) idx = idx * MAXL[bpath] + (j < bn ? len[j] - 1 : 0);
    key[k] = key_entry(best, bn, BASE[bpath] + idx);
  }
}

// ---------------------------------------------------------------- the per-thread decode
// 4 bits: msb of each byte of m.
UG_HD uint32_t msb4(uint32_t m) { return (((m & HI) >> 7) * 0x204081u) >> 21 & 0xFu; }
// 4 bits: byte k of x is not a continuation byte (10xxxxxx).
UG_HD uint32_t noncont4(uint32_t x) { return msb4(~(x & ~(x << 1))); }
// 4 bits: byte k of x is the last byte of a character starting at byte k - d, for the
// declared length d + 1 of that lead (0xxxxxxx, 110xxxxx, 1110xxxx, 11110xxx),
// returned as ends[d] (lead masks; the caller shifts them by d positions).
UG_HD void leads4(uint32_t x, uint32_t *a, uint32_t *l2, uint32_t *l3, uint32_t *l4) {
  const uint32_t x1 = x << 1, x2 = x << 2, x3 = x << 3, x4 = x << 4;
  *a = msb4(~x);
  *l2 = msb4(x & x1 & ~x2);
  *l3 = msb4(x & x1 & x2 & ~x3);
  *l4 = msb4(x & x1 & x2 & x3 & ~x4);
}

UG_HD int ctz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
  return __ffsll((long long)x) - 1;
#else
  return __builtin_ctzll(x);
#endif
}
UG_HD int msb32(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return 31 - __clz(x);
#else
  return 31 - __builtin_clz(x);
#endif
}

// Code point of a character of l bytes, b = its bytes, first byte lowest.
UG_HD uint32_t code_point(uint32_t b, int l) {
  const uint32_t b0 = b & 0xFFu, b1 = (b >> 8) & 0x3Fu, b2 = (b >> 16) & 0x3Fu,
                 b3 = (b >> 24) & 0x3Fu;
  if (l == 1) return b0;
  if (l == 2) return (b0 & 0x1Fu) << 6 | b1;
  if (l == 3) return (b0 & 0x0Fu) << 12 | b1 << 6 | b2;
  return (b0 & 0x07u) << 18 | b1 << 12 | b2 << 6 | b3;
}

// Thread's own bytes at img[0, 32), readable img[-4, 48), img 4-byte aligned; words = the
// same 40 bytes img[-4, 36) as ten words (prev, own 8, next).  Emits the units of own
// positions [lo, hi) into out[0, cap) (cap: the thread's count), returns the units emitted.
UG_HD int decode_thread(const uint8_t *img, const uint32_t *words, int lo, int hi,
                        const uint16_t *ktab, const uint32_t *stab, uint16_t *out, int cap) {
  // Character ends by DECLARED length (the lead bytes, "we can quickly determine
  // the leading bytes and thus the end of each character"): on a valid prefix the same as
  // "the next byte is not a continuation", and before the first error exactly a7's emission
  // points (utf8.cuh), which a corrupted byte after a character cannot move.
  uint64_t NC = 0, A = 0, L2 = 0, L3 = 0, L4 = 0;  // bit i + 4: position i in [-4, 36)
#pragma unroll
  for (int k = 0; k < 10; k++) {
    uint32_t a, l2, l3, l4;
    leads4(words[k], &a, &l2, &l3, &l4);
    NC |= (uint64_t)noncont4(words[k]) << (4 * k);
    A |= (uint64_t)a << (4 * k);
    L2 |= (uint64_t)l2 << (4 * k);
    L3 |= (uint64_t)l3 << (4 * k);
    L4 |= (uint64_t)l4 << (4 * k);
  }
  const uint64_t END = A | (L2 << 1) | (L3 << 2) | (L4 << 3);
  const uint64_t own = hi > lo ? (((1ull << (hi - lo)) - 1ull) << (lo + 4)) : 0ull;
  const uint64_t ENDa = END & own;
  int nout = 0;
  auto emit = [&](uint32_t u) {
    if (nout < cap) out[nout] = (uint16_t)u;
    nout++;
  };
  int p = lo;
  if (lo == 0 && hi > 0 && !(NC >> 4 & 1u)) {
    // head: byte 0 continues a character whose lead is the last non-continuation byte in
    // [-3, -1]; its end follows from the lead's declared length
    const uint32_t leads = (uint32_t)(NC & 0xEu);
    if (!leads) return nout;  // invalid (an error at or before position 0)
    const int p0 = msb32(leads) - 4;
    const uint32_t b = fsr(words[0], words[1], 8 * (p0 + 4));  // bytes p0 .. p0 + 3
    const uint32_t b0 = b & 0xFFu;
    const int l = 1 + (b0 >= 0xC0u) + (b0 >= 0xE0u) + (b0 >= 0xF0u);
    const int e0 = p0 + l - 1;
    if (e0 < 0) return nout;  // invalid: byte 0 is a stray continuation
    const uint32_t cp = code_point(b, l);
    if (l == 4) {
      if (p0 + 2 >= 0 && p0 + 2 < hi) emit(0xD7C0u + (cp >> 10));
      if (e0 < hi) emit(0xDC00u | (cp & 0x3FFu));
    } else if (e0 < hi) {
      emit(cp);
    }
    p = e0 + 1;
  }
  while (p < hi) {
#ifdef UG_KEYED_FASTPATHS
    {
    const uint32_t *wp = reinterpret_cast<const uint32_t *>(img + (p & ~3));
    const uint32_t sh = 8u * (uint32_t)(p & 3);
    const uint32_t r0 = wp[0], r1 = wp[1], r2 = wp[2], r3 = wp[3];
    const uint32_t w0 = fsr(r0, r1, sh), w1 = fsr(r1, r2, sh), w2 = fsr(r2, r3, sh);
    // the routine's three homogeneous fast paths: 16 ASCII bytes, 16 bytes of
    // two-byte characters, and (R23) 12 bytes of three-byte characters.  Off by default: on
    // the GPU they cost 11-16 % (the checks run every iteration; a lane that hits one still
    // waits for the lanes of its warp that do not)
    if (p + 16 <= hi) {
      const uint32_t w3 = fsr(r3, wp[4], sh);
      if (((w0 | w1 | w2 | w3) & HI) == 0u) {
        const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
          for (int b = 0; b < 4; b++) emit((w[k] >> (8 * b)) & 0xFFu);
        p += 16;
        continue;
      }
      if ((w0 & 0xC0E0C0E0u) == 0x80C080C0u && (w1 & 0xC0E0C0E0u) == 0x80C080C0u &&
          (w2 & 0xC0E0C0E0u) == 0x80C080C0u && (w3 & 0xC0E0C0E0u) == 0x80C080C0u) {
        const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
        for (int k = 0; k < 4; k++) {
          emit(((w[k] & 0x1Fu) << 6) | ((w[k] >> 8) & 0x3Fu));
          emit(((w[k] >> 10) & 0x7C0u) | ((w[k] >> 24) & 0x3Fu));
        }
        p += 16;
        continue;
      }
    }
    if (p + 12 <= hi && (w0 & 0xF0C0C0F0u) == 0xE08080E0u && (w1 & 0xC0F0C0C0u) == 0x80E08080u &&
        (w2 & 0xC0C0F0C0u) == 0x8080E080u) {
      emit(code_point(w0, 3));
      emit(code_point(fsr(w0, w1, 24), 3));
      emit(code_point(fsr(w1, w2, 16), 3));
      emit(code_point(w2 >> 8, 3));
      p += 12;
      continue;
    }
    }
#endif
    const uint32_t key = (uint32_t)(ENDa >> (p + 4)) & 0xFFFu;
    const uint32_t ke = ktab[key];
    const int consumed = (int)(ke & 15u);
    if (consumed == 0) break;
    const int nch = (int)(ke >> 4 & 7u);
    const uint32_t idx = ke >> 8;
    // the 12-byte window at p (aligned 4-byte loads + funnel shifts)
    const uint32_t *wp = reinterpret_cast<const uint32_t *>(img + (p & ~3));
    const uint32_t sh = 8u * (uint32_t)(p & 3);
    const uint32_t r0 = wp[0], r1 = wp[1], r2 = wp[2], r3 = wp[3];
    const uint32_t w0 = fsr(r0, r1, sh), w1 = fsr(r1, r2, sh), w2 = fsr(r2, r3, sh);
    const uint32_t *e = stab + idx * SHUF_WORDS;
    uint32_t v[4];
#pragma unroll
    for (int r = 0; r < 4; r++) v[r] = mux(e[4 + r], prmt(w0, w1, e[r]), prmt(w2, 0u, e[r] >> 16));
    if (idx < 64) {  // (a) six characters of 1-2 bytes, 16-bit lanes
#pragma unroll
      for (int r = 0; r < 3; r++) {
        const uint32_t u = ((v[r] >> 2) & 0x07C007C0u) | (v[r] & 0x007F007Fu);
        if (2 * r < nch) emit(u & 0xFFFFu);
        if (2 * r + 1 < nch) emit(u >> 16);
      }
    } else if (idx < 145) {  // (b) four characters of 1-3 bytes, 32-bit lanes
#pragma unroll
      for (int j = 0; j < 4; j++)
        if (j < nch) emit((v[j] & 0x7Fu) | ((v[j] >> 2) & 0x0FC0u) | ((v[j] >> 4) & 0xF000u));
    } else {  // (c) three characters of 1-4 bytes
#pragma unroll
      for (int j = 0; j < 3; j++) {
        if (j >= nch) break;
        uint32_t x = (v[j] & 0x7Fu) | ((v[j] >> 2) & 0xFC0u) | ((v[j] >> 4) & 0x3F000u) |
                     ((v[j] >> 6) & 0x1C0000u);
        if ((v[j] >> 24) == 0u) x &= 0xFFFFu;  // 1-3 bytes: drop the 3-byte lead's bit 5
        if (x >= 0x10000u) {
          emit(0xD7C0u + (x >> 10));
          emit(0xDC00u | (x & 0x3FFu));
        } else {
          emit(x);
        }
      }
    }
    p += consumed;
  }
  // tail: a 4-byte character whose third byte is owned but whose last byte is not
  if (p >= 0 && p + 2 < hi) {
    const uint32_t *wp = reinterpret_cast<const uint32_t *>(img + (p & ~3));
    const uint32_t b = fsr(wp[0], wp[1], 8u * (uint32_t)(p & 3));
    if ((b & 0xF8u) == 0xF0u) emit(0xD7C0u + (code_point(b, 4) >> 10));
  }
  return nout;
}

}  // namespace keyed
}  // namespace ug
