// utf16.cuh -- UTF-16LE arithmetic of the hot path.
//
//  * Pairing predicate (exact, no rescan needed): word i is in error iff it is a high
//    surrogate not followed by a low one, or a low surrogate not preceded by a high one
//    ("During validation, only the possible surrogate pairs require attention").
//  * Widths in UTF-8 bytes: 1 below 0x80, 2 below 0x800, 2 for each half of a surrogate pair
//    (the pair's 4 bytes split 2 + 2 so each word emits its own bytes), 3 otherwise; a lone
//    surrogate also gets 2.  At most 3 bytes per word on ANY input.
//  * Bytes: minimal UTF-8 encoding.  For a pair (h, l) the code point is
//    0x10000 + ((h & 0x3FF) << 10 | (l & 0x3FF)), so bytes 1-2 depend only on h
//    (cp >> 10 = 0x40 + (h & 0x3FF)) and bytes 3-4 on l and the low 2 bits of h.
#pragma once
#include <cstdint>

#include "swar.cuh"

namespace ug {
namespace u16 {

UG_HD bool is_high(uint32_t u) { return (u & 0xFC00u) == 0xD800u; }
UG_HD bool is_low(uint32_t u) { return (u & 0xFC00u) == 0xDC00u; }

// UTF-8 bytes emitted for word u: the same rule as widths() / len16_word (a surrogate 2, so a
// pair 4, a lone surrogate 2 as well).  On a valid prefix this is the minimal encoding length.
UG_HD uint32_t width(uint32_t u) {
  const bool two = u < 0x800u || (u & 0xF800u) == 0xD800u;
  return 1u + (u >= 0x80u ? 1u : 0u) + (two ? 0u : 1u);
}

UG_HD bool err_at(uint32_t prev, uint32_t u, uint32_t next) {
  return (is_high(u) && !is_low(next)) || (is_low(u) && !is_high(prev));
}



// ---------------------------------------------------------------- byte-SWAR, 4 words per op
// The 4 words of two registers (wa = words 0, 1; wb = words 2, 3) are split into their low
// and high bytes (2 PRMT), so every class test, width and output byte below is one byte lane
// per word.  Masks are msb-per-byte.
//  * widths (a5): w = 1 + [u >= 0x80] + [u >= 0x800 and u not a surrogate]: a surrogate
//    emits 2 bytes, so a pair emits its 4 and every word at most 3 on ANY input
//    (SPEC.md S:175).  The same rule gives utf8_length_from_utf16le.
//  * output (a7), first / second / third byte of each word:
//      u < 0x80     : u
//      u < 0x800    : C0 | u >> 6,          80 | u & 3F
//      other BMP    : E0 | u >> 12,         80 | (u >> 6) & 3F,   80 | u & 3F
//      high h (pair): F0 | h' >> 8,         80 | (h' >> 2) & 3F            h' = (h & 3FF) + 40
//      low l (pair) : 80 | (h & 3) << 4 | (l >> 6) & F,   80 | l & 3F      (h: previous word)
struct Cls4 {
  uint32_t lo, hi;              // low / high bytes of the 4 words
  uint32_t ge80, ge800, S, H;   // u >= 0x80, u >= 0x800, surrogate, high surrogate
  uint32_t L;                   // low surrogate
};
// BE: the words are stored big-endian (UTF-16BE): the byte order is folded
// into the split by swapping the two selectors, everything after it is unchanged.
template <bool BE = false>
UG_HD Cls4 classes4(uint32_t wa, uint32_t wb) {
  Cls4 c;
  c.lo = prmt(wa, wb, BE ? 0x7531u : 0x6420u);
  c.hi = prmt(wa, wb, BE ? 0x6420u : 0x7531u);
  // (the byte adds are IMADs: the FMA pipe has room, the ALU pipe is the busy one)
  const uint32_t h7 = c.hi & 0x7F7F7F7Fu;
  c.ge800 = (mad(h7, 1u, 0x78787878u) | c.hi) & HI;         // hi >= 8 (7-bit adds)
  c.ge80 = (mad(h7, 1u, 0x7F7F7F7Fu) | c.hi | c.lo) & HI;    // hi != 0 or lo >= 0x80
  const uint32_t z = (c.hi & 0xF8F8F8F8u) ^ 0xD8D8D8D8u;
  c.S = ~(mad(z & 0x7F7F7F7Fu, 1u, 0x7F7F7F7Fu) | z) & HI;  // hi in D8..DF
  const uint32_t b2 = c.hi << 5;                        // bit 2 of hi: DC..DF
  c.L = c.S & b2;
  c.H = c.S & ~b2;
  return c;
}
// width - 1 per byte lane (0..2)
UG_HD uint32_t wm1(const Cls4 &c) { return (c.ge80 >> 7) + ((c.ge800 & ~c.S) >> 7); }
// width per byte lane (1..3), both shifts and adds on the FMA pipe (IMAD.HI accumulate)
UG_HD uint32_t widths(const Cls4 &c) {
  return mad_hi(c.ge800 & ~c.S, 1u << 25, mad_hi(c.ge80, 1u << 25, 0x01010101u));
}
// byte mask (0xFF per lane) from an msb-per-byte mask
UG_HD uint32_t bmask(uint32_t m) { return prmt(m, 0u, 0xBA98u); }

// Output byte planes of the 4 words: byte j of *O0 / *O1 / *O2 = first / second / third
// output byte of word j (meaningful up to its width).  lp: low byte of the previous word
// in each lane (the high surrogate's low bits for a low surrogate).
UG_HD void encode4(const Cls4 &c, uint32_t lp, uint32_t *O0, uint32_t *O1, uint32_t *O2) {
  const uint32_t U6 = muxc<0xFCFCFCFCu>(c.hi << 2, c.lo >> 6);  // (u >> 6) & 0xFF
  const uint32_t T = (c.lo & 0x3F3F3F3Fu) | HI;                 // 80 | u & 3F
  // first byte
  const uint32_t vB = U6 | 0xC0C0C0C0u;
  const uint32_t vC = ((c.hi >> 4) & 0x0F0F0F0Fu) | 0xE0E0E0E0u;
  const uint32_t cy = shr_fma<7>(c.lo & (c.lo << 1) & HI);      // lo >= 0xC0: h' carries
  const uint32_t vH = mad(c.hi & 0x03030303u, 1u, cy) | 0xF0F0F0F0u;
  const uint32_t vL = ((lp << 4) & 0x30303030u) | (U6 & 0x0F0F0F0Fu) | HI;
  const uint32_t mS = bmask(c.S), mH = bmask(c.H);
  const uint32_t mB = bmask(c.ge80 & ~c.ge800), mA = bmask(~c.ge80 & HI);
  uint32_t x = mux(mH, vH, vL);
  x = mux(mS, x, vC);
  x = mux(mB, vB, x);
  *O0 = mux(mA, c.lo, x);
  // second byte
  const uint32_t vH1 = (mad(shr_fma<2>(c.lo) & 0x3F3F3F3Fu, 1u, 0x10101010u) & 0x3F3F3F3Fu) | HI;
  const uint32_t mC = bmask(c.ge800 & ~c.S);
  *O1 = mux(mC, (U6 & 0x3F3F3F3Fu) | HI, mux(mH, vH1, T));
  // third byte
  *O2 = T;
}

// ---------------------------------------------------------------- surrogate-free fast path
// (the BMP-only case).  A group whose words hold no
// surrogate cannot be invalid (only surrogates need attention), and every word is
// a 1-, 2- or 3-byte character: only the low / high byte split and two class masks are needed.
struct Bmp4 {
  uint32_t lo, hi;      // low / high bytes of the 4 words
  uint32_t ge80, ge800;  // u >= 0x80, u >= 0x800 (msb per byte)
};
template <bool BE = false>
UG_HD Bmp4 classes4_bmp(uint32_t wa, uint32_t wb) {
  Bmp4 c;
  c.lo = prmt(wa, wb, BE ? 0x7531u : 0x6420u);
  c.hi = prmt(wa, wb, BE ? 0x6420u : 0x7531u);
  const uint32_t h7 = c.hi & 0x7F7F7F7Fu;
  c.ge800 = (mad(h7, 1u, 0x78787878u) | c.hi) & HI;
  c.ge80 = (mad(h7, 1u, 0x7F7F7F7Fu) | c.hi | c.lo) & HI;
  return c;
}
UG_HD uint32_t widths_bmp(const Bmp4 &c) {
  return mad_hi(c.ge800, 1u << 25, mad_hi(c.ge80, 1u << 25, 0x01010101u));
}
// Output byte planes as encode4, for surrogate-free words.
UG_HD void encode4_bmp(const Bmp4 &c, uint32_t *O0, uint32_t *O1, uint32_t *O2) {
  const uint32_t U6 = muxc<0xFCFCFCFCu>(c.hi << 2, c.lo >> 6);  // (u >> 6) & 0xFF
  const uint32_t T = (c.lo & 0x3F3F3F3Fu) | HI;                 // 80 | u & 3F
  const uint32_t vB = U6 | 0xC0C0C0C0u;                          // 2-byte lead
  const uint32_t vC = ((c.hi >> 4) & 0x0F0F0F0Fu) | 0xE0E0E0E0u; // 3-byte lead
  const uint32_t mC = bmask(c.ge800), mA = bmask(~c.ge80 & HI);
  *O0 = mux(mA, c.lo, mux(mC, vC, vB));
  *O1 = mux(mC, (U6 & 0x3F3F3F3Fu) | HI, T);
  *O2 = T;
}

}  // namespace u16
}  // namespace ug
