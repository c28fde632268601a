// utf16.cuh -- UTF-16LE arithmetic of the hot path.
//
//  * Pairing predicate (exact, no rescan needed): word i is in error iff it is a high
//    surrogate not followed by a low one, or a low surrogate not preceded by a high one
//    ("During validation, only the possible surrogate pairs require attention").
//  * Widths in UTF-8 bytes: 1 below 0x80, 2 below 0x800, 2 for each half of a surrogate pair
//    (the pair's 4 bytes split 2 + 2 so each word emits its own bytes), 3 otherwise; a lone
//    high gets 2 and a lone low 3.  At most 3 bytes per word on ANY input.
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

UG_HD uint32_t width(uint32_t u, uint32_t prev) {
  const bool two = u < 0x800u || is_high(u) || (is_low(u) && is_high(prev));
  return 1u + (u >= 0x80u ? 1u : 0u) + (two ? 0u : 1u);
}

UG_HD bool err_at(uint32_t prev, uint32_t u, uint32_t next) {
  return (is_high(u) && !is_low(next)) || (is_low(u) && !is_high(prev));
}

// UTF-8 bytes of word u (little-endian packed, width(u, prev) of them are meaningful).
// Branch-free: all candidates computed, then selected.
UG_HD uint32_t utf8_bytes(uint32_t u, uint32_t prev) {
  const uint32_t t6 = 0x80u | (u & 0x3Fu);         // last continuation byte
  const uint32_t m6 = 0x80u | ((u >> 6) & 0x3Fu);  // middle continuation byte
  const uint32_t b2 = (0xC0u | (u >> 6)) | (t6 << 8);
  const uint32_t b3 = (0xE0u | (u >> 12)) | (m6 << 8) | (t6 << 16);
  const uint32_t h10 = (u & 0x3FFu) + 0x40u;       // cp >> 10 of a pair
  const uint32_t bh = (0xF0u | (h10 >> 8)) | ((0x80u | ((h10 >> 2) & 0x3Fu)) << 8);
  const uint32_t bl = (0x80u | ((prev & 3u) << 4) | ((u >> 6) & 0xFu)) | (t6 << 8);
  uint32_t v = b3;
  v = (is_low(u) && is_high(prev)) ? bl : v;
  v = is_high(u) ? bh : v;
  v = (u < 0x800u) ? b2 : v;
  v = (u < 0x80u) ? u : v;
  return v;
}

#if defined(__CUDACC__)
// ---------------------------------------------------------------- SWAR (two words per op)
// Masks carry one bit per 16-bit lane, at bit 15 (low word) and bit 31 (high word).
constexpr uint32_t LANE_TOP = 0x80008000u;
// lane == 0 -> top bit set (exact per lane: no borrow across lanes)
__device__ __forceinline__ uint32_t zero_lanes(uint32_t x) {
  return ~(((x & 0x7FFF7FFFu) + 0x7FFF7FFFu) | x) & LANE_TOP;
}
// top-bit lane masks -> 0xFFFF per selected lane (PRMT sign replication of bytes 1 and 3)
__device__ __forceinline__ uint32_t lanes16(uint32_t m) {
  uint32_t d;
  asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(d) : "r"(m));
  return d;
}

struct Cls2 {
  uint32_t A;   // u < 0x80
  uint32_t B;   // u < 0x800
  uint32_t H;   // high surrogate
  uint32_t L;   // low surrogate
};
// Per-lane compares without cross-lane carries: (u & 0x7FFF) + (0x8000 - k) sets bit 15 iff
// (u & 0x7FFF) >= k; OR-ing u's own bit 15 gives u >= k for k <= 0x8000.
__device__ __forceinline__ Cls2 classes2(uint32_t r) {
  Cls2 c;
  const uint32_t lo15 = r & 0x7FFF7FFFu;
  c.A = ~((lo15 + 0x7F807F80u) | r) & LANE_TOP;          // u < 0x80
  c.B = ~((lo15 + 0x78007800u) | r) & LANE_TOP;          // u < 0x800
  const uint32_t S = zero_lanes((r & 0xF800F800u) ^ 0xD800D800u);  // D800..DFFF
  const uint32_t b10 = (r << 5) & LANE_TOP;              // bit 10: low (DC00..) vs high
  c.H = S & ~b10;
  c.L = S & b10;
  return c;
}
// three-byte lanes (a5): not < 0x800, not a high surrogate, not a low one after a high one
__device__ __forceinline__ uint32_t three2(const Cls2 &c, uint32_t Hp) {
  return ~(c.B | c.H | (c.L & Hp)) & LANE_TOP;
}

// UTF-8 byte streams of the two words of r: lane k of B0/B1/B2 holds the
// first / second / third byte of word k (only the first width(word) are meaningful).
// pl = the two previous words ([word before lane 0, lane 0]); Hp = previous word is high.
__device__ __forceinline__ void encode2(uint32_t r, uint32_t pl, const Cls2 &c, uint32_t Hp,
                                        uint32_t *B0, uint32_t *B1, uint32_t *B2) {
  const uint32_t r6 = r >> 6;
  const uint32_t t6 = (r & 0x003F003Fu) | 0x00800080u;
  const uint32_t m6 = (r6 & 0x003F003Fu) | 0x00800080u;
  const uint32_t c2 = (r6 & 0x001F001Fu) | 0x00C000C0u;
  const uint32_t e3 = ((r >> 12) & 0x000F000Fu) | 0x00E000E0u;
  const uint32_t h10 = (r & 0x03FF03FFu) + 0x00400040u;  // cp >> 10 of a pair
  const uint32_t hl = ((h10 >> 8) & 0x00070007u) | 0x00F000F0u;
  const uint32_t hm = ((h10 >> 2) & 0x003F003Fu) | 0x00800080u;
  const uint32_t ll = ((pl & 0x00030003u) << 4) | (r6 & 0x000F000Fu) | 0x00800080u;
  const uint32_t mB = lanes16(c.B), mA = lanes16(c.A), mH = lanes16(c.H);
  const uint32_t mLp = lanes16(c.L & Hp);
  uint32_t b0 = (c2 & mB) | (e3 & ~mB);
  b0 = (r & mA) | (b0 & ~mA);
  b0 = (hl & mH) | (b0 & ~mH);
  *B0 = (ll & mLp) | (b0 & ~mLp);
  const uint32_t mT = mB | mLp;
  uint32_t b1 = (t6 & mT) | (m6 & ~mT);
  *B1 = (hm & mH) | (b1 & ~mH);
  *B2 = t6;
}


#endif  // __CUDACC__

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
  const uint32_t h7 = c.hi & 0x7F7F7F7Fu;
  c.ge800 = ((h7 + 0x78787878u) | c.hi) & HI;         // hi >= 8 (no carries: 7-bit adds)
  c.ge80 = ((h7 + 0x7F7F7F7Fu) | c.hi | c.lo) & HI;    // hi != 0 or lo >= 0x80
  const uint32_t z = (c.hi & 0xF8F8F8F8u) ^ 0xD8D8D8D8u;
  c.S = ~(((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) & HI;  // hi in D8..DF
  const uint32_t b2 = c.hi << 5;                        // bit 2 of hi: DC..DF
  c.L = c.S & b2;
  c.H = c.S & ~b2;
  return c;
}
// width - 1 per byte lane (0..2)
UG_HD uint32_t wm1(const Cls4 &c) { return (c.ge80 >> 7) + ((c.ge800 & ~c.S) >> 7); }
// byte mask (0xFF per lane) from an msb-per-byte mask
UG_HD uint32_t bmask(uint32_t m) { return prmt(m, 0u, 0xBA98u); }

// Output byte planes of the 4 words: byte j of *O0 / *O1 / *O2 = first / second / third
// output byte of word j (meaningful up to its width).  lp: low byte of the previous word
// in each lane (the high surrogate's low bits for a low surrogate).
UG_HD void encode4(const Cls4 &c, uint32_t lp, uint32_t *O0, uint32_t *O1, uint32_t *O2) {
  const uint32_t U6 = mux(0xFCFCFCFCu, c.hi << 2, c.lo >> 6);   // (u >> 6) & 0xFF
  const uint32_t T = (c.lo & 0x3F3F3F3Fu) | HI;                 // 80 | u & 3F
  // first byte
  const uint32_t vB = U6 | 0xC0C0C0C0u;
  const uint32_t vC = ((c.hi >> 4) & 0x0F0F0F0Fu) | 0xE0E0E0E0u;
  const uint32_t cy = (c.lo & (c.lo << 1) & HI) >> 7;           // lo >= 0xC0: h' carries
  const uint32_t vH = ((c.hi & 0x03030303u) + cy) | 0xF0F0F0F0u;
  const uint32_t vL = ((lp << 4) & 0x30303030u) | (U6 & 0x0F0F0F0Fu) | HI;
  const uint32_t mS = bmask(c.S), mH = bmask(c.H);
  const uint32_t mB = bmask(c.ge80 & ~c.ge800), mA = bmask(~c.ge80 & HI);
  uint32_t x = mux(mH, vH, vL);
  x = mux(mS, x, vC);
  x = mux(mB, vB, x);
  *O0 = mux(mA, c.lo, x);
  // second byte
  const uint32_t vH1 = ((((c.lo >> 2) & 0x3F3F3F3Fu) + 0x10101010u) & 0x3F3F3F3Fu) | HI;
  const uint32_t mC = bmask(c.ge800 & ~c.S);
  *O1 = mux(mC, (U6 & 0x3F3F3F3Fu) | HI, mux(mH, vH1, T));
  // third byte
  *O2 = T;
}

}  // namespace u16
}  // namespace ug
