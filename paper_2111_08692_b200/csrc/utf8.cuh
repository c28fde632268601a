// utf8.cuh -- UTF-8 arithmetic of the hot path, SWAR over 32-bit words (4 bytes per op).
//
//  * classify(): the validation classifier.  Six value rules (plus the C0/C1
//    and F5..FF leads that can only fail them) come from three 16-entry nibble tables keyed by
//    hi(prev1), lo(prev1), hi(cur) and AND-ed (the "three-nibble lookup-table classification"
//    of BASELINE north_star; PAPER.md:98 cites Keiser-Lemire for it).  The tables live in
//    REGISTERS and are read with PRMT (one byte permute = four 8-entry lookups).  The
//    structural rules (too short, too long) and the continuation-count check
//    are plain LOP3 bit logic.  Derivation and its brute-force check: DESIGN.md D3,
//    tests/test_derivations.py.  A position flags iff the input is invalid, and the first
//    flagged position r satisfies e <= r <= e+3 for the first error e.
//  * widths: units a position emits in UTF-16: 1 per non-continuation
//    byte, and 1 for a continuation byte that directly follows a byte >= F0 (it emits the
//    surrogate pair's second unit).  Exactly 0 or 1 unit per input byte on ANY input, so
//    out_cap = n is always safe, and every position is a fixed-size slot.
//  * decode(): code point assembly, and the UTF-16 encoding of PAPER.md:87.
//  * err_at(): the exact local first-error predicate (D2), used only to rescan
//    flagged tiles.
#pragma once
#include <cstdint>

namespace ug {
namespace u8 {

constexpr uint32_t HI = 0x80808080u;

// Kinds (same numbering as include/unigpu.h).
enum { OK = 0, HEADER_BITS = 1, TOO_SHORT = 2, TOO_LONG = 3, OVERLONG = 4, TOO_LARGE = 5,
       SURROGATE = 6 };

// Class bits: 0 overlong-2 (C0/C1 + cont), 1 overlong-3 (E0 80..9F), 2 surrogate (ED A0..BF),
// 3 overlong-4 (F0 80..8F), 4 too-large (F4 90..BF), 5 too-large lead (F5..FF + cont).
// T1 / T3 are indexed by (hi nibble ^ 8): 8..F -> entries 0..7, ASCII nibbles 0..7 -> PRMT
// sign mode on bytes whose msb is 0 -> 0x00.  T2 (lo nibble) needs all 16 entries: two PRMTs,
// the second with the selector's bit 3 flipped, OR-ed (each contributes 0x00 in sign mode).
constexpr uint32_t T1_A = 0x00000000u;  // hi(prev1) 8,9,A,B
constexpr uint32_t T1_B = 0x38060001u;  // hi(prev1) C,D,E,F
constexpr uint32_t T2_0 = 0x0000010Bu;  // lo(prev1) 0..3
constexpr uint32_t T2_1 = 0x20202010u;  // lo(prev1) 4..7
constexpr uint32_t T2_2 = 0x20202020u;  // lo(prev1) 8..B
constexpr uint32_t T2_3 = 0x20202420u;  // lo(prev1) C..F
constexpr uint32_t T3_A = 0x3535332Bu;  // hi(cur) 8,9,A,B
constexpr uint32_t T3_B = 0x00000000u;  // hi(cur) C..F

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// byte k of x -> nibble k of the result (low 16 bits), for the hi / lo nibbles of each byte
__device__ __forceinline__ uint32_t sel_hi(uint32_t x) {
  uint32_t z = (x >> 4) & 0x0F0F0F0Fu;
  return prmt(z | (z >> 4), 0u, 0x4420u);
}
__device__ __forceinline__ uint32_t sel_lo(uint32_t x) {
  uint32_t z = x & 0x0F0F0F0Fu;
  return prmt(z | (z >> 4), 0u, 0x4420u);
}

// Per-word quantities carried from one word to the next.
struct WordMasks {
  uint32_t x;   // the bytes
  uint32_t K;   // continuation bytes (10xxxxxx), msb per byte
  uint32_t L;   // >= C0
  uint32_t E;   // >= E0
  uint32_t F;   // >= F0
  uint32_t t1;  // T1[hi(byte)]
  uint32_t t2;  // T2[lo(byte)]
  uint32_t t3;  // T3[hi(byte)]
};

__device__ __forceinline__ WordMasks masks(uint32_t x, bool tables) {
  WordMasks m;
  uint32_t s1 = x << 1, s2 = x << 2, s3 = x << 3;
  m.x = x;
  m.K = x & ~s1 & HI;
  m.L = x & s1 & HI;
  m.E = m.L & s2;
  m.F = m.E & s3;
  if (tables) {
    uint32_t sh = sel_hi(x) ^ 0x8888u;
    uint32_t sl = sel_lo(x);
    m.t1 = prmt(T1_A, T1_B, sh);
    m.t3 = prmt(T3_A, T3_B, sh);
    m.t2 = prmt(T2_0, T2_1, sl) | prmt(T2_2, T2_3, sl ^ 0x8888u);
  } else {
    m.t1 = m.t2 = m.t3 = 0;
  }
  return m;
}

// Error bits (nonzero iff some position of word `c` flags) given the previous word `p`.
__device__ __forceinline__ uint32_t classify(const WordMasks &p, const WordMasks &c) {
  uint32_t p1 = __funnelshift_l(p.x, c.x, 8);     // byte i-1 for each byte i
  uint32_t Kp1 = __funnelshift_l(p.K, c.K, 8);
  uint32_t Lp1 = __funnelshift_l(p.L, c.L, 8);
  uint32_t Ep2 = __funnelshift_l(p.E, c.E, 16);
  uint32_t Fp3 = __funnelshift_l(p.F, c.F, 24);
  // rule 2 (lead then non-continuation) | rule 3 (ASCII then continuation)
  uint32_t structural = (Lp1 & ~c.K) | (c.K & ~p1);
  // continuation-count check: the 2nd continuation of a 3/4-byte lead must follow exactly
  // when prev2 >= E0 or prev3 >= F0
  uint32_t count = (Kp1 & c.K) ^ (Ep2 | Fp3);
  // value rules: T1[hi(prev1)] & T2[lo(prev1)] & T3[hi(cur)]
  uint32_t t1 = __funnelshift_l(p.t1, c.t1, 8);
  uint32_t t2 = __funnelshift_l(p.t2, c.t2, 8);
  return structural | count | (t1 & t2 & c.t3);
}

// Emit bits of word c (previous word p): msb of byte j set iff position j emits a UTF-16 unit
// (a non-continuation byte, or a continuation byte right after a byte >= F0).
__device__ __forceinline__ uint32_t emit_bits(const WordMasks &p, const WordMasks &c) {
  uint32_t Fp1 = __funnelshift_l(p.F, c.F, 8);  // byte j-1 >= F0
  return (~c.K & HI) | (c.K & Fp1);
}

// Decode the character whose lead is the low byte of x (bytes b0..b3 = x, little endian) and
// encode it as UTF-16.  Returns the first unit; *u1 = second unit.
__device__ __forceinline__ uint32_t decode_units(uint32_t x, uint32_t *u1) {
  uint32_t b0 = x & 0xFFu;
  uint32_t v2 = ((b0 & 0x1Fu) << 6) | ((x >> 8) & 0x3Fu);
  uint32_t v3 = ((b0 & 0x0Fu) << 12) | ((x >> 2) & 0x0FC0u) | ((x >> 16) & 0x3Fu);
  uint32_t cp = ((b0 & 0x07u) << 18) | ((x << 4) & 0x3F000u) | ((x >> 10) & 0x0FC0u) |
                ((x >> 24) & 0x3Fu);
  *u1 = 0xDC00u | (cp & 0x3FFu);
  uint32_t hi = 0xD7C0u + (cp >> 10);
  return b0 < 0x80u ? b0 : (b0 < 0xE0u ? v2 : (b0 < 0xF0u ? v3 : hi));
}

// ---------------------------------------------------------------- SWAR decode (a7)
// Code-unit candidates for the 4 positions of word x (bytes b0..b3; b4.. from xn), two
// positions per 32-bit op in 16-bit lanes: "even" lanes hold positions 0 and 2, "odd" lanes
// positions 1 and 3.  With c_j = b_j & 0x3F and P(j) = c_j << 6 | c_{j+1}:
//   ASCII      u = b_j
//   2-byte     u = P(j)                                  (b_j & 0x3F has bit 5 clear)
//   3-byte     u = (b_j & 0xF) << 12 | P(j+1)
//   4-byte     hi = 0xD7C0 + ((b_j & 7) << 8 | P(j+1) >> 4),  lo = 0xDC00 | P(j+2)
// Pe / Po are P at the even / odd positions of this word; Pe2 / Po2 the same two positions
// later (they need the next word's P).
__device__ __forceinline__ uint32_t pair_payload(uint32_t s) {
  // s holds, per 16-bit lane, [c_{j+1}, c_j]; returns c_j << 6 | c_{j+1} per lane
  return (s & 0x003F003Fu) | ((s >> 2) & 0x0FC00FC0u);
}
__device__ __forceinline__ uint32_t payload_even(uint32_t c) { return pair_payload(prmt(c, 0u, 0x2301u)); }
__device__ __forceinline__ uint32_t payload_odd(uint32_t c, uint32_t cn) {
  return pair_payload(prmt(c, cn, 0x3412u));
}
// per-16-bit-lane masks (0xFFFF) from per-byte top-bit masks, even / odd positions
__device__ __forceinline__ uint32_t lanes_even(uint32_t m) { return prmt(m, 0u, 0xAA88u); }
__device__ __forceinline__ uint32_t lanes_odd(uint32_t m) { return prmt(m, 0u, 0xBB99u); }
__device__ __forceinline__ uint32_t mux(uint32_t m, uint32_t a, uint32_t b) {
  return (a & m) | (b & ~m);
}

// The unit emitted at each of the 4 positions (ue: positions 0 and 2, uo: 1 and 3).  A
// continuation byte right after a 4-byte lead emits the low surrogate 0xDC00 | P(i+1).
// x: bytes of this word; Pe, Po: P at even / odd positions; Pe2: P at positions 2 and 4;
// L/E/F: >= C0 / E0 / F0 top-bit masks; LO: continuation-after-F0 top-bit mask.
__device__ __forceinline__ void units4(uint32_t x, uint32_t Pe, uint32_t Po, uint32_t Pe2,
                                       uint32_t L, uint32_t E, uint32_t F, uint32_t LO,
                                       uint32_t *ue, uint32_t *uo) {
  const uint32_t asc_e = prmt(x, 0u, 0x4240u), asc_o = prmt(x, 0u, 0x4341u);
  const uint32_t u3_e = ((x << 12) & 0xF000F000u) | Po;
  const uint32_t u3_o = ((x << 4) & 0xF000F000u) | Pe2;
  const uint32_t hi_e = (((x << 8) & 0x07000700u) | ((Po >> 4) & 0x00FF00FFu)) + 0xD7C0D7C0u;
  const uint32_t hi_o = ((x & 0x07000700u) | ((Pe2 >> 4) & 0x00FF00FFu)) + 0xD7C0D7C0u;
  uint32_t e = mux(lanes_even(L), Pe, asc_e);
  e = mux(lanes_even(E), u3_e, e);
  e = mux(lanes_even(F), hi_e, e);
  *ue = mux(lanes_even(LO), Po | 0xDC00DC00u, e);  // 0xDC00 has bits 10-11 set
  uint32_t o = mux(lanes_odd(L), Po, asc_o);
  o = mux(lanes_odd(E), u3_o, o);
  o = mux(lanes_odd(F), hi_o, o);
  *uo = mux(lanes_odd(LO), Pe2 | 0xDC00DC00u, o);
}

// ---------------------------------------------------------------- exact (cold) path
// All bytes are passed in registers (little-endian words): no local arrays.
__device__ __forceinline__ uint32_t byte_of(uint32_t x, int k) { return (x >> (8 * k)) & 0xFFu; }

// Kind of the failure of a sequential decoder whose window is x = s[0..3] (rules in the order
// of DESIGN.md R2); bytes past the end of the input are 0x00 (not continuation bytes).
__device__ __forceinline__ int decode_kind(uint32_t x) {
  uint32_t b = x & 0xFFu;
  if (b < 0x80u) return OK;
  if (b < 0xC0u) return TOO_LONG;
  if (b >= 0xF8u) return HEADER_BITS;
  int L = b < 0xE0u ? 2 : (b < 0xF0u ? 3 : 4);
  uint32_t cp = b & (0x7Fu >> L);
#pragma unroll
  for (int k = 1; k < 4; k++) {
    if (k < L) {
      uint32_t c = byte_of(x, k);
      if ((c & 0xC0u) != 0x80u) return TOO_SHORT;
      cp = (cp << 6) | (c & 0x3Fu);
    }
  }
  uint32_t minv = L == 2 ? 0x80u : (L == 3 ? 0x800u : 0x10000u);
  if (cp < minv) return OVERLONG;
  if (cp > 0x10FFFFu) return TOO_LARGE;
  if (cp >= 0xD800u && cp <= 0xDFFFu) return SURROGATE;
  return OK;
}

__device__ __forceinline__ int declared_len(uint32_t b) {
  return b < 0x80u ? 1 : (b < 0xC0u ? 0 : (b < 0xE0u ? 2 : (b < 0xF0u ? 3 : (b < 0xF8u ? 4 : 0))));
}

// Exact local predicate at position i (D2 / SURVEY.md C.4(i)): back = s[i-4..i-1],
// fwd = s[i..i+3].  A(i): a non-continuation byte whose character fails to decode.  B(i): a
// continuation byte with no lead within the 3 previous bytes that declares it.
__device__ __forceinline__ bool err_at(uint32_t back, uint32_t fwd) {
  uint32_t c = fwd & 0xFFu;
  if ((c & 0xC0u) != 0x80u) return decode_kind(fwd) != OK;
#pragma unroll
  for (int d = 1; d <= 3; d++) {
    uint32_t b = byte_of(back, 4 - d);
    if ((b & 0xC0u) != 0x80u) return !(declared_len(b) > d);
  }
  return true;
}

}  // namespace u8
}  // namespace ug
