// utf8.cuh -- UTF-8 arithmetic of the hot path (host-compilable: tests/emu/kernel_math_emu.cpp).
//
// Two representations, each used where it is cheapest (D3/D4):
//
//  * VALIDATION on BIT PLANES.  A thread's 32 bytes are transposed (PRMT 4x4 byte transposes +
//    three delta swaps) into eight 32-bit planes, P[b] bit i = bit b of byte i.  Every rule is
//    then one LOP3/SHF per 32 positions:
//      - structure (rules 2 and 3, plus the continuation count): with
//        L = lead >= C0, E = lead >= E0, F = lead >= F0 and K = continuation byte, the bytes
//        that must be continuations are R = S1(L) | S2(E) | S3(F) (Sd = shift by d positions,
//        carrying the 3 bytes before the chunk); any position where R != K is in error;
//      - value (rules 4-6 and the C0/C1, F5..FF leads): the lead bytes E0, F0
//        need a second byte >= A0 / >= 90, ED, F4 need one < A0 / < 90, and C0, C1, F5..FF
//        are always wrong; flagged at the lead, looking one byte ahead.
//    A position flags iff the input is invalid there, and the first flagged position r obeys
//    e <= r <= e + 3 for the first error e (e is the start of the offending sequence, DESIGN
//    R1), so a tile that flags rescans its own positions with the exact predicate err_at().
//  * TRANSCODING in BYTE-SWAR at END positions (4 positions per 32-bit op).  Each character
//    emits its UTF-16 unit at its LAST byte e (a 4-byte character emits its high surrogate at
//    its third byte and its low surrogate at its fourth), so every emitted unit is a function
//    of bytes e-2..e only, and its low byte always has the same form:
//      lb = (b[e-1] << 6 | b[e] & 0x3F) & 0xFF        (ASCII: b[e])
//      hb = (b[e-1] & 0x3F) >> 2  |  (b[e-2] & 0xF) << 4 if b[e-2] >= E0   (ASCII: 0)
//    (the code point is the concatenation of the payload bits, the
//    surrogate pair).  The low surrogate is 0xDC00 | (G & 0x3FF) and the high surrogate
//    0xD800 | ((G >> 4) - 0x40) of the same G = hb:lb.  Each position emits 0 or 1 unit on ANY
//    input, so out_cap = n always suffices.
#pragma once
#include <cstdint>

#include "swar.cuh"

namespace ug {
namespace u8 {

// Kinds (same numbering as include/unigpu.h).
enum { OK = 0, HEADER_BITS = 1, TOO_SHORT = 2, TOO_LONG = 3, OVERLONG = 4, TOO_LARGE = 5,
       SURROGATE = 6 };

// ---------------------------------------------------------------- bit planes
// t_j = byte j of a, b, c, d (a 4x4 byte transpose, 8 PRMT).
UG_HD void tr4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t &t0, uint32_t &t1,
               uint32_t &t2, uint32_t &t3) {
  const uint32_t ab0 = prmt(a, b, 0x5140u), ab1 = prmt(a, b, 0x7362u);
  const uint32_t cd0 = prmt(c, d, 0x5140u), cd1 = prmt(c, d, 0x7362u);
  t0 = prmt(ab0, cd0, 0x5410u);
  t1 = prmt(ab0, cd0, 0x7632u);
  t2 = prmt(ab1, cd1, 0x5410u);
  t3 = prmt(ab1, cd1, 0x7632u);
}
// Exchange bit b (b & D set) of every byte of a with bit b - D of the same byte of c.
// Written as two bit-selects (one LOP3 each) of the operands shifted by D, the shifts on the
// FMA pipe (IMAD.HI / IMAD): the integer ALU pipe is the one the classifier saturates.
template <int D>
UG_HD void dswap(uint32_t &a, uint32_t &c) {
  constexpr uint32_t M = D == 1 ? 0x55555555u : (D == 2 ? 0x33333333u : 0x0F0F0F0Fu);
  const uint32_t ad = shr_fma<D>(a), cu = mad(c, 1u << D, 0u);
  const uint32_t c2 = muxc<M>(ad, c);
  a = muxc<(M << D)>(cu, a);
  c = c2;
}
// w[0..7] = 32 bytes (position 4r + k = byte k of w[r]) -> P[b] bit i = bit b of byte i.
// R[r] gathers positions r, 8+r, 16+r, 24+r; the delta swaps then transpose every byte lane's
// 8x8 (register, bit) matrix, so bit 8k + r of P[b] is bit b of position 8k + r.
UG_HD void planes32(const uint32_t w[8], uint32_t P[8]) {
  tr4(w[0], w[2], w[4], w[6], P[0], P[1], P[2], P[3]);
  tr4(w[1], w[3], w[5], w[7], P[4], P[5], P[6], P[7]);
  dswap<1>(P[0], P[1]); dswap<1>(P[2], P[3]); dswap<1>(P[4], P[5]); dswap<1>(P[6], P[7]);
  dswap<2>(P[0], P[2]); dswap<2>(P[1], P[3]); dswap<2>(P[4], P[6]); dswap<2>(P[5], P[7]);
  dswap<4>(P[0], P[4]); dswap<4>(P[1], P[5]); dswap<4>(P[2], P[6]); dswap<4>(P[3], P[7]);
}

// msb-per-byte masks of a word: lead >= C0, >= E0, >= F0.
UG_HD uint32_t lead_c0(uint32_t x) { return x & (x << 1) & HI; }

// Carry words for the bit-plane shifts: bits 31, 30, 29 = the mask at positions -1, -2, -3
// (bytes 3, 2, 1 of `prev`), from msb-per-byte form by one multiply (bit 23 -> 30, 15 -> 29).
UG_HD uint32_t carry3(uint32_t msb_mask) { return msb_mask * 0x4081u; }

// Validation of one 32-byte chunk (a3) and its emit mask (a5).
//   w: the 32 bytes; prev: the 4 bytes before (byte 3 = position -1); nxt: the 4 bytes after.
//   Returns the error flags (bit i = position i; nonzero iff some position flags).
//   *emit: bit i set iff position i emits a UTF-16 unit (end-position rule above).
//   tail: also flag continuation bytes missing at positions 32..34 (the last chunk of a tile).
UG_HD uint32_t analyze32(const uint32_t w[8], uint32_t prev, uint32_t nxt, bool tail,
                         uint32_t *emit, uint32_t *fany = nullptr) {
  uint32_t P[8];
  planes32(w, P);
  const uint32_t L = P[7] & P[6], E = L & P[5], F = E & P[4];
  const uint32_t K = P[7] & ~P[6];
  const uint32_t pL = lead_c0(prev), pE = pL & (prev << 2), pF = pE & (prev << 3);
  const uint32_t cL = carry3(pL), cE = carry3(pE), cF = carry3(pF);
  const uint32_t S2E = fsl(cE, E, 2), S3F = fsl(cF, F, 3);
  // structure: required continuations == continuation bytes
  uint32_t err = (fsl(cL, L, 1) | S2E | S3F) ^ K;
  // values, at the lead, against the next byte's bits 5 and 4 (Q: next >= A0 after an E lead,
  // next >= 90 after an F lead)
  const uint32_t E3 = E & ~P[4], F3 = F & ~P[3];
  const uint32_t Z3 = ~(P[3] | P[2] | P[1]);
  const uint32_t T0 = Z3 & ~P[0] & (E3 | F3);                    // E0, F0: need Q
  const uint32_t T1 = (P[3] & P[2] & ~P[1] & P[0] & E3) |         // ED
                      (P[2] & ~P[1] & ~P[0] & F3);                // F4: need !Q
  const uint32_t AE = (P[2] & (P[1] | P[0]) & F3) | (F & P[3]) |  // F5..F7, F8..FF
                      (L & ~P[5] & ~P[4] & Z3);                   // C0, C1
  const uint32_t N5 = fsr(P[5], nxt >> 5, 1), N4 = fsr(P[4], nxt >> 4, 1);
  const uint32_t Q = N5 | (N4 & F);
  err |= (T0 & ~Q) | (T1 & Q) | AE;
  if (tail) {
    // leads at positions 29..31 whose continuations (positions 32..34) are missing
    const uint32_t Rt = (L >> 31) | (E >> 30) | (F >> 29);
    const uint32_t Kn = nxt & ~(nxt << 1) & 0x00808080u;
    const uint32_t Knb = ((Kn >> 7) & 1u) | ((Kn >> 14) & 2u) | ((Kn >> 21) & 4u);
    if (Rt & ~Knb) err |= 0x80000000u;
  }
  *emit = ~P[7] | fsl(cL & ~cE, L & ~E, 1) | S2E | S3F;
  if (fany) *fany = F | cF;  // nonzero iff a >= F0 lead lies in the chunk or the 3 bytes before
  return err;
}

// ---------------------------------------------------------------- transcoding (a5, a7)
// Carried from one word to the next: the previous word and its lead masks.
struct Carry {
  uint32_t x, L2, E, F;  // bytes; 2-byte leads (C0..DF); >= E0; >= F0  (msb per byte)
};
UG_HD Carry carry_of(uint32_t x) {
  const uint32_t L = lead_c0(x), E = L & (x << 2);
  return Carry{x, L & ~E, E, E & (x << 3)};
}

// The 4 positions of word x (previous word in c, updated): units of positions 0 / 1 in the
// low / high half of *u01, positions 2 / 3 in *u23.  Returns the emit mask, 1 in the lsb of
// every emitting byte.  Units at non-emitting positions are garbage.
// The class masks are taken in lsb-per-byte form straight from a funnel shift by 8d + 1
// (d = distance to the lead), so every per-byte constant is one multiply (FMA pipe).
// BE: units stored big-endian (UTF-16BE output): the two PRMT that pair
// low and high bytes into units take the bytes in the other order - no extra instruction.
template <bool BE = false>
UG_HD uint32_t units4(uint32_t x, Carry &c, uint32_t *u01, uint32_t *u23) {
  const Carry n = carry_of(x);
  const uint32_t bp1 = fsl(c.x, x, 8), bp2 = fsl(c.x, x, 16);  // bytes e-1, e-2
  const uint32_t s1l2 = fsl(c.L2, n.L2, 1);                    // end of a 2-byte character
  const uint32_t s2e = fsl(c.E, n.E, 9);                       // end of 3-byte / high surrogate
  const uint32_t s2f = fsl(c.F, n.F, 9);                       // high surrogate
  const uint32_t s3f = fsl(c.F, n.F, 17);                      // low surrogate
  c = n;
  const uint32_t n7 = (x >> 7) & 0x01010101u;  // 1 in every non-ASCII byte
  const uint32_t em = ((n7 ^ 0x01010101u) | s1l2 | s2e | s3f);
  uint32_t lb = mux(n7 * 0xC0u, bp1 << 6, x);
  // (right shifts on the FMA pipe as IMAD.HI where the ALU pipe is the bottleneck).  At a low
  // surrogate the payload bits are (b[e-1] >> 2) & 3, but OR-ing all four bits of
  // (b[e-1] >> 2) & 0xF into 0xDC is the same: 0xDC already has bits 2 and 3 set.
  uint32_t hb = (shr_fma<2>(bp1) & (n7 * 15u)) | (s3f * 0xDCu) | ((bp2 << 4) & (s2e * 0xF0u));
  // high surrogate: G = hb:lb = cp >> 6, unit = 0xD800 | ((G >> 4) - 0x40)
  const uint32_t Mh = s2f * 0xFFu;
  const uint32_t hbm = (hb | HI) - 0x04040404u;  // per byte 0x80 + hb - 4, no borrows
  lb = mux(Mh, muxc<0xF0F0F0F0u>(hbm << 4, shr_fma<4>(lb)), lb);
  hb = mux(Mh, (shr_fma<4>(hbm) & 0x03030303u) | 0xD8D8D8D8u, hb);
  *u01 = prmt(lb, hb, BE ? 0x1504u : 0x5140u);
  *u23 = prmt(lb, hb, BE ? 0x3726u : 0x7362u);
  return em;
}

// units4 for a warp whose 1 KiB and the 3 bytes before hold no >= F0 lead (no 4-byte
// character: no surrogate pair to emit, f1 for UTF-8): the same units and emit mask on such
// input without the surrogate terms.
template <bool BE = false>
UG_HD uint32_t units4_nof(uint32_t x, Carry &c, uint32_t *u01, uint32_t *u23) {
  const Carry n = carry_of(x);
  const uint32_t bp1 = fsl(c.x, x, 8), bp2 = fsl(c.x, x, 16);
  const uint32_t s1l2 = fsl(c.L2, n.L2, 1);
  const uint32_t s2e = fsl(c.E, n.E, 9);
  c = n;
  const uint32_t n7 = (x >> 7) & 0x01010101u;
  const uint32_t em = ((n7 ^ 0x01010101u) | s1l2 | s2e);
  const uint32_t lb = mux(n7 * 0xC0u, bp1 << 6, x);
  const uint32_t hb = (shr_fma<2>(bp1) & (n7 * 15u)) | ((bp2 << 4) & (s2e * 0xF0u));
  *u01 = prmt(lb, hb, BE ? 0x1504u : 0x5140u);
  *u23 = prmt(lb, hb, BE ? 0x3726u : 0x7362u);
  return em;
}

// ---------------------------------------------------------------- exact (cold) path
UG_HD uint32_t byte_of(uint32_t x, int k) { return (x >> (8 * k)) & 0xFFu; }

// Kind of the failure of a sequential decoder whose window is x = s[0..3] (rules in the order
// of DESIGN.md R2); bytes past the end of the input are 0x00 (not continuation bytes).
UG_HD int decode_kind(uint32_t x) {
  uint32_t b = x & 0xFFu;
  if (b < 0x80u) return OK;
  if (b < 0xC0u) return TOO_LONG;
  if (b >= 0xF8u) return HEADER_BITS;
  int L = b < 0xE0u ? 2 : (b < 0xF0u ? 3 : 4);
  uint32_t cp = b & (0x7Fu >> L);
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

UG_HD int declared_len(uint32_t b) {
  return b < 0x80u ? 1 : (b < 0xC0u ? 0 : (b < 0xE0u ? 2 : (b < 0xF0u ? 3 : (b < 0xF8u ? 4 : 0))));
}

// Exact local predicate at position i (D2 / SURVEY.md C.4(i)): back = s[i-4..i-1],
// fwd = s[i..i+3].  A(i): a non-continuation byte whose character fails to decode.  B(i): a
// continuation byte with no lead within the 3 previous bytes that declares it.
UG_HD bool err_at(uint32_t back, uint32_t fwd) {
  uint32_t c = fwd & 0xFFu;
  if ((c & 0xC0u) != 0x80u) return decode_kind(fwd) != OK;
  for (int d = 1; d <= 3; d++) {
    uint32_t b = byte_of(back, 4 - d);
    if ((b & 0xC0u) != 0x80u) return !(declared_len(b) > d);
  }
  return true;
}

// Emission rule at position i from bytes i-3..i (the cold finalize count, same rule as units4).
UG_HD uint32_t emits_at(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  // b0 = s[i], b1 = s[i-1], b2 = s[i-2], b3 = s[i-3]
  return (b0 < 0x80u || (b1 >= 0xC0u && b1 < 0xE0u) || b2 >= 0xE0u || b3 >= 0xF0u) ? 1u : 0u;
}

// The plan's arithmetic (kernels.cu k_plan8, DESIGN.md section 5 "planned").  Summed over
// positions, emits_at's four terms (ASCII at i, 2-byte lead at i-1, >= E0 at i-2, >= F0 at
// i-3) weigh each byte by plan_weight = [non-continuation] + [>= F0], the R15 length formula,
// but credit a lead's units to the positions that emit them, up to 3 bytes later; pending3 =
// the units that the leads in the 3 bytes before a cut q (b1 = s[q-1], b2 = s[q-2],
// b3 = s[q-3]) emit at q or later.  So sum of the terms over [a, b) = sum of plan_weight over
// [a, b) + pending3(at a) - pending3(at b); it equals emits_at's count where the terms never
// coincide (an error-free prefix) and exceeds it otherwise.
UG_HD uint32_t plan_weight(uint32_t b) { return ((b & 0xC0u) != 0x80u ? 1u : 0u) + (b >= 0xF0u ? 1u : 0u); }
UG_HD uint32_t pending3(uint32_t b1, uint32_t b2, uint32_t b3) {
  const uint32_t l2 = (b1 >= 0xC0u && b1 < 0xE0u) ? 1u : 0u;
  const uint32_t e1 = b1 >= 0xE0u ? 1u : 0u, f1 = b1 >= 0xF0u ? 1u : 0u;
  const uint32_t e2 = b2 >= 0xE0u ? 1u : 0u, f2 = b2 >= 0xF0u ? 1u : 0u;
  const uint32_t f3 = b3 >= 0xF0u ? 1u : 0u;
  return l2 + e1 + f1 + e2 + f2 + f3;
}

}  // namespace u8
}  // namespace ug
