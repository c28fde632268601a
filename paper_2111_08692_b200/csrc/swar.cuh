// swar.cuh -- the handful of sm_100a integer primitives the codec arithmetic is written in
// (PRMT, funnel shifts, POPC, IMAD.HI), each with a bit-exact host definition so the same
// per-thread code (utf8.cuh / utf16.cuh) can be compiled for the host by tests/emu/kernel_math_emu.cpp and
// checked against the oracle without a GPU.  Nothing here is method arithmetic.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define UG_HD __host__ __device__ __forceinline__
#else
#define UG_HD inline
#endif

namespace ug {

constexpr uint32_t HI = 0x80808080u;  // msb of every byte

// PRMT (byte permute): byte i of the result is byte (sel >> 4i) & 7 of {b:a}; if bit 3 of that
// selector nibble is set the msb of the chosen byte is replicated over the whole byte.
UG_HD uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
#else
  const uint64_t v = ((uint64_t)b << 32) | a;
  uint32_t d = 0;
  for (int i = 0; i < 4; i++) {
    const uint32_t s = (sel >> (4 * i)) & 0xFu;
    uint32_t byte = (uint32_t)(v >> (8 * (s & 7u))) & 0xFFu;
    if (s & 8u) byte = (byte & 0x80u) ? 0xFFu : 0u;
    d |= byte << (8 * i);
  }
  return d;
#endif
}

// Most significant 32 bits of (hi:lo) << s, s in [0, 31]  (SHF.L.W).
UG_HD uint32_t fsl(uint32_t lo, uint32_t hi, uint32_t s) {
#if defined(__CUDA_ARCH__)
  return __funnelshift_l(lo, hi, s);
#else
  s &= 31u;
  return s ? (hi << s) | (lo >> (32 - s)) : hi;
#endif
}
// Least significant 32 bits of (hi:lo) >> s, s in [0, 31]  (SHF.R.W).
UG_HD uint32_t fsr(uint32_t lo, uint32_t hi, uint32_t s) {
#if defined(__CUDA_ARCH__)
  return __funnelshift_r(lo, hi, s);
#else
  s &= 31u;
  return s ? (lo >> s) | (hi << (32 - s)) : lo;
#endif
}
UG_HD uint32_t popc(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)__popc(x);
#else
  return (uint32_t)__builtin_popcount(x);
#endif
}
// High 32 bits of a 32x32 product (IMAD.HI): x >> s written as umulhi(x, 1 << (32 - s)) runs on
// the FMA pipe instead of the ALU pipe.
UG_HD uint32_t umulhi(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}
// x >> S as IMAD.HI (FMA pipe, half rate): for code whose ALU pipe is the bottleneck.
template <int S>
UG_HD uint32_t shr_fma(uint32_t x) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "n"(1u << (32 - S)));
  return d;
#else
  return x >> S;
#endif
}
// a * b + c on the FMA pipe (IMAD).
UG_HD uint32_t mad(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
#else
  return a * b + c;
#endif
}
// (a * b >> 32) + c on the FMA pipe (IMAD.HI with accumulate).
UG_HD uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
#else
  return (uint32_t)(((uint64_t)a * b) >> 32) + c;
#endif
}
// (a & m) | (b & ~m): one LOP3.
UG_HD uint32_t mux(uint32_t m, uint32_t a, uint32_t b) { return (a & m) | (b & ~m); }
// mux with a constant mask, forced into ONE LOP3 (mask as its immediate; left to itself the
// compiler splits a constant-mask select into two).
template <uint32_t M>
UG_HD uint32_t muxc(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "n"(M));
  return d;
#else
  return (a & M) | (b & ~M);
#endif
}

}  // namespace ug
