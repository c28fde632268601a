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

namespace ug {
namespace u16 {

__device__ __forceinline__ bool is_high(uint32_t u) { return (u & 0xFC00u) == 0xD800u; }
__device__ __forceinline__ bool is_low(uint32_t u) { return (u & 0xFC00u) == 0xDC00u; }

__device__ __forceinline__ uint32_t width(uint32_t u, uint32_t prev) {
  const bool two = u < 0x800u || is_high(u) || (is_low(u) && is_high(prev));
  return 1u + (u >= 0x80u ? 1u : 0u) + (two ? 0u : 1u);
}

__device__ __forceinline__ bool err_at(uint32_t prev, uint32_t u, uint32_t next) {
  return (is_high(u) && !is_low(next)) || (is_low(u) && !is_high(prev));
}

// UTF-8 bytes of word u (little-endian packed, width(u, prev) of them are meaningful).
// Branch-free: all candidates computed, then selected.
__device__ __forceinline__ uint32_t utf8_bytes(uint32_t u, uint32_t prev) {
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

}  // namespace u16
}  // namespace ug
