/*
 * oracle.c -- plain scalar reference codec.  TEST INFRASTRUCTURE ONLY (see oracle.h header):
 * only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load liboracle.so.
 *
 * Written from PAPER.md Section 3 (lines 61-87), step by step, with no SIMD, no tables and no
 * blocking.  Compiled with -O2 -fno-tree-vectorize.  Shares nothing with the CUDA path.
 *
 * Readings of points the paper leaves open are DESIGN.md section 3 (R1..R12); the ones used
 * here are cited inline.
 */
#include "oracle.h"

#include <string.h>

/* ------------------------------------------------------------------------------------------
 * decode8 -- PAPER.md:67-83.  Steps in the order of DESIGN.md R2 (kind precedence):
 *   lead class (rule 3 TooLong, rule 1 HeaderBits), then rule 2 TooShort, then rule 4
 *   Overlong, then rule 5 TooLarge, then rule 6 Surrogate.
 * ---------------------------------------------------------------------------------------- */
int ugo_decode_utf8_at(const uint8_t *s, size_t n, size_t p, uint32_t *cp_out, int *len_out) {
  uint32_t b = s[p];
  int L;
  /* PAPER.md:69 "If the most significant bit is zero, we have a sequence of one byte". */
  if (b < 0x80) {
    *cp_out = b;
    *len_out = 1;
    return UGO_OK;
  }
  /* PAPER.md:74 continuation bytes are 10xxxxxx; one in lead position violates rule 3
   * ("A continuation byte must be preceded by a leading byte"). */
  if (b <= 0xBF) return UGO_TOO_LONG;
  /* PAPER.md:77 rule 1: "The five most significant bits of any byte cannot be all ones." */
  if (b >= 0xF8) return UGO_HEADER_BITS;
  /* 110xxxxx -> 2, 1110xxxx -> 3, 11110xxx -> 4. */
  if (b <= 0xDF)
    L = 2;
  else if (b <= 0xEF)
    L = 3;
  else
    L = 4;
  /* PAPER.md:78 rule 2: "The leading byte must be followed by the right number of
   * continuation bytes."  End of buffer counts as a missing byte (R4). */
  for (int k = 1; k < L; k++) {
    if (p + (size_t)k >= n) return UGO_TOO_SHORT;
    if ((s[p + k] & 0xC0) != 0x80) return UGO_TOO_SHORT;
  }
  /* payload bits, most significant in the lead byte, then 6 bits per
   * continuation byte.  The lead keeps its low 7-L bits. */
  uint32_t cp = b & (0x7Fu >> L);
  for (int k = 1; k < L; k++) cp = (cp << 6) | (s[p + k] & 0x3Fu);
  /* PAPER.md:80 rule 4: larger than 7F / 7FF / FFFF for 2 / 3 / 4-byte sequences. */
  if ((L == 2 && cp <= 0x7F) || (L == 3 && cp <= 0x7FF) || (L == 4 && cp <= 0xFFFF))
    return UGO_OVERLONG;
  /* PAPER.md:81 rule 5: "must be less than 1114112" (R8). */
  if (cp >= 1114112u) return UGO_TOO_LARGE;
  /* PAPER.md:82 rule 6: not in D800..DFFF. */
  if (cp >= 0xD800 && cp <= 0xDFFF) return UGO_SURROGATE;
  *cp_out = cp;
  *len_out = L;
  return UGO_OK;
}

/* Minimal encoding, PAPER.md:67-75 read in reverse: 1 byte up to 7F, 2 up to 7FF, 3 up to
 * FFFF, else 4. */
int ugo_encode_utf8(uint32_t cp, uint8_t out[4]) {
  if (cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF)) return 0;
  if (cp <= 0x7F) {
    out[0] = (uint8_t)cp;
    return 1;
  }
  if (cp <= 0x7FF) {
    out[0] = (uint8_t)(0xC0 | (cp >> 6));
    out[1] = (uint8_t)(0x80 | (cp & 0x3F));
    return 2;
  }
  if (cp <= 0xFFFF) {
    out[0] = (uint8_t)(0xE0 | (cp >> 12));
    out[1] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
    out[2] = (uint8_t)(0x80 | (cp & 0x3F));
    return 3;
  }
  out[0] = (uint8_t)(0xF0 | (cp >> 18));
  out[1] = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
  out[2] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
  out[3] = (uint8_t)(0x80 | (cp & 0x3F));
  return 4;
}

/* decode16 -- PAPER.md:85-87.  Words outside D800..DFFF are characters; a word in D800..DBFF
 * followed by one in DC00..DFFF is a pair whose value is the 10 low bits of each word, the
 * second word least significant, plus 0x10000.  Anything else is a Surrogate error at p
 * (R4: a trailing high surrogate is an error at its own position). */
int ugo_decode_utf16_at(const uint16_t *u, size_t m, size_t p, uint32_t *cp_out, int *len_out) {
  uint32_t w = u[p];
  if (w < 0xD800 || w > 0xDFFF) {
    *cp_out = w;
    *len_out = 1;
    return UGO_OK;
  }
  if (w <= 0xDBFF && p + 1 < m) {
    uint32_t w2 = u[p + 1];
    if (w2 >= 0xDC00 && w2 <= 0xDFFF) {
      *cp_out = 0x10000u + (((w & 0x3FFu) << 10) | (w2 & 0x3FFu));
      *len_out = 2;
      return UGO_OK;
    }
  }
  return UGO_SURROGATE;
}

/* PAPER.md:85-87 inverted: BMP values are one word, supplementary values a pair. */
int ugo_encode_utf16(uint32_t cp, uint16_t out[2]) {
  if (cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF)) return 0;
  if (cp <= 0xFFFF) {
    out[0] = (uint16_t)cp;
    return 1;
  }
  uint32_t v = cp - 0x10000u;
  out[0] = (uint16_t)(0xD800u + (v >> 10));
  out[1] = (uint16_t)(0xDC00u + (v & 0x3FFu));
  return 2;
}

/* ------------------------------------------------------------------------------------------
 * Whole-buffer operations.  Result convention (R1, R5, R6):
 *   success      -> {OK, n, units written}
 *   first error  -> {kind, e, units for in[0..e)}, e = offset of the first code unit of the
 *                   sequence a left-to-right decoder fails on
 *   capacity     -> if the units for in[0..e) (e = first error, or n) exceed out_cap:
 *                   {OUTPUT_TOO_SMALL, required units, 0}; nothing is written past out_cap.
 * ---------------------------------------------------------------------------------------- */
static ugo_result mk(int32_t err, uint64_t pos, uint64_t wr) {
  ugo_result r;
  r.error = err;
  r.pad_ = 0;
  r.position = pos;
  r.written = wr;
  return r;
}

ugo_result ugo_utf8_validate(const uint8_t *in, size_t n) {
  size_t p = 0;
  while (p < n) {
    uint32_t cp;
    int len;
    int k = ugo_decode_utf8_at(in, n, p, &cp, &len);
    if (k != UGO_OK) return mk(k, p, 0);
    p += (size_t)len;
  }
  return mk(UGO_OK, n, 0);
}

ugo_result ugo_utf16le_validate(const uint16_t *in, size_t n) {
  size_t p = 0;
  while (p < n) {
    uint32_t cp;
    int len;
    int k = ugo_decode_utf16_at(in, n, p, &cp, &len);
    if (k != UGO_OK) return mk(k, p, 0);
    p += (size_t)len;
  }
  return mk(UGO_OK, n, 0);
}

ugo_result ugo_utf8_to_utf16le(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap) {
  size_t p = 0;
  uint64_t w = 0; /* units required so far */
  int kind = UGO_OK;
  while (p < n) {
    uint32_t cp;
    int len;
    int k = ugo_decode_utf8_at(in, n, p, &cp, &len);
    if (k != UGO_OK) {
      kind = k;
      break;
    }
    uint16_t units[2];
    int nu = ugo_encode_utf16(cp, units);
    for (int j = 0; j < nu; j++) {
      if (w < out_cap) out[w] = units[j];
      w++;
    }
    p += (size_t)len;
  }
  if (w > out_cap) return mk(UGO_OUTPUT_TOO_SMALL, w, 0);
  return mk(kind, p, w);
}

ugo_result ugo_utf16le_to_utf8(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap) {
  size_t p = 0;
  uint64_t w = 0;
  int kind = UGO_OK;
  while (p < n) {
    uint32_t cp;
    int len;
    int k = ugo_decode_utf16_at(in, n, p, &cp, &len);
    if (k != UGO_OK) {
      kind = k;
      break;
    }
    uint8_t bytes[4];
    int nb = ugo_encode_utf8(cp, bytes);
    for (int j = 0; j < nb; j++) {
      if (w < out_cap) out[w] = bytes[j];
      w++;
    }
    p += (size_t)len;
  }
  if (w > out_cap) return mk(UGO_OUTPUT_TOO_SMALL, w, 0);
  return mk(kind, p, w);
}

/* Length-from functions (not in the paper; BASELINE.json north_star names them).  Defined by
 * formula for ANY input (R15); on valid input they equal the transcoders' counts:
 * every non-continuation byte starts one character (one UTF-16 unit), and a 4-byte lead
 * (F0..F7) adds the second unit of its surrogate pair. */
uint64_t ugo_utf16_length_from_utf8(const uint8_t *in, size_t n) {
  uint64_t c = 0;
  for (size_t i = 0; i < n; i++) {
    if ((in[i] & 0xC0) != 0x80) c++;
    if (in[i] >= 0xF0) c++;
  }
  return c;
}

/* Each word contributes the UTF-8 length of the character it starts:
 * 1 below 0x80, 2 below 0x800, 3 for the rest of the BMP; each surrogate word contributes 2,
 * so a pair contributes 4. */
uint64_t ugo_utf8_length_from_utf16le(const uint16_t *in, size_t n) {
  uint64_t c = 0;
  for (size_t i = 0; i < n; i++) {
    uint32_t w = in[i];
    if (w < 0x80)
      c += 1;
    else if (w < 0x800)
      c += 2;
    else if (w >= 0xD800 && w <= 0xDFFF)
      c += 2;
    else
      c += 3;
  }
  return c;
}

/* ------------------------------------------------------------------------------------------
 * Exhaustive sweeps for the pinning tests.  They only enumerate inputs and call the
 * functions above.
 * ---------------------------------------------------------------------------------------- */
void ugo_sweep_utf8(int len, int part, int nparts, uint64_t *hist_kind, uint64_t *hist_off) {
  uint8_t s[4];
  uint64_t lo = 0, hi = 1;
  for (int k = 0; k < len; k++) hi *= 256;
  if (len == 4 && nparts > 0) {
    uint64_t span = hi / (uint64_t)nparts;
    lo = span * (uint64_t)part;
    hi = lo + span;
  }
  for (uint64_t x = lo; x < hi; x++) {
    /* byte 0 is the most significant digit of x */
    for (int k = 0; k < len; k++) s[k] = (uint8_t)(x >> (8 * (len - 1 - k)));
    ugo_result r = ugo_utf8_validate(s, (size_t)len);
    hist_kind[r.error]++;
    if (r.error != UGO_OK) hist_off[r.position]++;
  }
}

void ugo_sweep_utf8_offsets(int len, int8_t *off, int8_t *kind) {
  uint8_t s[4];
  uint64_t hi = 1;
  for (int k = 0; k < len; k++) hi *= 256;
  for (uint64_t x = 0; x < hi; x++) {
    for (int k = 0; k < len; k++) s[k] = (uint8_t)(x >> (8 * (len - 1 - k)));
    ugo_result r = ugo_utf8_validate(s, (size_t)len);
    off[x] = (int8_t)(r.error == UGO_OK ? -1 : (int)r.position);
    kind[x] = (int8_t)r.error;
  }
}

void ugo_sweep_utf16_pairs(int part, int nparts, uint64_t *valid, uint64_t *hist_off) {
  uint16_t u[2];
  uint32_t a0 = (uint32_t)(65536 / nparts) * (uint32_t)part, a1 = a0 + (uint32_t)(65536 / nparts);
  for (uint32_t a = a0; a < a1; a++) {
    u[0] = (uint16_t)a;
    for (uint32_t b = 0; b < 65536; b++) {
      u[1] = (uint16_t)b;
      ugo_result r = ugo_utf16le_validate(u, 2);
      if (r.error == UGO_OK)
        (*valid)++;
      else
        hist_off[r.position]++;
    }
  }
}
