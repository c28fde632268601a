/*
 * oracle.h -- the parity ORACLE for paper_2111_08692_b200.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load, call or link anything under oracle/.  The product path (include/unigpu.h,
 * paper_2111_08692_b200/) never includes this header and shares no code, tables or helpers
 * with it.
 *
 * What it is: a plain, branchy, sequential scalar codec that follows the paper's definition of
 * the two formats (D. Lemire, "Unicode at Gigabytes per Second", arXiv 2111.08692):
 *   - PAPER.md:67-83 (Section 3): UTF-8 lead-byte length classes, continuation bytes, payload
 *     layout and the six exhaustive validity rules;
 *   - PAPER.md:85-87 (Section 3): UTF-16 code units, surrogate ranges and the pair formula.
 * The result conventions (first-error offset = first code unit of the offending sequence, kind
 * precedence, truncation at end of buffer) are the readings listed in DESIGN.md section 3.
 *
 * Every function here is pinned by tests/test_oracle_*.py against things other than itself
 * (CPython's strict codecs, closed-form counts, exhaustive enumeration); see DESIGN.md.
 */
#ifndef UNIGPU_ORACLE_H
#define UNIGPU_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error kinds: one per validity rule of PAPER.md:76-82 (rule 1..6), plus lone UTF-16
 * surrogates folded into rule 6's kind. */
enum {
  UGO_OK = 0,
  UGO_HEADER_BITS = 1, /* rule 1: five most significant bits all ones (F8..FF)            */
  UGO_TOO_SHORT = 2,   /* rule 2: lead not followed by enough continuation bytes          */
  UGO_TOO_LONG = 3,    /* rule 3: continuation byte not preceded by a lead                */
  UGO_OVERLONG = 4,    /* rule 4: value not larger than 7F / 7FF / FFFF for 2 / 3 / 4 B     */
  UGO_TOO_LARGE = 5,   /* rule 5: value not less than 1114112 (0x110000)                  */
  UGO_SURROGATE = 6,   /* rule 6: value in D800..DFFF; also unpaired UTF-16 surrogates     */
  UGO_OUTPUT_TOO_SMALL = -3
};

typedef struct {
  int32_t error;     /* UGO_* kind, 0 on success                                          */
  uint32_t pad_;
  uint64_t position; /* success: input units consumed (= n); error: first-error offset    */
  uint64_t written;  /* output units written for in[0..position) (0 for validators)       */
} ugo_result;

/* ---- per-character primitives ---- */
/* Decode the UTF-8 sequence starting at s[p] (p < n).  Returns 0 and sets *cp, *len on
 * success, else the UGO_* kind of the violated rule. */
int ugo_decode_utf8_at(const uint8_t *s, size_t n, size_t p, uint32_t *cp, int *len);
/* Minimal UTF-8 encoding of a Unicode scalar value; returns its length 1..4, or 0 if cp is a
 * surrogate or > 0x10FFFF. */
int ugo_encode_utf8(uint32_t cp, uint8_t out[4]);
/* Decode the UTF-16 character starting at u[p] (p < m). */
int ugo_decode_utf16_at(const uint16_t *u, size_t m, size_t p, uint32_t *cp, int *len);
/* UTF-16 encoding of a scalar value; returns 1 or 2, or 0 for a surrogate / out of range. */
int ugo_encode_utf16(uint32_t cp, uint16_t out[2]);

/* ---- whole-buffer operations: the C-ABI contract of include/unigpu.h, on host memory ---- */
ugo_result ugo_utf8_validate(const uint8_t *in, size_t n);
ugo_result ugo_utf16le_validate(const uint16_t *in, size_t n);
ugo_result ugo_utf8_to_utf16le(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap);
ugo_result ugo_utf16le_to_utf8(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap);
uint64_t ugo_utf16_length_from_utf8(const uint8_t *in, size_t n);
uint64_t ugo_utf8_length_from_utf16le(const uint16_t *in, size_t n);

/* ---- exhaustive sweeps used by the pinning tests (enumerate, call the functions above) ---- */
/* All 256^len byte strings (len 1..4): kind histogram hist_kind[7] (index = kind) and
 * first-error-offset histogram hist_off[len] (valid strings are not counted there).
 * len == 4 is split into `nparts` slices; slice `part` enumerates first bytes
 * [part*256/nparts, (part+1)*256/nparts). */
void ugo_sweep_utf8(int len, int part, int nparts, uint64_t *hist_kind, uint64_t *hist_off);
/* Per-string first-error offsets (-1 if valid) and kinds of all 256^len strings, len <= 3,
 * indexed by the big-endian value of the string. */
void ugo_sweep_utf8_offsets(int len, int8_t *off, int8_t *kind);
/* All 65536^2 two-word UTF-16 strings (first word in slice `part` of `nparts`): valid count
 * and first-error-offset histogram. */
void ugo_sweep_utf16_pairs(int part, int nparts, uint64_t *valid, uint64_t *hist_off);

#ifdef __cplusplus
}
#endif
#endif
