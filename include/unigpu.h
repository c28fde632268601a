/*
 * unigpu.h -- C-ABI of paper_2111_08692_b200 (libunigpu.so): B200-native (sm_100a) UTF-8 /
 * UTF-16LE validation and validating transcoding, after D. Lemire, "Unicode at Gigabytes per
 * Second", arXiv 2111.08692.
 *
 * What each entry point computes is the paper's statement of the problem:
 *   - UTF-8 validity = the six exhaustive rules of PAPER.md:76-83 (Section 3);
 *   - UTF-16 validity = surrogate pairing, PAPER.md:85-87 ("only the possible surrogate pairs
 *     require attention");
 *   - transcoding = decode with the payload layout of PAPER.md:75 and re-encode with the
 *     surrogate-pair formula of PAPER.md:87 (or its inverse), validation fused in
 *     ("All of our transcoding tests include validation").
 * The result conventions the paper leaves open are DESIGN.md section 3 (R1..R21).
 *
 * Conventions shared by every function below
 * -------------------------------------------
 *  - Pointers named in/out are DEVICE pointers (cudaMalloc'd or torch CUDA tensors) on the
 *    current CUDA device, unless the name ends in _host.  The caller owns every input and
 *    output buffer; the library never allocates output.  It owns a small workspace per
 *    (device, stream) (tile status words, ticket counters, a result slot), allocated lazily on
 *    first use and reused; calls on different streams never share a workspace.
 *  - Lengths are in CODE UNITS: bytes for UTF-8, 16-bit words for UTF-16LE.  UTF-16LE is
 *    little-endian, the GPU's native order; a BOM is ordinary data (R7, R9).
 *    n <= 2^38 - 1 units per call (tile status words carry 38-bit counts); a larger n is API
 *    misuse (UG_ERR_ARG) - split the input with the sharded entry points instead.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *  - Validity failures are DATA, returned in ug_result, not API failures.
 *  - API misuse (NULL pointer with n > 0, odd address for a UTF-16 pointer, output capacity
 *    larger than the buffer can be checked for is the caller's duty) returns UG_ERR_ARG; CUDA
 *    failures return UG_ERR_CUDA.  n = 0 returns {UG_OK, 0, 0} without launching anything.
 *  - Synchronous functions enqueue on `stream`, then synchronise `stream` and return the
 *    result.  *_async functions only enqueue; they write the result into a caller-provided
 *    DEVICE (or pinned, device-mapped) pointer and return UG_OK or an API error code.
 *  - Nothing is ever written at or beyond out[out_cap].  out[0..written) is exact; output
 *    units beyond `written` are unspecified (R5).
 *  - Every device function is one kernel launch (no memset, no host round trip): per-call
 *    state is epoch-tagged and self-resetting.
 */
#ifndef UNIGPU_H
#define UNIGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UNIGPU_ABI_VERSION 1

/* Data verdicts: one per validity rule of PAPER.md:77-82, lone or
 * misordered UTF-16 surrogates reuse UG_SURROGATE.  Negative values are API
 * outcomes. */
typedef enum {
  UG_OK = 0,
  UG_HEADER_BITS = 1, /* rule 1: byte F8..FF                                         */
  UG_TOO_SHORT = 2,   /* rule 2: lead without enough continuation bytes (incl. at end) */
  UG_TOO_LONG = 3,    /* rule 3: continuation byte not preceded by a lead             */
  UG_OVERLONG = 4,    /* rule 4: value not larger than 7F / 7FF / FFFF                 */
  UG_TOO_LARGE = 5,   /* rule 5: value >= 0x110000                                     */
  UG_SURROGATE = 6,   /* rule 6 (D800..DFFF in UTF-8) and unpaired UTF-16 surrogates   */
  UG_ERR_ARG = -1,
  UG_ERR_CUDA = -2,
  UG_ERR_OUTPUT_TOO_SMALL = -3,
  UG_ERR_NCCL = -4 /* reserved for the collective layer; this library makes no
                      NCCL calls - the record all-gather runs in the caller's torch.distributed */
} ug_error;

/* 24-byte result, SPEC.md S:39-44 / BASELINE north_star ("output length or a validity
 * verdict with the first-error offset"):
 *   success:            error = UG_OK, position = n (input units consumed),
 *                       written = output units (0 for validators)
 *   invalid input:      error = kind of the first error, position = e, the offset of the
 *                       first code unit of the sequence a left-to-right decoder fails on
 *                       (R1), written = output units for in[0..e)
 *   output too small:   error = UG_ERR_OUTPUT_TOO_SMALL, position = units required for
 *                       in[0..e) (e = first error or n), written = 0
 *   API error:          error = UG_ERR_ARG / UG_ERR_CUDA, position = written = 0          */
typedef struct {
  int32_t error;
  uint32_t reserved;
  uint64_t position;
  uint64_t written;
} ug_result;

/* ------------------------------------------------------------------ synchronous, device
 * Validate UTF-8 in[0..n).  Read-only. */
ug_result utf8_validate(const uint8_t *in, size_t n, void *stream);

/* Validate UTF-16LE in[0..n) words.  `in` must be 2-byte aligned. */
ug_result utf16le_validate(const uint16_t *in, size_t n, void *stream);

/* Validate UTF-8 in[0..n) and transcode to UTF-16LE out[0..out_cap) words, in one fused pass
 * (PAPER.md:95-100 + 120).  out_cap = n always suffices (one unit per input byte at most,
 * SPEC.md S:175); utf16_length_from_utf8() gives the exact size for valid input.  `out` must
 * be 2-byte aligned. */
ug_result utf8_to_utf16le(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap,
                          void *stream);

/* Validate UTF-16LE in[0..n) and transcode to UTF-8 out[0..out_cap) bytes (PAPER.md:104-107
 * + 120).  out_cap = 3n always suffices; utf8_length_from_utf16le() is exact for valid
 * input. */
ug_result utf16le_to_utf8(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap,
                          void *stream);

/* Number of UTF-16 units the UTF-8 input transcodes to, for ANY input defined as
 * #(bytes b with (b & 0xC0) != 0x80) + #(bytes b >= 0xF0) (R15); equals
 * utf8_to_utf16le's `written` on valid input.  Read-only reduction. */
uint64_t utf16_length_from_utf8(const uint8_t *in, size_t n, void *stream);

/* Number of UTF-8 bytes the UTF-16LE input transcodes to, defined as the sum over words of
 * 1 (< 0x80), 2 (< 0x800), 2 (surrogate), 3 (other); exact on valid input. */
uint64_t utf8_length_from_utf16le(const uint16_t *in, size_t n, void *stream);

/* The two length-from functions with an error channel: return UG_OK and *len, or UG_ERR_ARG
 * (NULL `len`, NULL `in` with n > 0, odd UTF-16 pointer, n > 2^62) / UG_ERR_CUDA with
 * *len = 0.  (The plain forms above return 0 in those cases, indistinguishable from an empty
 * count.)  Synchronous. */
int ug_utf16_length_from_utf8_ex(const uint8_t *in, size_t n, uint64_t *len, void *stream);
int ug_utf8_length_from_utf16le_ex(const uint16_t *in, size_t n, uint64_t *len, void *stream);

/* ------------------------------------------------------------------ asynchronous, device
 * Same operations; the result is written by the GPU into *d_result (a device pointer, or
 * pinned host memory mapped into the device).  Return UG_OK once enqueued, or UG_ERR_ARG /
 * UG_ERR_CUDA (then nothing was enqueued and *d_result is untouched). */
int ug_utf8_validate_async(const uint8_t *in, size_t n, ug_result *d_result, void *stream);
int ug_utf16le_validate_async(const uint16_t *in, size_t n, ug_result *d_result, void *stream);
int ug_utf8_to_utf16le_async(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap,
                             ug_result *d_result, void *stream);
int ug_utf16le_to_utf8_async(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap,
                             ug_result *d_result, void *stream);
int ug_utf16_length_from_utf8_async(const uint8_t *in, size_t n, uint64_t *d_len, void *stream);
int ug_utf8_length_from_utf16le_async(const uint16_t *in, size_t n, uint64_t *d_len,
                                      void *stream);

/* ------------------------------------------------------------------ UTF-16BE
 * The same operations on big-endian UTF-16: word k of the buffer is the code unit
 * (byte[2k] << 8) | byte[2k + 1] ("utf16be file [0x00,0x41] -> words
 * [0x0041]").  Results, positions (in words), capacities and error conventions are exactly
 * those of the LE functions above on the byte-swapped buffer; no BOM handling (a BOM is data).
 * The kernels are the LE kernels with the byte order folded into their low/high byte split
 * (input) or unit packing (output), so they run at the LE speed. */
ug_result utf16be_validate(const uint16_t *in, size_t n, void *stream);
ug_result utf8_to_utf16be(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap,
                          void *stream);
ug_result utf16be_to_utf8(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap,
                          void *stream);
uint64_t utf8_length_from_utf16be(const uint16_t *in, size_t n, void *stream);
int ug_utf16be_validate_async(const uint16_t *in, size_t n, ug_result *d_result, void *stream);
int ug_utf8_to_utf16be_async(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap,
                             ug_result *d_result, void *stream);
int ug_utf16be_to_utf8_async(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap,
                             ug_result *d_result, void *stream);
int ug_utf8_length_from_utf16be_ex(const uint16_t *in, size_t n, uint64_t *len, void *stream);
int ug_utf8_length_from_utf16be_async(const uint16_t *in, size_t n, uint64_t *d_len,
                                      void *stream);

/* ------------------------------------------------------------------ sharded (multi-GPU)
 * One rank's share of a buffer cut at character boundaries (BASELINE
 * north_star item 3).  `in` points at the first OWNED code unit; the owned range is
 * in[0..n), which starts at offset `in_global_offset` of the whole (unsharded) input.
 * in[-halo_before .. -1] and in[n .. n+halo_after-1] must be readable context from the
 * neighbouring shards (0 at the global start / end; 3 bytes / 1 word suffice, more is
 * ignored).  Every per-position quantity reads only in[i-3 .. i+3] (D2), so the
 * counts and the first error are exact wherever the cuts fall.
 *
 * The kernel writes one 32-byte record to *d_rec (device memory):
 *   count     output units produced for the owned range (exact for valid input),
 *   first_err GLOBAL offset (in_global_offset + local) of the first error among owned
 *             positions, UINT64_MAX if none,
 *   written   output units for in[0..first_err) (0 if none),
 *   kind      ug_error kind at first_err (UG_OK if none).
 * Output goes to out[0..out_cap) of this rank (outputs stay sharded).  Ranks exchange the
 * records (one all-gather of 32 B per rank) and call ug_combine_records. */
typedef struct {
  uint64_t count;
  uint64_t first_err;
  uint64_t written;
  int32_t kind;
  int32_t reserved;
} ug_shard_record;

int ug_utf8_to_utf16le_shard_async(const uint8_t *in, size_t n, size_t halo_before,
                                   size_t halo_after, uint64_t in_global_offset, uint16_t *out,
                                   size_t out_cap, ug_shard_record *d_rec, void *stream);
int ug_utf16le_to_utf8_shard_async(const uint16_t *in, size_t n, size_t halo_before,
                                   size_t halo_after, uint64_t in_global_offset, uint8_t *out,
                                   size_t out_cap, ug_shard_record *d_rec, void *stream);
int ug_utf8_validate_shard_async(const uint8_t *in, size_t n, size_t halo_before,
                                 size_t halo_after, uint64_t in_global_offset,
                                 ug_shard_record *d_rec, void *stream);
int ug_utf16le_validate_shard_async(const uint16_t *in, size_t n, size_t halo_before,
                                    size_t halo_after, uint64_t in_global_offset,
                                    ug_shard_record *d_rec, void *stream);

/* Combine the all-gathered records of `nranks` shards (d_recs[0..nranks), device memory, in
 * rank order).  Writes the global result to *d_result: {OK, total_in, total count} if no rank
 * saw an error, else {kind, e, written} for the smallest first_err e, written = the output
 * offset of e's rank + that rank's local written.  total_in is the global input length.
 * Writes this rank's global output offset (exclusive prefix of counts) to *d_out_offset
 * (may be NULL).  One single-thread kernel; no host synchronisation. */
int ug_combine_records_async(const ug_shard_record *d_recs, int nranks, int rank,
                             uint64_t total_in, ug_result *d_result, uint64_t *d_out_offset,
                             void *stream);
/* The same combine on host memory (for hosts that gather records themselves). */
ug_result ug_combine_records_host(const ug_shard_record *recs, int nranks, int rank,
                                  uint64_t total_in, uint64_t *out_offset);

/* ------------------------------------------------------------------ two-pass (planned)
 * Reduce-then-scan form of the two transcoders (DESIGN.md section 5,
 * "planned").  A caller sizes the output with a length-from pass anyway; the *_plan_async
 * forms of that pass also write a PLAN into the caller's device buffer d_plan
 * (ug_plan_bytes() bytes, 8-byte aligned): the output count of each contiguous range of
 * tiles the transcoder's CTAs will take, under the transcoder's own emission rule.  The
 * *_planned_async transcoders then need no inter-CTA look-back: CTA c starts at the sum of
 * the earlier ranges' counts.  Results, outputs, capacities and error conventions are exactly
 * those of the plain calls.
 *   d_len     receives the length-from value (utf16_length_from_utf8 /
 *             utf8_length_from_utf16le; may be NULL);
 *   d_plan    must come from the plan call on the SAME input pointer, n and halos, on the same
 *             device, and stay unmodified until the planned call has run (stream order);
 *             a plan of another input makes the planned call's result {UG_ERR_ARG, 0, 0}
 *             (checked on the device against the plan's header);
 *   returns   UG_OK once enqueued, UG_ERR_ARG (NULL / misaligned pointers, n too large),
 *             UG_ERR_CUDA. */
size_t ug_plan_bytes(void);
int ug_utf16_length_from_utf8_plan_async(const uint8_t *in, size_t n, uint64_t *d_len,
                                         void *d_plan, void *stream);
int ug_utf8_length_from_utf16le_plan_async(const uint16_t *in, size_t n, uint64_t *d_len,
                                           void *d_plan, void *stream);
int ug_utf8_to_utf16le_planned_async(const uint8_t *in, size_t n, const void *d_plan,
                                     uint16_t *out, size_t out_cap, ug_result *d_result,
                                     void *stream);
int ug_utf16le_to_utf8_planned_async(const uint16_t *in, size_t n, const void *d_plan,
                                     uint8_t *out, size_t out_cap, ug_result *d_result,
                                     void *stream);

/* SURVEY 8(f) f4, research comparison: ug_utf8_to_utf16le_planned_async with the a7 decode
 * replaced by the paper's keyed 12-byte routine (section 4: a 12-bit key of
 * character ends indexes a table giving the bytes consumed and a shuffle index; index
 * [0, 64) = six characters of 1-2 bytes, [64, 145) = four of 1-3, [145, 209) = three of
 * 1-4).  Same arguments, plan (from ug_utf16_length_from_utf8_plan_async), results, outputs
 * and error conventions as ug_utf8_to_utf16le_planned_async; slower. */
int ug_utf8_to_utf16le_keyed_planned_async(const uint8_t *in, size_t n, const void *d_plan,
                                           uint16_t *out, size_t out_cap,
                                           ug_result *d_result, void *stream);
/* The f4 tables, built on the host (no GPU): key_table[4096] (bits 0-3 bytes consumed, 0 = no
 * whole character; bits 4-6 characters decoded; bits 8-15 shuffle index) and
 * shuffle_table[209 * 8] (per entry: four PRMT selector pairs A | B << 16 and four byte masks
 * M; output register r = mux(M_r, prmt(w0, w1, A_r), prmt(w2, 0, B_r)) of the 12-byte window
 * w0..w2).  Returns UG_OK, or UG_ERR_ARG for a NULL pointer. */
int ug_utf8_keyed_tables(uint16_t *key_table, uint32_t *shuffle_table);
/* Shard forms (the window conventions of ug_*_shard_async; the plan covers the owned range). */
int ug_utf8_shard_plan_async(const uint8_t *in, size_t n, size_t halo_before, size_t halo_after,
                             uint64_t *d_len, void *d_plan, void *stream);
int ug_utf16le_shard_plan_async(const uint16_t *in, size_t n, size_t halo_before,
                                size_t halo_after, uint64_t *d_len, void *d_plan, void *stream);
int ug_utf8_to_utf16le_shard_planned_async(const uint8_t *in, size_t n, size_t halo_before,
                                           size_t halo_after, uint64_t in_global_offset,
                                           const void *d_plan, uint16_t *out, size_t out_cap,
                                           ug_shard_record *d_rec, void *stream);
int ug_utf16le_to_utf8_shard_planned_async(const uint16_t *in, size_t n, size_t halo_before,
                                           size_t halo_after, uint64_t in_global_offset,
                                           const void *d_plan, uint8_t *out, size_t out_cap,
                                           ug_shard_record *d_rec, void *stream);

/* ------------------------------------------------------------------ multi-GPU, one process
 * The whole sharded step for a C caller that drives several devices from one process
 * (BASELINE north_star item 3): shard k runs on shards[k].device with its
 * stream; the 32-byte records are exchanged device to device (cudaMemcpyPeerAsync; a plain
 * device copy when two shards share a device) and every shard's device combines them
 * (k_combine), so each device ends with the global result and its own output offset.
 * Shards must be given in input order; each descriptor is exactly the arguments of the
 * matching ug_*_shard_async call (cuts at character starts, e.g. by
 * ug_utf8_cut_backoff), shard k + 1 starting where shard k ends (in_global_offset).
 * Positions in the result are in that global numbering (success: position = the end offset
 * of the last shard; error: the global first-error offset); `written` counts output units
 * from shard 0's output start.  Outputs stay sharded: shard k's units are out[0..count_k) at
 * global output offset out_offsets[k].
 *   ug_sharded_*():  synchronous; returns the global ug_result and, if out_offsets is not
 *                    NULL, each shard's global output offset (host array of nshards);
 *   errors:          UG_ERR_ARG (nshards < 1 or > 1024, bad descriptor: the shard call's own
 *                    checks), UG_ERR_CUDA (a launch, peer copy or synchronisation failed;
 *                    e.g. no peer access between two devices). */
typedef struct {
  int device;              /* CUDA device ordinal of this shard                            */
  const void *in;          /* first OWNED unit (device pointer on `device`)               */
  size_t n;                /* owned units                                                  */
  size_t halo_before;      /* readable context units before `in` (<= 3 / 1 used)           */
  size_t halo_after;       /* readable context units after in[n - 1]                       */
  uint64_t in_global_offset;  /* offset of in[0] in the whole input                        */
  void *out;               /* this shard's output (device pointer on `device`), or NULL    */
  size_t out_cap;          /* output capacity in units                                     */
  void *stream;            /* a stream of `device` (NULL = its legacy default stream)      */
} ug_shard_desc;

ug_result ug_sharded_utf8_to_utf16le(const ug_shard_desc *shards, int nshards,
                                     uint64_t *out_offsets);
ug_result ug_sharded_utf16le_to_utf8(const ug_shard_desc *shards, int nshards,
                                     uint64_t *out_offsets);
ug_result ug_sharded_utf8_validate(const ug_shard_desc *shards, int nshards);
ug_result ug_sharded_utf16le_validate(const ug_shard_desc *shards, int nshards);

/* Cut rule on HOST memory: how many units to move a nominal cut back
 * so that it falls on a character start.  `at` points at the unit at the nominal cut; up to
 * `avail_before` units before it are readable.  UTF-8: back off over at most 3 continuation
 * bytes (stop early at a non-continuation byte); UTF-16: back off 1 word off a low
 * surrogate. */
size_t ug_utf8_cut_backoff(const uint8_t *at, size_t avail_before);
size_t ug_utf16_cut_backoff(const uint16_t *at, size_t avail_before);
/* The same rule on big-endian UTF-16 words (f3). */
size_t ug_utf16be_cut_backoff(const uint16_t *at, size_t avail_before);

/* Sharded UTF-16BE variants (f3): the shard contract above, on big-endian words. */
int ug_utf8_to_utf16be_shard_async(const uint8_t *in, size_t n, size_t halo_before,
                                   size_t halo_after, uint64_t in_global_offset, uint16_t *out,
                                   size_t out_cap, ug_shard_record *d_rec, void *stream);
int ug_utf16be_to_utf8_shard_async(const uint16_t *in, size_t n, size_t halo_before,
                                   size_t halo_after, uint64_t in_global_offset, uint8_t *out,
                                   size_t out_cap, ug_shard_record *d_rec, void *stream);
int ug_utf16be_validate_shard_async(const uint16_t *in, size_t n, size_t halo_before,
                                    size_t halo_after, uint64_t in_global_offset,
                                    ug_shard_record *d_rec, void *stream);

/* ------------------------------------------------------------------ host buffers
 * End-to-end variants on HOST memory (pinned memory gives DMA-speed copies in both
 * directions at once).  Same result as the device functions on the same data.  The input is
 * processed as a pipeline of chunks of ug_set_host_chunk() input units cut at character starts
 * (DESIGN.md f2): chunk i is copied in on one copy stream, transcoded as a shard (the sharded
 * kernel is exact at any cut, D2) on `stream`, and its output copied out on a second
 * copy stream as soon as its 32-byte record has fixed its output offset, so host->device
 * copies, kernels and device->host copies overlap.  Chunks stream through 4 (ug_set_host_slots) library-owned
 * device staging slots per (device, stream) (a chunk with its halos + its worst-case output
 * each), reused round robin: device memory is O(chunk), not O(n), so inputs larger than HBM
 * stream through.  Synchronous (returns when the output is in out_host).
 * out_host[0..written) is exact; nothing at or beyond out_host[out_cap] is written.
 * Thread safety (all entry points): calls on one (device, stream) serialise on its workspace
 * mutex, a synchronous call holding it from its launch through its result read-back. */
ug_result utf8_to_utf16le_host(const uint8_t *in_host, size_t n, uint16_t *out_host,
                               size_t out_cap, void *stream);
ug_result utf16le_to_utf8_host(const uint16_t *in_host, size_t n, uint8_t *out_host,
                               size_t out_cap, void *stream);
/* UTF-16BE host-buffer variants (f3). */
ug_result utf8_to_utf16be_host(const uint8_t *in_host, size_t n, uint16_t *out_host,
                               size_t out_cap, void *stream);
ug_result utf16be_to_utf8_host(const uint16_t *in_host, size_t n, uint8_t *out_host,
                               size_t out_cap, void *stream);

/* Chunk size of the host-buffer pipeline, in input code units (default 64 Mi units); returns
 * the previous value.  0 restores the default.  Process-wide. */
size_t ug_set_host_chunk(size_t units);
/* Number of device staging slots of the host-buffer pipeline (chunks in flight; 2..16, default
 * 4; other values restore the default); returns the previous value.  Process-wide. */
int ug_set_host_slots(int slots);

/* f2, file form (SURVEY 8(f) f2 "input ... on NVMe"): validate + transcode the
 * file in_path (UTF-8 bytes / UTF-16LE words, no BOM handling: the bytes are the text) into the
 * file out_path (created or truncated), streaming through bounded memory: segments of
 * ug_set_file_segment() input units (default 128 Mi) are read with pread at character-start
 * cuts with their halos, the next segment's read overlapping the current one's pipeline (the
 * *_host chunk pipeline above: pinned host segment -> staging slots -> kernels -> output),
 * each segment's output appended to out_path.  Host memory: two input segments and one output
 * segment, pinned; device memory: the *_host staging.  Result as for the device call over the
 * whole file: {UG_OK, n, units} or {kind, e, units before e} (then out_path holds exactly those
 * units); UG_ERR_ARG for a NULL / unreadable / uncreatable path, a UTF-16 file of odd size, or a
 * read / write failure; UG_ERR_CUDA on a CUDA failure.  The pinned segment buffers are kept
 * for the next call (freed by ug_release_workspaces); concurrent file calls are serialised. */
ug_result ug_utf8_to_utf16le_file(const char *in_path, const char *out_path, void *stream);
ug_result ug_utf16le_to_utf8_file(const char *in_path, const char *out_path, void *stream);
/* Input units per file segment (0: default 128 Mi); returns the previous value. */
size_t ug_set_file_segment(size_t units);

/* ------------------------------------------------------------------ misc */
/* Human-readable name of a ug_error value (static string). */
const char *ug_error_name(int err);
/* Number of kernel launches this process has issued through the library (for the bench's
 * gpu_launches accounting). */
uint64_t ug_launch_count(void);
/* Free the workspaces of the current device (all streams). */
void ug_release_workspaces(void);
/* Input bytes per tile of the single-pass transcoding kernels (16 KiB in this build): tile t of a call
 * covers input bytes [t * T - lead, (t + 1) * T - lead) where lead = (input address mod 16).
 * Exposed so tests can place inputs across real tile edges. */
size_t ug_tile_bytes(void);
/* Input bytes per tile of the two-pass (planned) transcoders and of the plan's sub-ranges
 * (8 KiB in this build), with the same tiling rule as ug_tile_bytes. */
size_t ug_planned_tile_bytes(void);
/* Device bytes currently held by the library's workspace for (current device, stream): tile
 * status words, counters, result slots, and the host pipeline's staging slots (bounded:
 * 4 slots of one chunk each, whatever n is) and per-chunk records.  0 if none exists. */
size_t ug_workspace_bytes(void *stream);
int ug_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* UNIGPU_H */
