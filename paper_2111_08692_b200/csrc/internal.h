// internal.h -- declarations shared by kernels.cu (device code + launchers) and api.cu (the
// C-ABI).  Not part of the public interface (include/unigpu.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace ug {

// Device-side mirrors of the public structs (identical layout, checked in api.cu).
struct ResultDev {
  int32_t error;
  uint32_t reserved;
  unsigned long long position;
  unsigned long long written;
};
struct RecordDev {
  unsigned long long count;
  unsigned long long first_err;
  unsigned long long written;
  int32_t kind;
  int32_t reserved;  // 1 = this rank's output buffer was too small
};

constexpr int ERR_OUTPUT_TOO_SMALL = -3;

// Arguments of one tile-kernel launch (passed by value as the kernel parameter).
struct TileArgs {
  Window win;                   // byte positions (UTF-16: 2 bytes per word)
  void *out;                    // output buffer (uint16_t* or uint8_t*), may be null
  unsigned long long out_cap;   // in output units
  unsigned long long ntiles;
  uint64_t *status;             // tile status words (transcoders)
  uint32_t epoch;
  Counters *ctr;
  ResultDev *result;            // non-sharded result slot, or null
  RecordDev *rec;               // sharded record slot, or null
  unsigned long long global_off;  // sharded: global offset of position 0 (code units)
};

enum class Op : int {
  U8_VALIDATE = 0, U8_TO_U16 = 1, U16_VALIDATE = 2, U16_TO_U8 = 3,
  U16BE_VALIDATE = 4, U8_TO_U16BE = 5, U16BE_TO_U8 = 6  // UTF-16BE
};
constexpr int NUM_OPS = 7;
inline bool op_u16_input(Op op) {
  return op == Op::U16_VALIDATE || op == Op::U16_TO_U8 || op == Op::U16BE_VALIDATE ||
         op == Op::U16BE_TO_U8;
}
inline bool op_transcodes(Op op) {
  return op == Op::U8_TO_U16 || op == Op::U16_TO_U8 || op == Op::U8_TO_U16BE ||
         op == Op::U16BE_TO_U8;
}

size_t tile_smem_bytes(Op op);
int tile_threads(Op op);
unsigned long long tile_units(Op op, long long nbytes, long long lead, int *per_cta);
cudaError_t tile_configure(Op op);  // set max dynamic smem (idempotent)
cudaError_t tile_occupancy(Op op, int *blocks_per_sm);
cudaError_t launch_tile(Op op, const TileArgs &a, int grid, cudaStream_t s);

// planned (two-pass) path: plan kernels and the planned transcoders
constexpr int PLAN_HDR = 16;                // header words (kernels.cu plan_finish)
constexpr int PLAN_WORDS = PLAN_HDR + 8192;  // header + sub-range offsets
#ifndef UG_PLAN_SUBS
#define UG_PLAN_SUBS 8
#endif
constexpr int PLAN_SUBS_PER_CTA = UG_PLAN_SUBS;  // sub-ranges per planned-transcoder CTA (tickets)
size_t planned_smem_bytes(bool u16in);
cudaError_t planned_configure(Op op);
cudaError_t planned_occupancy(Op op, int *blocks_per_sm);
// f4: the planned forward with the keyed 12-byte decoder (utf8_keyed.cuh)
cudaError_t keyed_upload();  // tables to the current device + kernel attributes
cudaError_t keyed_occupancy(int *blocks_per_sm);
cudaError_t launch_planned_keyed(const TileArgs &a, const unsigned long long *plan, int grid,
                                 cudaStream_t s);
int planned_kernels(Op op);
cudaError_t launch_planned(Op op, const TileArgs &a, const unsigned long long *plan, int grid,
                           cudaStream_t s);
cudaError_t launch_plan(bool u16in, bool be, const Window &w, unsigned long long ntiles,
                        int nsub, unsigned long long tps, unsigned long long *plan,
                        Counters *ctr, unsigned long long *d_len, cudaStream_t s);

cudaError_t launch_len8(const uint8_t *in, unsigned long long n, Counters *ctr,
                        unsigned long long *d_len, int grid, cudaStream_t s);
cudaError_t launch_len16(const uint16_t *in, unsigned long long n, Counters *ctr,
                         unsigned long long *d_len, int grid, cudaStream_t s, bool be = false);
cudaError_t launch_combine(const RecordDev *recs, int nranks, int rank,
                           unsigned long long total_in, ResultDev *res,
                           unsigned long long *out_off, cudaStream_t s);
// host mirror of the combine kernel (same code path semantics)
void combine_host(const RecordDev *recs, int nranks, int rank, unsigned long long total_in,
                  ResultDev *res, unsigned long long *out_off);

#ifdef UG_TRACE
cudaError_t trace_read(void *host, size_t bytes);
cudaError_t dbg_read(void *host);
#endif
}  // namespace ug
