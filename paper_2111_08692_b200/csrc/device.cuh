// device.cuh -- sm_100a device primitives for libunigpu: TMA bulk copies + mbarriers, relaxed
// global atomics for the decoupled look-back, the epoch-tagged tile status word, the tile
// loader shared by all tile kernels, and block-level scan helpers.
//
// Nothing here computes the method itself; the UTF-8 / UTF-16 arithmetic lives in utf8.cuh /
// utf16.cuh.  Independent of oracle/ (shares no code with it).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef UG_MBAR_SUSPEND_NS
#define UG_MBAR_SUSPEND_NS 20000
#endif

namespace ug {

constexpr uint32_t FULL = 0xffffffffu;
constexpr uint64_t NONE = ~0ull;
#ifndef UG_NT
#define UG_NT 512
#endif
constexpr int NT = UG_NT;         // data threads per CTA for the tile kernels
constexpr int LNT = 512;          // threads per CTA for the length reductions
constexpr int TILE = NT * 32;     // input bytes per tile (32 per data thread)
#ifndef UG_CPS
#define UG_CPS (1024 / UG_NT)
#endif
constexpr int CTAS_PER_SM = UG_CPS;  // transcoder CTAs per SM (register budget)
constexpr int BPT = TILE / NT;    // 32 contiguous input bytes per thread
#ifndef UG_LB_PER_LANE
// measured (tools/exp/exp65-66.sh): 1 beats 2/3/4/8 on every config - wider rounds only add
// polling (each lane re-polls its unpublished words until the window resolves)
// (reverse c4 -6 %, ASCII -14 %; forward c4 -3 %, ASCII -10 % against 8)
#define UG_LB_PER_LANE 1
#endif
constexpr int LB_PER_LANE = UG_LB_PER_LANE;  // look-back window: 32 lanes x LB_PER_LANE tiles
constexpr int HALO = 16;          // bytes of context loaded before and after each tile
constexpr int INBUF = TILE + 2 * HALO;
// The two-pass (planned) transcoders run their own geometry: 256 threads x 32 bytes = 8 KiB
// tiles, 4 CTAs per SM (measured against 512 x 32 at 2 CTAs/SM: forward -1.4 %, reverse -2.5 %
// on config 4, -5..-7 % on ASCII; the same switch for every kernel slowed the validators and
// the single-pass kernels, which keep NT).
#ifndef UG_NTP
#define UG_NTP 256
#endif
#ifndef UG_PHALVES
#define UG_PHALVES 1
#endif
#ifndef UG_CPSP
#define UG_CPSP (1024 / UG_NTP / UG_PHALVES)
#endif
constexpr int NTP = UG_NTP;
constexpr int PHALVES = UG_PHALVES;     // 32-byte chunks per thread per planned tile
constexpr int HALFP = NTP * 32;         // one chunk of every thread (warps own 1 KiB each)
constexpr int TILEP = HALFP * PHALVES;  // input bytes per planned tile
constexpr int CPSP = UG_CPSP;

// ---------------------------------------------------------------- workspace counters
// One per (device, stream); zero-initialised once, self-resetting at the end of every call
// (the last CTA to finish resets them), so each API call is a single launch.
struct Counters {
  uint32_t ticket;    // dynamic tile tickets (decoupled look-back needs issue order)
  uint32_t done;      // CTAs finished
  unsigned long long err_min;  // smallest error position found (NONE = none)
  unsigned long long accum;    // reduction accumulator (length-from kernels)
  unsigned long long accf;     // second accumulator (the UTF-8 plan's >= F0 bytes)
  unsigned long long flags;    // bit 0: a planned transcoder was given a plan of other input
};

// ---------------------------------------------------------------- status words
// [63:40] call epoch (24 bits) | [39:38] flag | [37:0] value.  A word whose epoch is not the
// current call's reads as "not ready", so the array never needs clearing between calls.
constexpr uint32_t FLAG_AGG = 1, FLAG_PREFIX = 2;
__device__ __forceinline__ uint64_t pack_status(uint32_t epoch, uint32_t flag, uint64_t v) {
  return ((uint64_t)epoch << 40) | ((uint64_t)flag << 38) | (v & ((1ull << 38) - 1));
}

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  // try_wait with a suspend-time hint: the warp sleeps until the phase completes (or the hint
  // expires) instead of spinning on the issue slots the other warps need
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "UG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra UG_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity), "n"(UG_MBAR_SUSPEND_NS)
      : "memory");
}
// 1-D TMA bulk copy global -> shared, completing on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// 1-D TMA bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// order generic-proxy shared-memory writes before async-proxy (TMA) reads of them
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void sts8(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
template <int OFF>  // st.shared.u8 [addr + OFF] with the offset as an immediate
__device__ __forceinline__ void sts8o(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u8 [%0+%2], %1;" ::"r"(addr), "r"(v), "n"(OFF) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// ---------------------------------------------------------------- named barriers
// bar.arrive has release and bar.sync acquire semantics for the participating threads' shared
// memory accesses (producer / consumer hand-off between warp roles).
// Barrier ids are immediates so ptxas reserves only the ids actually used.
template <int ID, int N>
__device__ __forceinline__ void named_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
template <int ID, int N>
__device__ __forceinline__ void named_arrive() {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(N) : "memory");
}

// ---------------------------------------------------------------- warp / block helpers
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t = __shfl_up_sync(FULL, v, d);
    if (lane >= d) v += t;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
  return v;
}

// Byte-lane mask (0xFF per byte) of the 4 bytes at positions pos..pos+3 inside [lo, hi).
__device__ __forceinline__ uint32_t range_bytes(long long pos, long long lo, long long hi) {
  long long a = lo - pos, b = hi - pos;
  a = a < 0 ? 0 : (a > 4 ? 4 : a);
  b = b < 0 ? 0 : (b > 4 ? 4 : b);
  if (b <= a) return 0u;
  uint64_t m = ((1ull << (8 * b)) - 1) & ~((1ull << (8 * a)) - 1);
  return (uint32_t)m;
}

// ---------------------------------------------------------------- tile loader
// Input window of one call: positions are BYTE offsets from `base` (the first owned byte).
// Valid bytes are [lo_valid, hi_valid) = [-halo_before, n + halo_after); everything else reads
// as 0x00 (start / end of stream).  Tile t covers positions [t*TILE - lead, (t+1)*TILE - lead)
// so that tiles start on 16-byte boundaries in memory; its smem image holds positions
// [tile_pos - HALO, tile_pos + TILE + HALO).
struct Window {
  const uint8_t *base;
  long long lo_valid, hi_valid;
  long long lead;          // base % 16
  uintptr_t mem_lo, mem_hi;  // 16-byte aligned readable address range covering the window
  long long n;             // owned bytes
};

template <int TB = TILE>
__device__ __forceinline__ long long tile_pos(const Window &w, long long t) {
  return t * TB - w.lead;
}

// Issued by ONE thread: bulk-load the smem image of tile t into buf, completing on bar.
template <int TB = TILE>
__device__ __forceinline__ void issue_tile_load(const Window &w, long long t, uint8_t *buf,
                                                uint64_t *bar) {
  uintptr_t A = (uintptr_t)(w.base + tile_pos<TB>(w, t) - HALO);
  uintptr_t B = A + TB + 2 * HALO;
  uintptr_t a = A > w.mem_lo ? A : w.mem_lo;
  uintptr_t b = B < w.mem_hi ? B : w.mem_hi;
  uint32_t bytes = b > a ? (uint32_t)(b - a) : 0u;
  mbar_arrive_expect_tx(bar, bytes);
  if (bytes) bulk_g2s(buf + (a - A), (const void *)a, bytes, bar);
}

// Does tile t's smem image reach outside the valid window (needs fix_tile_edges)?
template <int TB = TILE>
__device__ __forceinline__ bool tile_at_edge(const Window &w, long long t) {
  const long long p0 = tile_pos<TB>(w, t) - HALO;
  return !(p0 >= w.lo_valid && p0 + TB + 2 * HALO <= w.hi_valid);
}

// After the load landed: zero every smem byte whose position lies outside the valid window
// (only tiles touching the window edges do any work).  Called by threads 0..nthreads-1; the
// caller syncs after.
template <int TB = TILE>
__device__ __forceinline__ void fix_tile_edges(const Window &w, long long t, uint8_t *buf,
                                               int nthreads, int first = -1) {
  constexpr int IB = TB + 2 * HALO;
  long long p0 = tile_pos<TB>(w, t) - HALO;
  if (p0 >= w.lo_valid && p0 + IB <= w.hi_valid) return;
  uint32_t *b32 = reinterpret_cast<uint32_t *>(buf);
  for (int q = first >= 0 ? first : (int)threadIdx.x; q < IB / 4; q += nthreads) {
    long long pos = p0 + 4 * q;
    if (pos >= w.lo_valid && pos + 4 <= w.hi_valid) continue;
    b32[q] &= range_bytes(pos, w.lo_valid, w.hi_valid);
  }
}

// ---------------------------------------------------------------- decoupled look-back
// Called by one full warp for tile t whose aggregate is already published (t > 0).  Returns the
// exclusive prefix (sum of all earlier tiles' aggregates) in every lane.  Each round reads a
// window of 32 x LB_PER_LANE predecessors (nearest first) with independent relaxed loads.
// One look-back round over K status words per lane: lane l examines tiles
// idx - K*l, ..., idx - K*l - K + 1 (nearest first).  Waits (re-polling only the words that
// are not yet published, with a back-off) until every word up to this lane's first inclusive
// prefix is published; returns true and the prefix if some lane saw one, else adds the whole
// window's aggregates to *excl.
template <int K>
__device__ __forceinline__ bool look_back_round(uint64_t *status, uint32_t epoch, long long idx,
                                                int lane, uint64_t *excl, int *polls) {
  const long long j0 = idx - (long long)K * lane;
  uint64_t s[K];
#pragma unroll
  for (int k = 0; k < K; k++) s[k] = (j0 - k >= 0) ? ld_relaxed(status + j0 - k) : 0;
  int spins = 0;
  while (true) {
    // ready: every word up to (and including) this lane's first PREFIX is published
    bool ready = true, stop = false;
#pragma unroll
    for (int k = 0; k < K; k++) {
      if (!stop && j0 - k >= 0) {
        const bool pub = (uint32_t)(s[k] >> 40) == epoch && ((s[k] >> 38) & 3u) != 0;
        if (!pub) ready = false;
        if (pub && ((s[k] >> 38) & 3u) == FLAG_PREFIX) stop = true;
      }
    }
    if (polls) ++*polls;
    if (__all_sync(FULL, ready)) break;
#ifndef UG_SLEEP0
#define UG_SLEEP0 128
#define UG_SLEEP1 512
#endif
    __nanosleep(spins < 2 ? UG_SLEEP0 : UG_SLEEP1);
    ++spins;
    bool stop2 = false;
#pragma unroll
    for (int k = 0; k < K; k++) {
      if (!stop2 && j0 - k >= 0) {
        const bool pub = (uint32_t)(s[k] >> 40) == epoch && ((s[k] >> 38) & 3u) != 0;
        if (!pub) s[k] = ld_relaxed(status + j0 - k);
        else if (((s[k] >> 38) & 3u) == FLAG_PREFIX) stop2 = true;
      }
    }
  }
  bool has_p = false;
  uint64_t lane_sum = 0;
#pragma unroll
  for (int k = 0; k < K; k++) {
    if (!has_p) {
      bool pre = (j0 - k < 0) || (((s[k] >> 38) & 3u) == FLAG_PREFIX);
      lane_sum += (j0 - k < 0) ? 0ull : (s[k] & ((1ull << 38) - 1));
      has_p = pre;
    }
  }
  const uint32_t pm = __ballot_sync(FULL, has_p);
  if (pm) {
    const int first = __ffs(pm) - 1;
    *excl += warp_sum64(lane <= first ? lane_sum : 0ull);
    return true;
  }
  *excl += warp_sum64(lane_sum);
  return false;
}

// Push-forward (after tile t's inclusive prefix `incl` is known): publish the inclusive
// prefixes of the run of successors t+1, t+2, ... (up to 32) whose aggregates are already
// published.  An inclusive prefix is unique, so a push racing with the tile's own look-back (or
// another push) writes the same value.  It kept the published-prefix frontier close behind the
// aggregate frontier when look-back rounds were 256 wide; with 32-wide rounds it only adds
// polling (measured 0.3-11 % slower), so it is compiled only with -DUG_PUSH.
__device__ __forceinline__ void push_forward(uint64_t *status, uint32_t epoch, long long t,
                                             long long ntiles, uint64_t incl, int lane) {
  const long long j = t + 1 + lane;
  uint64_t w = (j < ntiles) ? ld_relaxed(status + j) : 0ull;
  const uint32_t fl = ((uint32_t)(w >> 40) == epoch) ? (uint32_t)((w >> 38) & 3u) : 0u;
  // the run: lanes below the first lane that is unpublished or already an inclusive prefix
  const uint32_t stop = __ballot_sync(FULL, fl != FLAG_AGG);
  const int run = stop ? __ffs(stop) - 1 : 32;
  uint64_t v = (lane < run) ? (w & ((1ull << 38) - 1)) : 0ull;
  // inclusive scan of the aggregates over the run
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = __shfl_up_sync(FULL, v, d);
    if (lane >= d) v += o;
  }
  if (lane < run) st_relaxed(status + j, pack_status(epoch, FLAG_PREFIX, incl + v));
}

// Exclusive prefix of tile t (t > 0): the sum of all earlier tiles' aggregates, from the
// nearest inclusive prefix.  A first round probes only the 32 nearest predecessors (one
// status word per lane), later rounds LB_PER_LANE per lane: the look-backs of all CTAs poll
// L2 concurrently, so each round's request volume matters.
__device__ __forceinline__ uint64_t look_back(uint64_t *status, uint32_t epoch, long long t,
                                              int lane, int *rounds = nullptr,
                                              unsigned long long *t_first = nullptr,
                                              int *polls = nullptr) {
  uint64_t excl = 0;
  long long idx = t - 1;
  if (rounds) ++*rounds;
  if (look_back_round<1>(status, epoch, idx, lane, &excl, polls)) return excl;
#ifdef UG_TRACE
  if (t_first && *t_first == 0) {
    unsigned long long tt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
    *t_first = tt;
  }
#endif
  idx -= 32;
  while (true) {
    if (rounds) ++*rounds;
    if (look_back_round<LB_PER_LANE>(status, epoch, idx, lane, &excl, polls)) return excl;
    idx -= (long long)LB_PER_LANE * 32;
  }
}

}  // namespace ug
