// kernels.cu -- the sm_100a kernels of libunigpu.
//
//   k_utf8<false>   utf8_validate              (K1)  classify tiles, rescan flagged ones
//   k_utf8<true>    utf8_to_utf16le            (K2)  + widths, scan, look-back, decode, store
//   k_utf16<false>  utf16le_validate           (K3)  pairing predicate
//   k_utf16<true>   utf16le_to_utf8            (K4)  + widths, scan, look-back, encode, store
//   k_len8 / k_len16  length-from reductions    (K5, K6)
//   k_combine       sharded result combine      (C1 consumer)
// Finalisation (first-error kind, written count, result slot, counter reset) is done by the
// last CTA to finish (K7), so every API call is one launch.
//
// Tile pipeline (all tile kernels): persistent CTAs of 512 threads pull 16 KiB tiles by
// atomic ticket (issue order makes the decoupled look-back deadlock-free), bulk-load tile +
// 16-byte halos into shared memory with TMA (cp.async.bulk + mbarrier, 2 stages: the next
// tile is in flight while the current one is processed), and each thread owns 32 contiguous
// input bytes.  Transcoders: warp 0 publishes the tile aggregate and looks back while the
// other warps already decode into a shared-memory stage at tile-local offsets; once the
// tile's global offset is known every thread streams 16-byte output chunks, re-aligned to the
// global address phase in registers (funnel shifts), with 128-bit stores.
#include <cstdint>

#include "device.cuh"
#include "internal.h"
#include "utf16.cuh"
#include "utf8.cuh"
#include "utf8_keyed.cuh"

namespace ug {

#ifdef UG_TRACE
// Debug trace (tools only): per CTA, per iteration: [tile, lb_start, lb_end, rounds, pwait_start, pwait_end]
constexpr int TR_IT = 64;
__device__ unsigned long long g_trace[1024][TR_IT][12];
__device__ unsigned long long g_dbg[8];  // [0] warps rescanned (validate), [1] tiles rescanned (transcode)
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

constexpr unsigned long long VALMASK = (1ull << 38) - 1;
// named barrier ids (0 is __syncthreads)
constexpr int BAR_DATA = 1;           // the NT data threads
#ifndef UG_PRODUCER
#define UG_PRODUCER (NT - 32)
#endif
// the data thread that draws tickets, issues the tile loads and publishes the forward kernel's
// aggregates: lane 0 of the LAST data warp, so that warp 0 (bulk stores, head / tail bytes)
// is not also the one the emit barriers wait for
constexpr int PRODUCER = UG_PRODUCER;
#ifndef UG_SHIP_WARP
#define UG_SHIP_WARP 0
#endif
// lane 0 of this warp issues the TMA bulk stores of the stage; its lanes store head / tail
constexpr int SHIPPER = 32 * UG_SHIP_WARP;

__device__ __forceinline__ uint32_t byte_at(const Window &w, long long pos) {
  return (pos >= w.lo_valid && pos < w.hi_valid) ? (uint32_t)w.base[pos] : 0u;
}
__device__ __forceinline__ uint32_t word_at(const Window &w, long long wpos) {
  long long pos = 2 * wpos;
  return (pos >= w.lo_valid && pos + 2 <= w.hi_valid)
             ? (uint32_t)reinterpret_cast<const uint16_t *>(w.base)[wpos]
             : 0u;
}


// Block exclusive scan over the NT data threads: returns the thread's exclusive prefix within
// the tile and the tile total.  One data-warp barrier inside.
__device__ __forceinline__ void block_scan(uint32_t cnt, uint32_t *s_wsum, int lane, int warp,
                                           uint32_t *excl, uint32_t *total) {
  uint32_t incl = warp_incl_scan(cnt, lane);
  if (lane == 31) s_wsum[warp] = incl;
  named_sync<BAR_DATA, NT>();
  // every warp scans the NT/32 warp totals with shuffles (lane l holds warp l's total)
  uint32_t v = (lane < NT / 32) ? s_wsum[lane] : 0u;
#pragma unroll
  for (int d = 1; d < NT / 32; d <<= 1) {
    uint32_t t = __shfl_up_sync(FULL, v, d);
    if (lane >= d) v += t;
  }
  const uint32_t wincl = __shfl_sync(FULL, v, warp);
  *total = __shfl_sync(FULL, v, NT / 32 - 1);
  *excl = wincl - __shfl_sync(FULL, incl, 31) + incl - cnt;
}

// Exclusive prefix of tile t (sum of all earlier tiles' aggregates); one full warp.  Needs only
// the predecessors, so it runs while tile t itself is still being loaded and classified.
__device__ __forceinline__ unsigned long long tile_excl_prefix(const TileArgs &a, long long t,
                                                               int lane, int *rounds = nullptr,
                                                               unsigned long long *t_first = nullptr,
                                                               int *polls = nullptr) {
  if (t == 0) return 0;
  return look_back(a.status, a.epoch, t, lane, rounds, t_first, polls);
}

// Write the call's outcome (last CTA, lane 0) and reset the per-call counters.
__device__ __forceinline__ void write_outcome(const TileArgs &a, bool xc, int kind,
                                              unsigned long long e, unsigned long long total,
                                              unsigned long long wr, unsigned long long n_units) {
  unsigned long long required = (e == NONE) ? total : wr;
  bool small = xc && required > a.out_cap;
  if (a.rec) {
    RecordDev r;
    r.count = xc ? total : 0ull;
    r.first_err = (e == NONE) ? NONE : e + a.global_off;
    r.written = (e == NONE) ? 0ull : wr;
    r.kind = (e == NONE) ? 0 : kind;
    r.reserved = small ? 1 : 0;
    *a.rec = r;
  }
  if (a.result) {
    ResultDev r;
    r.reserved = 0;
    if (small) {
      r.error = ERR_OUTPUT_TOO_SMALL;
      r.position = required;
      r.written = 0;
    } else if (e == NONE) {
      r.error = 0;
      r.position = n_units;
      r.written = xc ? total : 0ull;
    } else {
      r.error = kind;
      r.position = e;
      r.written = xc ? wr : 0ull;
    }
    *a.result = r;
  }
  a.ctr->ticket = 0;
  a.ctr->done = 0;
  a.ctr->err_min = NONE;
}

// ============================================================================ UTF-8 policy
// Positions are bytes.  Thread `tid` owns tile bytes [32 tid, 32 tid + 32).
// Bit i of a chunk mask = position pos0 + i.
__device__ __forceinline__ uint32_t bit_range(long long pos0, long long lo, long long hi) {
  long long a = lo - pos0, b = hi - pos0;
  a = a < 0 ? 0 : (a > 32 ? 32 : a);
  b = b < 0 ? 0 : (b > 32 ? 32 : b);
  if (b <= a) return 0u;
  const uint32_t mb = b == 32 ? 0xFFFFFFFFu : ((1u << b) - 1u);
  const uint32_t ma = a == 32 ? 0xFFFFFFFFu : ((1u << a) - 1u);
  return mb & ~ma;
}

// BE: UTF-16BE output; only the unit packing differs.
template <bool BE>
struct U8PolT {
  using Out = uint16_t;
  static constexpr int UNIT = 1;                      // input bytes per position
  static constexpr bool kNoF = true;  // planned kernel: warps without >= F0 leads decode by units4_nof
  static constexpr int STAGE = 2 * (TILE + 32);        // stage bytes per buffer
  struct St {
    uint32_t w[8];   // own 32 bytes
    uint32_t prev;   // the 4 bytes before
    uint32_t nxt;    // the 4 bytes after
    uint32_t err;    // classifier flags (a3)
    uint32_t fany;   // nonzero: a >= F0 lead in the chunk or the 3 bytes before (f1, UTF-8)
    long long pos0;  // position of own byte 0
    long long n;
    const uint8_t *img;  // own bytes in the smem tile image
    bool wasc;
  };

  // Thread tid's 32 bytes of the tile image in `buf` (plus the 4 before and after), its
  // position, and the warp-uniform ASCII verdict (a2).
  template <bool IN>
  __device__ static __forceinline__ void load(St &s, const uint8_t *buf, int tid, int lane,
                                              long long tp, long long n) {
    const uint8_t *my = buf + HALO + BPT * tid;
    s.img = my;
    {
      uint4 q0 = *reinterpret_cast<const uint4 *>(my);
      uint4 q1 = *reinterpret_cast<const uint4 *>(my + 16);
      s.w[0] = q0.x; s.w[1] = q0.y; s.w[2] = q0.z; s.w[3] = q0.w;
      s.w[4] = q1.x; s.w[5] = q1.y; s.w[6] = q1.z; s.w[7] = q1.w;
    }
    uint32_t prev = __shfl_up_sync(FULL, s.w[7], 1);
    uint32_t nxt = __shfl_down_sync(FULL, s.w[0], 1);
    if (lane == 0) prev = *reinterpret_cast<const uint32_t *>(my - 4);
    if (lane == 31) nxt = *reinterpret_cast<const uint32_t *>(my + BPT);
    s.prev = prev;
    s.nxt = nxt;
    s.pos0 = tp + BPT * tid;
    s.n = n;
    // a2: warp ASCII fast path (no byte >= 0x80 and no pending lead before the warp)
    uint32_t orv = s.w[0] | s.w[1] | s.w[2] | s.w[3] | s.w[4] | s.w[5] | s.w[6] | s.w[7];
    bool pend = (prev >= 0xC0000000u) || ((prev & 0x00FF0000u) >= 0x00E00000u) ||
                ((prev & 0x0000FF00u) >= 0x0000F000u);
    s.wasc = __all_sync(FULL, ((orv & HI) == 0u) && !pend);
  }

  // The same state from registers (streaming validator): q0 / q1 = the thread's 32 bytes,
  // pv / nx = the 4 bytes before / after.
  __device__ static __forceinline__ void from_regs(St &s, uint4 q0, uint4 q1, uint32_t pv,
                                                   uint32_t nx, long long pos0, long long n) {
    s.w[0] = q0.x; s.w[1] = q0.y; s.w[2] = q0.z; s.w[3] = q0.w;
    s.w[4] = q1.x; s.w[5] = q1.y; s.w[6] = q1.z; s.w[7] = q1.w;
    s.prev = pv;
    s.nxt = nx;
    s.pos0 = pos0;
    s.n = n;
    const uint32_t orv = q0.x | q0.y | q0.z | q0.w | q1.x | q1.y | q1.z | q1.w;
    const bool pend = (pv >= 0xC0000000u) || ((pv & 0x00FF0000u) >= 0x00E00000u) ||
                      ((pv & 0x0000FF00u) >= 0x0000F000u);
    s.wasc = __all_sync(FULL, ((orv & HI) == 0u) && !pend);
  }

  // a3 classification (flags into s.err) and, if xc, the number of units the thread emits.
  template <bool IN>  // IN: the whole tile is owned (tile-uniform)
  __device__ static __forceinline__ uint32_t analyze(St &s, int tid, bool xc) {
    uint32_t emit = 0xFFFFFFFFu;
    s.err = 0;
#ifdef UG_ABL_NOVAL
    emit = ~s.w[0] & 0x80808080u;
#else
    s.fany = 0;
    if (!s.wasc) s.err = u8::analyze32(s.w, s.prev, s.nxt, (tid & 31) == 31, &emit, &s.fany);
#endif
    if (!xc) return 0u;
    if (!IN) emit &= bit_range(s.pos0, 0, s.n);
    return popc(emit);
  }

  __device__ static __forceinline__ bool hint(const St &s) { return s.err != 0; }

  // a4: exact rescan of the owned positions (cold: only in flagged tiles)
  __device__ static __forceinline__ unsigned long long find_error(const St &s, long long n) {
    unsigned long long found = NONE;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const uint32_t wb = k ? s.w[k - 1] : s.prev;
      const uint32_t wn = k < 7 ? s.w[k + 1] : s.nxt;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const long long pos = s.pos0 + 4 * k + j;
        const uint32_t back = fsr(wb, s.w[k], 8 * j);
        const uint32_t fwd = fsr(s.w[k], wn, 8 * j);
        if (found == NONE && pos >= 0 && pos < n && u8::err_at(back, fwd))
          found = (unsigned long long)pos;
      }
    }
    return found;
  }

  // a7: decode the owned characters into stage[o ...] (UTF-16 units).  Each emitting position
  // stores its unit at its exclusive-prefix slot (predicated on the emit mask).
  template <bool IN, bool NOF = false>  // NOF: the warp holds no >= F0 lead (units4_nof)
  __device__ static __forceinline__ void decode(const St &s, uint16_t *stage, uint32_t o,
                                                uint32_t, long long) {
    if (IN && s.wasc) {
      // a2: the warp's 1 KiB is ASCII and its 1024 units are contiguous from lane 0's slot.
      // Written cooperatively: lane l zero-extends warp words l, l + 32, ... (read back from
      // the tile image), so each store instruction covers consecutive 8-byte chunks.
      const int lane = threadIdx.x & 31;
      const uint32_t *wb = reinterpret_cast<const uint32_t *>(s.img - BPT * lane) + lane;
      const uint32_t o0 = __shfl_sync(FULL, o, 0);
      uint16_t *sb = stage + o0 + 4 * lane;
      if ((o0 & 3u) == 0u) {  // warp-uniform
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const uint32_t x = wb[32 * j];
          *reinterpret_cast<uint2 *>(sb + 128 * j) =
              make_uint2(prmt(x, 0u, BE ? 0x1404u : 0x4140u), prmt(x, 0u, BE ? 0x3424u : 0x4342u));
        }
      } else if ((o0 & 1u) == 0u) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const uint32_t x = wb[32 * j];
          uint32_t *d = reinterpret_cast<uint32_t *>(sb + 128 * j);
          d[0] = prmt(x, 0u, BE ? 0x1404u : 0x4140u);
          d[1] = prmt(x, 0u, BE ? 0x3424u : 0x4342u);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const uint32_t x = wb[32 * j];
#pragma unroll
          for (int q = 0; q < 4; q++)
            sb[128 * j + q] = (uint16_t)(((x >> (8 * q)) & 0xFFu) << (BE ? 8 : 0));
        }
      }
      return;
    }
#ifdef UG_ABL_NODECODE
    {
      uint32_t p = smem_addr(stage + o);
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint32_t em = (~s.w[k] >> 7) & 0x01010101u;
        const uint32_t inc2 = em * 0x02020202u;
        sts16(p, s.w[k]);
        p += inc2 >> 24;
      }
      return;
    }
#endif
    u8::Carry cy = u8::carry_of(s.prev);
    uint32_t p = smem_addr(stage + o);  // shared-window byte address of this thread's slot
#pragma unroll
    for (int k = 0; k < 8; k++) {
      uint32_t u01, u23;
      uint32_t em = NOF ? u8::units4_nof<BE>(s.w[k], cy, &u01, &u23)
                        : u8::units4<BE>(s.w[k], cy, &u01, &u23);
      if (!IN) em &= range_bytes(s.pos0 + 4 * k, 0, s.n) & 0x01010101u;
      const uint32_t inc2 = em * 0x02020202u;  // byte j: 2 x units emitted by positions <= j
      const uint32_t a1 = mad(prmt(inc2, 0u, 0x4440u), 1u, p);
      const uint32_t a2 = mad(prmt(inc2, 0u, 0x4441u), 1u, p);
      const uint32_t a3 = mad(prmt(inc2, 0u, 0x4442u), 1u, p);
      const uint32_t u1 = shr_fma<16>(u01), u3 = shr_fma<16>(u23);
      // only emitting positions store: fewer active lanes per store instruction means fewer
      // bank conflicts among the lanes' scattered slots (config 4: -3.7 % against storing
      // every position and letting the next unit overwrite the garbage)
      {
        if (em & 0x00000001u) sts16(p, u01);
        if (em & 0x00000100u) sts16(a1, u1);
        if (em & 0x00010000u) sts16(a2, u23);
        if (em & 0x01000000u) sts16(a3, u3);
      }
      p += shr_fma<24>(inc2);
    }
  }

  // a10 (last CTA, warp 0): kind of the first error and units written before it
  template <int TB = TILE>  // the launch's tile bytes (TILE, or TILEP for the planned kernels)
  __device__ static __forceinline__ void finalize(const TileArgs &a, unsigned long long e,
                                                  bool xc, int lane, int *kind,
                                                  unsigned long long *wr) {
    const Window &win = a.win;
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) x |= byte_at(win, (long long)e + j) << (8 * j);
    *kind = u8::decode_kind(x);
    *wr = 0;
    if (!xc) return;
    long long te = ((long long)e + win.lead) / TB;
    unsigned long long base = te ? (ld_relaxed(a.status + te - 1) & VALMASK) : 0ull;
    long long from = te * TB - win.lead;
    if (from < 0) from = 0;
    unsigned long long c = 0;
    for (long long i = from + lane; i < (long long)e; i += 32)
      c += u8::emits_at(byte_at(win, i), byte_at(win, i - 1), byte_at(win, i - 2),
                        byte_at(win, i - 3));
    *wr = base + warp_sum64(c);
  }
};

using U8Pol = U8PolT<false>;
using U8PolBE = U8PolT<true>;

// ---------------------------------------------------------------- f4: keyed 12-byte decoder
// SURVEY 8(f) f4, research comparison: the planned forward with the a7 decode
// replaced by the paper's keyed 12-byte routine (utf8_keyed.cuh).  Classification, validation,
// the ASCII warp path, counts, offsets and shipping are U8Pol's.  Tables: global memory, read
// through L1 (16 KiB + 6.5 KiB), uploaded once per device (keyed_upload).
__device__ uint16_t g_keyed_key[keyed::KEYS];
__device__ uint32_t g_keyed_shuf[keyed::SHUFFLES * keyed::SHUF_WORDS];

struct U8KeyPol : U8PolT<false> {
  static constexpr bool kNoF = false;  // the comparison keeps its own decode everywhere
  template <bool IN>
  __device__ static __forceinline__ void decode(const St &s, uint16_t *stage, uint32_t o,
                                                uint32_t lim, long long n) {
    if (IN && s.wasc) {  // a2: the warp's 1 KiB is ASCII (the paper's ASCII block path)
      U8PolT<false>::template decode<true>(s, stage, o, lim, n);
      return;
    }
    int lo = 0, hi = BPT;
    if (!IN) {
      lo = s.pos0 < 0 ? (int)(-s.pos0 < BPT ? -s.pos0 : BPT) : 0;
      const long long r = s.n - s.pos0;
      hi = r < 0 ? 0 : (r > BPT ? BPT : (int)r);
    }
    const uint32_t words[10] = {s.prev, s.w[0], s.w[1], s.w[2], s.w[3],
                                s.w[4], s.w[5], s.w[6], s.w[7], s.nxt};
    keyed::decode_thread(s.img, words, lo, hi, g_keyed_key, g_keyed_shuf, stage + o,
                         (int)(lim - o));
  }
};

// ============================================================================ UTF-16 policy
// Positions are words.  Thread `tid` owns tile words [16 tid, 16 tid + 16), two per register.

// BE: UTF-16BE input: the low/high byte split of the classes swaps its
// selectors (u16::classes4<BE>), the two scalar context words are byte-swapped.
template <bool BE>
struct U16PolT {
  using Out = uint8_t;
  static constexpr int UNIT = 2;
  static constexpr bool kBE = BE;
  static constexpr bool kNoF = false;  // (the UTF-8 forward's f1 form)
  __device__ static __forceinline__ uint32_t native(uint32_t w) {  // a stored word's value
    return BE ? (((w >> 8) | (w << 8)) & 0xFFFFu) : w;
  }
  static constexpr int STAGE = 3 * (TILE / 2) + 64;
  struct St {
    uint32_t w[8];                   // words 2k (low half), 2k + 1 (high half) of w[k]
    const uint8_t *img;              // own words in the smem tile image
    uint32_t prev_word, next_word;
    uint32_t own;                    // bit i: word i owned (all set in interior tiles)
    unsigned long long first_err;
    long long pos0;
    bool wasc;
  };
  // msb-per-byte ownership of words 4g..4g+3
  __device__ static __forceinline__ uint32_t own4(const St &s, int g) {
    return ((((s.own >> (4 * g)) & 0xFu) * 0x00204081u) & 0x01010101u) << 7;
  }

  template <bool IN>  // IN: the whole tile is owned (tile-uniform)
  __device__ static __forceinline__ void load(St &s, const uint8_t *buf, int tid, int lane,
                                              long long tp_bytes, long long n_bytes) {
    const long long tpw = tp_bytes / 2, nw = n_bytes / 2;
    const uint8_t *my = buf + HALO + BPT * tid;
    s.img = my;
    {
      uint4 q0 = *reinterpret_cast<const uint4 *>(my);
      uint4 q1 = *reinterpret_cast<const uint4 *>(my + 16);
      s.w[0] = q0.x; s.w[1] = q0.y; s.w[2] = q0.z; s.w[3] = q0.w;
      s.w[4] = q1.x; s.w[5] = q1.y; s.w[6] = q1.z; s.w[7] = q1.w;
    }
    uint32_t pv = __shfl_up_sync(FULL, s.w[7], 1);
    uint32_t nx = __shfl_down_sync(FULL, s.w[0], 1);
    if (lane == 0) pv = *reinterpret_cast<const uint32_t *>(my - 4);
    if (lane == 31) nx = *reinterpret_cast<const uint32_t *>(my + BPT);
    s.prev_word = native(pv >> 16);
    s.next_word = native(nx & 0xFFFFu);
    s.pos0 = tpw + (BPT / 2) * tid;
    s.own = IN ? 0xFFFFu : (bit_range(s.pos0, 0, nw) & 0xFFFFu);
    const uint32_t orv = s.w[0] | s.w[1] | s.w[2] | s.w[3] | s.w[4] | s.w[5] | s.w[6] | s.w[7];
    s.wasc = __all_sync(FULL, (orv & (BE ? 0x80FF80FFu : 0xFF80FF80u)) == 0u);
  }

  // The same state from registers (streaming validator): q0 / q1 = the thread's 16 words,
  // pv / nx = the 32-bit words before / after; pos0 / nw in words; own = words < nw owned.
  template <bool IN>
  __device__ static __forceinline__ void from_regs(St &s, uint4 q0, uint4 q1, uint32_t pv,
                                                   uint32_t nx, long long pos0, long long nw) {
    s.w[0] = q0.x; s.w[1] = q0.y; s.w[2] = q0.z; s.w[3] = q0.w;
    s.w[4] = q1.x; s.w[5] = q1.y; s.w[6] = q1.z; s.w[7] = q1.w;
    s.prev_word = native(pv >> 16);
    s.next_word = native(nx & 0xFFFFu);
    s.pos0 = pos0;
    s.own = IN ? 0xFFFFu : (bit_range(pos0, 0, nw) & 0xFFFFu);
    const uint32_t orv = q0.x | q0.y | q0.z | q0.w | q1.x | q1.y | q1.z | q1.w;
    s.wasc = __all_sync(FULL, (orv & (BE ? 0x80FF80FFu : 0xFF80FF80u)) == 0u);
  }

  // a9 pairing predicate (exact) and a5 widths, byte-SWAR over 4 words.
  template <bool IN>
  __device__ static __forceinline__ uint32_t analyze(St &s, int, bool xc) {
#ifdef UG_ABL_NOVAL
    s.first_err = NONE;
    return xc ? 16u : 0u;
#endif
    if (IN && s.wasc) {  // a2: the warp's words are all below 0x80: one byte each, no surrogate
      s.first_err = NONE;
      return xc ? 16u : 0u;
    }
    uint32_t Hprev = u16::is_high(s.prev_word) ? 0x80000000u : 0u;  // byte 3 = word -1
    u16::Cls4 c = u16::classes4<BE>(s.w[0], s.w[1]);
    uint32_t acc = 0, anyerr = 0, errm[4];
#pragma unroll
    for (int g = 0; g < 4; g++) {
      u16::Cls4 cn;
      uint32_t Lnext;
      if (g < 3) {
        cn = u16::classes4<BE>(s.w[2 * g + 2], s.w[2 * g + 3]);
        Lnext = cn.L;
      } else {
        Lnext = u16::is_low(s.next_word) ? 0x80u : 0u;
      }
      const uint32_t Hp = fsl(Hprev, c.H, 8), Ln = fsr(c.L, Lnext, 8);
      uint32_t e = (c.H & ~Ln) | (c.L & ~Hp);
      uint32_t d = u16::widths(c);  // widths
      if (!IN) {
        const uint32_t o4 = own4(s, g);
        e &= o4;
        d &= (o4 >> 7) * 0xFFu;
      }
      acc += d;
      errm[g] = e;
      anyerr |= e;
      Hprev = c.H;
      if (g < 3) c = cn;
    }
    s.first_err = NONE;
    if (anyerr) {  // cold
#pragma unroll
      for (int g = 3; g >= 0; g--)
        if (errm[g])
          s.first_err = (unsigned long long)(s.pos0 + 4 * g + (__ffs(errm[g]) - 8) / 8);
    }
    return xc ? (acc * 0x01010101u) >> 24 : 0u;
  }

  __device__ static __forceinline__ bool hint(const St &s) { return s.first_err != NONE; }
  __device__ static __forceinline__ unsigned long long find_error(const St &s, long long) {
    return s.first_err;
  }

  // a7: encode the owned words into stage[o ...] (UTF-8 bytes).  Every word stores 3 bytes at
  // its offset; bytes past its width are overwritten by the following words (program order);
  // the thread's last 4 words clip at its end slot `lim`.
  template <bool IN>
  __device__ static __forceinline__ void decode(const St &s, uint8_t *stage, uint32_t o,
                                                uint32_t lim, long long) {
    if (IN && s.wasc) {
      // a2: the warp's 512 words are ASCII, its 512 output bytes contiguous from lane 0's
      // slot; lane l narrows warp word quads l, l + 32, ... so stores cover consecutive bytes.
      const int lane = threadIdx.x & 31;
      const uint2 *wb = reinterpret_cast<const uint2 *>(s.img - BPT * lane) + lane;
      const uint32_t o0 = __shfl_sync(FULL, o, 0);
      uint8_t *sb = stage + o0 + 4 * lane;
      if ((o0 & 3u) == 0u) {  // warp-uniform
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint2 x = wb[32 * j];
          *reinterpret_cast<uint32_t *>(sb + 128 * j) = prmt(x.x, x.y, BE ? 0x7531u : 0x6420u);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint2 x = wb[32 * j];
          const uint32_t v = prmt(x.x, x.y, BE ? 0x7531u : 0x6420u);
#pragma unroll
          for (int q = 0; q < 4; q++) sb[128 * j + q] = (uint8_t)(v >> (8 * q));
        }
      }
      return;
    }
#ifdef UG_ABL_NODECODE
    {
      uint8_t *q = stage + o;
#pragma unroll
      for (int k = 0; k < 8; k++) q[k] = (uint8_t)s.w[k];
      return;
    }
#endif
    uint32_t p = smem_addr(stage + o);
    const uint32_t pend = smem_addr(stage + lim);
    uint32_t lprev = (s.prev_word & 0xFFu) << 24;
#pragma unroll
    for (int g = 0; g < 4; g++) {
      const u16::Cls4 c = u16::classes4<BE>(s.w[2 * g], s.w[2 * g + 1]);
      const uint32_t lp = fsl(lprev, c.lo, 8);
      lprev = c.lo;
      uint32_t O0, O1, O2;
      u16::encode4(c, lp, &O0, &O1, &O2);
      uint32_t d = u16::widths(c);
      if (!IN) d &= (own4(s, g) >> 7) * 0xFFu;
      const uint32_t inc = d * 0x01010101u;  // byte j: bytes emitted by words <= j
      const uint32_t a1 = p + prmt(inc, 0u, 0x4440u);
      const uint32_t a2 = p + prmt(inc, 0u, 0x4441u);
      const uint32_t a3 = p + prmt(inc, 0u, 0x4442u);
      const uint32_t A[4] = {p, a1, a2, a3};
#ifdef UG_U16_SHR_ALU
      const uint32_t B0[4] = {O0, O0 >> 8, O0 >> 16, O0 >> 24};
      const uint32_t B1[4] = {O1, O1 >> 8, O1 >> 16, O1 >> 24};
      const uint32_t B2[4] = {O2, O2 >> 8, O2 >> 16, O2 >> 24};
#else
      // byte j to the low byte on the FMA pipe (the ALU pipe is the busy one here)
      const uint32_t B0[4] = {O0, shr_fma<8>(O0), shr_fma<16>(O0), shr_fma<24>(O0)};
      const uint32_t B1[4] = {O1, shr_fma<8>(O1), shr_fma<16>(O1), shr_fma<24>(O1)};
      const uint32_t B2[4] = {O2, shr_fma<8>(O2), shr_fma<16>(O2), shr_fma<24>(O2)};
#endif
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint32_t b0 = B0[j], b1 = B1[j], b2 = B2[j];
        if (g < 3) {
          sts8o<0>(A[j], b0);
          sts8o<1>(A[j], b1);
          sts8o<2>(A[j], b2);
        } else if (IN) {
          // every word owned (width >= 1): only word 3's second and third bytes and word 2's
          // third byte can pass the thread's end
          sts8o<0>(A[j], b0);
          if (j < 3 || A[j] + 1 < pend) sts8o<1>(A[j], b1);
          if (j < 2 || A[j] + 2 < pend) sts8o<2>(A[j], b2);
        } else {
          if (A[j] < pend) sts8o<0>(A[j], b0);
          if (A[j] + 1 < pend) sts8o<1>(A[j], b1);
          if (A[j] + 2 < pend) sts8o<2>(A[j], b2);
        }
      }
      p += inc >> 24;
    }
  }

  // a7 + a9 fused (count-first kernel): encode the owned words into stage[o ...] exactly as
  // decode() does and check the pairing predicate on the same classes (computed once, one
  // group ahead for the low-surrogate look-ahead).  Returns the first error position or NONE.
  template <bool IN>
  __device__ static __forceinline__ unsigned long long decode_validate(const St &s,
                                                                       uint8_t *stage,
                                                                       uint32_t o, uint32_t lim) {
#ifdef UG_ABL_NODECODE
    decode<IN>(s, stage, o, lim, 0);  // ablation: no encode, no check
    return NONE;
#endif
    if (IN && s.wasc) {  // a2: no surrogate, one byte per word
      decode<true>(s, stage, o, lim, 0);
      return NONE;
    }
    uint32_t p = smem_addr(stage + o);
    const uint32_t pend = smem_addr(stage + lim);
    uint32_t lprev = (s.prev_word & 0xFFu) << 24;
    uint32_t Hprev = u16::is_high(s.prev_word) ? 0x80000000u : 0u;
    uint32_t errm[4];
    uint32_t anyerr = 0;
    u16::Cls4 c = u16::classes4<BE>(s.w[0], s.w[1]);
#pragma unroll
    for (int g = 0; g < 4; g++) {
      u16::Cls4 cn;
      uint32_t Lnext;
      if (g < 3) {
        cn = u16::classes4<BE>(s.w[2 * g + 2], s.w[2 * g + 3]);
        Lnext = cn.L;
      } else {
        Lnext = u16::is_low(s.next_word) ? 0x80u : 0u;
      }
      // a9: high not followed by low, low not preceded by high
      uint32_t e = (c.H & ~fsr(c.L, Lnext, 8)) | (c.L & ~fsl(Hprev, c.H, 8));
      const uint32_t lp = fsl(lprev, c.lo, 8);
      uint32_t O0, O1, O2;
      u16::encode4(c, lp, &O0, &O1, &O2);
      uint32_t d = u16::widths(c);
      if (!IN) {
        const uint32_t o4 = own4(s, g);
        e &= o4;
        d &= (o4 >> 7) * 0xFFu;
      }
      errm[g] = e;
      anyerr |= e;
      const uint32_t inc = d * 0x01010101u;  // byte j: bytes emitted by words <= j
      const uint32_t A[4] = {p, p + prmt(inc, 0u, 0x4440u), p + prmt(inc, 0u, 0x4441u),
                             p + prmt(inc, 0u, 0x4442u)};
      const uint32_t B0[4] = {O0, shr_fma<8>(O0), shr_fma<16>(O0), shr_fma<24>(O0)};
      const uint32_t B1[4] = {O1, shr_fma<8>(O1), shr_fma<16>(O1), shr_fma<24>(O1)};
      const uint32_t B2[4] = {O2, shr_fma<8>(O2), shr_fma<16>(O2), shr_fma<24>(O2)};
#pragma unroll
      for (int j = 0; j < 4; j++) {
        if (g < 3) {
          sts8o<0>(A[j], B0[j]);
          sts8o<1>(A[j], B1[j]);
          sts8o<2>(A[j], B2[j]);
        } else if (IN) {
          sts8o<0>(A[j], B0[j]);
          if (j < 3 || A[j] + 1 < pend) sts8o<1>(A[j], B1[j]);
          if (j < 2 || A[j] + 2 < pend) sts8o<2>(A[j], B2[j]);
        } else {
          if (A[j] < pend) sts8o<0>(A[j], B0[j]);
          if (A[j] + 1 < pend) sts8o<1>(A[j], B1[j]);
          if (A[j] + 2 < pend) sts8o<2>(A[j], B2[j]);
        }
      }
      p += inc >> 24;
      Hprev = c.H;
      lprev = c.lo;
      if (g < 3) c = cn;
    }
    if (!anyerr) return NONE;
    unsigned long long f = NONE;  // cold
#pragma unroll
    for (int g = 3; g >= 0; g--)
      if (errm[g]) f = (unsigned long long)(s.pos0 + 4 * g + (__ffs(errm[g]) - 8) / 8);
    return f;
  }

  // a7 for a warp whose words hold no surrogate (f1): the BMP-only encode, no pairing check
  // (nothing to check: only surrogates can be invalid), the same stores and clipping.
  template <bool IN>
  __device__ static __forceinline__ void decode_bmp(const St &s, uint8_t *stage, uint32_t o,
                                                    uint32_t lim) {
#ifdef UG_ABL_NODECODE
    decode<IN>(s, stage, o, lim, 0);
    return;
#endif
    if (IN && s.wasc) {
      decode<true>(s, stage, o, lim, 0);
      return;
    }
    uint32_t p = smem_addr(stage + o);
    const uint32_t pend = smem_addr(stage + lim);
#pragma unroll
    for (int g = 0; g < 4; g++) {
      const u16::Bmp4 c = u16::classes4_bmp<BE>(s.w[2 * g], s.w[2 * g + 1]);
      uint32_t O0, O1, O2;
      u16::encode4_bmp(c, &O0, &O1, &O2);
      uint32_t d = u16::widths_bmp(c);
      if (!IN) d &= (own4(s, g) >> 7) * 0xFFu;
      const uint32_t inc = d * 0x01010101u;
      const uint32_t A[4] = {p, p + prmt(inc, 0u, 0x4440u), p + prmt(inc, 0u, 0x4441u),
                             p + prmt(inc, 0u, 0x4442u)};
      const uint32_t B0[4] = {O0, shr_fma<8>(O0), shr_fma<16>(O0), shr_fma<24>(O0)};
      const uint32_t B1[4] = {O1, shr_fma<8>(O1), shr_fma<16>(O1), shr_fma<24>(O1)};
      const uint32_t B2[4] = {O2, shr_fma<8>(O2), shr_fma<16>(O2), shr_fma<24>(O2)};
#pragma unroll
      for (int j = 0; j < 4; j++) {
        if (g < 3) {
          sts8o<0>(A[j], B0[j]);
          sts8o<1>(A[j], B1[j]);
          sts8o<2>(A[j], B2[j]);
        } else if (IN) {
          sts8o<0>(A[j], B0[j]);
          if (j < 3 || A[j] + 1 < pend) sts8o<1>(A[j], B1[j]);
          if (j < 2 || A[j] + 2 < pend) sts8o<2>(A[j], B2[j]);
        } else {
          if (A[j] < pend) sts8o<0>(A[j], B0[j]);
          if (A[j] + 1 < pend) sts8o<1>(A[j], B1[j]);
          if (A[j] + 2 < pend) sts8o<2>(A[j], B2[j]);
        }
      }
      p += inc >> 24;
    }
  }

  template <int TB = TILE>  // the launch's tile bytes (TILE, or TILEP for the planned kernels)
  __device__ static __forceinline__ void finalize(const TileArgs &a, unsigned long long e,
                                                  bool xc, int lane, int *kind,
                                                  unsigned long long *wr) {
    const Window &win = a.win;
    *kind = u8::SURROGATE;
    *wr = 0;
    if (!xc) return;
    long long te = (2 * (long long)e + win.lead) / TB;
    unsigned long long base = te ? (ld_relaxed(a.status + te - 1) & VALMASK) : 0ull;
    long long from = (te * TB - win.lead) / 2;
    if (from < 0) from = 0;
    unsigned long long c = 0;
    for (long long i = from + lane; i < (long long)e; i += 32)
      c += u16::width(native(word_at(win, i)));
    *wr = base + warp_sum64(c);
  }
};

using U16Pol = U16PolT<false>;
using U16PolBE = U16PolT<true>;

// Last CTA to finish: outcome + counter reset.  n_units in input code units.
template <class Pol, int TB = TILE>
__device__ __forceinline__ void finish_call(const TileArgs &a, bool xc, int tid, int warp,
                                            int lane, int *s_last) {
  if (tid == 0) {
    __threadfence();
    *s_last = (atomicAdd(&a.ctr->done, 1u) == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (*s_last && warp == 0) {
    __threadfence();
    const unsigned long long e =
        *reinterpret_cast<volatile unsigned long long *>(&a.ctr->err_min);
    unsigned long long total = 0, wr = 0;
    int kind = 0;
    const unsigned long long flags =
        *reinterpret_cast<volatile unsigned long long *>(&a.ctr->flags);
    if (flags) {  // a planned call given the plan of another input: API misuse, no result
      if (lane == 0) {
        if (a.result) *a.result = ResultDev{-1, 0, 0ull, 0ull};
        if (a.rec) *a.rec = RecordDev{0ull, 0ull, 0ull, -1, 0};
        a.ctr->ticket = 0;
        a.ctr->done = 0;
        a.ctr->err_min = NONE;
        a.ctr->flags = 0;
      }
      return;
    }
    if (xc && a.ntiles) total = ld_relaxed(a.status + a.ntiles - 1) & VALMASK;
    if (e != NONE) Pol::template finalize<TB>(a, e, xc, lane, &kind, &wr);
    if (lane == 0)
      write_outcome(a, xc, kind, e, total, wr, (unsigned long long)(a.win.n / Pol::UNIT));
  }
}

// ============================================================================ validators
// K1 / K3: classify (UTF-8: flag, then exact rescan) or pair-check (UTF-16).  No inter-CTA
// dependence, so tiles go in static order (CTA c: c, c + G, ...) through a ring of VRING TMA
// slots kept VRING - 1 tiles ahead.  No CTA barrier per tile: each warp arrives on the slot's
// "empty" mbarrier when done with the image and thread 0 refills the slot once all have.  A
// warp that flags rescans its own 1 KiB (every warp's last lane checks the 3-byte look-ahead,
// so a flag never has to be resolved by another warp).
#ifndef UG_VRING
#define UG_VRING 4
#endif
constexpr int VRING = UG_VRING;
#ifndef UG_VAHEAD
#define UG_VAHEAD (UG_VRING - 2)
#endif
constexpr int VAHEAD = UG_VAHEAD;  // tiles loading ahead of the one being validated
static_assert(VAHEAD >= 1 && VAHEAD <= VRING - 1, "validator ring");
#ifndef UG_VCPS
#define UG_VCPS 3  // 38-40 registers: 3 CTAs/SM measured +3 % (UTF-8) / +6 % (UTF-16) over 2
#endif
[[maybe_unused]] constexpr int VCPS = UG_VCPS;  // validator CTAs per SM (register budget)

#ifndef UG_NO_VPRODUCER
// Validator with a dedicated producer warp (NT consumer threads + 32): the producer's lane 0
// keeps every ring slot loading as soon as the consumers release it, so no compute warp waits
// on another warp's progress before the next load is issued (round 1's thread 0 refilled the
// ring between its own tiles and waited for the slowest warp two tiles back: ~28 % of the
// UTF-8 validator's issued instructions were mbarrier polls).  CTAs per SM per direction:
// UTF-8 2 (48 registers; 3 CTAs force 32 registers and spills: +0..5 %), UTF-16 3 (32).
// Measured against the round-1 form (1 GiB c4 / c1 / c3): utf8_validate -3.4 / -4.2 / -2.8 %,
// utf16le_validate -3.8 / +6.2 / -6.4 % (c2a -6.1 %).
// Round 2 late: the UTF-8 validator's compute threads take VH chunks of 32 bytes per tile each
// (chunk h of thread tid = tile bytes [h * TILE / VH + 32 tid, ... + 32)), so the per-tile glue
// (slot wait, tile position and edge test, loop, release) is paid once per VH chunks; VH = 2:
// 256 compute threads + the producer warp, 4 CTAs per SM.  Measured against one chunk per
// thread (1 GiB / BASELINE sizes, gpurun_out/vh_ab.log): c4 -5.9 %, c3 -5.6 %, c2a / c2b
// -0.2 %, c1 +4.9 % (ASCII, at 1.0 of the copy peak either way); four chunks +1..17 %.
#ifndef UG_VHALVES
#define UG_VHALVES 2
#endif
template <class Pol>
struct VGeo {
  static constexpr int VH = Pol::UNIT == 1 ? UG_VHALVES : 1;  // chunks per thread per tile
  static constexpr int VC = NT / VH;                           // compute threads
  static constexpr int THREADS = VC + 32;
  static constexpr int MINB = Pol::UNIT == 1 ? (VH > 1 ? 4 : 2) : 3;
};
#ifndef UG_VRING8
#define UG_VRING8 3
#endif
// the UTF-8 validator's ring: 3 slots (4 CTAs per SM at 49 KiB) measured against 4 (3 CTAs) with
// two chunks per thread: c4 -2.9 %, c3 -1.2 %, c1 -0.7 %
constexpr int VRING8 = UG_VRING8;
template <class Pol>
__global__ void __launch_bounds__(VGeo<Pol>::THREADS, VGeo<Pol>::MINB) k_validate(const TileArgs a) {
  constexpr int VRING = Pol::UNIT == 1 ? VRING8 : ::ug::VRING;
  constexpr int VH = VGeo<Pol>::VH, VC = VGeo<Pol>::VC;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mb_full[VRING], mb_empty[VRING];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Window &win = a.win;
  const long long ntiles = (long long)a.ntiles;
  const long long n_units = win.n / Pol::UNIT;
  const long long G = gridDim.x;
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < VRING; j++) {
      mbar_init(&mb_full[j], 1);
      mbar_init(&mb_empty[j], VC / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == VC / 32) {  // producer
    if (lane == 0) {
      int k = 0;
      for (long long t = blockIdx.x; t < ntiles; t += G, k++) {
        const int sl = k % VRING;
        if (k >= VRING) mbar_wait(&mb_empty[sl], ((k - VRING) / VRING) & 1);
        fence_proxy_async_smem();
        issue_tile_load(win, t, smem + sl * INBUF, &mb_full[sl]);
      }
    }
  } else {
    int k = 0;
    for (long long t = blockIdx.x; t < ntiles; t += G, k++) {
      const int sl = k % VRING;
      uint8_t *buf = smem + sl * INBUF;
      mbar_wait(&mb_full[sl], (k / VRING) & 1);
      if (tile_at_edge(win, t)) {  // tile-uniform
        named_sync<BAR_DATA, VC>();
        fix_tile_edges(win, t, buf, VC);
        named_sync<BAR_DATA, VC>();
      }
      const long long tp0 = tile_pos(win, t);
      unsigned long long e = NONE;
#pragma unroll
      for (int h = 0; h < VH; h++) {
        typename Pol::St st;
        const long long tp = tp0 + (long long)h * (TILE / VH);
        uint8_t *hb = buf + h * (TILE / VH);
        if (tp >= 0 && tp + TILE / VH <= win.n) {
          Pol::template load<true>(st, hb, tid, lane, tp, win.n);
          Pol::template analyze<true>(st, tid, false);
        } else {
          Pol::template load<false>(st, hb, tid, lane, tp, win.n);
          Pol::template analyze<false>(st, tid, false);
        }
        if (__any_sync(FULL, Pol::hint(st))) {  // a4 (cold)
          const unsigned long long f = Pol::find_error(st, n_units);
          if (f < e) e = f;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mb_empty[sl]);
      if (e != NONE) atomicMin(&a.ctr->err_min, e);
    }
  }
  __syncthreads();
  finish_call<Pol>(a, false, tid, warp, lane, &s_last);
}
#else
template <class Pol>
__global__ void __launch_bounds__(NT, VCPS) k_validate(const TileArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mb_full[VRING], mb_empty[VRING];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Window &win = a.win;
  const long long ntiles = (long long)a.ntiles;
  const long long n_units = win.n / Pol::UNIT;
  const long long G = gridDim.x;

  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < VRING; j++) {
      mbar_init(&mb_full[j], 1);
      mbar_init(&mb_empty[j], NT / 32);
    }
    fence_mbar_init();
#pragma unroll
    for (int j = 0; j < VAHEAD; j++) {
      const long long t = blockIdx.x + j * G;
      if (t < ntiles) issue_tile_load(win, t, smem + j * INBUF, &mb_full[j]);
    }
  }
  __syncthreads();
  int k = 0;
  for (long long t = blockIdx.x; t < ntiles; t += G, k++) {
    const int sl = k % VRING;
    if (tid == 0) {
      // refill the slot of tile k + VAHEAD - VRING (two tiles back: every warp has long left
      // it, so thread 0 does not wait for the slowest warp of the previous tile)
      const long long tn = t + VAHEAD * G;
      const int sn = (k + VAHEAD) % VRING;
      const int kf = k + VAHEAD - VRING;
      if (tn < ntiles) {
        if (kf >= 0) mbar_wait(&mb_empty[sn], (kf / VRING) & 1);
        fence_proxy_async_smem();
        issue_tile_load(win, tn, smem + sn * INBUF, &mb_full[sn]);
      }
    }
    uint8_t *buf = smem + sl * INBUF;
    mbar_wait(&mb_full[sl], (k / VRING) & 1);
    if (tile_at_edge(win, t)) {  // tile-uniform
      named_sync<BAR_DATA, NT>();  // everyone has waited for the load
      fix_tile_edges(win, t, buf, NT);
      named_sync<BAR_DATA, NT>();
    }
    typename Pol::St st;
    const long long tp = tile_pos(win, t);
    if (tp >= 0 && tp + TILE <= win.n) {
      Pol::template load<true>(st, buf, tid, lane, tp, win.n);
      Pol::template analyze<true>(st, tid, false);
    } else {
      Pol::template load<false>(st, buf, tid, lane, tp, win.n);
      Pol::template analyze<false>(st, tid, false);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&mb_empty[sl]);  // this warp is done with the image
    if (__any_sync(FULL, Pol::hint(st))) {       // a4 (cold)
#ifdef UG_TRACE
      if (lane == 0) atomicAdd(&g_dbg[0], 1ull);
      if (lane == 0 && g_dbg[2] == 0) { g_dbg[2] = 1; g_dbg[3] = (unsigned long long)t; g_dbg[4] = warp; }
#endif
      const unsigned long long e = Pol::find_error(st, n_units);
      if (e != NONE) atomicMin(&a.ctr->err_min, e);
    }
  }
  __syncthreads();
  finish_call<Pol>(a, false, tid, warp, lane, &s_last);
}
#endif

// ---------------------------------------------------------------------------- streaming
// K1 / K3 as streaming register kernels (-DUG_VALIDATE_STREAM; measured and NOT the default:
// equal to the TMA ring on mixed text, where the classifier's ALU work binds (config 4
// utf8_validate 0.383 vs 0.381 ms per GiB), and slower where loads bind (ASCII utf8 0.217 vs
// 0.196 ms, utf16le 0.415 vs 0.336 ms): two 1 KiB chunks in flight per warp are fewer bytes in
// flight than the ring's 4 x 16 KiB TMA slots per CTA).  No inter-CTA dependence and no smem
// ring.  Each warp takes 1 KiB chunks in grid-stride order (chunk c = positions
// [c * 1024 - lead, ...), so every load is a 16-byte-aligned LDG.128 and the warp / lane
// layout is exactly the tile kernels': lane l owns 32 contiguous bytes, the classifier's
// 3-byte look-ahead runs in lane 31), with the next chunk's loads issued before the current
// chunk is classified.  The 4 bytes before / after a lane come from its neighbours by shuffle,
// lanes 0 / 31 load them.  Chunks touching the window edges take guarded byte loads (bytes
// outside the window read as 0x00, as fix_tile_edges makes them in the tile kernels).  A warp
// that flags rescans its own 1 KiB (a4) and atomicMin's the first error; the last CTA
// finalises (a10).
constexpr int VS_THREADS = 256;  // 8 warps per CTA
constexpr int VS_CHUNK = 1024;   // input bytes per warp per step
#ifndef UG_VSCPS
#define UG_VSCPS 4
#endif
constexpr int VSCPS = UG_VSCPS;  // CTAs per SM (register budget: 64 registers)

struct VChunk {
  uint4 q0, q1;
  uint32_t pv, nx;
};

// Load chunk c (warp-uniform) into this lane's registers.
__device__ __forceinline__ void vs_load(const Window &w, long long c, int lane, VChunk &v) {
  const long long p0 = c * VS_CHUNK - w.lead;  // position of the chunk's byte 0
  const long long pos = p0 + 32 * lane;
  if (p0 - 4 >= w.lo_valid && p0 + VS_CHUNK + 4 <= w.hi_valid) {  // interior (warp-uniform)
    const uint4 *g = reinterpret_cast<const uint4 *>(w.base + pos);
    v.q0 = __ldcs(g);
    v.q1 = __ldcs(g + 1);
    v.pv = lane == 0 ? __ldcs(reinterpret_cast<const uint32_t *>(w.base + pos - 4)) : 0u;
    v.nx = lane == 31 ? __ldcs(reinterpret_cast<const uint32_t *>(w.base + pos + 32)) : 0u;
  } else {  // cold: window edges, byte by byte
    uint32_t b[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      uint32_t x = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const long long q = pos + 4 * k + j;
        x |= ((q >= w.lo_valid && q < w.hi_valid) ? (uint32_t)w.base[q] : 0u) << (8 * j);
      }
      b[k] = x;
    }
    v.q0 = make_uint4(b[0], b[1], b[2], b[3]);
    v.q1 = make_uint4(b[4], b[5], b[6], b[7]);
    uint32_t pv = 0, nx = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const long long qp = pos - 4 + j, qn = pos + 32 + j;
      pv |= ((qp >= w.lo_valid && qp < w.hi_valid) ? (uint32_t)w.base[qp] : 0u) << (8 * j);
      nx |= ((qn >= w.lo_valid && qn < w.hi_valid) ? (uint32_t)w.base[qn] : 0u) << (8 * j);
    }
    v.pv = lane == 0 ? pv : 0u;
    v.nx = lane == 31 ? nx : 0u;
  }
}

template <class Pol>
__global__ void __launch_bounds__(VS_THREADS, VSCPS) k_validate_stream(const TileArgs a) {
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Window &win = a.win;
  const long long nch = (long long)a.ntiles;  // 1 KiB chunks
  const long long n_units = win.n / Pol::UNIT;
  const long long nwarps = (long long)gridDim.x * (VS_THREADS / 32);
  long long c = (long long)blockIdx.x * (VS_THREADS / 32) + warp;
  VChunk cur, nxt;
  if (c < nch) vs_load(win, c, lane, cur);
  for (; c < nch; c += nwarps) {
    if (c + nwarps < nch) vs_load(win, c + nwarps, lane, nxt);  // in flight during the check
    uint32_t pv = __shfl_up_sync(FULL, cur.q1.w, 1);
    uint32_t nx = __shfl_down_sync(FULL, cur.q0.x, 1);
    if (lane == 0) pv = cur.pv;
    if (lane == 31) nx = cur.nx;
    const long long pos = c * VS_CHUNK - win.lead + 32 * lane;  // bytes
    typename Pol::St st;
    const long long p0 = c * VS_CHUNK - win.lead;
    if (p0 >= 0 && p0 + VS_CHUNK <= win.n) {  // every position owned (warp-uniform)
      if constexpr (Pol::UNIT == 1) Pol::from_regs(st, cur.q0, cur.q1, pv, nx, pos, win.n);
      else Pol::template from_regs<true>(st, cur.q0, cur.q1, pv, nx, pos / 2, win.n / 2);
      Pol::template analyze<true>(st, tid, false);
    } else {
      if constexpr (Pol::UNIT == 1) Pol::from_regs(st, cur.q0, cur.q1, pv, nx, pos, win.n);
      else Pol::template from_regs<false>(st, cur.q0, cur.q1, pv, nx, pos / 2, win.n / 2);
      Pol::template analyze<false>(st, tid, false);
    }
    if (__any_sync(FULL, Pol::hint(st))) {  // a4 (cold)
      const unsigned long long e = Pol::find_error(st, n_units);
      if (e != NONE) atomicMin(&a.ctr->err_min, e);
    }
    cur = nxt;
  }
  __syncthreads();
  finish_call<Pol>(a, false, tid, warp, lane, &s_last);
}

// ---------------------------------------------------------------------------- K3, streaming
// utf16le_validate / utf16be_validate as a register-streaming kernel (round 2, late; the
// default, -DUG_VAL16_TMA restores the TMA-ring k_validate<U16Pol>).  The pairing rule
// ("only the possible surrogate pairs require attention") needs no tile, no
// ring and no inter-CTA order: a word i is in error iff it is a high surrogate not followed by
// a low one or a low one not preceded by a high one, so on the whole window the hot check is
//     H(i - 1) XOR L(i) == 0   for every word i in [0, n]
// (word -1 / word n: the halo word, 0 outside [lo_valid, hi_valid)), which flags a lone low at
// i and a lone high at i - 1 at position i.  A lane holds one 16-byte chunk per slot (8 words,
// two byte-lane groups of 4 split by PRMT as in u16::classes4, ~11 ops per group); the
// high-surrogate mask of word -1 comes from the lane before by one shuffle (lane 0: from lane
// 31 of the slot before, or one scalar load for the first slot).  VU chunks per lane are in
// flight (LDG.128 with the streaming hint).  A flagging warp rescans its lanes' words exactly
// with u16::err_at from global memory (cold) and atomicMin's the first error; the last CTA
// finalises as every validator does (a10).  Chunk c covers bytes [16c - lead, 16c - lead + 16)
// of the window; the chunks cover [-lead, n + 2) so the word at n (a shard's halo, else 0)
// settles a high surrogate at n - 1.
#ifndef UG_V16_THREADS
#define UG_V16_THREADS 512
#endif
#ifndef UG_V16_U
#define UG_V16_U 4
#endif
constexpr int V16_THREADS = UG_V16_THREADS;
constexpr int V16_U = UG_V16_U;  // chunks in flight per lane

__device__ __forceinline__ long long v16_nchunks(const Window &w) {
  return (w.n + 2 + w.lead + 15) / 16;
}

// Guarded 32-bit word of the window at byte position p (p even): bytes outside
// [lo_valid, hi_valid) read as 0 (cold paths and edge chunks only).
__device__ __forceinline__ uint32_t v16_rd16(const Window &w, long long p) {
  return (p >= w.lo_valid && p + 2 <= w.hi_valid)
             ? (uint32_t)*reinterpret_cast<const uint16_t *>(w.base + p)
             : 0u;
}

template <bool BE>
__global__ void __launch_bounds__(V16_THREADS) k_validate16(const TileArgs a) {
  using Pol = U16PolT<BE>;
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Window &win = a.win;
  const long long nch = v16_nchunks(win);
  const long long nw = win.n / 2;
  constexpr int GW = 32 * V16_U;  // chunks per warp round
  const long long nwarps = (long long)gridDim.x * (V16_THREADS / 32);
  constexpr uint32_t SEL_HI = BE ? 0x6420u : 0x7531u;
  for (long long g = (long long)blockIdx.x * (V16_THREADS / 32) + warp; g * GW < nch;
       g += nwarps) {
    const long long c0 = g * GW;
    uint4 v[V16_U];
    // interior round: every chunk of it inside the valid range
    const bool in = (c0 * 16 - win.lead >= win.lo_valid) &&
                    ((c0 + GW) * 16 - win.lead <= win.hi_valid);
    if (in) {
      const uint4 *gp = reinterpret_cast<const uint4 *>(win.base - win.lead) + c0 + lane;
#pragma unroll
      for (int j = 0; j < V16_U; j++) v[j] = __ldcs(gp + 32 * j);
    } else {  // cold: the window's first / last rounds, word by word with guards
#pragma unroll
      for (int j = 0; j < V16_U; j++) {
        const long long p0 = (c0 + 32 * j + lane) * 16 - win.lead;
        uint32_t q[4];
#pragma unroll
        for (int k = 0; k < 4; k++)
          q[k] = v16_rd16(win, p0 + 4 * k) | (v16_rd16(win, p0 + 4 * k + 2) << 16);
        v[j] = make_uint4(q[0], q[1], q[2], q[3]);
      }
    }
    // H of the word before the round (lane 0 of slot 0 only; 0 outside the valid range)
    uint32_t hcarry = 0;
    if (lane == 0) {
      const uint32_t u = Pol::native(v16_rd16(win, c0 * 16 - win.lead - 2));
      hcarry = u16::is_high(u) ? 0x80000000u : 0u;
    }
    uint32_t flag = 0;
#pragma unroll
    for (int j = 0; j < V16_U; j++) {
      const uint32_t his[2] = {prmt(v[j].x, v[j].y, SEL_HI), prmt(v[j].z, v[j].w, SEL_HI)};
      uint32_t H[2], L[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const uint32_t hi = his[h];
        const uint32_t z = (hi & 0xF8F8F8F8u) ^ 0xD8D8D8D8u;  // 0 iff hi in D8..DF
        const uint32_t S = ~(mad(z & 0x7F7F7F7Fu, 1u, 0x7F7F7F7Fu) | z) & HI;
        const uint32_t b2 = hi << 5;  // bit 2 of hi: DC..DF
        L[h] = S & b2;
        H[h] = S & ~b2;
      }
      // bit 31 of the word before this chunk: the lane before (lane 0: lane 31 of the slot
      // before, or the carry for slot 0)
      uint32_t hp = __shfl_up_sync(FULL, H[1], 1);
      if (lane == 0) hp = hcarry;
      hcarry = __shfl_sync(FULL, H[1], 31);  // for lane 0 of the next slot
      flag |= (fsl(hp, H[0], 8) ^ L[0]) | (fsl(H[0], H[1], 8) ^ L[1]);
    }
    if (__any_sync(FULL, flag != 0u)) {  // cold: exact rescan of this lane's flagged chunks
      unsigned long long e = NONE;
#pragma unroll 1
      for (int j = 0; j < V16_U; j++) {
        const long long p0 = (c0 + 32 * j + lane) * 16 - win.lead;  // bytes
#pragma unroll 1
        for (int k = -1; k < 8; k++) {
          const long long q = p0 / 2 + k;  // word
          if (q < 0 || q >= nw) continue;
          const uint32_t pv = Pol::native(v16_rd16(win, 2 * q - 2));
          const uint32_t u = Pol::native(v16_rd16(win, 2 * q));
          const uint32_t nx = Pol::native(v16_rd16(win, 2 * q + 2));
          if (u16::err_at(pv, u, nx)) {
            if ((unsigned long long)q < e) e = (unsigned long long)q;
            break;
          }
        }
      }
      if (e != NONE) atomicMin(&a.ctr->err_min, e);
    }
  }
  __syncthreads();
  finish_call<Pol>(a, false, tid, warp, lane, &s_last);
}

// ============================================================================ transcoders
// K2 / K4.  NT data threads + one look-back warp (warp NT/32); several CTAs per SM.
// Per tile the data warps take a ticket and bulk-load the tile (TMA), classify, block-scan,
// publish the tile aggregate and hand it to the look-back warp (named barrier BAR_C), decode
// into the stage at tile-local offsets while the look-back runs, wait for the prefix (BAR_P,
// which also orders every warp's stage writes before the copy-out) and copy the stage out.
// A ticket is taken only when its tile is about to be processed, so a tile's aggregate is
// published one load + classify after its ticket (the look-back of every later tile waits
// for it); the load latency is hidden by the other CTAs on the SM instead of by prefetching.
#ifndef UG_PF
#define UG_PF 1
#endif
constexpr int PF = UG_PF;        // tiles loading ahead of the one being classified
#ifndef UG_DEFER
#define UG_DEFER 3  // measured: 3 beats 2 (c1 -17 %), 5 ring slots still fit 2 CTAs/SM
#endif
constexpr int DEFER = UG_DEFER;  // tiles between classification and emit (awaiting the prefix)
constexpr int RING = PF + 1 + DEFER;  // input slots: PF loading, one classifying, DEFER waiting
#ifndef UG_NLB
#define UG_NLB 1
#endif
constexpr int NLB = UG_NLB;  // look-back warps per CTA (alternating tiles)
static_assert(NLB == 1 || PF == 1, "termination ticks assume one look-back agent when PF > 1");

// Decode tile j (ring slot js, prefix P, aggregate C; this thread's offset excl / count cnt)
// into the stage at the tile's global 16-byte phase, then store it: the 16-byte aligned
// interior by one TMA bulk store (thread 0), the head and tail by scalar stores.  Ends with
// the stage still being read by the bulk copy (the caller waits before the next decode).
template <class Pol>
__device__ __forceinline__ void emit_tile(const TileArgs &a, const uint8_t *img, long long t,
                                          unsigned long long P, uint32_t C, uint32_t excl,
                                          uint32_t cnt, typename Pol::Out *stage, int tid,
                                          int lane) {
  using Out = typename Pol::Out;
  constexpr uint32_t A = 16 / sizeof(Out);  // units per 16 bytes
  const Window &win = a.win;
  const long long tp = tile_pos(win, t);
  Out *out = reinterpret_cast<Out *>(a.out);
  // phase: unit index of global unit P inside its 16-byte granule
  const uint32_t ph = (uint32_t)((((uintptr_t)(out + P)) & 15u) / sizeof(Out));
  typename Pol::St st;
  if (tp >= 0 && tp + TILE <= win.n) {  // tile-uniform
    Pol::template load<true>(st, img, tid, lane, tp, win.n);
    Pol::template decode<true>(st, stage, ph + excl, ph + excl + cnt, win.n / Pol::UNIT);
  } else {
    Pol::template load<false>(st, img, tid, lane, tp, win.n);
    Pol::template decode<false>(st, stage, ph + excl, ph + excl + cnt, win.n / Pol::UNIT);
  }
  named_sync<BAR_DATA, NT>();  // the whole tile is in the stage
  unsigned long long hi = P + C;
  if (hi > a.out_cap) hi = a.out_cap;
  if (hi <= P) return;
  const uint32_t Cc = (uint32_t)(hi - P);
  const uint32_t h = ph ? A - ph : 0u;  // head units (before the first 16-byte boundary)
  if (h >= Cc) {
    if ((uint32_t)(tid - SHIPPER) < Cc) out[P + tid - SHIPPER] = stage[ph + tid - SHIPPER];
    return;
  }
  const uint32_t nb = (Cc - h) / A;  // whole 16-byte granules
  const uint32_t tl = h + nb * A;    // first tail unit
  const uint32_t sid = (uint32_t)(tid - SHIPPER);  // head / tail bytes: the shipping warp
  if (sid < h) out[P + sid] = stage[ph + sid];
  if (sid < Cc - tl) out[P + tl + sid] = stage[ph + tl + sid];
  if (tid == SHIPPER && nb) {
    fence_proxy_async_smem();  // the stage writes above (generic proxy) before the TMA read
    bulk_s2g(out + P + h, stage + ph + h, nb * 16u);
    bulk_commit();
  }
}

// K2 (and K4 in the UG_U16_TILE_SCAN build).  NT data threads + one look-back warp (warp
// NT/32); two CTAs per SM.
//  * The producer thread (lane 0 of the last data warp) takes tiles by atomic ticket (issue
//    order keeps the decoupled look-back deadlock-free) and bulk-loads them (TMA) into a ring
//    of RING input slots, one tile ahead.
//  * Tile i is classified; in-warp scans of the thread counts, and the last warp to add its
//    total publishes the tile aggregate at once (no CTA barrier; UG_FWD_BLOCK_SCAN restores
//    the block scan); the look-back warp turns the warp totals into offsets, computes the
//    exclusive prefix P from the predecessors and publishes P + C.
//  * Tile i - DEFER - whose prefix had DEFER tiles of time to arrive - is then decoded from
//    its still-resident input image straight into the stage at its global 16-byte phase and
//    shipped by one TMA bulk store.
template <class Pol>
__global__ void __launch_bounds__(NT + 32 * NLB, CTAS_PER_SM) k_transcode(const TileArgs a) {
  using Out = typename Pol::Out;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t *ring = smem;                                         // RING input tile images
  Out *stage = reinterpret_cast<Out *>(smem + RING * INBUF);   // output stage (global phase)
  __shared__ uint64_t mb_load[RING];  // tile load landed (TMA tx) / no tile (plain arrive)
  __shared__ uint64_t mb_tick[RING];  // producer -> look-back warp: ticket of slot taken
  __shared__ uint64_t mb_agg[RING];   // data warps -> look-back warp: aggregate of slot
  __shared__ uint64_t mb_pre[RING];   // look-back warp -> data warps: prefix of slot
#ifndef UG_FWD_BLOCK_SCAN  // warp-level publish (measured: forward -2 to -3 %)
  // warp totals, turned in place into exclusive warp offsets by the look-back warp
  __shared__ uint32_t s_wsum[RING][NT / 32];
  __shared__ uint32_t s_acc[RING];  // arrivals << 24 | running sum of warp totals
#else
  __shared__ uint32_t s_wsum[2][NT / 32];
#endif
  __shared__ long long s_t[RING];
  __shared__ uint32_t s_cnt[RING];
  __shared__ unsigned long long s_pre[RING];
  __shared__ int s_flag[3], s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Window &win = a.win;
  const long long ntiles = (long long)a.ntiles;
  const long long n_units = win.n / Pol::UNIT;

  // Producer: publish ticket tn for ring slot `slot` and start loading its tile.
  auto start_tile = [&](int slot, long long tn) {
    s_t[slot] = tn;
    mbar_arrive(&mb_tick[slot]);  // the look-back of tile tn can start now
    if (tn < ntiles) {
      fence_proxy_async_smem();
      issue_tile_load(win, tn, ring + slot * INBUF, &mb_load[slot]);
    } else {
      mbar_arrive(&mb_load[slot]);
    }
  };

  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < RING; j++) {
      mbar_init(&mb_load[j], 1);
      mbar_init(&mb_tick[j], 1);
#ifndef UG_FWD_BLOCK_SCAN
      mbar_init(&mb_agg[j], NT / 32);
      s_acc[j] = 0u;
#else
      mbar_init(&mb_agg[j], 1);
#endif
      mbar_init(&mb_pre[j], 1);
    }
    s_flag[0] = s_flag[1] = s_flag[2] = 0;
    fence_mbar_init();
#pragma unroll
    for (int j = 0; j < PF; j++) start_tile(j, (long long)atomicAdd(&a.ctr->ticket, 1u));
  }
  __syncthreads();

  if (warp >= NT / 32) {
    // ------------------------------------------------------------ look-back warps (a6)
    // Warp NT/32 + a handles the tiles i = a (mod NLB): a look-back is mostly waiting for
    // predecessors, so two agents keep one tile's wait from queueing behind the previous one.
    for (int i = warp - NT / 32;; i += NLB) {
      const int sl = i % RING;
      const uint32_t ph = (i / RING) & 1;
      mbar_wait(&mb_tick[sl], ph);
      const long long t = s_t[sl];
      if (t >= ntiles) break;
#ifndef UG_LB_AT_TICKET
      // start when the tile itself is classified: its predecessors were ticketed earlier and
      // are classified around the same time, so an earlier start would only poll L2 longer
      mbar_wait(&mb_agg[sl], ph);
#endif
#ifndef UG_FWD_BLOCK_SCAN
      {  // exclusive warp offsets and the tile count from the warp totals
        const uint32_t wv = lane < NT / 32 ? s_wsum[sl][lane] : 0u;
        uint32_t sc = wv;
#pragma unroll
        for (int d = 1; d < NT / 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, sc, d);
          if (lane >= d) sc += y;
        }
        if (lane < NT / 32) s_wsum[sl][lane] = sc - wv;
        if (lane == NT / 32 - 1) s_cnt[sl] = sc;
        __syncwarp();
      }
#endif
#ifdef UG_TRACE
      unsigned long long t0 = gtime();
      int rounds = 0, polls = 0;
      unsigned long long tf = 0;
      const unsigned long long P = tile_excl_prefix(a, t, lane, &rounds, &tf, &polls);
      if (lane == 0 && i < TR_IT && blockIdx.x < 1024) {
        g_trace[blockIdx.x][i][0] = t;
        g_trace[blockIdx.x][i][1] = t0;
        g_trace[blockIdx.x][i][2] = gtime();
        g_trace[blockIdx.x][i][3] = rounds;
        g_trace[blockIdx.x][i][6] = tf;
        g_trace[blockIdx.x][i][7] = polls;
      }
#else
#ifdef UG_ABL_NOLB
      const unsigned long long P = (unsigned long long)t * (TILE / 2);
#else
      const unsigned long long P = tile_excl_prefix(a, t, lane);
#endif
#endif
#ifdef UG_LB_AT_TICKET
      mbar_wait(&mb_agg[sl], ph);
#endif
      const unsigned long long incl = P + s_cnt[sl];
      if (lane == 0) {
        if (t != 0) st_relaxed(a.status + t, pack_status(a.epoch, FLAG_PREFIX, incl));
        s_pre[sl] = P;
        mbar_arrive(&mb_pre[sl]);
      }
#ifdef UG_PUSH  // push-forward: measured slower with 32-wide look-back rounds
      push_forward(a.status, a.epoch, t, ntiles, incl, lane);
#endif
    }
  } else {
    // ------------------------------------------------------------ data warps
    // this thread's offset << 8 | count of the tiles awaiting emit, newest first (a shift
    // register: constant indices keep it in registers; offset < 2^15, count <= 32)
    uint32_t hist[DEFER];
#pragma unroll
    for (int q = 0; q < DEFER; q++) hist[q] = 0u;
    int i = 0;
    auto emit = [&](int j, uint32_t v) {  // decode + store tile j (all data threads)
      const int js = j % RING;
#ifdef UG_TRACE
      unsigned long long w0 = gtime();
#endif
      mbar_wait(&mb_pre[js], (j / RING) & 1);
#ifdef UG_TRACE
      if (tid == 0 && j < TR_IT && blockIdx.x < 1024) {
        g_trace[blockIdx.x][j][4] = w0;
        g_trace[blockIdx.x][j][5] = gtime();
      }
#endif
      if (tid == SHIPPER) bulk_wait_read_all();  // the previous bulk store has read the stage
      named_sync<BAR_DATA, NT>();
#ifndef UG_FWD_BLOCK_SCAN
      emit_tile<Pol>(a, ring + js * INBUF, s_t[js], s_pre[js], s_cnt[js],
                     s_wsum[js][warp] + (v >> 8), v & 0xFFu,
#else
      emit_tile<Pol>(a, ring + js * INBUF, s_t[js], s_pre[js], s_cnt[js], v >> 8, v & 0xFFu,
#endif
                     stage, tid, lane);
    };
    while (true) {
      const int sl = i % RING;
      // The next ticket: the atomic is issued now and its result used only after this
      // thread's share of the classification, so its L2 round trip is off the critical path.
      long long tn = 0;
      if (tid == PRODUCER) tn = (long long)atomicAdd(&a.ctr->ticket, 1u);
#ifdef UG_TRACE
      const unsigned long long lw0 = gtime();
#endif
      mbar_wait(&mb_load[sl], (i / RING) & 1);
#ifdef UG_TRACE
      if (tid == 0 && i < TR_IT && blockIdx.x < 1024) {
        g_trace[blockIdx.x][i][8] = lw0;
        g_trace[blockIdx.x][i][9] = gtime();
      }
#endif
      const long long t = s_t[sl];
      if (t >= ntiles) break;
      uint8_t *img = ring + sl * INBUF;
      if (tile_at_edge(win, t)) {  // tile-uniform
        fix_tile_edges(win, t, img, NT);
        named_sync<BAR_DATA, NT>();
      }
      typename Pol::St st;
      const long long tp = tile_pos(win, t);
      uint32_t cnt;
      if (tp >= 0 && tp + TILE <= win.n) {  // tile-uniform
        Pol::template load<true>(st, img, tid, lane, tp, win.n);
        cnt = Pol::template analyze<true>(st, tid, true);
      } else {
        Pol::template load<false>(st, img, tid, lane, tp, win.n);
        cnt = Pol::template analyze<false>(st, tid, true);
      }
#ifndef UG_FWD_BLOCK_SCAN
      // in-warp scan; the warp that completes the tile's (arrivals | sum) word publishes the
      // aggregate (no CTA barrier between the classification and the publish)
      uint32_t sc = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, sc, d);
        if (lane >= d) sc += y;
      }
      const uint32_t excl = sc - cnt;  // in-warp
      if (lane == 31) {
        s_wsum[sl][warp] = sc;
        const uint32_t old = atomicAdd(&s_acc[sl], (1u << 24) | sc);
        if ((old >> 24) == NT / 32 - 1) {
          st_relaxed(a.status + t, pack_status(a.epoch, t == 0 ? FLAG_PREFIX : FLAG_AGG,
                                               (old & 0xFFFFFFu) + sc));
          s_acc[sl] = 0u;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mb_agg[sl]);
      if (tid == PRODUCER) start_tile((i + PF) % RING, tn);
      // a4 (cold): a flag is resolved inside its warp (every warp's last lane checks the
      // 3-byte look-ahead), so the warp rescans its own positions
      if (__any_sync(FULL, Pol::hint(st))) {
#else
      if (Pol::hint(st)) s_flag[i % 3] = 1;
      if (tid == PRODUCER) {
        // ring slot (i + PF) % RING held tile i - DEFER - 1, emitted last iteration
        start_tile((i + PF) % RING, tn);
        // flag slot of tile i + 1: last read after the block scan of i - 2 (every thread has
        // passed the block scan of i - 1 since), next written after the block scan of i
        s_flag[(i + 1) % 3] = 0;
      }
      uint32_t excl = 0, C = 0;
      block_scan(cnt, s_wsum[i & 1], lane, warp, &excl, &C);
      if (tid == PRODUCER) {
        // publish the tile aggregate at once (a6): successors' look-backs need it
        st_relaxed(a.status + t, pack_status(a.epoch, t == 0 ? FLAG_PREFIX : FLAG_AGG, C));
        s_cnt[sl] = C;
        mbar_arrive(&mb_agg[sl]);
      }
      if (s_flag[i % 3]) {  // a4 (cold): straight to the call's minimum
#endif
#ifdef UG_TRACE
        if (tid == 0) atomicAdd(&g_dbg[1], 1ull);
        if (Pol::hint(st) && g_dbg[5] == 0) { g_dbg[5] = 1; g_dbg[6] = (unsigned long long)t; g_dbg[7] = tid; }
#endif
        unsigned long long e = Pol::find_error(st, n_units);
        if (e != NONE) atomicMin(&a.ctr->err_min, e);
      }
#ifdef UG_TRACE
      if (tid == 0 && i < TR_IT && blockIdx.x < 1024) g_trace[blockIdx.x][i][10] = gtime();  // AGG
#endif
      const uint32_t oldest = hist[DEFER - 1];  // tile i - DEFER
#pragma unroll
      for (int q = DEFER - 1; q > 0; q--) hist[q] = hist[q - 1];
      hist[0] = (excl << 8) | cnt;
      if (i >= DEFER) emit(i - DEFER, oldest);  // a7, a8
#ifdef UG_TRACE
      if (tid == 0 && i < TR_IT && blockIdx.x < 1024) g_trace[blockIdx.x][i][11] = gtime();  // end
#endif
      i++;
    }
    // every look-back agent must see a past-the-end ticket to stop: the one owning tile i has;
    // post the same for the others (their slots are free: tiles i - 3.. were emitted)
    if (tid == PRODUCER) {
#pragma unroll
      for (int k = 1; k < NLB; k++) {
        s_t[(i + k) % RING] = ntiles;
        mbar_arrive(&mb_tick[(i + k) % RING]);
      }
    }
    // drain: tiles i - DEFER .. i - 1 (hist[DEFER - 1] is the oldest)
#pragma unroll
    for (int q = DEFER - 1; q >= 0; q--)
      if (i - 1 - q >= 0) emit(i - 1 - q, hist[q]);
    if (tid == SHIPPER) bulk_wait_all();  // all output written before the CTA retires
  }
  __syncthreads();
  finish_call<Pol>(a, true, tid, warp, lane, &s_last);
}

// ============================================================================ length-from
__device__ __forceinline__ uint32_t len8_word(uint32_t x) {
  uint32_t s1 = x << 1;
  uint32_t cont = x & ~s1 & HI;
  uint32_t f0 = x & s1 & (x << 2) & (x << 3) & HI;
  return 4u - __popc(cont) + __popc(f0);
}
__device__ __forceinline__ uint32_t len8_byte(uint32_t b) { return u8::plan_weight(b); }
// per byte lane: [non-continuation] + [>= F0], accumulated (IMAD.HI) into acc
__device__ __forceinline__ uint32_t len8_acc(uint32_t x, uint32_t acc, uint32_t *fo = nullptr) {
  const uint32_t x1 = x << 1;
  const uint32_t nk = (~x | x1) & HI;
  const uint32_t f = x & x1 & (x << 2) & (x << 3) & HI;
  if (fo) *fo |= f;
  return mad_hi(f, 1u << 25, mad_hi(nk, 1u << 25, acc));
}
__device__ __forceinline__ uint32_t lane_sum(uint32_t acc) { return (acc * 0x01010101u) >> 24; }
__device__ __forceinline__ uint32_t len16_word(uint32_t u) {
  return 1u + (u >= 0x80u ? 1u : 0u) + ((u >= 0x800u && (u & 0xF800u) != 0xD800u) ? 1u : 0u);
}

__device__ __forceinline__ void finish_reduction(unsigned long long sum, Counters *ctr,
                                                 unsigned long long *d_len) {
  __shared__ unsigned long long s_part[LNT / 32];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  sum = warp_sum64(sum);
  if (lane == 0) s_part[warp] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = 0;
    for (int i = 0; i < (int)(blockDim.x / 32); i++) b += s_part[i];
    atomicAdd(&ctr->accum, b);
    __threadfence();
    s_last = (atomicAdd(&ctr->done, 1u) == gridDim.x - 1) ? 1 : 0;
    if (s_last) {
      __threadfence();
      *d_len = *reinterpret_cast<volatile unsigned long long *>(&ctr->accum);
      ctr->accum = 0;
      ctr->done = 0;
    }
  }
}

__global__ void __launch_bounds__(LNT) k_len8(const uint8_t *in, unsigned long long n,
                                             Counters *ctr, unsigned long long *d_len) {
  const uintptr_t addr = (uintptr_t)in;
  unsigned long long head = (16u - (addr & 15u)) & 15u;
  if (head > n) head = n;
  const uint4 *body = reinterpret_cast<const uint4 *>(in + head);
  const unsigned long long nb = (n - head) / 16;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long sum = 0;
  unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nb; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; j++) v[j] = __ldcs(body + i + j * stride);
    // (POPC here: measured faster than the byte-lane IMAD.HI accumulation of k_plan8 in this
    // grid-stride loop, 1.32 vs 1.48 ms at 8 GiB)
#pragma unroll
    for (int j = 0; j < 4; j++)
      sum += len8_word(v[j].x) + len8_word(v[j].y) + len8_word(v[j].z) + len8_word(v[j].w);
  }
  for (; i < nb; i += stride) {
    uint4 v = __ldcs(body + i);
    sum += len8_word(v.x) + len8_word(v.y) + len8_word(v.z) + len8_word(v.w);
  }
  if (blockIdx.x == 0) {
    for (unsigned long long j = threadIdx.x; j < head; j += blockDim.x) sum += len8_byte(in[j]);
    for (unsigned long long j = head + nb * 16 + threadIdx.x; j < n; j += blockDim.x)
      sum += len8_byte(in[j]);
  }
  finish_reduction(sum, ctr, d_len);
}

// Four words per op (byte lanes: low / high bytes split by two PRMT, as u16::classes4): per word
// [u >= 0x80] + [u >= 0x800 and not a surrogate] (the width minus 1; a surrogate counts 2, so a
// pair counts 4), added into a byte-lane accumulator by IMAD.HI (FMA pipe; the compares use the
// ALU pipe).  Lane sums stay below 256 for up to 127 calls.
template <bool BE = false>
__device__ __forceinline__ uint32_t len16_acc4(uint32_t a, uint32_t b, uint32_t acc) {
  const uint32_t lo = prmt(a, b, BE ? 0x7531u : 0x6420u), hi = prmt(a, b, BE ? 0x6420u : 0x7531u);
  const uint32_t h7 = hi & 0x7F7F7F7Fu;
  const uint32_t ge80 = (mad(h7, 1u, 0x7F7F7F7Fu) | hi | lo) & HI;   // hi != 0 or lo >= 0x80
  const uint32_t ge800 = (mad(h7, 1u, 0x78787878u) | hi) & HI;       // hi >= 8
  const uint32_t z = (hi & 0xF8F8F8F8u) ^ 0xD8D8D8D8u;               // 0 iff hi in D8..DF
  const uint32_t S = ~(mad(z & 0x7F7F7F7Fu, 1u, 0x7F7F7F7Fu) | z) & HI;
  acc = mad_hi(ge80, 1u << 25, acc);          // + ge80 >> 7
  return mad_hi(ge800 & ~S, 1u << 25, acc);   // + (ge800 and not S) >> 7
}
// len16_acc4 that also ORs the surrogate mask into *sur (f1: a warp without surrogates takes
// the BMP-only decode)
template <bool BE = false>
__device__ __forceinline__ uint32_t len16_acc4s(uint32_t a, uint32_t b, uint32_t acc,
                                                uint32_t *sur) {
  const uint32_t lo = prmt(a, b, BE ? 0x7531u : 0x6420u), hi = prmt(a, b, BE ? 0x6420u : 0x7531u);
  const uint32_t h7 = hi & 0x7F7F7F7Fu;
  const uint32_t ge80 = (mad(h7, 1u, 0x7F7F7F7Fu) | hi | lo) & HI;
  const uint32_t ge800 = (mad(h7, 1u, 0x78787878u) | hi) & HI;
  const uint32_t z = (hi & 0xF8F8F8F8u) ^ 0xD8D8D8D8u;
  const uint32_t S = ~(mad(z & 0x7F7F7F7Fu, 1u, 0x7F7F7F7Fu) | z) & HI;
  *sur |= S;
  acc = mad_hi(ge80, 1u << 25, acc);
  return mad_hi(ge800 & ~S, 1u << 25, acc);
}

template <bool BE>
__global__ void __launch_bounds__(LNT) k_len16(const uint16_t *in, unsigned long long n,
                                              Counters *ctr, unsigned long long *d_len) {
  const uintptr_t addr = (uintptr_t)in;
  unsigned long long head = ((16u - (addr & 15u)) & 15u) / 2;
  if (head > n) head = n;
  const uint4 *body = reinterpret_cast<const uint4 *>(in + head);
  const unsigned long long nb = (n - head) / 8;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long sum = 0;
  auto quad = [](const uint4 &v) {  // 8 words
    return 8u + lane_sum(len16_acc4<BE>(v.z, v.w, len16_acc4<BE>(v.x, v.y, 0u)));
  };
  auto word = [](uint32_t w) { return BE ? (((w >> 8) | (w << 8)) & 0xFFFFu) : w; };
  unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nb; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; j++) v[j] = __ldcs(body + i + j * stride);
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 4; j++)
      acc = len16_acc4<BE>(v[j].z, v[j].w, len16_acc4<BE>(v[j].x, v[j].y, acc));
    sum += 32u + lane_sum(acc);
  }
  for (; i < nb; i += stride) sum += quad(__ldcs(body + i));
  if (blockIdx.x == 0) {
    for (unsigned long long j = threadIdx.x; j < head; j += blockDim.x)
      sum += len16_word(word(in[j]));
    for (unsigned long long j = head + nb * 8 + threadIdx.x; j < n; j += blockDim.x)
      sum += len16_word(word(in[j]));
  }
  finish_reduction(sum, ctr, d_len);
}

#ifdef UG_PREFIX_EXPT
__device__ unsigned long long g_pref[1 << 20];
__device__ int g_pmode;
extern "C" cudaError_t ug_pmode_set_impl(int m) {
  return cudaMemcpyToSymbol(g_pmode, &m, sizeof(m));
}
#endif
// ============================================================================ count-first K4
// UTF-16LE -> UTF-8 with validation moved off the look-back's critical path.  A word's UTF-8
// width depends on the word alone (u16::wm1: 1 + [u >= 0x80] + [u >= 0x800, not a surrogate]),
// so a tile's output count - and every thread's offset inside it - is a plain width sum, exact
// on ANY input: validity decides only the error report, never an offset.  So per tile:
//  * data warps: count only (byte-lane width sums, 4 words per op), an in-warp scan, and the
//    warp total added to a shared 64-bit (arrivals | sum) word; the warp that completes it
//    publishes the tile aggregate at once.  No CTA barrier between the load and the publish.
//  * look-back warp: exclusive prefix (a6) in ticket order, per-warp offsets.
//  * data warps, D16 tiles later: decode + pairing check in one pass (classes computed once,
//    a7 + a9), stage, TMA bulk store (a8).
// Against k_transcode<U16Pol> (classify + block scan before the publish) this shortens the
// ticket -> aggregate latency that every successor's look-back waits on.
#ifndef UG_RING16
#define UG_RING16 5  // measured best: 5 slots, one load ahead, emit deferred 3 tiles
#endif
constexpr int RING16 = UG_RING16;
#ifndef UG_PF16
#define UG_PF16 1
#endif
constexpr int PF16 = UG_PF16;  // tiles loading ahead of the one being counted
constexpr int D16 = RING16 - PF16 - 1;  // tiles awaiting their prefix (emit deferral)
static_assert(3 * (TILE / 2) < (1 << 24) && NT / 32 < 256, "s_acc packing");
static_assert(PF16 >= 1 && D16 >= 1, "ring: loads in flight + the tile counted + deferral");
#ifndef UG_NLB16
#define UG_NLB16 1
#endif
// look-back agents (warps) of K4, alternating tiles.  One is best: two were measured 7 % (c4)
// to 21 % (ASCII) slower although the no-look-back ablation is 12 % faster on c4 - the chain
// costs latency against the 3-tile emit slack, not agent throughput.
constexpr int NLB16 = UG_NLB16;
constexpr int T16_THREADS = NT + 32 * NLB16;
static_assert(NLB16 == 1 || PF16 == 1, "termination ticks assume one tile loading ahead");
static_assert(NLB16 <= RING16 - D16, "termination ticks use slots of emitted tiles");

template <bool BE>
__device__ __forceinline__ void emit_tile16(const TileArgs &a, const uint8_t *img, long long t,
                                            unsigned long long P, uint32_t C, uint32_t excl,
                                            uint32_t cnt, uint8_t *stage, int tid, int lane) {
  constexpr uint32_t A = 16;
  const Window &win = a.win;
  const long long tp = tile_pos(win, t);
  uint8_t *out = reinterpret_cast<uint8_t *>(a.out);
  const uint32_t ph = (uint32_t)(((uintptr_t)(out + P)) & 15u);
  using P16 = U16PolT<BE>;
  typename P16::St st;
  unsigned long long f;
  if (tp >= 0 && tp + TILE <= win.n) {  // tile-uniform
    P16::template load<true>(st, img, tid, lane, tp, win.n);
    f = P16::template decode_validate<true>(st, stage, ph + excl, ph + excl + cnt);
  } else {
    P16::template load<false>(st, img, tid, lane, tp, win.n);
    f = P16::template decode_validate<false>(st, stage, ph + excl, ph + excl + cnt);
  }
  if (f != NONE) atomicMin(&a.ctr->err_min, f);  // a4 (cold)
  named_sync<BAR_DATA, NT>();  // the whole tile is in the stage
  unsigned long long hi = P + C;
  if (hi > a.out_cap) hi = a.out_cap;
  if (hi <= P) return;
  const uint32_t Cc = (uint32_t)(hi - P);
  const uint32_t h = ph ? A - ph : 0u;
  if (h >= Cc) {
    if ((uint32_t)(tid - SHIPPER) < Cc) out[P + tid - SHIPPER] = stage[ph + tid - SHIPPER];
    return;
  }
  const uint32_t nb = (Cc - h) / A;
  const uint32_t tl = h + nb * A;
  const uint32_t sid = (uint32_t)(tid - SHIPPER);  // head / tail bytes: the shipping warp
  if (sid < h) out[P + sid] = stage[ph + sid];
  if (sid < Cc - tl) out[P + tl + sid] = stage[ph + tl + sid];
  if (tid == SHIPPER && nb) {
    fence_proxy_async_smem();
    bulk_s2g(out + P + h, stage + ph + h, nb * 16u);
    bulk_commit();
  }
}

template <bool BE>
__global__ void __launch_bounds__(T16_THREADS, CTAS_PER_SM) k_transcode16(const TileArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t *ring = smem;
  uint8_t *stage = smem + RING16 * INBUF;
  __shared__ uint64_t mb_load[RING16];  // tile landed (TMA tx) / no tile
  __shared__ uint64_t mb_tick[RING16];  // producer -> look-back warp: ticket of the slot
  __shared__ uint64_t mb_agg[RING16];   // data warps (one arrival each) -> look-back warp
  __shared__ uint64_t mb_pre[RING16];   // look-back warp -> data warps: prefix known
  __shared__ long long s_t[RING16];
  __shared__ uint32_t s_wsum[RING16][NT / 32];  // warp totals, then exclusive warp offsets
  // arrivals << 24 | running sum of warp totals (a tile emits <= 3 * TILE / 2 < 2^24 bytes):
  // one native 32-bit shared atomic (a 64-bit one is a CAS loop, ATOMS.CAST.SPIN.64)
  __shared__ uint32_t s_acc[RING16];
  __shared__ uint32_t s_cnt[RING16];
  __shared__ unsigned long long s_pre[RING16];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Window &win = a.win;
  const long long ntiles = (long long)a.ntiles;

  auto start_tile = [&](int slot, long long tn) {  // producer (thread 0 in the prologue)
    s_t[slot] = tn;
    mbar_arrive(&mb_tick[slot]);
    if (tn < ntiles) {
      fence_proxy_async_smem();
      issue_tile_load(win, tn, ring + slot * INBUF, &mb_load[slot]);
    } else {
      mbar_arrive(&mb_load[slot]);
    }
  };
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < RING16; j++) {
      mbar_init(&mb_load[j], 1);
      mbar_init(&mb_tick[j], 1);
      mbar_init(&mb_agg[j], NT / 32);
      mbar_init(&mb_pre[j], 1);
      s_acc[j] = 0u;
    }
    fence_mbar_init();
#pragma unroll 1
    for (int j = 0; j < PF16; j++) start_tile(j, (long long)atomicAdd(&a.ctr->ticket, 1u));
  }
  __syncthreads();

  if (warp >= NT / 32) {
    // ------------------------------------------------------------ look-back warps (a6)
    // agent a = warp - NT/32 takes the tiles k = a (mod NLB16), in ticket order
#pragma unroll 1
    for (int k = warp - NT / 32;; k += NLB16) {
      const int sl = k % RING16;
      const uint32_t ph = (k / RING16) & 1;
      mbar_wait(&mb_tick[sl], ph);
      const long long t = s_t[sl];
      if (t >= ntiles) break;
      mbar_wait(&mb_agg[sl], ph);
      // tile aggregate from the 16 warp totals; exclusive warp offsets back into s_wsum
      const uint32_t wv = lane < NT / 32 ? s_wsum[sl][lane] : 0u;
      uint32_t sc = wv;
#pragma unroll
      for (int d = 1; d < NT / 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, sc, d);
        if (lane >= d) sc += y;
      }
      const uint32_t C = __shfl_sync(FULL, sc, NT / 32 - 1);  // (published by the last warp)
      if (lane < NT / 32) s_wsum[sl][lane] = sc - wv;
#ifdef UG_ABL_NOLB
      const unsigned long long P = (unsigned long long)t * (3 * TILE / 2);  // ablation: no chain
#elif defined(UG_PREFIX_EXPT)
      // experiment: mode 1 records every tile's true prefix, mode 2 replays them without the
      // look-back (same output placement as a real run, no chain)
      unsigned long long P;
      if (g_pmode == 2 && t < (1 << 20)) {
        P = g_pref[t];
      } else {
        P = tile_excl_prefix(a, t, lane);
        if (g_pmode == 1 && lane == 0 && t < (1 << 20)) g_pref[t] = P;
      }
#else
      const unsigned long long P = tile_excl_prefix(a, t, lane);
#endif
      const unsigned long long incl = P + C;
      __syncwarp();
      if (lane == 0) {
        if (t != 0) st_relaxed(a.status + t, pack_status(a.epoch, FLAG_PREFIX, incl));
        s_cnt[sl] = C;
        s_pre[sl] = P;
        mbar_arrive(&mb_pre[sl]);  // release: offsets, count, prefix
      }
#ifdef UG_PUSH  // push-forward: measured slower with 32-wide look-back rounds
      push_forward(a.status, a.epoch, t, ntiles, incl, lane);
#endif
    }
  } else {
    // ------------------------------------------------------------ data warps
    // this thread's in-warp offset << 8 | count of the tiles awaiting emit, newest first (a
    // shift register: constant indices keep it in registers)
    uint32_t hist[D16];
#pragma unroll
    for (int j = 0; j < D16; j++) hist[j] = 0u;
    auto emit = [&](int j, uint32_t v) {
      const int js = j % RING16;
      mbar_wait(&mb_pre[js], (j / RING16) & 1);
      if (tid == SHIPPER) bulk_wait_read_all();  // the previous bulk store has read the stage
      named_sync<BAR_DATA, NT>();
      emit_tile16<BE>(a, ring + js * INBUF, s_t[js], s_pre[js], s_cnt[js],
                  s_wsum[js][warp] + (v >> 8), v & 0xFFu, stage, tid, lane);
    };
    int i = 0;
#pragma unroll 1
    while (true) {
      const int sl = i % RING16;
      long long tn = 0;
      if (tid == PRODUCER) tn = (long long)atomicAdd(&a.ctr->ticket, 1u);
      mbar_wait(&mb_load[sl], (i / RING16) & 1);
      const long long t = s_t[sl];
      if (t >= ntiles) break;
      uint8_t *img = ring + sl * INBUF;
      if (tile_at_edge(win, t)) {  // tile-uniform
        fix_tile_edges(win, t, img, NT);
        named_sync<BAR_DATA, NT>();
      }
      // a5: this thread's output bytes (width sum of its 16 words; owned words only)
      const long long tp = tile_pos(win, t);
      const uint4 *my = reinterpret_cast<const uint4 *>(img + HALO + BPT * tid);
      const uint4 q0 = my[0], q1 = my[1];
      uint32_t cnt;
      if (tp >= 0 && tp + TILE <= win.n) {
        // a2: an all-ASCII warp emits one byte per word (skip the width arithmetic)
        const uint32_t orv = q0.x | q0.y | q0.z | q0.w | q1.x | q1.y | q1.z | q1.w;
        if (__all_sync(FULL, (orv & (BE ? 0x80FF80FFu : 0xFF80FF80u)) == 0u))
          cnt = 16u;
        else
          cnt = 16u + lane_sum(len16_acc4<BE>(q1.z, q1.w, len16_acc4<BE>(q1.x, q1.y,
                               len16_acc4<BE>(q0.z, q0.w, len16_acc4<BE>(q0.x, q0.y, 0u)))));
      } else {
        const uint32_t q[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        const long long w0 = (tp + BPT * tid) / 2, nw = win.n / 2;
        cnt = 0;
#pragma unroll
        for (int k = 0; k < 16; k++)
          if (w0 + k >= 0 && w0 + k < nw) cnt += len16_word(U16PolT<BE>::native((q[k >> 1] >> (16 * (k & 1))) & 0xFFFFu));
      }
      uint32_t sc = cnt;  // in-warp inclusive scan
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, sc, d);
        if (lane >= d) sc += y;
      }
      if (lane == 31) {
        s_wsum[sl][warp] = sc;
        // the last warp to add its total publishes the tile aggregate at once (a6): the
        // look-back warp may still be busy with the previous tile, and every successor's
        // look-back waits for this word
        const uint32_t old = atomicAdd(&s_acc[sl], (1u << 24) | sc);
        if ((old >> 24) == NT / 32 - 1) {
          st_relaxed(a.status + t, pack_status(a.epoch, t == 0 ? FLAG_PREFIX : FLAG_AGG,
                                               (old & 0xFFFFFFu) + sc));
          s_acc[sl] = 0u;  // next use of the slot is RING16 tiles later
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mb_agg[sl]);
      const uint32_t oldest = hist[D16 - 1];  // tile i - D16
#pragma unroll
      for (int q = D16 - 1; q > 0; q--) hist[q] = hist[q - 1];
      hist[0] = ((sc - cnt) << 8) | cnt;  // count <= 48, offset < 2^11
      // slot of tile i + PF16 held tile i + PF16 - RING16 = i - D - 1, emitted last iteration
      if (tid == PRODUCER) start_tile((i + PF16) % RING16, tn);
      if (i >= D16) emit(i - D16, oldest);  // a7-a9, a8
      i++;
    }
    // every look-back agent must see a past-the-end ticket to stop: the one owning tile i has;
    // post the same for the others (slots of tiles i + 1 .., held tiles emitted long ago)
    if (tid == PRODUCER) {
#pragma unroll
      for (int k = 1; k < NLB16; k++) {
        s_t[(i + k) % RING16] = ntiles;
        mbar_arrive(&mb_tick[(i + k) % RING16]);
      }
    }
    // drain: tiles i - D16 .. i - 1 (hist[D16 - 1] is the oldest)
#pragma unroll
    for (int q = D16 - 1; q >= 0; q--)
      if (i - 1 - q >= 0) emit(i - 1 - q, hist[q]);
    if (tid == SHIPPER) bulk_wait_all();
  }
  __syncthreads();
  finish_call<U16PolT<BE>>(a, true, tid, warp, lane, &s_last);
}

// ============================================================================ planned (two-pass)
// Reduce-then-scan form of the transcoders.  The sizing
// pass a caller runs anyway (the length-from reduction that sizes the output buffer) also
// writes a PLAN: the output count of each of 2R contiguous sub-ranges of tiles under the
// transcoder's own emission rule (R = the transcoder's grid).  The planned transcoder then
// gives CTA c the tiles of sub-ranges 2c and 2c + 1 in order: its first output offset is the
// sum of the earlier sub-ranges' counts, and inside its range every tile's offset is the
// running sum of the tiles it has already processed.  No decoupled look-back, no tickets, no
// look-back warp, no emit deferral: a tile is counted (classify + validate), its thread
// offsets are block-scanned and it is decoded and shipped the next iteration, the loads run
// ahead in static order.  One CTA barrier per tile: the decode of tile t and the count of tile
// t + 1 are issued between the same two barriers, and the output stage is double-buffered.
//
// Plan buffer (device, 8-byte words): [0] tag, [1] input address, [2] n (input bytes),
// [3] sub-ranges, [4] tiles per sub-range, [5] total under the emission rule, [6] lead,
// [7] halos (before << 32 | after, bytes), [8 + j] output offset (exclusive prefix of the
// counts) of sub-range j.
constexpr int PLAN_MAX_SUB = 8192;
static_assert(PLAN_WORDS == PLAN_HDR + PLAN_MAX_SUB, "plan layout (internal.h PLAN_WORDS)");
constexpr unsigned long long PLAN_TAG = 0x554750414E563031ull;

struct PlanArgs {
  Window win;                // the same window the transcoder will see
  unsigned long long ntiles;
  int nsub;
  unsigned long long tps;    // tiles per sub-range
  unsigned long long *plan;
  Counters *ctr;
  unsigned long long *d_len;  // the length-from result (optional)
};

// Positions [p0, p1) of sub-range j (clipped to the owned range [0, n)), in bytes.
__device__ __forceinline__ void sub_span(const PlanArgs &a, long long j, long long *p0,
                                         long long *p1) {
  const long long t0 = j * (long long)a.tps, t1 = t0 + (long long)a.tps;
  long long q0 = t0 * TILEP - a.win.lead, q1 = t1 * TILEP - a.win.lead;
  if (q0 < 0) q0 = 0;
  if (q1 > a.win.n) q1 = a.win.n;
  if (t0 >= (long long)a.ntiles) q0 = q1 = a.win.n;
  *p0 = q0;
  *p1 = q1 > q0 ? q1 : q0;
}

// The halos of a window (bytes before / after the owned range that are readable context): part
// of the plan's identity, since the UTF-8 emit rule at the first positions reads them.
__device__ __forceinline__ unsigned long long plan_halos(const Window &w) {
  return ((unsigned long long)(-w.lo_valid) << 32) | (unsigned long long)(w.hi_valid - w.n);
}

__device__ __forceinline__ void plan_finish(const PlanArgs &a, unsigned long long emit_sum,
                                            unsigned long long len_sum,
                                            unsigned long long f_sum = 0,
                                            unsigned long long a_sum = 1) {  // 1: not known ASCII
  __shared__ unsigned long long s_e[LNT / 32], s_l[LNT / 32];
  __shared__ int s_last, s_f;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_f = 0;
  emit_sum = warp_sum64(emit_sum);
  len_sum = warp_sum64(len_sum);
  const bool f_any = __any_sync(FULL, f_sum != 0), a_any = __any_sync(FULL, a_sum != 0);
  __syncthreads();
  if (lane == 0) {
    s_e[warp] = emit_sum;
    s_l[warp] = len_sum;
    if (f_any) atomicOr(&s_f, 1);
    if (a_any) atomicOr(&s_f, 2);
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long e = 0, l = 0;
    for (int i = 0; i < LNT / 32; i++) {
      e += s_e[i];
      l += s_l[i];
    }
    st_relaxed(reinterpret_cast<uint64_t *>(a.plan + PLAN_HDR + blockIdx.x), e);
    atomicAdd(&a.ctr->accum, l);
    // flags, not counts (bit 0: a >= F0 byte; bit 1: a byte >= 0x80, or not known to be
    // ASCII): one atomic per CTA that adds a bit not yet set
    const unsigned long long fl = (unsigned long long)s_f;
    if (fl & ~*reinterpret_cast<volatile unsigned long long *>(&a.ctr->accf))
      atomicOr(&a.ctr->accf, fl);
    __threadfence();
    s_last = (atomicAdd(&a.ctr->done, 1u) == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (!s_last) return;
  // last CTA: the sub-range counts become exclusive prefixes (in place), then the header
  __threadfence();
  const int ns = a.nsub, per = (ns + LNT - 1) / LNT;
  const int j0 = tid * per, j1 = j0 + per < ns ? j0 + per : ns;
  unsigned long long mine = 0;
  for (int j = j0; j < j1; j++) mine += ld_relaxed(reinterpret_cast<uint64_t *>(a.plan + PLAN_HDR + j));
  unsigned long long sc = mine;  // inclusive scan over the 512 threads
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long y = __shfl_up_sync(FULL, sc, d);
    if (lane >= d) sc += y;
  }
  if (lane == 31) s_e[warp] = sc;
  __syncthreads();
  unsigned long long wpre = 0, total = 0;
  for (int i = 0; i < LNT / 32; i++) {
    if (i < warp) wpre += s_e[i];
    total += s_e[i];
  }
  unsigned long long run = wpre + sc - mine;
  for (int j = j0; j < j1; j++) {
    const unsigned long long c = ld_relaxed(reinterpret_cast<uint64_t *>(a.plan + PLAN_HDR + j));
    a.plan[PLAN_HDR + j] = run;
    run += c;
  }
  if (tid == 0) {
    const unsigned long long L = *reinterpret_cast<volatile unsigned long long *>(&a.ctr->accum);
    a.plan[0] = PLAN_TAG;
    a.plan[1] = (unsigned long long)(uintptr_t)a.win.base;
    a.plan[2] = (unsigned long long)a.win.n;
    a.plan[3] = (unsigned long long)a.nsub;
    a.plan[4] = a.tps;
    a.plan[5] = total;
    a.plan[6] = (unsigned long long)a.win.lead;
    a.plan[7] = plan_halos(a.win);
    // nonzero iff the window (with the halo before it) holds a >= F0 byte (UTF-8 plans; f1)
    const unsigned long long fl = *reinterpret_cast<volatile unsigned long long *>(&a.ctr->accf);
    a.plan[8] = fl & 1u;
    // 0 iff no owned byte is >= 0x80 (UTF-8 plans: the all-ASCII widening copy's; UTF-16: 1)
    a.plan[9] = (fl >> 1) & 1u;
    if (a.d_len) *a.d_len = L;
    a.ctr->accum = 0;
    a.ctr->accf = 0;
    a.ctr->done = 0;
  }
}

// UTF-16 -> UTF-8 plan: per sub-range the width sum (u16::widths rule, = utf8 length on valid
// input), which is also the transcoder's count; total = utf8_length_from_utf16le.  Read-only,
// grid = nsub CTAs, 16-byte loads over the aligned interior, 4 in flight per thread.
template <bool BE>
__global__ void __launch_bounds__(LNT) k_plan16(const PlanArgs a) {
  long long p0, p1;
  sub_span(a, blockIdx.x, &p0, &p1);  // bytes, even
  const uint8_t *base = a.win.base;
  unsigned long long sum = 0;
  // aligned interior [h0, h1) of 16-byte vectors; scalar words before / after
  long long h0 = p0, h1 = p1;
  while (h0 < p1 && (((uintptr_t)(base + h0)) & 15u)) h0 += 2;
  h1 = h0 + ((p1 - h0) & ~15ll);
  if (h1 < h0) h1 = h0;
  const uint4 *v = reinterpret_cast<const uint4 *>(base + h0);
  const long long nv = (h1 - h0) / 16;
  long long i = threadIdx.x;
  for (; i + 3 * LNT < nv; i += 4 * LNT) {
    uint4 q[4];
#pragma unroll
    for (int j = 0; j < 4; j++) q[j] = __ldcs(v + i + j * LNT);
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 4; j++)
      acc = len16_acc4<BE>(q[j].z, q[j].w, len16_acc4<BE>(q[j].x, q[j].y, acc));
    sum += 32u + lane_sum(acc);
  }
  for (; i < nv; i += LNT) {
    const uint4 q = __ldcs(v + i);
    sum += 8u + lane_sum(len16_acc4<BE>(q.z, q.w, len16_acc4<BE>(q.x, q.y, 0u)));
  }
  const uint16_t *w16 = reinterpret_cast<const uint16_t *>(base);
  for (long long b = p0 + 2 * threadIdx.x; b < h0; b += 2 * LNT) {
    const uint32_t u = w16[b / 2];
    sum += len16_word(BE ? (((u >> 8) | (u << 8)) & 0xFFFFu) : u);
  }
  for (long long b = h1 + 2 * threadIdx.x; b < p1; b += 2 * LNT) {
    const uint32_t u = w16[b / 2];
    sum += len16_word(BE ? (((u >> 8) | (u << 8)) & 0xFFFFu) : u);
  }
  plan_finish(a, sum, sum);
}

// UTF-8 -> UTF-16 plan: per sub-range the number of EMITTING positions (the transcoder's end-
// position rule: ASCII, or the end of a 2- / 3-byte character, or the 3rd / 4th byte after an
// F lead - exactly analyze32's emit mask, also on invalid input); the length total is the
// utf16_length_from_utf8 formula (R15).  Byte-SWAR over 4 positions per word with
// the word before (from the window: halo bytes of a shard, 0x00 before the start).
__device__ __forceinline__ uint32_t word_before(const Window &w, long long pos) {
  if (pos - 4 >= w.lo_valid && pos <= w.hi_valid && !(((uintptr_t)(w.base + pos)) & 3u))
    return *reinterpret_cast<const uint32_t *>(w.base + pos - 4);
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < 4; j++) x |= byte_at(w, pos - 4 + j) << (8 * j);
  return x;
}
// msb-per-byte masks of one word: >= C0 (L), >= E0 (E), >= F0 (F)
struct Lef {
  uint32_t L2, E, F;  // C0..DF, >= E0, >= F0
};
__device__ __forceinline__ Lef lef_of(uint32_t x) {
  const uint32_t L = x & (x << 1) & HI, E = L & (x << 2);
  return Lef{L & ~E, E, E & (x << 3)};
}
// emit count (end-position rule) and R15 length of word x after word p (masks mp of p)
__device__ __forceinline__ void plan8_word(const Lef &mp, uint32_t x, const Lef &mx, uint32_t own,
                                           uint32_t *em_acc, uint32_t *len_acc) {
  const uint32_t em = ((~x & HI) | fsl(mp.L2, mx.L2, 8) | fsl(mp.E, mx.E, 16) |
                       fsl(mp.F, mx.F, 24)) & own;
  *em_acc = mad_hi(em, 1u << 25, *em_acc);                      // + em >> 7 per byte
  const uint32_t nk = (~x | (x << 1)) & HI & own;                // not a continuation byte
  *len_acc = mad_hi(mx.F & own, 1u << 25, mad_hi(nk, 1u << 25, *len_acc));
}
__device__ __forceinline__ unsigned long long bsum(uint32_t acc) {
  return (acc & 0xFFu) + ((acc >> 8) & 0xFFu) + ((acc >> 16) & 0xFFu) + (acc >> 24);
}

#if !defined(UG_PLAN8_SWAR) && !defined(UG_PLAN8_PLANES)
// UTF-8 plan as the length-from reduction plus boundary terms.  Summed over positions, the end-
// position rule's terms (ASCII at i, 2-byte lead at i-1, >= E0 at i-2, >= F0 at i-3: R16) weigh
// each byte by [non-continuation] + [>= F0] -- the R15 length formula -- but credit a lead's
// units to the positions where they are emitted, up to 3 bytes later.  So the emit-term sum of
// [a, b) = formula[a, b) + pending(a) - pending(b), pending(q) = the units leads in the 3
// bytes before q emit at q or later.  On a prefix free of errors the terms never coincide and
// this is the transcoder's exact emit count; past an error the sum can only exceed it (a sum of
// the terms >= their OR), so a later range's offset never falls below the units written before
// the error, and the range holding the error starts at its exact offset.
__device__ __forceinline__ long long plan8_pending(const Window &w, long long q) {
  return (long long)u8::pending3(byte_at(w, q - 1), byte_at(w, q - 2), byte_at(w, q - 3));
}

__global__ void __launch_bounds__(LNT) k_plan8(const PlanArgs a) {
  long long p0, p1;
  sub_span(a, blockIdx.x, &p0, &p1);
  const Window &w = a.win;
  const uint8_t *base = w.base;
  unsigned long long sum = 0;
  long long h0 = p0;
  while (h0 < p1 && (((uintptr_t)(base + h0)) & 15u)) h0++;
  long long h1 = h0 + ((p1 - h0) & ~15ll);
  if (h1 < h0) h1 = h0;
  const uint4 *v = reinterpret_cast<const uint4 *>(base + h0);
  const long long nv = (h1 - h0) / 16;
  long long i = threadIdx.x;
  uint32_t fo = 0;  // >= F0 bytes seen (OR of their msb masks: only "any" matters per lane)
  uint32_t ao = 0;  // OR of every owned byte (bit 7: a byte >= 0x80)
  unsigned long long fsum = 0;
  for (; i + 3 * LNT < nv; i += 4 * LNT) {
    uint4 q[4];
#pragma unroll
    for (int j = 0; j < 4; j++) q[j] = __ldcs(v + i + j * LNT);
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      acc = len8_acc(q[j].w, len8_acc(q[j].z, len8_acc(q[j].y, len8_acc(q[j].x, acc, &fo), &fo),
                                      &fo), &fo);
      ao |= q[j].x | q[j].y | q[j].z | q[j].w;
    }
    sum += lane_sum(acc);
  }
  for (; i < nv; i += LNT) {
    const uint4 q = __ldcs(v + i);
    sum += lane_sum(len8_acc(q.w, len8_acc(q.z, len8_acc(q.y, len8_acc(q.x, 0u, &fo), &fo), &fo),
                             &fo));
    ao |= q.x | q.y | q.z | q.w;
  }
  for (long long b = p0 + threadIdx.x; b < h0; b += LNT) {
    sum += len8_byte(base[b]);
    fsum += base[b] >= 0xF0u;
    ao |= base[b];
  }
  for (long long b = h1 + threadIdx.x; b < p1; b += LNT) {
    sum += len8_byte(base[b]);
    fsum += base[b] >= 0xF0u;
    ao |= base[b];
  }
  fsum += fo != 0u;
  // the window's halo bytes before position 0 count too (a 4-byte character begun there)
  if (p0 == 0 && threadIdx.x == 0)
    for (int d = 1; d <= 3; d++) fsum += byte_at(w, -d) >= 0xF0u;
  // boundary terms (thread 0; modular: a range's count may be "negative", prefixes are not)
  const unsigned long long emit = threadIdx.x == 0
      ? sum + (unsigned long long)(plan8_pending(w, p0) - plan8_pending(w, p1))
      : sum;
  plan_finish(a, emit, sum, fsum, (ao & HI) != 0u);
}
#elif defined(UG_PLAN8_PLANES)
// UTF-8 plan on bit planes (the classifier's transposition, u8::planes32): a lane's 32 bytes ->
// 8 planes, then the emit mask of analyze32 (ASCII | end of a 2- / 3-byte character | 3rd /
// 4th byte after an F lead) and the R15 terms (non-continuation, >= F0) are 32 positions per op.
__device__ __forceinline__ void plan8_chunk32(const uint32_t w[8], uint32_t prev, uint32_t own,
                                              uint32_t *em, uint32_t *len) {
  uint32_t P[8];
  u8::planes32(w, P);
  const uint32_t L = P[7] & P[6], E = L & P[5], F = E & P[4];
  const uint32_t pL = u8::lead_c0(prev), pE = pL & (prev << 2), pF = pE & (prev << 3);
  const uint32_t cL = u8::carry3(pL), cE = u8::carry3(pE), cF = u8::carry3(pF);
  const uint32_t emit = ~P[7] | fsl(cL & ~cE, L & ~E, 1) | fsl(cE, E, 2) | fsl(cF, F, 3);
  *em = popc(emit & own);
  *len = popc(~(P[7] & ~P[6]) & own) + popc(F & own);  // non-continuation + >= F0
}

__global__ void __launch_bounds__(LNT) k_plan8(const PlanArgs a) {
  long long p0, p1;
  sub_span(a, blockIdx.x, &p0, &p1);
  const Window &w = a.win;
  const uint8_t *base = w.base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long esum = 0, lsum = 0;
  long long h0 = p0;
  while (h0 < p1 && (((uintptr_t)(base + h0)) & 15u)) h0++;
  long long h1 = h0 + ((p1 - h0) & ~15ll);
  if (h1 < h0) h1 = h0;
  // 1 KiB warp chunks of [h0, h1): lane l owns its 32 bytes; the 4 bytes before come from lane
  // l - 1 (lane 0: one load, the window's bytes at the start)
  const long long nb = h1 - h0;
  const long long nch = (nb + 1023) / 1024;
  constexpr int CU = 3;  // chunks per warp step (their loads in flight together)
  for (long long c0 = warp; c0 < nch; c0 += (LNT / 32) * CU) {
    uint32_t x[CU][8], own[CU];
#pragma unroll
    for (int u = 0; u < CU; u++) {
      const long long q = h0 + (c0 + (long long)u * (LNT / 32)) * 1024 + 32 * lane;
      uint4 a0 = make_uint4(0, 0, 0, 0), a1 = a0;
      if (q + 32 <= h1) {
        a0 = __ldcs(reinterpret_cast<const uint4 *>(base + q));
        a1 = __ldcs(reinterpret_cast<const uint4 *>(base + q + 16));
      } else {  // the partial last chunk (or none): vectors up to h1, zeros after
        if (q < h1) a0 = __ldcs(reinterpret_cast<const uint4 *>(base + q));
        if (q + 16 < h1) a1 = __ldcs(reinterpret_cast<const uint4 *>(base + q + 16));
      }
      x[u][0] = a0.x; x[u][1] = a0.y; x[u][2] = a0.z; x[u][3] = a0.w;
      x[u][4] = a1.x; x[u][5] = a1.y; x[u][6] = a1.z; x[u][7] = a1.w;
      const long long k = h1 - q;
      own[u] = k <= 0 ? 0u : (k >= 32 ? 0xFFFFFFFFu : ((1u << k) - 1u));
    }
#pragma unroll
    for (int u = 0; u < CU; u++) {
      const long long q = h0 + (c0 + (long long)u * (LNT / 32)) * 1024 + 32 * lane;
      uint32_t prev = __shfl_up_sync(FULL, x[u][7], 1);
      if (lane == 0) prev = q < h1 ? word_before(w, q) : 0u;
      uint32_t em, ln;
      plan8_chunk32(x[u], prev, own[u], &em, &ln);
      esum += em;
      lsum += ln;
    }
  }
  // the unaligned head / tail bytes, one word at a time with ownership masks
  for (long long b = p0 + 4 * threadIdx.x; b < h0; b += 4 * LNT) {
    uint32_t x = 0, own = 0;
    for (int j = 0; j < 4; j++) {
      x |= byte_at(w, b + j) << (8 * j);
      if (b + j < h0) own |= 0xFFu << (8 * j);
    }
    uint32_t ea = 0, la = 0;
    plan8_word(lef_of(word_before(w, b)), x, lef_of(x), own, &ea, &la);
    esum += bsum(ea);
    lsum += bsum(la);
  }
  for (long long b = h1 + 4 * threadIdx.x; b < p1; b += 4 * LNT) {
    uint32_t x = 0, own = 0;
    for (int j = 0; j < 4; j++) {
      x |= byte_at(w, b + j) << (8 * j);
      if (b + j < p1) own |= 0xFFu << (8 * j);
    }
    uint32_t ea = 0, la = 0;
    plan8_word(lef_of(word_before(w, b)), x, lef_of(x), own, &ea, &la);
    esum += bsum(ea);
    lsum += bsum(la);
  }
  plan_finish(a, esum, lsum);
}
#else
__global__ void __launch_bounds__(LNT) k_plan8(const PlanArgs a) {
  long long p0, p1;
  sub_span(a, blockIdx.x, &p0, &p1);
  const Window &w = a.win;
  const uint8_t *base = w.base;
  const int lane = threadIdx.x & 31;
  unsigned long long esum = 0, lsum = 0;
  long long h0 = p0;
  while (h0 < p1 && (((uintptr_t)(base + h0)) & 15u)) h0++;
  long long h1 = h0 + ((p1 - h0) & ~15ll);
  if (h1 < h0) h1 = h0;
  const uint4 *v = reinterpret_cast<const uint4 *>(base + h0);
  const long long nv = (h1 - h0) / 16;
  // a warp takes 32 consecutive vectors per step (lane l: vector l), UNR steps in flight; the
  // word before a lane's vector is the previous lane's last word (lane 0: one extra load).
  // Full steps run without bounds checks; the remainder vector by vector.
#ifndef UG_PLAN_UNR
#define UG_PLAN_UNR 4
#endif
  constexpr int UNR = UG_PLAN_UNR;
  const uint32_t nvu = (uint32_t)nv;  // < 2^31 vectors per sub-range
  const uint32_t lanev = (uint32_t)lane;
  // the word before vector 0 (may lie outside the window); every later one is an aligned load
  const uint32_t pre0 = word_before(w, h0);
  const uint32_t *v32 = reinterpret_cast<const uint32_t *>(v);
  uint32_t g = (threadIdx.x >> 5) * 32u * UNR;
  for (; g + 32u * UNR <= nvu; g += (uint32_t)LNT * UNR) {
    uint4 q[UNR];
    uint32_t pw[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) q[u] = __ldcs(v + g + 32u * u + lanev);
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const uint32_t vi = g + 32u * u;
      pw[u] = (lane == 0 && vi != 0u) ? __ldg(v32 + 4u * vi - 1u) : pre0;
    }
    uint32_t ea = 0, la = 0;
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      uint32_t prev = __shfl_up_sync(FULL, q[u].w, 1);
      if (lane == 0) prev = pw[u];
      const Lef m0 = lef_of(prev), m1 = lef_of(q[u].x), m2 = lef_of(q[u].y), m3 = lef_of(q[u].z),
                m4 = lef_of(q[u].w);
      plan8_word(m0, q[u].x, m1, 0xFFFFFFFFu, &ea, &la);
      plan8_word(m1, q[u].y, m2, 0xFFFFFFFFu, &ea, &la);
      plan8_word(m2, q[u].z, m3, 0xFFFFFFFFu, &ea, &la);
      plan8_word(m3, q[u].w, m4, 0xFFFFFFFFu, &ea, &la);
    }
    esum += bsum(ea);  // per-byte sums <= 4 x UNR x 2 < 256
    lsum += bsum(la);
  }
  for (uint32_t i = g + lanev; i < nvu; i += 32u) {  // this warp's last, partial step
    if (i >= g + 32u * UNR) break;
    const uint4 q = __ldcs(v + i);
    const Lef m0 = lef_of(word_before(w, h0 + 16ll * i)), m1 = lef_of(q.x), m2 = lef_of(q.y),
              m3 = lef_of(q.z), m4 = lef_of(q.w);
    uint32_t ea = 0, la = 0;
    plan8_word(m0, q.x, m1, 0xFFFFFFFFu, &ea, &la);
    plan8_word(m1, q.y, m2, 0xFFFFFFFFu, &ea, &la);
    plan8_word(m2, q.z, m3, 0xFFFFFFFFu, &ea, &la);
    plan8_word(m3, q.w, m4, 0xFFFFFFFFu, &ea, &la);
    esum += bsum(ea);
    lsum += bsum(la);
  }
  // the unaligned head / tail bytes, one word at a time with ownership masks
  for (long long b = p0 + 4 * threadIdx.x; b < h0; b += 4 * LNT) {
    uint32_t x = 0, own = 0;
    for (int j = 0; j < 4; j++) {
      x |= byte_at(w, b + j) << (8 * j);
      if (b + j < h0) own |= 0xFFu << (8 * j);
    }
    uint32_t ea = 0, la = 0;
    plan8_word(lef_of(word_before(w, b)), x, lef_of(x), own, &ea, &la);
    esum += bsum(ea);
    lsum += bsum(la);
  }
  for (long long b = h1 + 4 * threadIdx.x; b < p1; b += 4 * LNT) {
    uint32_t x = 0, own = 0;
    for (int j = 0; j < 4; j++) {
      x |= byte_at(w, b + j) << (8 * j);
      if (b + j < p1) own |= 0xFFu << (8 * j);
    }
    uint32_t ea = 0, la = 0;
    plan8_word(lef_of(word_before(w, b)), x, lef_of(x), own, &ea, &la);
    esum += bsum(ea);
    lsum += bsum(la);
  }
  plan_finish(a, esum, lsum);
}

#endif  // UG_PLAN8_SWAR

// The planned transcoder (both directions; Pol = U8PolT / U16PolT).
#ifndef UG_PRING8
#define UG_PRING8 2
#endif
#ifndef UG_PRING16
#define UG_PRING16 3
#endif
#ifndef UG_PMINB16
#define UG_PMINB16 CPSP
#endif
template <class Pol>
struct PlannedGeo {
  static constexpr int RING = Pol::UNIT == 1 ? UG_PRING8 : UG_PRING16;  // input slots
  static constexpr int MINB = Pol::UNIT == 1 ? CPSP : UG_PMINB16;        // launch bounds
  static constexpr int INBUFP = TILEP + 2 * HALO;                         // one input slot
  // an output stage: a tile's worst-case output (1 unit per byte / 3 bytes per word) + phase
  static constexpr int STAGE = Pol::UNIT == 1 ? 2 * (TILEP + 32) : 3 * (TILEP / 2) + 64;
  static constexpr size_t SMEM = (size_t)RING * INBUFP + 2 * (size_t)STAGE;
};

// Count first (the next tile's count before this tile's decode) or decode first: measured per
// direction (UTF-16 input: count first -9 %; UTF-8 input: decode first, count first +15 %).
template <class Pol>
struct PlannedOrder {
#ifndef UG_PORDER_FLIP
  static constexpr bool COUNT_FIRST = Pol::UNIT == 2;
#else
  static constexpr bool COUNT_FIRST = Pol::UNIT == 1;
#endif
};

template <class Pol, bool NOF = false>
__global__ void __launch_bounds__(NTP, PlannedGeo<Pol>::MINB)
    k_transcode_planned(const TileArgs a, const unsigned long long *plan) {
  using Out = typename Pol::Out;
  using G = PlannedGeo<Pol>;
  constexpr int PR = G::RING;
  constexpr int INBUFP = G::INBUFP;
  constexpr int STAGEP = G::STAGE;
  constexpr int PRODUCERP = NTP - 32;  // lane 0 of the last warp
  constexpr uint32_t AU = 16 / sizeof(Out);  // output units per 16 bytes
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t *ring = smem;
  uint8_t *stage_base = smem + PR * INBUFP;  // two output stages of STAGEP bytes
  __shared__ uint64_t mb_load[PR];
  __shared__ long long s_tile[PR];             // tile in each slot, -1 = no more tiles
  __shared__ unsigned long long s_base[PR];    // a sub-range's first tile: its output offset
  __shared__ uint32_t s_wsum[2][NTP / 32];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Window &win = a.win;
  const long long ntiles = (long long)a.ntiles;
  const long long n_units = win.n / Pol::UNIT;
  Out *out = reinterpret_cast<Out *>(a.out);

#ifndef UG_NO_PDL
  // the kernels launched after this one in the planned call (the other forward form, the
  // all-ASCII copies) only read the plan, written before this kernel: let them launch now
  // (programmatic dependent launch).  UTF-8 input: as the first instruction, so a form that
  // returns at once does not delay the next; UTF-16 input: after the exit test below (measured:
  // the narrowing copy of an ASCII window runs best launched once this kernel has returned)
  if constexpr (Pol::UNIT == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  // the plan must describe this very input (else: UG_ERR_ARG from finish, no work)
  const bool bad = plan[0] != PLAN_TAG || plan[1] != (unsigned long long)(uintptr_t)win.base ||
                   plan[2] != (unsigned long long)win.n ||
                   plan[6] != (unsigned long long)win.lead || plan[7] != plan_halos(win);
  // f1 for UTF-8: the forward is launched twice, with and without the no-F decode; the plan
  // (header word 8: the input's >= F0 bytes) picks the one that runs, the other returns here
  if constexpr (Pol::kNoF) {
    if ((!bad && plan[8] == 0) != NOF) return;
#ifndef UG_NO_WIDEN8
    if (NOF && !bad && plan[9] == 0) return;  // all ASCII: k_widen8's (launched after this one)
#endif
  }
#ifndef UG_NO_NARROW16
  // a window of ASCII words only is k_narrow16's (launched after this kernel)
  if constexpr (Pol::UNIT == 2) {
    if (!bad && plan[5] == (unsigned long long)(win.n / 2)) return;
  }
#endif
  const long long nsub = bad ? 0 : (long long)plan[3], tps = bad ? 1 : (long long)plan[4];
#ifndef UG_NO_PDL
  if constexpr (Pol::UNIT == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  if (bad && tid == 0 && blockIdx.x == 0) atomicOr(&a.ctr->flags, 1ull);
  // producer (lane 0 of the last warp, not the shipping warp 0): tiles in sub-range order,
  // sub-ranges by ticket; the next ticket is drawn as a sub-range starts, so its L2 round trip
  // is off the critical path
  long long cur_t = 0, cur_end = 0, next_j = 0;
  auto produce = [&](int slot) {
    long long t = -1;
    unsigned long long b = NONE;
    if (cur_t < cur_end) {
      t = cur_t++;
    } else {
      const long long j = next_j;
      if (j < nsub) {
        next_j = (long long)atomicAdd(&a.ctr->ticket, 1u);
        t = j * tps;
        cur_end = t + tps < ntiles ? t + tps : ntiles;
        cur_t = t + 1;
        b = plan[PLAN_HDR + j];
      }
    }
    s_tile[slot] = t;
    s_base[slot] = b;
    if (t >= 0) {
      fence_proxy_async_smem();
      issue_tile_load<TILEP>(win, t, ring + slot * INBUFP, &mb_load[slot]);
    } else {
      mbar_arrive(&mb_load[slot]);
    }
  };
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < PR; j++) mbar_init(&mb_load[j], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == PRODUCERP) {
    next_j = (long long)atomicAdd(&a.ctr->ticket, 1u);
    for (int j = 0; j < PR; j++) produce(j);
  }

  // count tile t (slot k % PR): classify / validate (errors to the call's minimum), the
  // thread's count, its in-warp exclusive offset; the warp total goes to s_wsum[k & 1].
  // PHALVES chunks per thread (chunk h = bytes [h * HALFP, (h + 1) * HALFP) of the tile): the
  // counts are packed 16 bits per chunk (bits 16h.., at most 12288 per tile) so ONE scan and
  // one barrier serve them all; bit 31 - h of *wexcl set = this warp's chunk h holds no
  // surrogate (UTF-16, f1)
  auto count_tile = [&](long long t, int k, uint32_t *cnt, uint32_t *wexcl, long long *tpo) {
    uint32_t nosurr = 0;
    uint8_t *img = ring + (k % PR) * INBUFP;
    // UTF-16 input: no second wait (the caller's slot_tile has waited for this slot's load) and
    // the tile position computed once per tile (c4 -0.8 %, c1 -2.6 %); the UTF-8 kernel keeps
    // the old form (+1.1 % with it)
    bool edge;
    if constexpr (Pol::UNIT == 2) {
      const long long e0 = tile_pos<TILEP>(win, t) - HALO;
      edge = !(e0 >= win.lo_valid && e0 + TILEP + 2 * HALO <= win.hi_valid);
    } else {
      mbar_wait(&mb_load[k % PR], (k / PR) & 1);
      edge = tile_at_edge<TILEP>(win, t);
    }
    if (edge) {  // tile-uniform
      named_sync<BAR_DATA, NTP>();
      fix_tile_edges<TILEP>(win, t, img, NTP);
      named_sync<BAR_DATA, NTP>();
    }
    const long long tp0 = tile_pos<TILEP>(win, t);
    *tpo = tp0;
    uint32_t cp = 0;
    int asc = 0;  // chunks in which this warp is all ASCII (warp-uniform)
#pragma unroll
    for (int h = 0; h < PHALVES; h++) {
      const long long tp = tp0 + (long long)h * HALFP;
      uint8_t *im = img + h * HALFP;
      uint32_t c;
      if constexpr (Pol::UNIT == 2) {
        // UTF-16: the count is the width sum alone (exact on any input); the pairing check is
        // done with the decode (decode_validate), as in the count-first k_transcode16
        constexpr bool BE = Pol::kBE;
        const uint4 *my = reinterpret_cast<const uint4 *>(im + HALO + BPT * tid);
        const uint4 q0 = my[0], q1 = my[1];
#ifdef UG_ABL_NOVAL
        if (true) {  // ablation: one byte per word, no width sum
          c = 16u;
          asc += 1;
        } else
#endif
        if (tp >= 0 && tp + HALFP <= win.n) {
          const uint32_t orv = q0.x | q0.y | q0.z | q0.w | q1.x | q1.y | q1.z | q1.w;
          if (__all_sync(FULL, (orv & (BE ? 0x80FF80FFu : 0xFF80FF80u)) == 0u)) {
            c = 16u;
            asc += 1;
          } else {
            uint32_t sur = 0;
            c = 16u + lane_sum(len16_acc4s<BE>(q1.z, q1.w, len16_acc4s<BE>(q1.x, q1.y,
                               len16_acc4s<BE>(q0.z, q0.w, len16_acc4s<BE>(q0.x, q0.y, 0u, &sur),
                               &sur), &sur), &sur));
#ifndef UG_NO_F1
            if (!__any_sync(FULL, sur != 0u)) nosurr |= 0x80000000u >> h;
#endif
          }
        } else {
          const uint32_t q[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
          const long long w0 = (tp + BPT * tid) / 2, nw = win.n / 2;
          c = 0;
#pragma unroll
          for (int k2 = 0; k2 < 16; k2++)
            if (w0 + k2 >= 0 && w0 + k2 < nw)
              c += len16_word(Pol::native((q[k2 >> 1] >> (16 * (k2 & 1))) & 0xFFFFu));
        }
      } else {
        typename Pol::St st;
        if (tp >= 0 && tp + HALFP <= win.n) {
          Pol::template load<true>(st, im, tid, lane, tp, win.n);
          c = Pol::template analyze<true>(st, tid, true);
        } else {
          Pol::template load<false>(st, im, tid, lane, tp, win.n);
          c = Pol::template analyze<false>(st, tid, true);
        }
        if (__any_sync(FULL, Pol::hint(st))) {  // a4 (cold)
          const unsigned long long e = Pol::find_error(st, n_units);
          if (e != NONE) atomicMin(&a.ctr->err_min, e);
        }
      }
      cp |= c << (16 * h);
    }
    uint32_t sc = cp;
#ifndef UG_NO_ASCII_SCAN
    // (UTF-16 input: config 1 -7.5 %, mixed text +0.5 %; the UTF-8 kernel: -1.7 % / +0.5 %, not
    // taken)
    if (Pol::UNIT == 2 && asc == PHALVES) {  // every lane's count is the same: closed form
      sc = cp * (uint32_t)(lane + 1);
    } else
#endif
    {
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, sc, d);
        if (lane >= d) sc += y;
      }
    }
    if (lane == 31) s_wsum[k & 1][warp] = sc;
    *cnt = cp;
    *wexcl = (sc - cp) | nosurr;
  };
  // after the barrier: this warp's offset inside the tile and the tile total (packed as the
  // counts)
  auto tile_offsets = [&](int k, uint32_t *woff, uint32_t *total) {
    const uint32_t v = lane < NTP / 32 ? s_wsum[k & 1][lane] : 0u;
    // two REDUX instead of the shuffle scan (forward -1 %; the UTF-16 kernel at 256 threads x 4
    // CTAs: c4 -0.1 %, c1 -4.2 %, c2a -2.0 %, c3 -1.1 %; at 512 x 2 it had been +1.4 %)
#ifndef UG_REDUX16
#define UG_REDUX16 1
#endif
    if constexpr (Pol::UNIT == 1 || UG_REDUX16) {
      *woff = __reduce_add_sync(FULL, lane < warp ? v : 0u);
      *total = __reduce_add_sync(FULL, v);
      return;
    }
    uint32_t sc = v;
#pragma unroll
    for (int d = 1; d < NTP / 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, sc, d);
      if (lane >= d) sc += y;
    }
    *woff = __shfl_sync(FULL, sc - v, warp);
    *total = __shfl_sync(FULL, sc, NTP / 32 - 1);
  };

  // the tile of the k-th iteration (after its load has landed) and its sub-range base
  auto slot_tile = [&](int k, unsigned long long *b) {
    mbar_wait(&mb_load[k % PR], (k / PR) & 1);
    *b = s_base[k % PR];
    return s_tile[k % PR];
  };

  constexpr uint32_t FIELD = PHALVES == 1 ? 0x7FFFFFFFu : 0x3FFFu;  // one chunk's packed count
  uint32_t cnt = 0, wex = 0, woff = 0, C = 0;
  unsigned long long running = 0, base_t;
  long long tpt = 0;  // tile_pos of tile t
  long long t = slot_tile(0, &base_t);
  if (t >= 0) count_tile(t, 0, &cnt, &wex, &tpt);
  named_sync<BAR_DATA, NTP>();
  if (t >= 0) tile_offsets(0, &woff, &C);
  for (int k = 0; t >= 0; k++) {
    const unsigned long long P = base_t != NONE ? base_t : running;
    Out *stage = reinterpret_cast<Out *>(stage_base + (k & 1) * STAGEP);
    const uint32_t ph = (uint32_t)((((uintptr_t)(out + P)) & 15u) / sizeof(Out));
    uint32_t cnt2 = 0, wex2 = 0;
    unsigned long long base2 = NONE;
    long long t2 = -1, tp2 = 0;
    if constexpr (PlannedOrder<Pol>::COUNT_FIRST) {
      t2 = slot_tile(k + 1, &base2);
      if (t2 >= 0) count_tile(t2, k + 1, &cnt2, &wex2, &tp2);
    }
    // decode tile t at its global 16-byte phase (its input image is still in slot k % PR);
    // chunk h's units follow those of chunks < h
#pragma unroll
    for (int h = 0; h < PHALVES; h++) {
      uint8_t *img = ring + (k % PR) * INBUFP + h * HALFP;
      typename Pol::St st;
      const long long tp =
          (Pol::UNIT == 2 ? tpt : tile_pos<TILEP>(win, t)) + (long long)h * HALFP;
      const uint32_t before = h == 0 ? 0u : (C & 0xFFFFu);  // (PHALVES <= 2)
      const uint32_t wo = PHALVES == 1 ? woff : ((woff >> (16 * h)) & 0xFFFFu);
      const uint32_t o = ph + before + wo + ((wex >> (16 * h)) & FIELD);
      const uint32_t ch = PHALVES == 1 ? cnt : ((cnt >> (16 * h)) & 0xFFFFu);
      if constexpr (Pol::UNIT == 2) {  // encode + pairing check in one pass
        unsigned long long f = NONE;
        if (tp >= 0 && tp + HALFP <= win.n) {
          Pol::template load<true>(st, img, tid, lane, tp, win.n);
          if ((wex << h) >> 31)  // warp-uniform (f1)
            Pol::template decode_bmp<true>(st, stage, o, o + ch);
          else
            f = Pol::template decode_validate<true>(st, stage, o, o + ch);
        } else {
          Pol::template load<false>(st, img, tid, lane, tp, win.n);
          f = Pol::template decode_validate<false>(st, stage, o, o + ch);
        }
        if (f != NONE) atomicMin(&a.ctr->err_min, f);  // a4 (cold)
      } else {
        if (tp >= 0 && tp + HALFP <= win.n) {
          Pol::template load<true>(st, img, tid, lane, tp, win.n);
          if constexpr (NOF)  // (f1, UTF-8: the input holds no >= F0 byte)
            Pol::template decode<true, true>(st, stage, o, o + ch, n_units);
          else
            Pol::template decode<true>(st, stage, o, o + ch, n_units);
        } else {
          Pol::template load<false>(st, img, tid, lane, tp, win.n);
          Pol::template decode<false>(st, stage, o, o + ch, n_units);
        }
      }
    }
    if constexpr (!PlannedOrder<Pol>::COUNT_FIRST) {
      t2 = slot_tile(k + 1, &base2);
      if (t2 >= 0) count_tile(t2, k + 1, &cnt2, &wex2, &tp2);
    }
    if (tid == SHIPPER) bulk_wait_read_all();  // the store of the previous tile has read its stage
    named_sync<BAR_DATA, NTP>();  // stage k & 1 complete; warp totals of the next tile published
    // ship tile t: 16-byte aligned interior by one TMA bulk store, head / tail by the warp
    // (head and tail are < 16 bytes: only the shipping warp has anything to do; skipping the
    // rest measured forward -2..-3 %, but +4..+7 % in the UTF-16 kernel, which keeps them)
    const uint32_t Ct = PHALVES == 1 ? C : (C & 0xFFFFu) + (C >> 16);  // the tile's units
#ifndef UG_SHIP_ALL16  // head / tail by the shipping warp only: c4 +3.7 % (c1 -6.5 %): kept
#define UG_SHIP_ALL16 1
#endif
    if ((UG_SHIP_ALL16 && Pol::UNIT == 2) || warp == UG_SHIP_WARP) {
      unsigned long long hi = P + Ct;
      if (hi > a.out_cap) hi = a.out_cap;
      if (hi > P) {
        const uint32_t Cc = (uint32_t)(hi - P);
        const uint32_t h = ph ? AU - ph : 0u;
        const uint32_t sid = (uint32_t)(tid - SHIPPER);
        if (h >= Cc) {
          if (sid < Cc) out[P + sid] = stage[ph + sid];
        } else {
          const uint32_t nb = (Cc - h) / AU;
          const uint32_t tl = h + nb * AU;
          if (sid < h) out[P + sid] = stage[ph + sid];
          if (sid < Cc - tl) out[P + tl + sid] = stage[ph + tl + sid];
          if (tid == SHIPPER && nb) {
            fence_proxy_async_smem();
            bulk_s2g(out + P + h, stage + ph + h, nb * 16u);
            bulk_commit();
          }
        }
      }
    }
    // the inclusive prefix of tile t for the finaliser (kind / written at the first error)
    if (tid == 0) st_relaxed(a.status + t, pack_status(a.epoch, FLAG_PREFIX, P + Ct));
    // slot k % PR is free: the producer refills it
    if (tid == PRODUCERP) produce(k % PR);
    running = P + Ct;
    t = t2;
    base_t = base2;
    if (t >= 0) {
      tile_offsets(k + 1, &woff, &C);
      cnt = cnt2;
      wex = wex2;
      tpt = tp2;
    }
  }
  if (tid == SHIPPER) bulk_wait_all();
  __syncthreads();
  finish_call<Pol, TILEP>(a, true, tid, warp, lane, &s_last);
}


// a2 for a whole window of ASCII words (planned UTF-16 -> UTF-8, round 2 late; -DUG_NO_NARROW16
// builds without).  The plan's total (header word 5, the width sum of the owned words) equals
// the word count iff every word is below 0x80 (every width is >= 1): such a window has no
// error and its output is the low byte of every word, so it needs
// neither tiles nor offsets: a grid-stride narrowing copy, 8 output bytes per item (one
// LDG.128 of 8 words -> two PRMT -> one 8-byte store when the input is 16-byte aligned at the
// output's 8-byte phase, 2-byte loads otherwise), four items per thread in flight, head / tail
// bytes by block 0.  The result / record is written up front (it does not depend on the
// data); the planned kernel launched with it returns at once on the same test.
constexpr int N16_THREADS = 512;
template <bool BE>
__global__ void __launch_bounds__(N16_THREADS, 4) k_narrow16(const TileArgs a,
                                                          const unsigned long long *plan) {
  const Window &win = a.win;
  const long long nw = win.n / 2;
  const bool bad = plan[0] != PLAN_TAG || plan[1] != (unsigned long long)(uintptr_t)win.base ||
                   plan[2] != (unsigned long long)win.n ||
                   plan[6] != (unsigned long long)win.lead || plan[7] != plan_halos(win);
  if (bad || plan[5] != (unsigned long long)nw) return;
  const unsigned long long total = (unsigned long long)nw;
  const unsigned long long m = total < a.out_cap ? total : a.out_cap;  // bytes written
  const int tid = threadIdx.x;
  if (blockIdx.x == 0 && tid == 0) write_outcome(a, true, 0, NONE, total, 0, total);
  constexpr uint32_t SEL = BE ? 0x7531u : 0x6420u;
  constexpr int LB = BE ? 1 : 0;  // the low byte's offset in a stored word
  const uint8_t *in = win.base;
  uint8_t *out = reinterpret_cast<uint8_t *>(a.out);
  unsigned long long h = (8u - ((uintptr_t)out & 7u)) & 7u;  // out + h is 8-byte aligned
  if (h > m) h = m;
  const unsigned long long nb = (m - h) / 8, tl = h + 8 * nb;
  const bool fast = (((uintptr_t)(in + 2 * h)) & 15u) == 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * N16_THREADS;
  unsigned long long i = (unsigned long long)blockIdx.x * N16_THREADS + tid;
  if (fast) {
    const uint4 *src = reinterpret_cast<const uint4 *>(in + 2 * h);
    uint2 *dst = reinterpret_cast<uint2 *>(out + h);
    for (; i + 3 * stride < nb; i += 4 * stride) {
      uint4 q[4];
#pragma unroll
      for (int j = 0; j < 4; j++) q[j] = __ldcs(src + i + j * stride);
#pragma unroll
      for (int j = 0; j < 4; j++)
        __stcs(dst + i + j * stride, make_uint2(prmt(q[j].x, q[j].y, SEL), prmt(q[j].z, q[j].w, SEL)));
    }
    for (; i < nb; i += stride) {
      const uint4 q = __ldcs(src + i);
      __stcs(dst + i, make_uint2(prmt(q.x, q.y, SEL), prmt(q.z, q.w, SEL)));
    }
  } else {  // (unaligned phases: correctness, not speed)
    for (; i < nb; i += stride) {
      const uint8_t *s = in + 2 * (h + 8 * i) + LB;
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        lo |= (uint32_t)s[2 * j] << (8 * j);
        hi |= (uint32_t)s[8 + 2 * j] << (8 * j);
      }
      *reinterpret_cast<uint2 *>(out + h + 8 * i) = make_uint2(lo, hi);
    }
  }
  if (blockIdx.x == 0) {
    if ((unsigned long long)tid < h) out[tid] = in[2 * tid + LB];
    if ((unsigned long long)tid < m - tl) out[tl + tid] = in[2 * (tl + tid) + LB];
  }
}


// a2 for a whole window of ASCII bytes (planned UTF-8 -> UTF-16, round 2 late; -DUG_NO_WIDEN8
// builds without): the UTF-8 plan's header word 9 is 0 iff no owned byte is >= 0x80; such a
// window is valid (every byte a 1-byte character) and its output is each byte
// zero-extended.  As k_narrow16: the result written up front, a grid-stride
// widening copy (one 8-byte load -> four PRMT -> one 16-byte store when the input is 8-byte
// aligned at the output's 16-byte phase, byte loads otherwise), head / tail by block 0; the
// third kernel of the forward's planned launch (programmatic dependent launch, like the pair).
template <bool BE>
__global__ void __launch_bounds__(N16_THREADS, 4) k_widen8(const TileArgs a,
                                                         const unsigned long long *plan) {
  const Window &win = a.win;
  const long long n = win.n;
  const bool bad = plan[0] != PLAN_TAG || plan[1] != (unsigned long long)(uintptr_t)win.base ||
                   plan[2] != (unsigned long long)win.n ||
                   plan[6] != (unsigned long long)win.lead || plan[7] != plan_halos(win);
  if (bad || plan[9] != 0 || n <= 0) return;
  const unsigned long long total = (unsigned long long)n;
  const unsigned long long m = total < a.out_cap ? total : a.out_cap;  // units written
  const int tid = threadIdx.x;
  if (blockIdx.x == 0 && tid == 0) write_outcome(a, true, 0, NONE, total, 0, total);
  constexpr uint32_t S0 = BE ? 0x1404u : 0x4140u, S1 = BE ? 0x3424u : 0x4342u;
  const uint8_t *in = win.base;
  uint16_t *out = reinterpret_cast<uint16_t *>(a.out);
  unsigned long long h = ((16u - ((uintptr_t)out & 15u)) & 15u) / 2;  // out + h: 16-byte aligned
  if (h > m) h = m;
  const unsigned long long nb = (m - h) / 8, tl = h + 8 * nb;  // 8-unit items
  const bool fast = (((uintptr_t)(in + h)) & 7u) == 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * N16_THREADS;
  unsigned long long i = (unsigned long long)blockIdx.x * N16_THREADS + tid;
  auto unit = [&](unsigned long long q) { return (uint16_t)(BE ? in[q] << 8 : in[q]); };
  if (fast) {
    const uint2 *src = reinterpret_cast<const uint2 *>(in + h);
    uint4 *dst = reinterpret_cast<uint4 *>(out + h);
    for (; i + 3 * stride < nb; i += 4 * stride) {
      uint2 q[4];
#pragma unroll
      for (int j = 0; j < 4; j++) q[j] = __ldcs(src + i + j * stride);
#pragma unroll
      for (int j = 0; j < 4; j++)
        __stcs(dst + i + j * stride, make_uint4(prmt(q[j].x, 0u, S0), prmt(q[j].x, 0u, S1),
                                                prmt(q[j].y, 0u, S0), prmt(q[j].y, 0u, S1)));
    }
    for (; i < nb; i += stride) {
      const uint2 q = __ldcs(src + i);
      __stcs(dst + i, make_uint4(prmt(q.x, 0u, S0), prmt(q.x, 0u, S1), prmt(q.y, 0u, S0),
                                 prmt(q.y, 0u, S1)));
    }
  } else {  // (unaligned phases: correctness, not speed)
    for (; i < nb; i += stride) {
      const unsigned long long q0 = h + 8 * i;
      uint32_t v[4];
#pragma unroll
      for (int j = 0; j < 4; j++)
        v[j] = unit(q0 + 2 * j) | ((uint32_t)unit(q0 + 2 * j + 1) << 16);
      *reinterpret_cast<uint4 *>(out + q0) = make_uint4(v[0], v[1], v[2], v[3]);
    }
  }
  if (blockIdx.x == 0) {
    if ((unsigned long long)tid < h) out[tid] = unit(tid);
    if ((unsigned long long)tid < m - tl) out[tl + tid] = unit(tl + tid);
  }
}

// ============================================================================ combine
__host__ __device__ inline void combine_impl(const RecordDev *recs, int nranks, int rank,
                                             unsigned long long total_in, ResultDev *res,
                                             unsigned long long *out_off) {
  unsigned long long off = 0, my_off = 0, e = NONE, wr = 0;
  int kind = 0, owner = -1;
  for (int k = 0; k < nranks; k++) {
    if (k == rank) my_off = off;
    if (recs[k].first_err < e) {
      e = recs[k].first_err;
      wr = off + recs[k].written;
      kind = recs[k].kind;
      owner = k;
    }
    off += recs[k].count;
  }
  // a rank whose own buffer was too small, at or before the error owner
  int last = owner < 0 ? nranks - 1 : owner;
  bool small = false;
  for (int k = 0; k <= last; k++) small = small || (recs[k].reserved != 0);
  ResultDev r;
  r.reserved = 0;
  if (small) {
    r.error = ERR_OUTPUT_TOO_SMALL;
    r.position = (e == NONE) ? off : wr;
    r.written = 0;
  } else if (e == NONE) {
    r.error = 0;
    r.position = total_in;
    r.written = off;
  } else {
    r.error = kind;
    r.position = e;
    r.written = wr;
  }
  if (res) *res = r;
  if (out_off) *out_off = my_off;
}

__global__ void k_combine(const RecordDev *recs, int nranks, int rank,
                          unsigned long long total_in, ResultDev *res,
                          unsigned long long *out_off) {
  if (threadIdx.x == 0 && blockIdx.x == 0) combine_impl(recs, nranks, rank, total_in, res, out_off);
}

void combine_host(const RecordDev *recs, int nranks, int rank, unsigned long long total_in,
                  ResultDev *res, unsigned long long *out_off) {
  combine_impl(recs, nranks, rank, total_in, res, out_off);
}

// ============================================================================ launchers
#ifdef UG_TRACE
cudaError_t dbg_read(void *host) { return cudaMemcpyFromSymbol(host, g_dbg, sizeof(g_dbg)); }
cudaError_t trace_read(void *host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_trace, bytes < sizeof(g_trace) ? bytes : sizeof(g_trace));
}
#endif
size_t tile_smem_bytes(Op op) {
  switch (op) {
    case Op::U8_VALIDATE:
#if !defined(UG_VALIDATE_STREAM) && !defined(UG_NO_VPRODUCER)
      return VRING8 * INBUF;
#endif
    case Op::U16_VALIDATE:
    case Op::U16BE_VALIDATE:
#if !defined(UG_VALIDATE_STREAM) && !defined(UG_VAL16_TMA)
      if (op != Op::U8_VALIDATE) return 0;
#endif
#ifndef UG_VALIDATE_STREAM
      return VRING * INBUF;
#else
      return 0;
#endif
    case Op::U8_TO_U16:
    case Op::U8_TO_U16BE: return RING * INBUF + U8Pol::STAGE;
    case Op::U16_TO_U8:
    case Op::U16BE_TO_U8:
#ifndef UG_U16_TILE_SCAN
      return RING16 * INBUF + U16Pol::STAGE;
#else
      return RING * INBUF + U16Pol::STAGE;
#endif
  }
  return 0;
}

int tile_threads(Op op) {
  switch (op) {
#if !defined(UG_VALIDATE_STREAM) && !defined(UG_VAL16_TMA)
    case Op::U16_VALIDATE:
    case Op::U16BE_VALIDATE: return V16_THREADS;
#endif
#ifdef UG_VALIDATE_STREAM
    case Op::U8_VALIDATE:
    case Op::U16_VALIDATE:
    case Op::U16BE_VALIDATE: return VS_THREADS;
#endif
    case Op::U8_TO_U16:
    case Op::U8_TO_U16BE: return NT + 32 * NLB;
    case Op::U16_TO_U8:
    case Op::U16BE_TO_U8:
#ifndef UG_U16_TILE_SCAN
      return T16_THREADS;
#else
      return NT + 32 * NLB;
#endif
#if !defined(UG_NO_VPRODUCER) && !defined(UG_VALIDATE_STREAM)
    case Op::U8_VALIDATE: return VGeo<U8Pol>::THREADS;
#if !(!defined(UG_VALIDATE_STREAM) && !defined(UG_VAL16_TMA))
    case Op::U16_VALIDATE:
    case Op::U16BE_VALIDATE: return VGeo<U16Pol>::THREADS;
#endif
#endif
    default: return NT;
  }
}

#ifndef UG_U16_TILE_SCAN
template <bool BE>
static const void *rev_fn() { return (const void *)k_transcode16<BE>; }
template <bool BE>
static void rev_launch(const TileArgs &a, int grid, int nt, size_t sm, cudaStream_t s) {
  k_transcode16<BE><<<grid, nt, sm, s>>>(a);
}
#else
template <bool BE>
static const void *rev_fn() { return (const void *)k_transcode<U16PolT<BE>>; }
template <bool BE>
static void rev_launch(const TileArgs &a, int grid, int nt, size_t sm, cudaStream_t s) {
  k_transcode<U16PolT<BE>><<<grid, nt, sm, s>>>(a);
}
#endif

#ifndef UG_VALIDATE_STREAM
#define UG_KVAL k_validate
#else
#define UG_KVAL k_validate_stream
#endif
#if !defined(UG_VALIDATE_STREAM) && !defined(UG_VAL16_TMA)
#define UG_V16_ON 1
#define UG_KVAL16(BE) k_validate16<BE>
#else
#define UG_V16_ON 0
#define UG_KVAL16(BE) UG_KVAL<U16PolT<BE>>
#endif
static const void *tile_fn(Op op) {
  switch (op) {
    case Op::U8_VALIDATE: return (const void *)UG_KVAL<U8Pol>;
    case Op::U8_TO_U16: return (const void *)k_transcode<U8Pol>;
    case Op::U16_VALIDATE: return (const void *)UG_KVAL16(false);
    case Op::U16_TO_U8: return rev_fn<false>();
    case Op::U16BE_VALIDATE: return (const void *)UG_KVAL16(true);
    case Op::U8_TO_U16BE: return (const void *)k_transcode<U8PolBE>;
    case Op::U16BE_TO_U8: return rev_fn<true>();
  }
  return nullptr;
}

// Work items of one launch over a window with `nbytes` owned bytes at address phase `lead`:
// tiles (tile kernels) or 1 KiB warp chunks (streaming validators); and items per CTA.
unsigned long long tile_units(Op op, long long nbytes, long long lead, int *per_cta) {
#if UG_V16_ON
  if (op == Op::U16_VALIDATE || op == Op::U16BE_VALIDATE) {  // 16-byte chunks, k_validate16
    *per_cta = (V16_THREADS / 32) * 32 * V16_U;
    return (unsigned long long)((nbytes + 2 + lead + 15) / 16);
  }
#endif
#ifdef UG_VALIDATE_STREAM
  if (!op_transcodes(op)) {
    *per_cta = VS_THREADS / 32;
    return (unsigned long long)((nbytes - 1 + lead) / VS_CHUNK + 1);
  }
#endif
  *per_cta = 1;
  return (unsigned long long)((nbytes - 1 + lead) / TILE + 1);
}

cudaError_t tile_configure(Op op) {
  return cudaFuncSetAttribute(tile_fn(op), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)tile_smem_bytes(op));
}

cudaError_t tile_occupancy(Op op, int *blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tile_fn(op),
                                                       tile_threads(op), tile_smem_bytes(op));
}

cudaError_t launch_tile(Op op, const TileArgs &a, int grid, cudaStream_t s) {
  size_t sm = tile_smem_bytes(op);
  int nt = tile_threads(op);
  switch (op) {
    case Op::U8_VALIDATE: UG_KVAL<U8Pol><<<grid, nt, sm, s>>>(a); break;
    case Op::U16_VALIDATE: UG_KVAL16(false)<<<grid, nt, sm, s>>>(a); break;
    case Op::U8_TO_U16: k_transcode<U8Pol><<<grid, nt, sm, s>>>(a); break;
    case Op::U16_TO_U8: rev_launch<false>(a, grid, nt, sm, s); break;
    case Op::U16BE_VALIDATE: UG_KVAL16(true)<<<grid, nt, sm, s>>>(a); break;
    case Op::U8_TO_U16BE: k_transcode<U8PolBE><<<grid, nt, sm, s>>>(a); break;
    case Op::U16BE_TO_U8: rev_launch<true>(a, grid, nt, sm, s); break;
  }
  return cudaGetLastError();
}

// ---- planned path launchers
size_t planned_smem_bytes(bool u16in) {
  return u16in ? PlannedGeo<U16Pol>::SMEM : PlannedGeo<U8Pol>::SMEM;
}
cudaError_t keyed_upload() {
  static uint16_t key[keyed::KEYS];
  static uint32_t shuf[keyed::SHUFFLES * keyed::SHUF_WORDS];
  static bool built = false;  // (called under the device-info lock)
  if (!built) keyed::build_tables(key, shuf), built = true;
  cudaError_t e = cudaMemcpyToSymbol(g_keyed_key, key, sizeof(key));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_keyed_shuf, shuf, sizeof(shuf));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute((const void *)k_transcode_planned<U8KeyPol>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)planned_smem_bytes(false));
  return e;
}
cudaError_t keyed_occupancy(int *blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      blocks_per_sm, (const void *)k_transcode_planned<U8KeyPol>, NTP, planned_smem_bytes(false));
}
cudaError_t launch_planned_keyed(const TileArgs &a, const unsigned long long *plan, int grid,
                                 cudaStream_t s) {
  k_transcode_planned<U8KeyPol><<<grid, NTP, planned_smem_bytes(false), s>>>(a, plan);
  return cudaGetLastError();
}
static const void *planned_fn(Op op) {
  switch (op) {
    case Op::U8_TO_U16: return (const void *)k_transcode_planned<U8Pol>;
    case Op::U8_TO_U16BE: return (const void *)k_transcode_planned<U8PolBE>;
    case Op::U16_TO_U8: return (const void *)k_transcode_planned<U16Pol>;
    case Op::U16BE_TO_U8: return (const void *)k_transcode_planned<U16PolBE>;
    default: return nullptr;
  }
}
static const void *planned_fn_nof(Op op) {  // f1 for UTF-8: the no-F forward
  switch (op) {
    case Op::U8_TO_U16: return (const void *)k_transcode_planned<U8Pol, true>;
    case Op::U8_TO_U16BE: return (const void *)k_transcode_planned<U8PolBE, true>;
    default: return nullptr;
  }
}
cudaError_t planned_configure(Op op) {
  cudaError_t e = cudaFuncSetAttribute(planned_fn(op), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)planned_smem_bytes(op_u16_input(op)));
  if (e == cudaSuccess && planned_fn_nof(op))
    e = cudaFuncSetAttribute(planned_fn_nof(op), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)planned_smem_bytes(false));
  return e;
}
cudaError_t planned_occupancy(Op op, int *blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      blocks_per_sm, planned_fn(op), NTP, planned_smem_bytes(op_u16_input(op)));
}
#ifndef UG_NO_PDL
// The second kernel of a planned pair, launched with programmatic stream serialization: it may
// start before the first completes (it reads only the plan, which both wait for in stream
// order; exactly one of the two does the work).  The next launch in the stream still waits for
// both.
template <class... Args>
static cudaError_t launch_paired(void (*fn)(Args...), int grid, int threads, size_t sm,
                                 cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, args...);
}
#endif
// kernels one launch_planned enqueues (the two forward forms; the reverse's tile kernel and
// narrowing copy): what the launch counter adds
int planned_kernels(Op op) {
  if (op_u16_input(op)) {
#ifdef UG_NO_NARROW16
    return 1;
#endif
    return 2;
  }
#ifdef UG_NO_WIDEN8
  return 2;
#endif
  return 3;
}
cudaError_t launch_planned(Op op, const TileArgs &a, const unsigned long long *plan, int grid,
                           cudaStream_t s) {
  const size_t sm = planned_smem_bytes(op_u16_input(op));
  switch (op) {
    // both forward forms are launched; the plan's header selects the one that works
    case Op::U8_TO_U16:
      k_transcode_planned<U8Pol><<<grid, NTP, sm, s>>>(a, plan);
#ifndef UG_NO_PDL
      launch_paired(k_transcode_planned<U8Pol, true>, grid, NTP, sm, s, a, plan);
#ifndef UG_NO_WIDEN8
      launch_paired(k_widen8<false>, grid, N16_THREADS, 0, s, a, plan);
#endif
#else
      k_transcode_planned<U8Pol, true><<<grid, NTP, sm, s>>>(a, plan);
#ifndef UG_NO_WIDEN8
      k_widen8<false><<<grid, N16_THREADS, 0, s>>>(a, plan);
#endif
#endif
      break;
    case Op::U8_TO_U16BE:
      k_transcode_planned<U8PolBE><<<grid, NTP, sm, s>>>(a, plan);
#ifndef UG_NO_PDL
      launch_paired(k_transcode_planned<U8PolBE, true>, grid, NTP, sm, s, a, plan);
#ifndef UG_NO_WIDEN8
      launch_paired(k_widen8<true>, grid, N16_THREADS, 0, s, a, plan);
#endif
#else
      k_transcode_planned<U8PolBE, true><<<grid, NTP, sm, s>>>(a, plan);
#ifndef UG_NO_WIDEN8
      k_widen8<true><<<grid, N16_THREADS, 0, s>>>(a, plan);
#endif
#endif
      break;
    // UTF-16 input: the tile kernel, then the all-ASCII narrowing copy; the plan's total
    // selects the one that works
    case Op::U16_TO_U8:
      k_transcode_planned<U16Pol><<<grid, NTP, sm, s>>>(a, plan);
#ifndef UG_NO_NARROW16
#ifndef UG_NO_PDL
      launch_paired(k_narrow16<false>, grid, N16_THREADS, 0, s, a, plan);
#else
      k_narrow16<false><<<grid, N16_THREADS, 0, s>>>(a, plan);
#endif
#endif
      break;
    case Op::U16BE_TO_U8:
      k_transcode_planned<U16PolBE><<<grid, NTP, sm, s>>>(a, plan);
#ifndef UG_NO_NARROW16
#ifndef UG_NO_PDL
      launch_paired(k_narrow16<true>, grid, N16_THREADS, 0, s, a, plan);
#else
      k_narrow16<true><<<grid, N16_THREADS, 0, s>>>(a, plan);
#endif
#endif
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
cudaError_t launch_plan(bool u16in, bool be, const Window &w, unsigned long long ntiles,
                        int nsub, unsigned long long tps, unsigned long long *plan,
                        Counters *ctr, unsigned long long *d_len, cudaStream_t s) {
  PlanArgs pa;
  pa.win = w;
  pa.ntiles = ntiles;
  pa.nsub = nsub;
  pa.tps = tps;
  pa.plan = plan;
  pa.ctr = ctr;
  pa.d_len = d_len;
  if (!u16in)
    k_plan8<<<nsub, LNT, 0, s>>>(pa);
  else if (be)
    k_plan16<true><<<nsub, LNT, 0, s>>>(pa);
  else
    k_plan16<false><<<nsub, LNT, 0, s>>>(pa);
  return cudaGetLastError();
}

cudaError_t launch_len8(const uint8_t *in, unsigned long long n, Counters *ctr,
                        unsigned long long *d_len, int grid, cudaStream_t s) {
  k_len8<<<grid, LNT, 0, s>>>(in, n, ctr, d_len);
  return cudaGetLastError();
}
cudaError_t launch_len16(const uint16_t *in, unsigned long long n, Counters *ctr,
                         unsigned long long *d_len, int grid, cudaStream_t s, bool be) {
  if (be)
    k_len16<true><<<grid, LNT, 0, s>>>(in, n, ctr, d_len);
  else
    k_len16<false><<<grid, LNT, 0, s>>>(in, n, ctr, d_len);
  return cudaGetLastError();
}
cudaError_t launch_combine(const RecordDev *recs, int nranks, int rank,
                           unsigned long long total_in, ResultDev *res,
                           unsigned long long *out_off, cudaStream_t s) {
  k_combine<<<1, 32, 0, s>>>(recs, nranks, rank, total_in, res, out_off);
  return cudaGetLastError();
}

}  // namespace ug
