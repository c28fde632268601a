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
// Tile pipeline (all tile kernels): persistent CTAs of 256 threads pull 8 KiB tiles by
// atomic ticket (issue order makes the decoupled look-back deadlock-free), bulk-load tile +
// 16-byte halos into shared memory with TMA (cp.async.bulk + mbarrier, 2 stages: the next
// tile is in flight while the current one is processed), and each thread owns 32 contiguous
// input bytes.  Output is staged in shared memory at the global address phase and leaves
// through one TMA bulk store (cp.async.bulk.global.shared::cta) plus <16 head/tail units.
#include <cstdint>

#include "device.cuh"
#include "internal.h"
#include "utf16.cuh"
#include "utf8.cuh"

namespace ug {

constexpr unsigned long long VALMASK = (1ull << 38) - 1;
constexpr int STAGE8_UNITS = TILE + 16;            // UTF-16 units staged per UTF-8 tile
constexpr int STAGE16_BYTES = 3 * (TILE / 2) + 32;   // UTF-8 bytes staged per UTF-16 tile

__device__ __forceinline__ uint32_t byte_at(const Window &w, long long pos) {
  return (pos >= w.lo_valid && pos < w.hi_valid) ? (uint32_t)w.base[pos] : 0u;
}
__device__ __forceinline__ uint32_t word_at(const Window &w, long long wpos) {
  long long pos = 2 * wpos;
  return (pos >= w.lo_valid && pos + 2 <= w.hi_valid)
             ? (uint32_t)reinterpret_cast<const uint16_t *>(w.base)[wpos]
             : 0u;
}

// Copy staged units [phase, phase + C) to out[P, P + C) (clipped at cap): aligned interior
// by one TMA bulk store, the < A-unit head and tail by plain stores.  A = units per 16 B.
template <typename T>
__device__ __forceinline__ void copy_out(T *out, unsigned long long cap, unsigned long long P,
                                         uint32_t C, uint32_t phase, const T *stage, int tid) {
  constexpr unsigned long long A = 16 / sizeof(T);
  unsigned long long lo = P, hi = P + C;
  if (hi > cap) hi = cap;
  if (hi <= lo) return;
  unsigned long long ua = P - phase;  // stage index k <-> unit ua + k; out + ua is 16B-aligned
  unsigned long long a_lo = phase ? ua + A : ua;
  unsigned long long a_hi = ua + ((hi - ua) / A) * A;
  if (a_lo < a_hi) {
    if (tid == 0) {
      fence_proxy_async_smem();
      bulk_s2g(out + a_lo, stage + (a_lo - ua), (uint32_t)((a_hi - a_lo) * sizeof(T)));
      bulk_commit();
    }
    long long nh = (long long)(a_lo - lo);
    if (tid < nh) out[lo + tid] = stage[phase + tid];
    long long nt = (long long)(hi - a_hi);
    if (tid >= 64 && tid - 64 < nt) out[a_hi + (tid - 64)] = stage[(a_hi - ua) + (tid - 64)];
  } else {
    long long m = (long long)(hi - lo);
    if (tid < m) out[lo + tid] = stage[phase + tid];
  }
}

// Block exclusive scan of per-thread counts: returns the thread's exclusive prefix within the
// tile and the tile total.  One __syncthreads inside.
__device__ __forceinline__ void block_scan(uint32_t cnt, uint32_t *s_wsum, int lane, int warp,
                                           uint32_t *excl, uint32_t *total) {
  uint32_t incl = warp_incl_scan(cnt, lane);
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0, C = 0;
#pragma unroll
  for (int i = 0; i < NT / 32; i++) {
    uint32_t v = s_wsum[i];
    wpre += (i < warp) ? v : 0u;
    C += v;
  }
  *excl = wpre + incl - cnt;
  *total = C;
}

// Publish tile t's aggregate, look back, publish its inclusive prefix; warp 0 only.
__device__ __forceinline__ unsigned long long tile_prefix(const TileArgs &a, long long t,
                                                          uint32_t C, int lane) {
  unsigned long long P;
  if (t == 0) {
    P = 0;
    if (lane == 0) st_relaxed(a.status, pack_status(a.epoch, FLAG_PREFIX, C));
  } else {
    if (lane == 0) st_relaxed(a.status + t, pack_status(a.epoch, FLAG_AGG, C));
    P = look_back(a.status, a.epoch, t, lane);
    if (lane == 0) st_relaxed(a.status + t, pack_status(a.epoch, FLAG_PREFIX, P + C));
  }
  return P;
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

// ============================================================================ UTF-8 tiles
template <bool XC>
__global__ void __launch_bounds__(NT) k_utf8(const TileArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t *inbuf = smem;
  uint16_t *stage = reinterpret_cast<uint16_t *>(smem + 2 * INBUF);
  __shared__ uint64_t bar[2];
  __shared__ uint32_t s_wsum[NT / 32];
  __shared__ long long s_next[2];
  __shared__ unsigned long long s_excl, s_emin;
  __shared__ int s_flag, s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Window &win = a.win;
  const long long ntiles = (long long)a.ntiles;
  const long long n = win.n;
  uint16_t *out = reinterpret_cast<uint16_t *>(a.out);
  const uint32_t out_mis = (uint32_t)(((uintptr_t)out >> 1) & 7u);

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    long long t0 = (long long)atomicAdd(&a.ctr->ticket, 1u);
    s_next[0] = t0;
    if (t0 < ntiles) issue_tile_load(win, t0, inbuf, &bar[0]);
  }
  __syncthreads();
  long long t = s_next[0];
  int s = 0;
  uint32_t parity = 0;

  while (t < ntiles) {
    if (tid == 0) {
      long long tn = (long long)atomicAdd(&a.ctr->ticket, 1u);
      s_next[s ^ 1] = tn;
      if (tn < ntiles) {
        fence_proxy_async_smem();
        issue_tile_load(win, tn, inbuf + (s ^ 1) * INBUF, &bar[s ^ 1]);
      }
      s_flag = 0;
      s_emin = NONE;
      if (XC) bulk_wait_read_all();  // previous tile's bulk store has read `stage`
    }
    mbar_wait(&bar[s], (parity >> s) & 1u);
    parity ^= 1u << s;
    uint8_t *buf = inbuf + s * INBUF;
    fix_tile_edges(win, t, buf);
    __syncthreads();

    // ---------------------------------------------------------------- a1: this thread's bytes
    const long long tp = tile_pos(win, t);
    const uint8_t *my = buf + HALO + BPT * tid;
    uint32_t w[9];
    {
      uint4 q0 = *reinterpret_cast<const uint4 *>(my);
      uint4 q1 = *reinterpret_cast<const uint4 *>(my + 16);
      w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
      w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
    }
    uint32_t prev = __shfl_up_sync(FULL, w[7], 1);
    uint32_t nxt = __shfl_down_sync(FULL, w[0], 1);
    if (lane == 0) prev = *reinterpret_cast<const uint32_t *>(my - 4);
    if (lane == 31) nxt = *reinterpret_cast<const uint32_t *>(my + BPT);
    w[8] = nxt;
    const long long mypos = tp + BPT * tid;
    const bool interior = (tp >= 0) && (tp + TILE + 1 <= n);

    // ---------------------------------------------------------------- a2: warp ASCII path
    uint32_t orv = w[0] | w[1] | w[2] | w[3] | w[4] | w[5] | w[6] | w[7];
    bool pend = (prev >= 0xC0000000u) || ((prev & 0x00FF0000u) >= 0x00E00000u) ||
                ((prev & 0x0000FF00u) >= 0x0000F000u);
    const bool wasc = __all_sync(FULL, ((orv & u8::HI) == 0u) && !pend);

    // ---------------------------------------------------------------- a3/a5: classify, widths
    uint32_t err = 0;
    uint32_t cm[8];
    if (wasc) {
#pragma unroll
      for (int k = 0; k < 8; k++) cm[k] = u8::HI;
    } else {
      u8::WordMasks pm = u8::masks(prev, true);
      u8::WordMasks cur = u8::masks(w[0], true);
#pragma unroll
      for (int k = 0; k < 8; k++) {
        u8::WordMasks nx = u8::masks(w[k + 1], true);
        err |= u8::classify(pm, cur);
        cm[k] = XC ? u8::width_bits(cur, nx.K) : 0u;
        pm = cur;
        cur = nx;
      }
      if (tid == NT - 1) err |= u8::classify(pm, cur);  // look-ahead: positions TILE..TILE+3
    }
    uint32_t cnt = 0;
    if (XC) {
      if (!interior) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
          long long pos = mypos + 4 * k;
          uint32_t own = range_bytes(pos, 0, n) & u8::HI;
          uint32_t own1 = (range_bytes(pos, 0, n - 1) & u8::HI) >> 1;
          cm[k] &= own | own1;
        }
      }
#pragma unroll
      for (int k = 0; k < 8; k++) cnt += __popc(cm[k]);
    }
    if (err) s_flag = 1;

    // ---------------------------------------------------------------- a6: scan + look-back
    uint32_t excl_local = 0, C = 0;
    if (XC) {
      block_scan(cnt, s_wsum, lane, warp, &excl_local, &C);
    } else {
      __syncthreads();
    }
    const bool flagged = s_flag != 0;
    if (XC && warp == 0) {
      unsigned long long P = tile_prefix(a, t, C, lane);
      if (lane == 0) s_excl = P;
    }
    // ---------------------------------------------------------------- a4: exact rescan (cold)
    if (flagged) {
      uint32_t l32[10];
      const uint8_t *loc = reinterpret_cast<const uint8_t *>(l32);
      l32[0] = prev;
#pragma unroll
      for (int k = 0; k < 9; k++) l32[k + 1] = w[k];
      for (int i = 0; i < BPT; i++) {
        long long pos = mypos + i;
        if (pos < 0 || pos >= n) continue;
        if (u8::err_at(loc + 4 + i)) {
          atomicMin(&s_emin, (unsigned long long)pos);
          break;
        }
      }
    }
    __syncthreads();
    if (flagged && tid == 0 && s_emin != NONE) atomicMin(&a.ctr->err_min, s_emin);

    if (XC) {
      // -------------------------------------------------------------- a7: decode into stage
      const unsigned long long P = s_excl;
      const uint32_t phase = (out_mis + (uint32_t)P) & 7u;
      uint32_t o = phase + excl_local;
      if (wasc && interior) {
        if ((o & 1u) == 0u) {
          uint32_t *st32 = reinterpret_cast<uint32_t *>(stage + o);
#pragma unroll
          for (int k = 0; k < 8; k++) {
            st32[2 * k] = u8::prmt(w[k], 0u, 0x4140u);
            st32[2 * k + 1] = u8::prmt(w[k], 0u, 0x4342u);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 8; k++)
#pragma unroll
            for (int j = 0; j < 4; j++) stage[o + 4 * k + j] = (uint16_t)((w[k] >> (8 * j)) & 0xFFu);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const uint32_t c = cm[k];
          uint32_t lead = c & u8::HI;
          while (lead) {
            const int b = __ffs(lead) - 1;  // 7, 15, 23 or 31
            lead &= lead - 1u;
            const uint32_t sh = (uint32_t)(b - 7);
            const uint32_t x = __funnelshift_r(w[k], w[k + 1], sh);
            uint32_t u1;
            const uint32_t u0 = u8::decode_units(x, &u1);
            const uint32_t off = o + __popc(c & ((1u << sh) - 1u));
            stage[off] = (uint16_t)u0;
            if (c & (1u << (b - 1))) stage[off + 1] = (uint16_t)u1;
          }
          o += __popc(c);
        }
      }
      __syncthreads();
      // -------------------------------------------------------------- a8: store
      copy_out<uint16_t>(out, a.out_cap, P, C, phase, stage, tid);
    }
    __syncthreads();
    t = s_next[s ^ 1];
    s ^= 1;
  }

  // -------------------------------------------------------------------- a10: finalize
  if (tid == 0) {
    if (XC) bulk_wait_all();
    __threadfence();
    s_last = (atomicAdd(&a.ctr->done, 1u) == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (s_last && warp == 0) {
    __threadfence();
    unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&a.ctr->err_min);
    unsigned long long total = 0, wr = 0;
    int kind = 0;
    if (XC && a.ntiles) total = ld_relaxed(a.status + a.ntiles - 1) & VALMASK;
    if (e != NONE) {
      uint8_t b[4];
#pragma unroll
      for (int j = 0; j < 4; j++) b[j] = (uint8_t)byte_at(win, (long long)e + j);
      kind = u8::decode_kind(b);
      if (XC) {
        long long te = ((long long)e + win.lead) / TILE;
        unsigned long long base = te ? (ld_relaxed(a.status + te - 1) & VALMASK) : 0ull;
        long long from = te * TILE - win.lead;
        if (from < 0) from = 0;
        unsigned long long c = 0;
        for (long long i = from + lane; i < (long long)e; i += 32) {
          uint32_t bi = byte_at(win, i), bn = byte_at(win, i + 1);
          c += ((bi & 0xC0u) != 0x80u) ? 1u : 0u;
          c += (bi >= 0xF0u && (bn & 0xC0u) == 0x80u && i + 1 < n) ? 1u : 0u;
        }
        wr = base + warp_sum64(c);
      }
    }
    if (lane == 0) write_outcome(a, XC, kind, e, total, wr, (unsigned long long)n);
  }
}

// ============================================================================ UTF-16 tiles
template <bool XC>
__global__ void __launch_bounds__(NT) k_utf16(const TileArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t *inbuf = smem;
  uint8_t *stage = smem + 2 * INBUF;
  __shared__ uint64_t bar[2];
  __shared__ uint32_t s_wsum[NT / 32];
  __shared__ long long s_next[2];
  __shared__ unsigned long long s_excl, s_emin;
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Window &win = a.win;  // byte positions
  const long long ntiles = (long long)a.ntiles;
  const long long nw = win.n / 2;  // owned words
  uint8_t *out = reinterpret_cast<uint8_t *>(a.out);
  const uint32_t out_mis = (uint32_t)((uintptr_t)out & 15u);

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    long long t0 = (long long)atomicAdd(&a.ctr->ticket, 1u);
    s_next[0] = t0;
    if (t0 < ntiles) issue_tile_load(win, t0, inbuf, &bar[0]);
  }
  __syncthreads();
  long long t = s_next[0];
  int s = 0;
  uint32_t parity = 0;

  while (t < ntiles) {
    if (tid == 0) {
      long long tn = (long long)atomicAdd(&a.ctr->ticket, 1u);
      s_next[s ^ 1] = tn;
      if (tn < ntiles) {
        fence_proxy_async_smem();
        issue_tile_load(win, tn, inbuf + (s ^ 1) * INBUF, &bar[s ^ 1]);
      }
      s_emin = NONE;
      if (XC) bulk_wait_read_all();
    }
    mbar_wait(&bar[s], (parity >> s) & 1u);
    parity ^= 1u << s;
    uint8_t *buf = inbuf + s * INBUF;
    fix_tile_edges(win, t, buf);
    __syncthreads();

    const long long tpw = tile_pos(win, t) / 2;  // word position of the tile's first word
    const uint8_t *my = buf + HALO + BPT * tid;
    uint32_t w[8];
    {
      uint4 q0 = *reinterpret_cast<const uint4 *>(my);
      uint4 q1 = *reinterpret_cast<const uint4 *>(my + 16);
      w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
      w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
    }
    uint32_t pv = __shfl_up_sync(FULL, w[7], 1);
    uint32_t nx = __shfl_down_sync(FULL, w[0], 1);
    if (lane == 0) pv = *reinterpret_cast<const uint32_t *>(my - 4);
    if (lane == 31) nx = *reinterpret_cast<const uint32_t *>(my + BPT);
    const uint32_t prev_word = pv >> 16, next_word = nx & 0xFFFFu;
    const long long mypos = tpw + (BPT / 2) * tid;  // word position of this thread's first word
    const bool interior = (tpw >= 0) && (tpw + TILE / 2 <= nw);

    // any surrogate among the thread's words and neighbours?  (SWAR on word pairs)
    uint32_t sur = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      uint32_t x = (w[k] & 0xF800F800u) ^ 0xD800D800u;  // zero half <=> surrogate
      sur |= ((x & 0xFFFFu) == 0u) | ((x >> 16) == 0u);
    }
    uint32_t orv = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) orv |= w[k];
    const bool wasc = __all_sync(FULL, (orv & 0xFF80FF80u) == 0u);

    // ---------------------------------------------------------------- a9 + a5
    uint32_t cnt = 0;
    unsigned long long first_err = NONE;
    if (sur || ((prev_word & 0xF800u) == 0xD800u) || ((next_word & 0xF800u) == 0xD800u) ||
        XC) {
      uint32_t p = prev_word;
#pragma unroll
      for (int i = 0; i < 16; i++) {
        uint32_t u = (w[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
        uint32_t q = (i < 15) ? ((w[(i + 1) >> 1] >> (16 * ((i + 1) & 1))) & 0xFFFFu) : next_word;
        long long pos = mypos + i;
        bool own = interior || (pos >= 0 && pos < nw);
        if (own) {
          if (first_err == NONE && u16::err_at(p, u, q)) first_err = (unsigned long long)pos;
          if (XC) cnt += u16::width(u, p);
        }
        p = u;
      }
    }
    if (first_err != NONE) atomicMin(&s_emin, first_err);

    uint32_t excl_local = 0, C = 0;
    if (XC) {
      block_scan(cnt, s_wsum, lane, warp, &excl_local, &C);
      if (warp == 0) {
        unsigned long long P = tile_prefix(a, t, C, lane);
        if (lane == 0) s_excl = P;
      }
    }
    __syncthreads();
    if (tid == 0 && s_emin != NONE) atomicMin(&a.ctr->err_min, s_emin * 2);  // byte position

    if (XC) {
      // -------------------------------------------------------------- a7: encode into stage
      const unsigned long long P = s_excl;
      const uint32_t phase = (out_mis + (uint32_t)P) & 15u;
      uint32_t o = phase + excl_local;
      if (wasc && interior) {
        if ((o & 3u) == 0u) {
          uint32_t *st32 = reinterpret_cast<uint32_t *>(stage + o);
#pragma unroll
          for (int k = 0; k < 4; k++) st32[k] = u8::prmt(w[2 * k], w[2 * k + 1], 0x6420u);
        } else {
#pragma unroll
          for (int i = 0; i < 16; i++) stage[o + i] = (uint8_t)(w[i >> 1] >> (16 * (i & 1)));
        }
      } else {
        uint32_t p = prev_word;
#pragma unroll
        for (int i = 0; i < 16; i++) {
          uint32_t u = (w[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
          long long pos = mypos + i;
          bool own = interior || (pos >= 0 && pos < nw);
          if (own) {
            uint32_t wd = u16::width(u, p);
            uint32_t v = u16::utf8_bytes(u, p);
            stage[o] = (uint8_t)v;
            if (wd > 1) stage[o + 1] = (uint8_t)(v >> 8);
            if (wd > 2) stage[o + 2] = (uint8_t)(v >> 16);
            o += wd;
          }
          p = u;
        }
      }
      __syncthreads();
      copy_out<uint8_t>(out, a.out_cap, P, C, phase, stage, tid);
    }
    __syncthreads();
    t = s_next[s ^ 1];
    s ^= 1;
  }

  if (tid == 0) {
    if (XC) bulk_wait_all();
    __threadfence();
    s_last = (atomicAdd(&a.ctr->done, 1u) == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (s_last && warp == 0) {
    __threadfence();
    unsigned long long eb = *reinterpret_cast<volatile unsigned long long *>(&a.ctr->err_min);
    unsigned long long e = (eb == NONE) ? NONE : eb / 2;  // word position
    unsigned long long total = 0, wr = 0;
    if (XC && a.ntiles) total = ld_relaxed(a.status + a.ntiles - 1) & VALMASK;
    if (e != NONE && XC) {
      long long te = (2 * (long long)e + win.lead) / TILE;
      unsigned long long base = te ? (ld_relaxed(a.status + te - 1) & VALMASK) : 0ull;
      long long from = (te * TILE - win.lead) / 2;
      if (from < 0) from = 0;
      unsigned long long c = 0;
      for (long long i = from + lane; i < (long long)e; i += 32)
        c += u16::width(word_at(win, i), word_at(win, i - 1));
      wr = base + warp_sum64(c);
    }
    if (lane == 0)
      write_outcome(a, XC, e == NONE ? 0 : (int)u8::SURROGATE, e, total, wr,
                    (unsigned long long)nw);
  }
}

// ============================================================================ length-from
__device__ __forceinline__ uint32_t len8_word(uint32_t x) {
  uint32_t s1 = x << 1;
  uint32_t cont = x & ~s1 & u8::HI;
  uint32_t f0 = x & s1 & (x << 2) & (x << 3) & u8::HI;
  return 4u - __popc(cont) + __popc(f0);
}
__device__ __forceinline__ uint32_t len8_byte(uint32_t b) {
  return ((b & 0xC0u) != 0x80u ? 1u : 0u) + (b >= 0xF0u ? 1u : 0u);
}
__device__ __forceinline__ uint32_t len16_word(uint32_t u) {
  return 1u + (u >= 0x80u ? 1u : 0u) + ((u >= 0x800u && (u & 0xF800u) != 0xD800u) ? 1u : 0u);
}

__device__ __forceinline__ void finish_reduction(unsigned long long sum, Counters *ctr,
                                                 unsigned long long *d_len) {
  __shared__ unsigned long long s_part[NT / 32];
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

__global__ void __launch_bounds__(NT) k_len8(const uint8_t *in, unsigned long long n,
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

__global__ void __launch_bounds__(NT) k_len16(const uint16_t *in, unsigned long long n,
                                              Counters *ctr, unsigned long long *d_len) {
  const uintptr_t addr = (uintptr_t)in;
  unsigned long long head = ((16u - (addr & 15u)) & 15u) / 2;
  if (head > n) head = n;
  const uint4 *body = reinterpret_cast<const uint4 *>(in + head);
  const unsigned long long nb = (n - head) / 8;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long sum = 0;
  auto pair = [](uint32_t x) { return len16_word(x & 0xFFFFu) + len16_word(x >> 16); };
  unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nb; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; j++) v[j] = __ldcs(body + i + j * stride);
#pragma unroll
    for (int j = 0; j < 4; j++) sum += pair(v[j].x) + pair(v[j].y) + pair(v[j].z) + pair(v[j].w);
  }
  for (; i < nb; i += stride) {
    uint4 v = __ldcs(body + i);
    sum += pair(v.x) + pair(v.y) + pair(v.z) + pair(v.w);
  }
  if (blockIdx.x == 0) {
    for (unsigned long long j = threadIdx.x; j < head; j += blockDim.x) sum += len16_word(in[j]);
    for (unsigned long long j = head + nb * 8 + threadIdx.x; j < n; j += blockDim.x)
      sum += len16_word(in[j]);
  }
  finish_reduction(sum, ctr, d_len);
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
size_t tile_smem_bytes(Op op) {
  switch (op) {
    case Op::U8_VALIDATE:
    case Op::U16_VALIDATE: return 2 * INBUF;
    case Op::U8_TO_U16: return 2 * INBUF + 2 * STAGE8_UNITS;
    case Op::U16_TO_U8: return 2 * INBUF + STAGE16_BYTES;
  }
  return 0;
}

static const void *tile_fn(Op op) {
  switch (op) {
    case Op::U8_VALIDATE: return (const void *)k_utf8<false>;
    case Op::U8_TO_U16: return (const void *)k_utf8<true>;
    case Op::U16_VALIDATE: return (const void *)k_utf16<false>;
    case Op::U16_TO_U8: return (const void *)k_utf16<true>;
  }
  return nullptr;
}

cudaError_t tile_configure(Op op) {
  return cudaFuncSetAttribute(tile_fn(op), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)tile_smem_bytes(op));
}

cudaError_t tile_occupancy(Op op, int *blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, tile_fn(op), NT,
                                                       tile_smem_bytes(op));
}

cudaError_t launch_tile(Op op, const TileArgs &a, int grid, cudaStream_t s) {
  size_t sm = tile_smem_bytes(op);
  switch (op) {
    case Op::U8_VALIDATE: k_utf8<false><<<grid, NT, sm, s>>>(a); break;
    case Op::U8_TO_U16: k_utf8<true><<<grid, NT, sm, s>>>(a); break;
    case Op::U16_VALIDATE: k_utf16<false><<<grid, NT, sm, s>>>(a); break;
    case Op::U16_TO_U8: k_utf16<true><<<grid, NT, sm, s>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_len8(const uint8_t *in, unsigned long long n, Counters *ctr,
                        unsigned long long *d_len, int grid, cudaStream_t s) {
  k_len8<<<grid, NT, 0, s>>>(in, n, ctr, d_len);
  return cudaGetLastError();
}
cudaError_t launch_len16(const uint16_t *in, unsigned long long n, Counters *ctr,
                         unsigned long long *d_len, int grid, cudaStream_t s) {
  k_len16<<<grid, NT, 0, s>>>(in, n, ctr, d_len);
  return cudaGetLastError();
}
cudaError_t launch_combine(const RecordDev *recs, int nranks, int rank,
                           unsigned long long total_in, ResultDev *res,
                           unsigned long long *out_off, cudaStream_t s) {
  k_combine<<<1, 32, 0, s>>>(recs, nranks, rank, total_in, res, out_off);
  return cudaGetLastError();
}

}  // namespace ug
