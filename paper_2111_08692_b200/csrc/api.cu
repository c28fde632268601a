// api.cu -- the C-ABI of libunigpu.so (declared, with argument semantics and citations, in
// include/unigpu.h).  Host-side only: argument checks, the per-(device, stream) workspace,
// grid sizing, launches.  Every step of the path runs in kernels.cu; there is no CPU fallback:
// if a launch fails the call returns UG_ERR_CUDA.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <thread>
#ifdef UG_FILE_TRACE
#include <chrono>
#include <cstdio>
#endif
#include <vector>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include "../../include/unigpu.h"
#include "internal.h"
#include "utf8_keyed.cuh"

using namespace ug;

static_assert(sizeof(ResultDev) == sizeof(ug_result), "ug_result layout");
static_assert(sizeof(RecordDev) == sizeof(ug_shard_record), "ug_shard_record layout");
static_assert(sizeof(ug_shard_record) == 32, "record is 32 bytes");

namespace {

std::atomic<uint64_t> g_launches{0};
constexpr size_t HOST_CHUNK_DEFAULT = 64ull << 20;  // input units per pipelined host chunk (e2e sweep: 64 Mi +1.3 % over 32 Mi; slots 3-8 equal)
std::atomic<size_t> g_host_chunk{HOST_CHUNK_DEFAULT};
constexpr int HOST_SLOTS_MAX = 16;
std::atomic<int> g_host_slots{4};  // staging slots of the host pipeline (chunks in flight)
constexpr unsigned long long MAX_N = (1ull << 38) - 1;  // status words carry 38-bit values

struct Workspace {
  int device = -1;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  uint64_t *status = nullptr;
  size_t status_cap = 0;
  Counters *ctr = nullptr;
  ResultDev *d_res = nullptr;
  ResultDev *h_res = nullptr;  // pinned
  unsigned long long *d_len = nullptr;
  unsigned long long *h_len = nullptr;  // pinned
  uint32_t epoch = 0;
  void *d_in = nullptr;
  size_t d_in_cap = 0;
  void *d_out = nullptr;
  size_t d_out_cap = 0;
  // host-buffer pipeline (run_host): copy streams, per-chunk events and shard records
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_start = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_done, ev_free;  // per staging slot
  RecordDev *d_recs = nullptr;
  RecordDev *h_recs = nullptr;  // pinned
  size_t rec_cap = 0;
};

struct DeviceInfo {
  int sms = 0;
  int occ[NUM_OPS] = {};
  int occ_planned[2] = {};  // planned transcoders: UTF-8 input, UTF-16 input
  int occ_keyed = 0;        // f4: the planned forward with the keyed decoder
  bool configured = false;
};

std::mutex g_mu;
std::map<std::pair<int, uintptr_t>, Workspace *> g_ws;
std::map<int, DeviceInfo> g_dev;

cudaError_t device_info(int dev, DeviceInfo **out) {
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceInfo &d = g_dev[dev];
  if (!d.configured) {
    cudaError_t e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < NUM_OPS; i++) {
      e = tile_configure((Op)i);
      if (e != cudaSuccess) return e;
      e = tile_occupancy((Op)i, &d.occ[i]);
      if (e != cudaSuccess) return e;
      if (d.occ[i] < 1) d.occ[i] = 1;
    }
    for (int u = 0; u < 2; u++) {
      const Op op = u ? Op::U16_TO_U8 : Op::U8_TO_U16;
      e = planned_configure(op);
      if (e == cudaSuccess) e = planned_configure(u ? Op::U16BE_TO_U8 : Op::U8_TO_U16BE);
      if (e != cudaSuccess) return e;
      e = planned_occupancy(op, &d.occ_planned[u]);
      if (e != cudaSuccess) return e;
      if (d.occ_planned[u] < 1) d.occ_planned[u] = 1;
      if (d.occ_planned[u] > CPSP) d.occ_planned[u] = CPSP;
    }
    e = keyed_upload();
    if (e == cudaSuccess) e = keyed_occupancy(&d.occ_keyed);
    if (e != cudaSuccess) return e;
    if (d.occ_keyed < 1) d.occ_keyed = 1;
    if (d.occ_keyed > CPSP) d.occ_keyed = CPSP;
    d.configured = true;
  }
  *out = &d;
  return cudaSuccess;
}

cudaError_t get_ws(cudaStream_t s, Workspace **out) {
  int dev;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, (uintptr_t)s);
  auto it = g_ws.find(key);
  if (it != g_ws.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  Workspace *w = new Workspace();
  w->device = dev;
  w->stream = s;
  if ((e = cudaMalloc(&w->ctr, sizeof(Counters))) != cudaSuccess) return e;
  Counters init;
  std::memset(&init, 0, sizeof(init));
  init.err_min = NONE;
  if ((e = cudaMemcpy(w->ctr, &init, sizeof(init), cudaMemcpyHostToDevice)) != cudaSuccess)
    return e;
  if ((e = cudaMalloc(&w->d_res, sizeof(ResultDev))) != cudaSuccess) return e;
  if ((e = cudaMallocHost(&w->h_res, sizeof(ResultDev))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&w->d_len, sizeof(unsigned long long))) != cudaSuccess) return e;
  if ((e = cudaMallocHost(&w->h_len, sizeof(unsigned long long))) != cudaSuccess) return e;
  g_ws[key] = w;
  *out = w;
  return cudaSuccess;
}

cudaError_t ensure_status(Workspace *w, size_t ntiles) {
  if (ntiles <= w->status_cap) return cudaSuccess;
  size_t cap = w->status_cap * 2 > ntiles ? w->status_cap * 2 : ntiles;
  if (w->status) {
    cudaError_t e = cudaStreamSynchronize(w->stream);
    if (e != cudaSuccess) return e;
    cudaFree(w->status);
    w->status = nullptr;
    w->status_cap = 0;
  }
  cudaError_t e = cudaMalloc(&w->status, cap * sizeof(uint64_t));
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(w->status, 0, cap * sizeof(uint64_t), w->stream);
  if (e != cudaSuccess) return e;
  w->status_cap = cap;
  return cudaSuccess;
}

uint32_t next_epoch(Workspace *w) {
  w->epoch = (w->epoch + 1) & 0xFFFFFFu;
  if (w->epoch == 0) {  // wrapped: old words could alias the new epoch
    if (w->status) cudaMemsetAsync(w->status, 0, w->status_cap * sizeof(uint64_t), w->stream);
    w->epoch = 1;
  }
  return w->epoch;
}

Window make_window(const void *base, unsigned long long nbytes, unsigned long long hb,
                   unsigned long long ha) {
  Window w;
  w.base = reinterpret_cast<const uint8_t *>(base);
  w.n = (long long)nbytes;
  w.lo_valid = -(long long)hb;
  w.hi_valid = (long long)(nbytes + ha);
  w.lead = (long long)((uintptr_t)base & 15u);
  w.mem_lo = ((uintptr_t)base - hb) & ~(uintptr_t)15;
  w.mem_hi = ((uintptr_t)base + nbytes + ha + 15) & ~(uintptr_t)15;
  return w;
}

// API-misuse checks of a tile op (include/unigpu.h conventions), before any CUDA call.
int check_tile_args(Op op, const void *in, unsigned long long n, const void *out,
                    unsigned long long out_cap) {
  if (n > MAX_N) return UG_ERR_ARG;
  if (n > 0 && in == nullptr) return UG_ERR_ARG;
  if (op_u16_input(op) && ((uintptr_t)in & 1u)) return UG_ERR_ARG;
  if ((op == Op::U8_TO_U16 || op == Op::U8_TO_U16BE) && ((uintptr_t)out & 1u)) return UG_ERR_ARG;
  if (op_transcodes(op) && out == nullptr && out_cap > 0) return UG_ERR_ARG;
  return UG_OK;
}

// Enqueue one tile kernel on workspace w, whose mutex the CALLER holds (so a synchronous
// call keeps it from its launch through its result read-back: two host threads sharing a
// stream, e.g. torch's legacy default stream, cannot read each other's result slot).
// Units: n / halos in code units of the input encoding.
int enqueue_tile_ws(Workspace *w, DeviceInfo *di, Op op, const void *in, unsigned long long n,
                    unsigned long long hb, unsigned long long ha, unsigned long long global_off,
                    void *out, unsigned long long out_cap, ResultDev *d_result, RecordDev *d_rec,
                    cudaStream_t s) {
  const bool u16in = op_u16_input(op);
  const unsigned long long us = u16in ? 2 : 1;
  TileArgs a;
  std::memset(&a, 0, sizeof(a));
  a.win = make_window(in, n * us, hb * us, ha * us);
  int per_cta = 1;
  a.ntiles = tile_units(op, a.win.n, a.win.lead, &per_cta);
  a.out = out;
  a.out_cap = out ? out_cap : 0;
  if (op_transcodes(op)) {
    if (ensure_status(w, a.ntiles) != cudaSuccess) return UG_ERR_CUDA;
    a.status = w->status;
  }
  a.epoch = next_epoch(w);
  a.ctr = w->ctr;
  a.result = d_result;
  a.rec = d_rec;
  a.global_off = global_off;
  unsigned long long maxg = (unsigned long long)di->sms * (unsigned long long)di->occ[(int)op];
  const unsigned long long want = (a.ntiles + per_cta - 1) / per_cta;
  int grid = (int)(want < maxg ? want : maxg);
  if (launch_tile(op, a, grid, s) != cudaSuccess) return UG_ERR_CUDA;
  g_launches.fetch_add(1);
  return UG_OK;
}

// n = 0: the empty result / record without a launch.
int enqueue_empty(ResultDev *d_result, RecordDev *d_rec, cudaStream_t s) {
  if (d_result && cudaMemsetAsync(d_result, 0, sizeof(ResultDev), s) != cudaSuccess)
    return UG_ERR_CUDA;
  if (d_rec) {  // {count 0, first_err NONE, written 0, kind OK}
    if (cudaMemsetAsync(d_rec, 0, sizeof(RecordDev), s) != cudaSuccess ||
        cudaMemsetAsync(&d_rec->first_err, 0xFF, sizeof(d_rec->first_err), s) != cudaSuccess)
      return UG_ERR_CUDA;
  }
  return UG_OK;
}

// ---- planned (two-pass) path (kernels.cu "planned"): the plan call and the planned call must
// see the same window; both derive the transcoder grid R and the 2R sub-ranges from the
// device, so the plan's sub-ranges are exactly the planned kernel's CTA ranges.
struct PlanGeo {
  Window win;
  unsigned long long ntiles;
  int grid, nsub;
  unsigned long long tps;
};
PlanGeo plan_geo(DeviceInfo *di, bool u16in, const void *in, unsigned long long n,
                 unsigned long long hb, unsigned long long ha) {
  const unsigned long long us = u16in ? 2 : 1;
  PlanGeo g;
  g.win = make_window(in, n * us, hb * us, ha * us);
  g.ntiles = (unsigned long long)((g.win.n - 1 + g.win.lead) / TILEP + 1);
  g.grid = di->sms * di->occ_planned[u16in ? 1 : 0];
  // sub-ranges of tps tiles (taken by ticket: load balance), PLAN_SUBS_PER_CTA per
  // 16 KiB-tile CTA slot: the count does not grow with the planned kernels' CTA count, whose
  // tiles are smaller -- more sub-ranges only cost the sizing pass
  unsigned long long want = (unsigned long long)di->sms * CTAS_PER_SM * PLAN_SUBS_PER_CTA;
  if (want > (unsigned long long)(PLAN_WORDS - PLAN_HDR)) want = PLAN_WORDS - PLAN_HDR;
  if (want > g.ntiles) want = g.ntiles;
  g.tps = (g.ntiles + want - 1) / want;
  g.nsub = (int)((g.ntiles + g.tps - 1) / g.tps);
  return g;
}

int enqueue_plan(Op op, const void *in, unsigned long long n, unsigned long long hb,
                 unsigned long long ha, unsigned long long *d_len, void *d_plan, cudaStream_t s) {
  const bool u16in = op_u16_input(op);
  if (d_plan == nullptr) return UG_ERR_ARG;
  if (n > MAX_N || (n > 0 && in == nullptr) || (u16in && ((uintptr_t)in & 1u)) ||
      ((uintptr_t)d_plan & 7u))
    return UG_ERR_ARG;
  if (n == 0)
    return (d_len == nullptr || cudaMemsetAsync(d_len, 0, sizeof(*d_len), s) == cudaSuccess)
               ? UG_OK
               : UG_ERR_CUDA;
  Workspace *w;
  if (get_ws(s, &w) != cudaSuccess) return UG_ERR_CUDA;
  DeviceInfo *di;
  if (device_info(w->device, &di) != cudaSuccess) return UG_ERR_CUDA;
  std::lock_guard<std::mutex> lk(w->mu);
  const PlanGeo g = plan_geo(di, u16in, in, n, hb, ha);
  if (launch_plan(u16in, op == Op::U16BE_TO_U8, g.win, g.ntiles, g.nsub, g.tps,
                  (unsigned long long *)d_plan, w->ctr, d_len, s) != cudaSuccess)
    return UG_ERR_CUDA;
  g_launches.fetch_add(1);
  return UG_OK;
}

int enqueue_planned(Op op, const void *in, unsigned long long n, unsigned long long hb,
                    unsigned long long ha, unsigned long long global_off, const void *d_plan,
                    void *out, unsigned long long out_cap, ResultDev *d_result, RecordDev *d_rec,
                    cudaStream_t s, bool keyed = false) {
  const int rc = check_tile_args(op, in, n, out, out_cap);
  if (rc != UG_OK) return rc;
  if (d_plan == nullptr || ((uintptr_t)d_plan & 7u)) return UG_ERR_ARG;
  if (n == 0) return enqueue_empty(d_result, d_rec, s);
  Workspace *w;
  if (get_ws(s, &w) != cudaSuccess) return UG_ERR_CUDA;
  DeviceInfo *di;
  if (device_info(w->device, &di) != cudaSuccess) return UG_ERR_CUDA;
  std::lock_guard<std::mutex> lk(w->mu);
  const PlanGeo g = plan_geo(di, op_u16_input(op), in, n, hb, ha);
  TileArgs a;
  std::memset(&a, 0, sizeof(a));
  a.win = g.win;
  a.ntiles = g.ntiles;
  a.out = out;
  a.out_cap = out ? out_cap : 0;
  if (ensure_status(w, a.ntiles) != cudaSuccess) return UG_ERR_CUDA;
  a.status = w->status;
  a.epoch = next_epoch(w);
  a.ctr = w->ctr;
  a.result = d_result;
  a.rec = d_rec;
  a.global_off = global_off;
  if (keyed) {
    // same plan geometry (the plan fixes the sub-ranges); the grid may differ
    if (launch_planned_keyed(a, (const unsigned long long *)d_plan, di->sms * di->occ_keyed,
                             s) != cudaSuccess)
      return UG_ERR_CUDA;
  } else if (launch_planned(op, a, (const unsigned long long *)d_plan, g.grid, s) !=
             cudaSuccess) {
    return UG_ERR_CUDA;
  }
  g_launches.fetch_add(keyed ? 1 : planned_kernels(op));
  return UG_OK;
}

// The asynchronous entry points: argument checks, workspace, one launch under its mutex.
int enqueue_tile(Op op, const void *in, unsigned long long n, unsigned long long hb,
                 unsigned long long ha, unsigned long long global_off, void *out,
                 unsigned long long out_cap, ResultDev *d_result, RecordDev *d_rec,
                 cudaStream_t s) {
  const int rc = check_tile_args(op, in, n, out, out_cap);
  if (rc != UG_OK) return rc;
  if (n == 0) return enqueue_empty(d_result, d_rec, s);
  Workspace *w;
  if (get_ws(s, &w) != cudaSuccess) return UG_ERR_CUDA;
  DeviceInfo *di;
  if (device_info(w->device, &di) != cudaSuccess) return UG_ERR_CUDA;
  std::lock_guard<std::mutex> lk(w->mu);
  return enqueue_tile_ws(w, di, op, in, n, hb, ha, global_off, out, out_cap, d_result, d_rec, s);
}

ug_result make_result(int err, uint64_t pos, uint64_t wr) {
  ug_result r;
  r.error = err;
  r.reserved = 0;
  r.position = pos;
  r.written = wr;
  return r;
}

// Run a tile op into the workspace's result slot and wait for it; the workspace mutex is held
// from the launch through the read-back.
ug_result run_sync(Op op, const void *in, unsigned long long n, void *out,
                   unsigned long long out_cap, cudaStream_t s) {
  const int arc = check_tile_args(op, in, n, out, out_cap);
  if (arc != UG_OK) return make_result(arc, 0, 0);
  if (n == 0) return make_result(UG_OK, 0, 0);
  Workspace *w;
  if (get_ws(s, &w) != cudaSuccess) return make_result(UG_ERR_CUDA, 0, 0);
  DeviceInfo *di;
  if (device_info(w->device, &di) != cudaSuccess) return make_result(UG_ERR_CUDA, 0, 0);
  std::lock_guard<std::mutex> lk(w->mu);
  int rc = enqueue_tile_ws(w, di, op, in, n, 0, 0, 0, out, out_cap, w->d_res, nullptr, s);
  if (rc != UG_OK) return make_result(rc, 0, 0);
  if (cudaMemcpyAsync(w->h_res, w->d_res, sizeof(ResultDev), cudaMemcpyDeviceToHost, s) !=
          cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return make_result(UG_ERR_CUDA, 0, 0);
  ug_result r;
  std::memcpy(&r, w->h_res, sizeof(r));
  return r;
}

int check_len_args(bool u16in, const void *in, unsigned long long n) {
  if (n > 0 && in == nullptr) return UG_ERR_ARG;
  if (u16in && ((uintptr_t)in & 1u)) return UG_ERR_ARG;
  if (n > (1ull << 62)) return UG_ERR_ARG;  // byte counts must not overflow
  return UG_OK;
}

// Enqueue a length reduction into d_len on workspace w (caller holds w->mu).
int enqueue_len_ws(Workspace *w, DeviceInfo *di, bool u16in, const void *in,
                   unsigned long long n, unsigned long long *d_len, cudaStream_t s, bool be) {
  unsigned long long per_block = (unsigned long long)LNT * 16 * 4;  // bytes per block pass
  unsigned long long bytes = n * (u16in ? 2 : 1);
  unsigned long long want = (bytes + per_block - 1) / per_block;
  unsigned long long maxg = (unsigned long long)di->sms * 4;
  int grid = (int)(want < maxg ? (want ? want : 1) : maxg);
  cudaError_t e = u16in ? launch_len16((const uint16_t *)in, n, w->ctr, d_len, grid, s, be)
                        : launch_len8((const uint8_t *)in, n, w->ctr, d_len, grid, s);
  if (e != cudaSuccess) return UG_ERR_CUDA;
  g_launches.fetch_add(1);
  return UG_OK;
}

int enqueue_len(bool u16in, const void *in, unsigned long long n, unsigned long long *d_len,
                cudaStream_t s, bool be = false) {
  if (d_len == nullptr) return UG_ERR_ARG;
  const int rc = check_len_args(u16in, in, n);
  if (rc != UG_OK) return rc;
  if (n == 0) return cudaMemsetAsync(d_len, 0, sizeof(*d_len), s) == cudaSuccess ? UG_OK
                                                                                 : UG_ERR_CUDA;
  Workspace *w;
  if (get_ws(s, &w) != cudaSuccess) return UG_ERR_CUDA;
  DeviceInfo *di;
  if (device_info(w->device, &di) != cudaSuccess) return UG_ERR_CUDA;
  std::lock_guard<std::mutex> lk(w->mu);
  return enqueue_len_ws(w, di, u16in, in, n, d_len, s, be);
}

// Synchronous length: UG_OK and *len, or an error code (UG_ERR_ARG / UG_ERR_CUDA) and *len = 0.
int run_len(bool u16in, const void *in, unsigned long long n, cudaStream_t s, uint64_t *len,
            bool be = false) {
  if (len) *len = 0;
  if (len == nullptr) return UG_ERR_ARG;
  const int rc = check_len_args(u16in, in, n);
  if (rc != UG_OK) return rc;
  if (n == 0) return UG_OK;
  Workspace *w;
  if (get_ws(s, &w) != cudaSuccess) return UG_ERR_CUDA;
  DeviceInfo *di;
  if (device_info(w->device, &di) != cudaSuccess) return UG_ERR_CUDA;
  std::lock_guard<std::mutex> lk(w->mu);
  const int e = enqueue_len_ws(w, di, u16in, in, n, w->d_len, s, be);
  if (e != UG_OK) return e;
  if (cudaMemcpyAsync(w->h_len, w->d_len, sizeof(*w->h_len), cudaMemcpyDeviceToHost, s) !=
          cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return UG_ERR_CUDA;
  *len = *w->h_len;
  return UG_OK;
}

cudaError_t ensure_staging(Workspace *w, size_t in_bytes, size_t out_bytes) {
  cudaError_t e;
  if (in_bytes > w->d_in_cap) {
    if (w->d_in) {
      cudaStreamSynchronize(w->stream);
      cudaFree(w->d_in);
    }
    w->d_in = nullptr;
    w->d_in_cap = 0;
    if ((e = cudaMalloc(&w->d_in, in_bytes)) != cudaSuccess) return e;
    w->d_in_cap = in_bytes;
  }
  if (out_bytes > w->d_out_cap) {
    if (w->d_out) {
      cudaStreamSynchronize(w->stream);
      cudaFree(w->d_out);
    }
    w->d_out = nullptr;
    w->d_out_cap = 0;
    if ((e = cudaMalloc(&w->d_out, out_bytes)) != cudaSuccess) return e;
    w->d_out_cap = out_bytes;
  }
  return cudaSuccess;
}

// Per-slot resources of the host pipeline (up to HOST_SLOTS_MAX staging slots, reused round robin): two
// copy streams, input-landed / kernel-done / output-drained events per slot, and one shard
// record per chunk (device + pinned copy; 32 B each).
cudaError_t ensure_pipeline(Workspace *w, size_t nchunks) {
  cudaError_t e;
  if (!w->h2d) {
    if ((e = cudaStreamCreateWithFlags(&w->h2d, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&w->d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&w->ev_start, cudaEventDisableTiming)) != cudaSuccess)
      return e;
    for (int k = 0; k < HOST_SLOTS_MAX; k++) {
      cudaEvent_t ev[3];
      for (auto &x : ev)
        if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) return e;
      w->ev_in.push_back(ev[0]);
      w->ev_done.push_back(ev[1]);
      w->ev_free.push_back(ev[2]);
    }
  }
  if (nchunks > w->rec_cap) {
    cudaFree(w->d_recs);
    cudaFreeHost(w->h_recs);
    w->d_recs = nullptr;
    w->h_recs = nullptr;
    w->rec_cap = 0;
    if ((e = cudaMalloc(&w->d_recs, nchunks * sizeof(RecordDev))) != cudaSuccess) return e;
    if ((e = cudaMallocHost(&w->h_recs, nchunks * sizeof(RecordDev))) != cudaSuccess) return e;
    w->rec_cap = nchunks;
  }
  return cudaSuccess;
}

// Host-buffer transcode as a pipeline over chunks of the input cut at character starts
// (DESIGN.md f2), streamed through a fixed number of staging slots (ug_set_host_slots), so device memory is
// O(chunk), not O(n), and inputs larger than HBM stream through:
//   h2d stream:  copy chunk i WITH its halos ([lo - 3, hi + 3) bytes / [lo - 1, hi + 1) words,
//                clipped at the ends) into slot i % slots, once that slot's previous
//                chunk has been copied out;
//   `s`:         the fused kernel transcodes chunk i as a shard (exact at any cut, D2)
//                into the slot's output, and its 32-byte record is copied to pinned memory;
//   d2h stream:  the host waits for record i, which fixes chunk i's output offset (the prefix
//                of the earlier chunks' counts), and enqueues the copy of its output units;
//                then the slot is refilled with chunk i + slots.
// Copies in both directions and the kernels overlap (slots - 1 chunks ahead of the host);
// the result is combined from the records exactly as the unsharded kernel states it (first
// error, written, output too small).  The workspace mutex is held for the whole call.
// The pipeline over a WINDOW of a longer stream (the file form below): in_host[0, n) are units
// [goff, goff + n) of the stream, with HB units readable before in_host and HA after its end;
// positions in the result are stream positions.  run_host is the whole-buffer case.
ug_result run_host_window(Op op, const void *in_host, unsigned long long n, unsigned long long HB,
                          unsigned long long HA, unsigned long long goff, void *out_host,
                          unsigned long long out_cap, cudaStream_t s);
ug_result run_host(Op op, const void *in_host, unsigned long long n, void *out_host,
                   unsigned long long out_cap, cudaStream_t s) {
  return run_host_window(op, in_host, n, 0, 0, 0, out_host, out_cap, s);
}
ug_result run_host_window(Op op, const void *in_host, unsigned long long n, unsigned long long HB,
                          unsigned long long HA, unsigned long long goff, void *out_host,
                          unsigned long long out_cap, cudaStream_t s) {
  const bool u16in = op_u16_input(op);
  const size_t ius = u16in ? 2 : 1, ous = u16in ? 1 : 2;
  const unsigned long long ub = u16in ? 3 : 1;  // output units per input unit, at most
  const unsigned long long halo = u16in ? 1 : 3;
  if (n == 0) return make_result(UG_OK, goff, 0);
  if (in_host == nullptr || (out_host == nullptr && out_cap > 0))
    return make_result(UG_ERR_ARG, 0, 0);
  if (n > MAX_N || (u16in && ((uintptr_t)in_host & 1u)) || (!u16in && ((uintptr_t)out_host & 1u)))
    return make_result(UG_ERR_ARG, 0, 0);
  Workspace *w;
  if (get_ws(s, &w) != cudaSuccess) return make_result(UG_ERR_CUDA, 0, 0);
  DeviceInfo *di;
  if (device_info(w->device, &di) != cudaSuccess) return make_result(UG_ERR_CUDA, 0, 0);
  // chunk cuts at character starts (the kernel is exact at any cut; this keeps chunks whole)
  const unsigned long long C = g_host_chunk.load() ? g_host_chunk.load() : HOST_CHUNK_DEFAULT;
  std::vector<unsigned long long> cut;
  cut.push_back(0);
  for (unsigned long long c = C; c < n; c += C) {
    unsigned long long k =
        op == Op::U16BE_TO_U8 ? ug_utf16be_cut_backoff((const uint16_t *)in_host + c, c)
        : u16in               ? ug_utf16_cut_backoff((const uint16_t *)in_host + c, c)
                              : ug_utf8_cut_backoff((const uint8_t *)in_host + c, c);
    if (c - k > cut.back()) cut.push_back(c - k);
  }
  cut.push_back(n);
  const size_t nch = cut.size() - 1;
  unsigned long long maxlen = 0;
  for (size_t i = 0; i < nch; i++)
    if (cut[i + 1] - cut[i] > maxlen) maxlen = cut[i + 1] - cut[i];
  // one slot: a chunk plus both halos (input), its worst-case output; 16-byte strides
  const size_t in_slot = ((maxlen + 2 * halo) * ius + 15) & ~(size_t)15;
  const size_t out_slot = (maxlen * ub * ous + 15) & ~(size_t)15;
  const int hs = g_host_slots.load();
  const int slots = (int)(nch < (size_t)hs ? nch : (size_t)hs);
  std::lock_guard<std::mutex> lk(w->mu);
  if (ensure_staging(w, slots * in_slot, slots * out_slot) != cudaSuccess ||
      ensure_pipeline(w, nch) != cudaSuccess)
    return make_result(UG_ERR_CUDA, 0, 0);
  const uint8_t *hin = (const uint8_t *)in_host;
  uint8_t *din = (uint8_t *)w->d_in, *dout = (uint8_t *)w->d_out;
  // copy chunk i with its halos into slot i % slots and launch its shard kernel
  auto stage_chunk = [&](size_t i) -> int {
    const int k = (int)(i % slots);
    const unsigned long long lo = cut[i], hi = cut[i + 1];
    const unsigned long long hb = lo + HB < halo ? lo + HB : halo;
    const unsigned long long ha = n - hi + HA < halo ? n - hi + HA : halo;
    uint8_t *sin = din + k * in_slot, *sout = dout + k * out_slot;
    if (cudaMemcpyAsync(sin, hin + (lo - hb) * ius, (hi - lo + hb + ha) * ius,
                        cudaMemcpyHostToDevice, w->h2d) != cudaSuccess ||
        cudaEventRecord(w->ev_in[k], w->h2d) != cudaSuccess ||
        cudaStreamWaitEvent(s, w->ev_in[k], 0) != cudaSuccess)
      return UG_ERR_CUDA;
    int rc = enqueue_tile_ws(w, di, op, sin + hb * ius, hi - lo, hb, ha, goff + lo, sout,
                             (hi - lo) * ub, nullptr, w->d_recs + i, s);
    if (rc != UG_OK) return rc;
    if (cudaMemcpyAsync(w->h_recs + i, w->d_recs + i, sizeof(RecordDev), cudaMemcpyDeviceToHost,
                        s) != cudaSuccess ||
        cudaEventRecord(w->ev_done[k], s) != cudaSuccess)
      return UG_ERR_CUDA;
    return UG_OK;
  };
  // the input copies are ordered after earlier work on the caller's stream
  if (cudaEventRecord(w->ev_start, s) != cudaSuccess ||
      cudaStreamWaitEvent(w->h2d, w->ev_start, 0) != cudaSuccess)
    return make_result(UG_ERR_CUDA, 0, 0);
  int rc = UG_OK;
  for (size_t i = 0; i < (size_t)slots && rc == UG_OK; i++) rc = stage_chunk(i);
  if (rc != UG_OK) return make_result(rc, 0, 0);
  // as each record lands: place the chunk's output, then refill its slot
  unsigned long long prefix = 0, e = NONE, wr = 0;
  int kind = 0;
  bool fits = true, failed = false;
  for (size_t i = 0; i < nch && !failed; i++) {
    const int k = (int)(i % slots);
    if (cudaEventSynchronize(w->ev_done[k]) != cudaSuccess) {
      failed = true;
      break;
    }
    const RecordDev &r = w->h_recs[i];
    const unsigned long long units = r.first_err == NONE ? r.count : r.written;
    if (fits && prefix + units > out_cap) fits = false;
    if (fits && units) {
      if (cudaStreamWaitEvent(w->d2h, w->ev_done[k], 0) != cudaSuccess ||
          cudaMemcpyAsync((uint8_t *)out_host + prefix * ous, dout + k * out_slot, units * ous,
                          cudaMemcpyDeviceToHost, w->d2h) != cudaSuccess) {
        failed = true;
        break;
      }
    }
    if (r.first_err != NONE) {
      e = r.first_err;
      wr = prefix + r.written;
      kind = r.kind;
      break;
    }
    prefix += r.count;
    if (i + slots < nch) {  // slot k is free once its output has been copied out
      if (cudaEventRecord(w->ev_free[k], w->d2h) != cudaSuccess ||
          cudaStreamWaitEvent(w->h2d, w->ev_free[k], 0) != cudaSuccess ||
          stage_chunk(i + slots) != UG_OK) {
        failed = true;
        break;
      }
    }
  }
  // every stage drained before the staging buffers can be reused
  if (cudaStreamSynchronize(w->d2h) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess ||
      cudaStreamSynchronize(w->h2d) != cudaSuccess || failed)
    return make_result(UG_ERR_CUDA, 0, 0);
  const unsigned long long required = e == NONE ? prefix : wr;
  if (required > out_cap) return make_result(UG_ERR_OUTPUT_TOO_SMALL, required, 0);
  if (e == NONE) return make_result(UG_OK, goff + n, prefix);
  return make_result(kind, e, wr);
}

// ---------------------------------------------------------------- f2: file streaming
// in_path -> out_path through bounded host and device memory (DESIGN.md f2):
// the file is read in segments of g_file_segment units (cut at character starts by the shard
// rule, each read with its halos), the next segment's read overlapped (a reader thread) with
// the current one's pipeline (run_host_window: H2D / kernels / D2H of its chunks), its output
// appended to out_path.  Stops at the first error: out_path then holds the units before it.
std::atomic<size_t> g_file_segment{128ull << 20};  // input units per file segment
struct FileBuffers {
  std::mutex mu;
  void *in[2] = {nullptr, nullptr}, *out[2] = {nullptr, nullptr};
  size_t in_bytes = 0, out_bytes = 0;
  cudaError_t grow(void **b, size_t *have, size_t need) {
    if (*have >= need) return cudaSuccess;
    for (int k = 0; k < 2; k++) {
      if (b[k]) cudaFreeHost(b[k]);
      b[k] = nullptr;
    }
    *have = 0;
    for (int k = 0; k < 2; k++) {
      const cudaError_t e = cudaHostAlloc(&b[k], need, cudaHostAllocDefault);
      if (e != cudaSuccess) return e;
    }
    *have = need;
    return cudaSuccess;
  }
  void release() {
    std::lock_guard<std::mutex> lk(mu);
    for (int k = 0; k < 2; k++) {
      if (in[k]) cudaFreeHost(in[k]);
      if (out[k]) cudaFreeHost(out[k]);
      in[k] = out[k] = nullptr;
    }
    in_bytes = out_bytes = 0;
  }
};
FileBuffers g_file;

bool pread_all(int fd, void *buf, size_t bytes, unsigned long long off) {
  uint8_t *p = (uint8_t *)buf;
  while (bytes) {
    const ssize_t r = pread(fd, p, bytes, (off_t)off);
    if (r <= 0) return false;
    p += r, bytes -= (size_t)r, off += (unsigned long long)r;
  }
  return true;
}
bool pwrite_all(int fd, const void *buf, size_t bytes, unsigned long long off) {
  const uint8_t *p = (const uint8_t *)buf;
  while (bytes) {
    const ssize_t r = pwrite(fd, p, bytes, (off_t)off);
    if (r <= 0) return false;
    p += r, bytes -= (size_t)r, off += (unsigned long long)r;
  }
  return true;
}

// pread / pwrite of one large block by IO_THREADS threads (a single thread's page-cache copy
// tops out near 2-3 GB/s)
constexpr int IO_THREADS = 4;
bool io_par(bool rd, int fd, void *buf, size_t bytes, unsigned long long off) {
  if (bytes < (8u << 20))
    return rd ? pread_all(fd, buf, bytes, off) : pwrite_all(fd, buf, bytes, off);
  bool ok[IO_THREADS];
  std::thread th[IO_THREADS];
  const size_t part = (((bytes + IO_THREADS - 1) / IO_THREADS) + 4095) & ~(size_t)4095;
  for (int t = 0; t < IO_THREADS; t++) {
    const size_t a = (size_t)t * part, b = a + part < bytes ? a + part : bytes;
    ok[t] = true;
    if (a >= b) continue;
    th[t] = std::thread([&, t, a, b] {
      uint8_t *p = (uint8_t *)buf + a;
      ok[t] = rd ? pread_all(fd, p, b - a, off + a) : pwrite_all(fd, p, b - a, off + a);
    });
  }
  bool all = true;
  for (int t = 0; t < IO_THREADS; t++) {
    if (th[t].joinable()) th[t].join();
    all = all && ok[t];
  }
  return all;
}

ug_result run_file(Op op, const char *in_path, const char *out_path, cudaStream_t s) {
  const bool u16in = op_u16_input(op);
  const size_t ius = u16in ? 2 : 1, ous = u16in ? 1 : 2;
  const unsigned long long ub = u16in ? 3 : 1, halo = u16in ? 1 : 3;
  if (!in_path || !out_path) return make_result(UG_ERR_ARG, 0, 0);
  const int fin = open(in_path, O_RDONLY);
  if (fin < 0) return make_result(UG_ERR_ARG, 0, 0);
  struct stat st;
  if (fstat(fin, &st) != 0 || (u16in && (st.st_size & 1))) {
    close(fin);
    return make_result(UG_ERR_ARG, 0, 0);
  }
  const int fout = open(out_path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fout < 0) {
    close(fin);
    return make_result(UG_ERR_ARG, 0, 0);
  }
  const unsigned long long n = (unsigned long long)st.st_size / ius;
  const unsigned long long seg = g_file_segment.load() ? g_file_segment.load() : (128ull << 20);
  const unsigned long long seg_n = seg < n ? seg : n;
  // two input buffers (current / prefetch): a segment plus 2 halos and the cut look-ahead
  const size_t in_bytes = (size_t)(seg_n + 4 * halo + 8) * ius;
  const size_t out_bytes = (size_t)(seg_n * ub + 8) * ous;
  // pinned segment buffers, kept across calls (pinning ~1 GB costs a few hundred ms)
  std::lock_guard<std::mutex> flk(g_file.mu);
  void **hin = g_file.in, **hout = g_file.out;
  ug_result res = make_result(UG_OK, 0, 0);
  bool io_err = false;
  if (n > 0 && (g_file.grow(g_file.in, &g_file.in_bytes, in_bytes) != cudaSuccess ||
                g_file.grow(g_file.out, &g_file.out_bytes, out_bytes) != cudaSuccess)) {
    res = make_result(UG_ERR_CUDA, 0, 0);
  } else if (n > 0) {
    // read segment [lo, ...): stream units [lo - hb, min(n, lo + seg + 2 halo)) into buf;
    // returns its end hi (a character start, by the shard cut rule) and hb
    auto load = [&](int b, unsigned long long lo, unsigned long long *hi,
                    unsigned long long *hb) -> bool {
      *hb = lo < halo ? lo : halo;
      unsigned long long end = lo + seg + 2 * halo;
      if (end > n) end = n;
      if (!io_par(true, fin, hin[b], (size_t)(end - lo + *hb) * ius, (lo - *hb) * ius))
        return false;
      const unsigned long long c = lo + seg;
      if (c >= n) {
        *hi = n;
      } else {
        const uint8_t *at = (const uint8_t *)hin[b] + (c - lo + *hb) * ius;
        const unsigned long long k =
            op == Op::U16BE_TO_U8 ? ug_utf16be_cut_backoff((const uint16_t *)at, c)
            : u16in               ? ug_utf16_cut_backoff((const uint16_t *)at, c)
                                  : ug_utf8_cut_backoff(at, c);
        *hi = c - k > lo ? c - k : c;
      }
      return true;
    };
    // three stages overlap: the reader thread fetches segment k + 1, the GPU pipeline runs
    // segment k, the writer thread appends segment k - 1's output (double-buffered in / out)
    unsigned long long lo = 0, hi = 0, hb = 0, prefix = 0;
    int cur = 0;
    bool wok = true;
    std::thread writer;
    bool ok = load(cur, 0, &hi, &hb);
    if (!ok) io_err = true;
    while (ok) {
      unsigned long long hi2 = 0, hb2 = 0;
      bool ok2 = true;
      std::thread reader;
      if (hi < n) reader = std::thread([&, nxt = cur ^ 1, from = hi] {
        ok2 = load(nxt, from, &hi2, &hb2);
      });
      const unsigned long long ha = n - hi < halo ? n - hi : halo;
#ifdef UG_FILE_TRACE
      const auto t0 = std::chrono::steady_clock::now();
#endif
      const ug_result r = run_host_window(op, (const uint8_t *)hin[cur] + hb * ius, hi - lo, hb,
                                          ha, lo, hout[cur], (hi - lo) * ub, s);
#ifdef UG_FILE_TRACE
      const auto t1 = std::chrono::steady_clock::now();
#endif
      if (reader.joinable()) reader.join();
#ifdef UG_FILE_TRACE
      const auto t2 = std::chrono::steady_clock::now();
#endif
      if (writer.joinable()) writer.join();  // segment k - 1's output (the other buffer) is out
#ifdef UG_FILE_TRACE
      const auto t3 = std::chrono::steady_clock::now();
      fprintf(stderr, "seg %llu: gpu %.1f ms, read wait %.1f ms, write wait %.1f ms\n", lo,
              std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(t2 - t1).count(),
              std::chrono::duration<double, std::milli>(t3 - t2).count());
#endif
      if (!wok) {
        io_err = true;
        break;
      }
      if (r.error < 0) {
        res = r;
        break;
      }
      const unsigned long long units = r.written;
      if (units) writer = std::thread([&, b = cur, bytes = (size_t)units * ous,
                                       off = prefix * ous] {
        if (!io_par(false, fout, hout[b], bytes, off)) wok = false;
      });
      if (r.error != UG_OK) {
        res = make_result(r.error, r.position, prefix + units);
        break;
      }
      prefix += units;
      res = make_result(UG_OK, hi, prefix);
      if (hi >= n) break;
      if (!ok2) {
        io_err = true;
        break;
      }
      lo = hi, hi = hi2, hb = hb2, cur ^= 1;
    }
    if (writer.joinable()) writer.join();
    if (!wok) io_err = true;
  }

  if (close(fout) != 0) io_err = true;
  close(fin);
  if (io_err) return make_result(UG_ERR_ARG, 0, 0);
  return res;
}

}  // namespace

extern "C" {

ug_result utf8_validate(const uint8_t *in, size_t n, void *stream) {
  if (n > 0 && in == nullptr) return make_result(UG_ERR_ARG, 0, 0);
  return run_sync(Op::U8_VALIDATE, in, n, nullptr, 0, (cudaStream_t)stream);
}
ug_result utf16le_validate(const uint16_t *in, size_t n, void *stream) {
  if (n > 0 && in == nullptr) return make_result(UG_ERR_ARG, 0, 0);
  return run_sync(Op::U16_VALIDATE, in, n, nullptr, 0, (cudaStream_t)stream);
}
ug_result utf8_to_utf16le(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap,
                          void *stream) {
  if (n > 0 && in == nullptr) return make_result(UG_ERR_ARG, 0, 0);
  return run_sync(Op::U8_TO_U16, in, n, out, out_cap, (cudaStream_t)stream);
}
ug_result utf16le_to_utf8(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap,
                          void *stream) {
  if (n > 0 && in == nullptr) return make_result(UG_ERR_ARG, 0, 0);
  return run_sync(Op::U16_TO_U8, in, n, out, out_cap, (cudaStream_t)stream);
}
uint64_t utf16_length_from_utf8(const uint8_t *in, size_t n, void *stream) {
  uint64_t len;
  run_len(false, in, n, (cudaStream_t)stream, &len);
  return len;
}
uint64_t utf8_length_from_utf16le(const uint16_t *in, size_t n, void *stream) {
  uint64_t len;
  run_len(true, in, n, (cudaStream_t)stream, &len);
  return len;
}
int ug_utf16_length_from_utf8_ex(const uint8_t *in, size_t n, uint64_t *len, void *stream) {
  return run_len(false, in, n, (cudaStream_t)stream, len);
}
int ug_utf8_length_from_utf16le_ex(const uint16_t *in, size_t n, uint64_t *len, void *stream) {
  return run_len(true, in, n, (cudaStream_t)stream, len);
}
int ug_utf8_length_from_utf16be_ex(const uint16_t *in, size_t n, uint64_t *len, void *stream) {
  return run_len(true, in, n, (cudaStream_t)stream, len, true);
}

int ug_utf8_validate_async(const uint8_t *in, size_t n, ug_result *d_result, void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_tile(Op::U8_VALIDATE, in, n, 0, 0, 0, nullptr, 0, (ResultDev *)d_result,
                      nullptr, (cudaStream_t)stream);
}
int ug_utf16le_validate_async(const uint16_t *in, size_t n, ug_result *d_result, void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_tile(Op::U16_VALIDATE, in, n, 0, 0, 0, nullptr, 0, (ResultDev *)d_result,
                      nullptr, (cudaStream_t)stream);
}
int ug_utf8_to_utf16le_async(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap,
                             ug_result *d_result, void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_tile(Op::U8_TO_U16, in, n, 0, 0, 0, out, out_cap, (ResultDev *)d_result,
                      nullptr, (cudaStream_t)stream);
}
int ug_utf16le_to_utf8_async(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap,
                             ug_result *d_result, void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_tile(Op::U16_TO_U8, in, n, 0, 0, 0, out, out_cap, (ResultDev *)d_result,
                      nullptr, (cudaStream_t)stream);
}
int ug_utf16_length_from_utf8_async(const uint8_t *in, size_t n, uint64_t *d_len, void *stream) {
  return enqueue_len(false, in, n, (unsigned long long *)d_len, (cudaStream_t)stream);
}
int ug_utf8_length_from_utf16le_async(const uint16_t *in, size_t n, uint64_t *d_len,
                                      void *stream) {
  return enqueue_len(true, in, n, (unsigned long long *)d_len, (cudaStream_t)stream);
}

// ---- UTF-16BE: same kernels, byte order folded into the byte split / unit
// packing (DESIGN.md f3).
ug_result utf16be_validate(const uint16_t *in, size_t n, void *stream) {
  if (n > 0 && in == nullptr) return make_result(UG_ERR_ARG, 0, 0);
  return run_sync(Op::U16BE_VALIDATE, in, n, nullptr, 0, (cudaStream_t)stream);
}
ug_result utf8_to_utf16be(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap,
                          void *stream) {
  if (n > 0 && in == nullptr) return make_result(UG_ERR_ARG, 0, 0);
  return run_sync(Op::U8_TO_U16BE, in, n, out, out_cap, (cudaStream_t)stream);
}
ug_result utf16be_to_utf8(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap,
                          void *stream) {
  if (n > 0 && in == nullptr) return make_result(UG_ERR_ARG, 0, 0);
  return run_sync(Op::U16BE_TO_U8, in, n, out, out_cap, (cudaStream_t)stream);
}
uint64_t utf8_length_from_utf16be(const uint16_t *in, size_t n, void *stream) {
  uint64_t len;
  run_len(true, in, n, (cudaStream_t)stream, &len, true);
  return len;
}
int ug_utf16be_validate_async(const uint16_t *in, size_t n, ug_result *d_result, void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_tile(Op::U16BE_VALIDATE, in, n, 0, 0, 0, nullptr, 0, (ResultDev *)d_result,
                      nullptr, (cudaStream_t)stream);
}
int ug_utf8_to_utf16be_async(const uint8_t *in, size_t n, uint16_t *out, size_t out_cap,
                             ug_result *d_result, void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_tile(Op::U8_TO_U16BE, in, n, 0, 0, 0, out, out_cap, (ResultDev *)d_result,
                      nullptr, (cudaStream_t)stream);
}
int ug_utf16be_to_utf8_async(const uint16_t *in, size_t n, uint8_t *out, size_t out_cap,
                             ug_result *d_result, void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_tile(Op::U16BE_TO_U8, in, n, 0, 0, 0, out, out_cap, (ResultDev *)d_result,
                      nullptr, (cudaStream_t)stream);
}
int ug_utf8_length_from_utf16be_async(const uint16_t *in, size_t n, uint64_t *d_len,
                                      void *stream) {
  return enqueue_len(true, in, n, (unsigned long long *)d_len, (cudaStream_t)stream, true);
}

static size_t clamp_halo(size_t h, size_t maxh) { return h < maxh ? h : maxh; }

int ug_utf8_to_utf16le_shard_async(const uint8_t *in, size_t n, size_t halo_before,
                                   size_t halo_after, uint64_t in_global_offset, uint16_t *out,
                                   size_t out_cap, ug_shard_record *d_rec, void *stream) {
  if (!d_rec) return UG_ERR_ARG;
  return enqueue_tile(Op::U8_TO_U16, in, n, clamp_halo(halo_before, 3),
                      clamp_halo(halo_after, 3), in_global_offset, out, out_cap, nullptr,
                      (RecordDev *)d_rec, (cudaStream_t)stream);
}
int ug_utf16le_to_utf8_shard_async(const uint16_t *in, size_t n, size_t halo_before,
                                   size_t halo_after, uint64_t in_global_offset, uint8_t *out,
                                   size_t out_cap, ug_shard_record *d_rec, void *stream) {
  if (!d_rec) return UG_ERR_ARG;
  return enqueue_tile(Op::U16_TO_U8, in, n, clamp_halo(halo_before, 1),
                      clamp_halo(halo_after, 1), in_global_offset, out, out_cap, nullptr,
                      (RecordDev *)d_rec, (cudaStream_t)stream);
}
int ug_utf8_validate_shard_async(const uint8_t *in, size_t n, size_t halo_before,
                                 size_t halo_after, uint64_t in_global_offset,
                                 ug_shard_record *d_rec, void *stream) {
  if (!d_rec) return UG_ERR_ARG;
  return enqueue_tile(Op::U8_VALIDATE, in, n, clamp_halo(halo_before, 3),
                      clamp_halo(halo_after, 3), in_global_offset, nullptr, 0, nullptr,
                      (RecordDev *)d_rec, (cudaStream_t)stream);
}
int ug_utf16le_validate_shard_async(const uint16_t *in, size_t n, size_t halo_before,
                                    size_t halo_after, uint64_t in_global_offset,
                                    ug_shard_record *d_rec, void *stream) {
  if (!d_rec) return UG_ERR_ARG;
  return enqueue_tile(Op::U16_VALIDATE, in, n, clamp_halo(halo_before, 1),
                      clamp_halo(halo_after, 1), in_global_offset, nullptr, 0, nullptr,
                      (RecordDev *)d_rec, (cudaStream_t)stream);
}

int ug_combine_records_async(const ug_shard_record *d_recs, int nranks, int rank,
                             uint64_t total_in, ug_result *d_result, uint64_t *d_out_offset,
                             void *stream) {
  if (!d_recs || nranks < 1 || rank < 0 || rank >= nranks) return UG_ERR_ARG;
  if (launch_combine((const RecordDev *)d_recs, nranks, rank, total_in, (ResultDev *)d_result,
                     (unsigned long long *)d_out_offset, (cudaStream_t)stream) != cudaSuccess)
    return UG_ERR_CUDA;
  g_launches.fetch_add(1);
  return UG_OK;
}

ug_result ug_combine_records_host(const ug_shard_record *recs, int nranks, int rank,
                                  uint64_t total_in, uint64_t *out_offset) {
  if (!recs || nranks < 1 || rank < 0 || rank >= nranks) return make_result(UG_ERR_ARG, 0, 0);
  ResultDev r;
  unsigned long long off = 0;
  combine_host((const RecordDev *)recs, nranks, rank, total_in, &r, &off);
  if (out_offset) *out_offset = off;
  ug_result o;
  std::memcpy(&o, &r, sizeof(o));
  return o;
}

int ug_utf8_to_utf16be_shard_async(const uint8_t *in, size_t n, size_t halo_before,
                                   size_t halo_after, uint64_t in_global_offset, uint16_t *out,
                                   size_t out_cap, ug_shard_record *d_rec, void *stream) {
  if (!d_rec) return UG_ERR_ARG;
  return enqueue_tile(Op::U8_TO_U16BE, in, n, clamp_halo(halo_before, 3),
                      clamp_halo(halo_after, 3), in_global_offset, out, out_cap, nullptr,
                      (RecordDev *)d_rec, (cudaStream_t)stream);
}
int ug_utf16be_to_utf8_shard_async(const uint16_t *in, size_t n, size_t halo_before,
                                   size_t halo_after, uint64_t in_global_offset, uint8_t *out,
                                   size_t out_cap, ug_shard_record *d_rec, void *stream) {
  if (!d_rec) return UG_ERR_ARG;
  return enqueue_tile(Op::U16BE_TO_U8, in, n, clamp_halo(halo_before, 1),
                      clamp_halo(halo_after, 1), in_global_offset, out, out_cap, nullptr,
                      (RecordDev *)d_rec, (cudaStream_t)stream);
}
int ug_utf16be_validate_shard_async(const uint16_t *in, size_t n, size_t halo_before,
                                    size_t halo_after, uint64_t in_global_offset,
                                    ug_shard_record *d_rec, void *stream) {
  if (!d_rec) return UG_ERR_ARG;
  return enqueue_tile(Op::U16BE_VALIDATE, in, n, clamp_halo(halo_before, 1),
                      clamp_halo(halo_after, 1), in_global_offset, nullptr, 0, nullptr,
                      (RecordDev *)d_rec, (cudaStream_t)stream);
}

size_t ug_utf8_cut_backoff(const uint8_t *at, size_t avail_before) {
  // at[-k] is the candidate cut byte; step back while it is a continuation byte (<= 3 steps)
  size_t k = 0;
  while (k < 3 && k < avail_before && (at[-(ptrdiff_t)k] & 0xC0u) == 0x80u) k++;
  return k;
}
size_t ug_utf16_cut_backoff(const uint16_t *at, size_t avail_before) {
  return ((at[0] & 0xFC00u) == 0xDC00u && avail_before >= 1) ? 1 : 0;
}
size_t ug_utf16be_cut_backoff(const uint16_t *at, size_t avail_before) {
  const uint32_t w = ((at[0] >> 8) | (at[0] << 8)) & 0xFFFFu;  // the big-endian unit
  return ((w & 0xFC00u) == 0xDC00u && avail_before >= 1) ? 1 : 0;
}

// ---- planned (two-pass) entry points (include/unigpu.h "two-pass")
size_t ug_plan_bytes(void) { return (size_t)PLAN_WORDS * 8; }
int ug_utf16_length_from_utf8_plan_async(const uint8_t *in, size_t n, uint64_t *d_len,
                                         void *d_plan, void *stream) {
  return enqueue_plan(Op::U8_TO_U16, in, n, 0, 0, (unsigned long long *)d_len, d_plan,
                      (cudaStream_t)stream);
}
int ug_utf8_length_from_utf16le_plan_async(const uint16_t *in, size_t n, uint64_t *d_len,
                                           void *d_plan, void *stream) {
  return enqueue_plan(Op::U16_TO_U8, in, n, 0, 0, (unsigned long long *)d_len, d_plan,
                      (cudaStream_t)stream);
}
int ug_utf8_to_utf16le_planned_async(const uint8_t *in, size_t n, const void *d_plan,
                                     uint16_t *out, size_t out_cap, ug_result *d_result,
                                     void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_planned(Op::U8_TO_U16, in, n, 0, 0, 0, d_plan, out, out_cap,
                         (ResultDev *)d_result, nullptr, (cudaStream_t)stream);
}
int ug_utf8_to_utf16le_keyed_planned_async(const uint8_t *in, size_t n, const void *d_plan,
                                           uint16_t *out, size_t out_cap,
                                           ug_result *d_result, void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_planned(Op::U8_TO_U16, in, n, 0, 0, 0, d_plan, out, out_cap,
                         (ResultDev *)d_result, nullptr, (cudaStream_t)stream, true);
}
int ug_utf8_keyed_tables(uint16_t *key_table, uint32_t *shuffle_table) {
  if (!key_table || !shuffle_table) return UG_ERR_ARG;
  keyed::build_tables(key_table, shuffle_table);
  return UG_OK;
}
int ug_utf16le_to_utf8_planned_async(const uint16_t *in, size_t n, const void *d_plan,
                                     uint8_t *out, size_t out_cap, ug_result *d_result,
                                     void *stream) {
  if (!d_result) return UG_ERR_ARG;
  return enqueue_planned(Op::U16_TO_U8, in, n, 0, 0, 0, d_plan, out, out_cap,
                         (ResultDev *)d_result, nullptr, (cudaStream_t)stream);
}
int ug_utf8_shard_plan_async(const uint8_t *in, size_t n, size_t halo_before, size_t halo_after,
                             uint64_t *d_len, void *d_plan, void *stream) {
  return enqueue_plan(Op::U8_TO_U16, in, n, clamp_halo(halo_before, 3), clamp_halo(halo_after, 3),
                      (unsigned long long *)d_len, d_plan, (cudaStream_t)stream);
}
int ug_utf16le_shard_plan_async(const uint16_t *in, size_t n, size_t halo_before,
                                size_t halo_after, uint64_t *d_len, void *d_plan, void *stream) {
  return enqueue_plan(Op::U16_TO_U8, in, n, clamp_halo(halo_before, 1), clamp_halo(halo_after, 1),
                      (unsigned long long *)d_len, d_plan, (cudaStream_t)stream);
}
int ug_utf8_to_utf16le_shard_planned_async(const uint8_t *in, size_t n, size_t halo_before,
                                           size_t halo_after, uint64_t in_global_offset,
                                           const void *d_plan, uint16_t *out, size_t out_cap,
                                           ug_shard_record *d_rec, void *stream) {
  if (!d_rec) return UG_ERR_ARG;
  return enqueue_planned(Op::U8_TO_U16, in, n, clamp_halo(halo_before, 3),
                         clamp_halo(halo_after, 3), in_global_offset, d_plan, out, out_cap,
                         nullptr, (RecordDev *)d_rec, (cudaStream_t)stream);
}
int ug_utf16le_to_utf8_shard_planned_async(const uint16_t *in, size_t n, size_t halo_before,
                                           size_t halo_after, uint64_t in_global_offset,
                                           const void *d_plan, uint8_t *out, size_t out_cap,
                                           ug_shard_record *d_rec, void *stream) {
  if (!d_rec) return UG_ERR_ARG;
  return enqueue_planned(Op::U16_TO_U8, in, n, clamp_halo(halo_before, 1),
                         clamp_halo(halo_after, 1), in_global_offset, d_plan, out, out_cap,
                         nullptr, (RecordDev *)d_rec, (cudaStream_t)stream);
}

// ---- multi-GPU from one process (include/unigpu.h "multi-GPU, one process")
namespace {
constexpr int MAX_SHARDS = 1024;
struct DevCtx {  // per (device, stream): the gather buffer and per-shard results
  RecordDev *recs = nullptr;  // nshards records, the all-gather target on this device
  ResultDev *res = nullptr;   // per shard index (shards may share a device and a stream)
  unsigned long long *off = nullptr;
  ResultDev *h_res = nullptr;  // pinned
  unsigned long long *h_off = nullptr;
  int cap = 0;
};
std::mutex g_shard_mu;
std::map<std::pair<int, uintptr_t>, DevCtx> g_shard_ctx;  // (device, stream)

cudaError_t shard_ctx(int dev, cudaStream_t s, int nshards, DevCtx **out) {
  DevCtx &c = g_shard_ctx[std::make_pair(dev, (uintptr_t)s)];
  if (c.cap < nshards) {
    cudaError_t e;
    if (c.recs) {
      cudaStreamSynchronize(s);
      cudaFree(c.recs);
      cudaFree(c.res);
      cudaFree(c.off);
      cudaFreeHost(c.h_res);
      cudaFreeHost(c.h_off);
    }
    c = DevCtx();
    if ((e = cudaMalloc(&c.recs, nshards * sizeof(RecordDev))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c.res, nshards * sizeof(ResultDev))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&c.off, nshards * sizeof(unsigned long long))) != cudaSuccess) return e;
    if ((e = cudaMallocHost(&c.h_res, nshards * sizeof(ResultDev))) != cudaSuccess) return e;
    if ((e = cudaMallocHost(&c.h_off, nshards * sizeof(unsigned long long))) != cudaSuccess)
      return e;
    c.cap = nshards;
  }
  *out = &c;
  return cudaSuccess;
}

// All shards' kernels, the record all-gather (peer copies: shard j's record lands in slot j of
// every shard's gather buffer), every shard's combine, then the result / offsets read back.
ug_result run_sharded(Op op, const ug_shard_desc *sh, int ns, uint64_t *out_offsets) {
  if (!sh || ns < 1 || ns > MAX_SHARDS) return make_result(UG_ERR_ARG, 0, 0);
  const bool u16in = op_u16_input(op);
  const unsigned long long hmax = u16in ? 1 : 3;
  for (int k = 0; k < ns; k++) {
    const int rc = check_tile_args(op, sh[k].in, sh[k].n, sh[k].out, sh[k].out_cap);
    if (rc != UG_OK) return make_result(rc, 0, 0);
    if (k > 0 && sh[k].in_global_offset != sh[k - 1].in_global_offset + sh[k - 1].n)
      return make_result(UG_ERR_ARG, 0, 0);  // shards must tile the input in order
  }
  int prev_dev;
  if (cudaGetDevice(&prev_dev) != cudaSuccess) return make_result(UG_ERR_CUDA, 0, 0);
  std::lock_guard<std::mutex> lk(g_shard_mu);
  std::vector<DevCtx *> ctx(ns);
  std::vector<cudaEvent_t> done(ns, nullptr);
  int rc = UG_OK;
  auto fail = [&](int code) {
    rc = code;
    return code;
  };
  const unsigned long long total_in = sh[ns - 1].in_global_offset + sh[ns - 1].n -
                                      sh[0].in_global_offset;
  // 1. every shard's kernel writes its record into slot k of its own gather buffer
  for (int k = 0; k < ns && rc == UG_OK; k++) {
    const cudaStream_t s = (cudaStream_t)sh[k].stream;
    if (cudaSetDevice(sh[k].device) != cudaSuccess ||
        shard_ctx(sh[k].device, s, ns, &ctx[k]) != cudaSuccess ||
        cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming) != cudaSuccess) {
      fail(UG_ERR_CUDA);
      break;
    }
    const unsigned long long hb = sh[k].halo_before < hmax ? sh[k].halo_before : hmax;
    const unsigned long long ha = sh[k].halo_after < hmax ? sh[k].halo_after : hmax;
    const int e = enqueue_tile(op, sh[k].in, sh[k].n, hb, ha, sh[k].in_global_offset, sh[k].out,
                               sh[k].out ? sh[k].out_cap : 0, nullptr, ctx[k]->recs + k, s);
    if (e != UG_OK || cudaEventRecord(done[k], s) != cudaSuccess) fail(e != UG_OK ? e : UG_ERR_CUDA);
  }
  // 2. all-gather: record k from shard k's device into slot k of every other shard's buffer
  for (int j = 0; j < ns && rc == UG_OK; j++) {
    const cudaStream_t s = (cudaStream_t)sh[j].stream;
    if (cudaSetDevice(sh[j].device) != cudaSuccess) {
      fail(UG_ERR_CUDA);
      break;
    }
    for (int k = 0; k < ns && rc == UG_OK; k++) {
      if (k == j) continue;
      if (cudaStreamWaitEvent(s, done[k], 0) != cudaSuccess ||
          cudaMemcpyPeerAsync(ctx[j]->recs + k, sh[j].device, ctx[k]->recs + k, sh[k].device,
                              sizeof(RecordDev), s) != cudaSuccess)
        fail(UG_ERR_CUDA);
    }
    // 3. this shard's combine -> global result and its output offset, to pinned memory
    if (rc == UG_OK &&
        (launch_combine(ctx[j]->recs, ns, j, sh[0].in_global_offset + total_in, ctx[j]->res + j,
                        ctx[j]->off + j, s) != cudaSuccess ||
         cudaMemcpyAsync(ctx[j]->h_res + j, ctx[j]->res + j, sizeof(ResultDev),
                         cudaMemcpyDeviceToHost, s) != cudaSuccess ||
         cudaMemcpyAsync(ctx[j]->h_off + j, ctx[j]->off + j, sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost, s) != cudaSuccess))
      fail(UG_ERR_CUDA);
    if (rc == UG_OK) g_launches.fetch_add(1);
  }
  // 4. wait for every shard's stream (also after a failure: nothing may still be in flight)
  for (int j = 0; j < ns; j++) {
    if (cudaSetDevice(sh[j].device) == cudaSuccess) {
      if (cudaStreamSynchronize((cudaStream_t)sh[j].stream) != cudaSuccess) fail(UG_ERR_CUDA);
    }
    if (done[j]) cudaEventDestroy(done[j]);
  }
  cudaSetDevice(prev_dev);
  if (rc != UG_OK) return make_result(rc, 0, 0);
  ug_result r;
  std::memcpy(&r, ctx[0]->h_res, sizeof(r));
  for (int j = 0; j < ns; j++) {
    ug_result rj;
    std::memcpy(&rj, ctx[j]->h_res + j, sizeof(rj));
    if (rj.error != r.error || rj.written != r.written || rj.position != r.position)
      return make_result(UG_ERR_CUDA, 0, 0);  // the shards disagree: a transfer went wrong
    if (out_offsets) out_offsets[j] = ctx[j]->h_off[j];
  }
  return r;
}
}  // namespace

ug_result ug_sharded_utf8_to_utf16le(const ug_shard_desc *shards, int nshards,
                                     uint64_t *out_offsets) {
  return run_sharded(Op::U8_TO_U16, shards, nshards, out_offsets);
}
ug_result ug_sharded_utf16le_to_utf8(const ug_shard_desc *shards, int nshards,
                                     uint64_t *out_offsets) {
  return run_sharded(Op::U16_TO_U8, shards, nshards, out_offsets);
}
ug_result ug_sharded_utf8_validate(const ug_shard_desc *shards, int nshards) {
  return run_sharded(Op::U8_VALIDATE, shards, nshards, nullptr);
}
ug_result ug_sharded_utf16le_validate(const ug_shard_desc *shards, int nshards) {
  return run_sharded(Op::U16_VALIDATE, shards, nshards, nullptr);
}

ug_result utf8_to_utf16le_host(const uint8_t *in_host, size_t n, uint16_t *out_host,
                               size_t out_cap, void *stream) {
  return run_host(Op::U8_TO_U16, in_host, n, out_host, out_cap, (cudaStream_t)stream);
}
ug_result utf16le_to_utf8_host(const uint16_t *in_host, size_t n, uint8_t *out_host,
                               size_t out_cap, void *stream) {
  return run_host(Op::U16_TO_U8, in_host, n, out_host, out_cap, (cudaStream_t)stream);
}
ug_result utf8_to_utf16be_host(const uint8_t *in_host, size_t n, uint16_t *out_host,
                               size_t out_cap, void *stream) {
  return run_host(Op::U8_TO_U16BE, in_host, n, out_host, out_cap, (cudaStream_t)stream);
}
ug_result utf16be_to_utf8_host(const uint16_t *in_host, size_t n, uint8_t *out_host,
                               size_t out_cap, void *stream) {
  return run_host(Op::U16BE_TO_U8, in_host, n, out_host, out_cap, (cudaStream_t)stream);
}

ug_result ug_utf8_to_utf16le_file(const char *in_path, const char *out_path, void *stream) {
  return run_file(Op::U8_TO_U16, in_path, out_path, (cudaStream_t)stream);
}
ug_result ug_utf16le_to_utf8_file(const char *in_path, const char *out_path, void *stream) {
  return run_file(Op::U16_TO_U8, in_path, out_path, (cudaStream_t)stream);
}
size_t ug_set_file_segment(size_t units) {
  return g_file_segment.exchange(units ? units : (128ull << 20));
}
int ug_set_host_slots(int slots) {
  const int v = slots < 2 ? 4 : (slots > HOST_SLOTS_MAX ? HOST_SLOTS_MAX : slots);
  return g_host_slots.exchange(v);
}

size_t ug_set_host_chunk(size_t units) {
  size_t prev = g_host_chunk.exchange(units ? units : HOST_CHUNK_DEFAULT);
  return prev;
}

const char *ug_error_name(int err) {
  switch (err) {
    case UG_OK: return "OK";
    case UG_HEADER_BITS: return "HeaderBits";
    case UG_TOO_SHORT: return "TooShort";
    case UG_TOO_LONG: return "TooLong";
    case UG_OVERLONG: return "Overlong";
    case UG_TOO_LARGE: return "TooLarge";
    case UG_SURROGATE: return "Surrogate";
    case UG_ERR_ARG: return "ErrArg";
    case UG_ERR_CUDA: return "ErrCuda";
    case UG_ERR_OUTPUT_TOO_SMALL: return "OutputTooSmall";
    case UG_ERR_NCCL: return "ErrNccl";
  }
  return "Unknown";
}

uint64_t ug_launch_count(void) { return g_launches.load(); }

void ug_release_workspaces(void) {
  int dev;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  g_file.release();  // the file form's pinned segment buffers
  {  // the multi-device entry's gather buffers on this device
    std::lock_guard<std::mutex> lk(g_shard_mu);
    for (auto it = g_shard_ctx.begin(); it != g_shard_ctx.end();) {
      if (it->first.first == dev) {
        cudaStreamSynchronize((cudaStream_t)it->first.second);
        cudaFree(it->second.recs);
        cudaFree(it->second.res);
        cudaFree(it->second.off);
        cudaFreeHost(it->second.h_res);
        cudaFreeHost(it->second.h_off);
        it = g_shard_ctx.erase(it);
      } else {
        ++it;
      }
    }
  }
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto it = g_ws.begin(); it != g_ws.end();) {
    if (it->first.first == dev) {
      Workspace *w = it->second;
      cudaStreamSynchronize(w->stream);
      cudaFree(w->status);
      cudaFree(w->ctr);
      cudaFree(w->d_res);
      cudaFreeHost(w->h_res);
      cudaFree(w->d_len);
      cudaFreeHost(w->h_len);
      cudaFree(w->d_in);
      cudaFree(w->d_out);
      if (w->h2d) {
        cudaStreamSynchronize(w->h2d);
        cudaStreamSynchronize(w->d2h);
        cudaStreamDestroy(w->h2d);
        cudaStreamDestroy(w->d2h);
        cudaEventDestroy(w->ev_start);
      }
      for (cudaEvent_t ev : w->ev_in) cudaEventDestroy(ev);
      for (cudaEvent_t ev : w->ev_done) cudaEventDestroy(ev);
      for (cudaEvent_t ev : w->ev_free) cudaEventDestroy(ev);
      cudaFree(w->d_recs);
      cudaFreeHost(w->h_recs);
      delete w;
      it = g_ws.erase(it);
    } else {
      ++it;
    }
  }
}

int ug_abi_version(void) { return UNIGPU_ABI_VERSION; }
size_t ug_tile_bytes(void) { return (size_t)TILE; }
size_t ug_planned_tile_bytes(void) { return (size_t)TILEP; }

size_t ug_workspace_bytes(void *stream) {
  int dev;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_ws.find(std::make_pair(dev, (uintptr_t)stream));
  if (it == g_ws.end()) return 0;
  const Workspace *w = it->second;
  return w->status_cap * sizeof(uint64_t) + w->d_in_cap + w->d_out_cap +
         w->rec_cap * sizeof(RecordDev) + sizeof(Counters) + sizeof(ResultDev) +
         sizeof(unsigned long long);
}

#ifdef UG_PREFIX_EXPT
cudaError_t ug_pmode_set_impl(int m);
int ug_debug_prefix_mode(int m) { return (int)ug_pmode_set_impl(m); }
#endif
#ifdef UG_TRACE
cudaError_t ug_trace_read_impl(void *host, size_t bytes);
int ug_debug_trace(void *host, size_t bytes) { return (int)ug::trace_read(host, bytes); }
int ug_debug_counters(void *host) { return (int)ug::dbg_read(host); }
#endif
}  // extern "C"
