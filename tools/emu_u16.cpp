// Host emulation of the UTF-16 -> UTF-8 per-thread arithmetic (utf16.cuh, byte-SWAR over 4
// words) against the oracle: validation (first error), widths, and the bytes the overwrite-
// trick stores leave in the stage (16 words per thread, clipped at the thread's end slot).
// Build: g++ -O2 -std=c++17 -I paper_2111_08692_b200/csrc tools/emu_u16.cpp oracle/oracle.c
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "utf16.cuh"
extern "C" {
#include "../oracle/oracle.h"
}
using namespace ug;
static int fails = 0;
#define CHECK(c, ...) do { if (!(c)) { if (fails++ < 20) { printf("FAIL: " __VA_ARGS__); printf("\n"); } } } while (0)

static uint32_t wd(const std::vector<uint16_t> &u, long long i) {
  return (i >= 0 && i < (long long)u.size()) ? u[i] : 0u;
}

static void run(const std::vector<uint16_t> &u, const char *name) {
  const long long m = (long long)u.size();
  std::vector<uint8_t> ref(3 * m + 4);
  ugo_result r = ugo_utf16le_to_utf8(u.data(), m, ref.data(), 3 * m + 4);
  const long long e = r.error ? (long long)r.position : -1;
  const long long nch = (m + 15) / 16;
  std::vector<uint8_t> out(3 * m + 64, 0xEE);
  long long o = 0, first_err = -1;
  for (long long c = 0; c < nch; c++) {
    const long long p0 = c * 16;
    uint32_t w[8];
    for (int k = 0; k < 8; k++) w[k] = wd(u, p0 + 2 * k) | (wd(u, p0 + 2 * k + 1) << 16);
    const uint32_t pw = wd(u, p0 - 1), nw = wd(u, p0 + 16);
    u16::Cls4 g[4];
    for (int k = 0; k < 4; k++) g[k] = u16::classes4(w[2 * k], w[2 * k + 1]);
    // ownership (positions < m) per byte lane
    uint32_t own[4];
    for (int k = 0; k < 4; k++) {
      own[k] = 0;
      for (int j = 0; j < 4; j++) if (p0 + 4 * k + j < m) own[k] |= 0x80u << (8 * j);
    }
    uint32_t Hprev = u16::is_high(pw) ? 0x80000000u : 0u;
    uint32_t cnt = 0;
    for (int k = 0; k < 4; k++) {
      const uint32_t Lnext = k < 3 ? g[k + 1].L : (u16::is_low(nw) ? 0x80u : 0u);
      const uint32_t Hp = fsl(Hprev, g[k].H, 8), Ln = fsr(g[k].L, Lnext, 8);
      const uint32_t err = ((g[k].H & ~Ln) | (g[k].L & ~Hp)) & own[k];
      for (int j = 0; j < 4; j++)
        if (first_err < 0 && ((err >> (8 * j + 7)) & 1u)) first_err = p0 + 4 * k + j;
      const uint32_t wl = (u16::wm1(g[k]) + 0x01010101u) & ((own[k] >> 7) * 0xFFu);
      cnt += (wl * 0x01010101u) >> 24;
      Hprev = g[k].H;
    }
    // encode + overwrite-trick stores into out[o ...], clipped at o + cnt
    uint8_t *st = out.data() + o;
    uint32_t so = 0;
    uint32_t lprev = (pw & 0xFFu) << 24;
    for (int k = 0; k < 4; k++) {
      const uint32_t lp = fsl(lprev, g[k].lo, 8);
      lprev = g[k].lo;
      uint32_t O0, O1, O2;
      u16::encode4(g[k], lp, &O0, &O1, &O2);
      const uint32_t wl = (u16::wm1(g[k]) + 0x01010101u) & ((own[k] >> 7) * 0xFFu);
      const uint32_t inc = wl * 0x01010101u;
      for (int j = 0; j < 4; j++) {
        const uint32_t oj = so + (j ? ((inc >> (8 * (j - 1))) & 0xFFu) : 0u);
        const uint8_t b[3] = {(uint8_t)(O0 >> (8 * j)), (uint8_t)(O1 >> (8 * j)), (uint8_t)(O2 >> (8 * j))};
        for (int q = 0; q < 3; q++)
          if (k < 3 || oj + q < cnt) st[oj + q] = b[q];
      }
      so += inc >> 24;
    }
    CHECK(so == cnt, "%s: count mismatch", name);
    o += cnt;
  }
  CHECK(first_err == e, "%s: first error %lld vs oracle %lld", name, first_err, e);
  if (e < 0) CHECK(o == (long long)r.written, "%s: total %lld vs %llu", name, o, (unsigned long long)r.written);
  for (unsigned long long i = 0; i < r.written; i++)
    if (out[i] != ref[i]) { CHECK(false, "%s: byte %llu: %02x vs %02x (m=%lld e=%lld)", name, i, out[i], ref[i], m, e); break; }
}

static void put(std::vector<uint16_t> &u, uint32_t cp) {
  uint16_t b[2];
  int n = ugo_encode_utf16(cp, b);
  for (int i = 0; i < n; i++) u.push_back(b[i]);
}
int main(int argc, char **argv) {
  int iters = argc > 1 ? atoi(argv[1]) : 300;
  std::mt19937_64 g(7);
  for (int it = 0; it < iters; it++) {
    std::vector<uint16_t> u;
    size_t len = (it % 5 == 0) ? 20000 + g() % 20000 : g() % 2000;
    while (u.size() < len) {
      double x = std::uniform_real_distribution<double>(0, 1)(g);
      uint32_t cp;
      if (x < 0.5) cp = 0x20 + g() % 95;
      else if (x < 0.7) cp = 0x80 + g() % 0x780;
      else if (x < 0.85) { do cp = 0x800 + g() % 0xF800; while (cp >= 0xD800 && cp <= 0xDFFF); }
      else cp = 0x10000 + g() % 0x100000;
      put(u, cp);
    }
    run(u, "mixed");
    if (!u.empty()) {
      std::vector<uint16_t> t = u;
      t[g() % t.size()] = (uint16_t)(0xD800 + g() % 0x800);  // lone surrogate (maybe)
      run(t, "surr");
      std::vector<uint16_t> v(u.begin(), u.begin() + g() % u.size());
      run(v, "trunc");
    }
  }
  const uint16_t pool[] = {0x41, 0x7F, 0x80, 0x7FF, 0x800, 0xD7FF, 0xD800, 0xDBFF, 0xDC00, 0xDFFF, 0xE000, 0xFFFF, 0xFFFE, 0x0};
  for (int it = 0; it < iters * 50; it++) {
    std::vector<uint16_t> u;
    size_t pre = (it & 1) ? 12 + g() % 8 : 0;
    for (size_t i = 0; i < pre; i++) u.push_back('a');
    size_t len = g() % 40;
    for (size_t i = 0; i < len; i++) u.push_back(pool[g() % (sizeof(pool) / 2)]);
    run(u, "soup");
  }
  printf("%s (%d failures)\n", fails ? "FAILED" : "ok", fails);
  return fails ? 1 : 0;
}
