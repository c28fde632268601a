// Host emulation of the UTF-8 tile kernels' per-thread arithmetic (utf8.cuh compiled for the
// host) against the oracle.  Development tool: checks, on random and adversarial inputs, that
//   * valid input flags nothing; invalid input flags only at positions >= e, and some flag lies
//     in [e, e+3] (tile-end look-ahead counted at the tile end);
//   * the emitted units (overwrite-trick stores at exclusive-prefix slots, 32-byte chunks,
//     16 KiB tiles) equal the oracle's output on [0, written).
// Build: g++ -O2 -std=c++17 -I paper_2111_08692_b200/csrc tools/emu_u8.cpp oracle/oracle.c
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "utf8.cuh"
extern "C" {
#include "../oracle/oracle.h"
}

using namespace ug;
static const int TILE = 16384, CH = 32;

static uint32_t word_at(const std::vector<uint8_t> &s, long long p) {
  uint32_t x = 0;
  for (int k = 0; k < 4; k++) {
    long long q = p + k;
    uint32_t b = (q >= 0 && q < (long long)s.size()) ? s[q] : 0u;
    x |= b << (8 * k);
  }
  return x;
}

static int fails = 0;
#define CHECK(c, ...)                \
  do {                               \
    if (!(c)) {                      \
      if (fails++ < 20) {            \
        printf("FAIL: " __VA_ARGS__); \
        printf("\n");                \
      }                              \
    }                                \
  } while (0)

static void run(const std::vector<uint8_t> &s, const char *name) {
  const long long n = (long long)s.size();
  std::vector<uint16_t> ref(n + 1);
  ugo_result r = ugo_utf8_to_utf16le(s.data(), n, ref.data(), n + 1);
  const long long e = r.error ? (long long)r.position : -1;
  const long long nch = (n + CH - 1) / CH;
  std::vector<uint32_t> emitm(nch);
  long long first_flag = -1, min_flag = -1;
  for (long long c = 0; c < nch; c++) {
    uint32_t w[8];
    for (int k = 0; k < 8; k++) w[k] = word_at(s, c * CH + 4 * k);
    const uint32_t prev = word_at(s, c * CH - 4), nxt = word_at(s, c * CH + CH);
    const bool tail = getenv("TAIL_ALL") ? true : (((c + 1) * CH) % TILE == 0 || c == nch - 1);
    uint32_t em;
    uint32_t err = u8::analyze32(w, prev, nxt, tail, &em);
    // ownership: positions < n
    long long own = n - c * CH;
    if (own < 32) em &= (1u << own) - 1u;
    emitm[c] = em;
    uint32_t err_in = err;
    if (tail) {
      // recompute without the tail to separate the tail flag
      uint32_t em2;
      err_in = u8::analyze32(w, prev, nxt, false, &em2);
      if (err != err_in) {
        long long p = c * CH + CH;  // tail flag at positions 32..34: count as 32
        if (min_flag < 0 || p < min_flag) min_flag = p;
      }
    }
    for (int i = 0; i < 32; i++)
      if ((err_in >> i) & 1u) {
        long long p = c * CH + i;
        if (first_flag < 0) first_flag = p;
        if (min_flag < 0 || p < min_flag) min_flag = p;
      }
  }
  if (e < 0) {
    CHECK(min_flag < 0, "%s: valid input flagged at %lld", name, min_flag);
  } else {
    CHECK(min_flag >= e && min_flag <= e + 3, "%s: first flag %lld for error %lld (kind %d)", name,
          min_flag, e, r.error);
  }
  // decode with the overwrite trick, chunk by chunk
  std::vector<uint16_t> out(n + 64, 0xEEEE);
  long long o = 0;
  for (long long c = 0; c < nch; c++) {
    u8::Carry cy = u8::carry_of(word_at(s, c * CH - 4));
    uint16_t *st = out.data() + o;
    uint32_t so = 0;
    const uint32_t em_bits = emitm[c];
    for (int k = 0; k < 8; k++) {
      uint32_t u01, u23;
      uint32_t em = u8::units4(word_at(s, c * CH + 4 * k), cy, &u01, &u23);
      // ownership clip (positions >= n) as the kernel does for partial tiles
      uint32_t ownb = 0;
      for (int j = 0; j < 4; j++)
        if (c * CH + 4 * k + j < n) ownb |= 0x01u << (8 * j);
      em &= ownb;
      // the msb-form emit mask must equal the bit-plane one
      uint32_t nib = (em_bits >> (4 * k)) & 0xFu;
      uint32_t msb = (em & 1u) | ((em >> 7) & 2u) | ((em >> 14) & 4u) | ((em >> 21) & 8u);
      CHECK(nib == msb, "%s: emit mismatch chunk %lld word %d: %x vs %x", name, c, k, nib, msb);
      const uint32_t inc = em * 0x01010101u;
      if (k < 7) {
        st[so] = (uint16_t)u01;
        st[so + (inc & 0xFFu)] = (uint16_t)(u01 >> 16);
        st[so + ((inc >> 8) & 0xFFu)] = (uint16_t)u23;
        st[so + ((inc >> 16) & 0xFFu)] = (uint16_t)(u23 >> 16);
      } else {
        if (em & 0x1u) st[so] = (uint16_t)u01;
        if (em & 0x100u) st[so + (inc & 0xFFu)] = (uint16_t)(u01 >> 16);
        if (em & 0x10000u) st[so + ((inc >> 8) & 0xFFu)] = (uint16_t)u23;
        if (em & 0x1000000u) st[so + ((inc >> 16) & 0xFFu)] = (uint16_t)(u23 >> 16);
      }
      so += inc >> 24;
    }
    CHECK(so == ug::popc(em_bits) || c * CH >= n, "%s: count mismatch chunk %lld", name, c);
    o += so;
  }
  const long long wr = (long long)r.written;
  if (e < 0) CHECK(o == wr, "%s: total units %lld vs oracle %lld", name, o, wr);
  for (long long i = 0; i < wr; i++)
    if (out[i] != ref[i]) {
      CHECK(false, "%s: unit %lld: %04x vs oracle %04x (n=%lld, e=%lld)", name, i, out[i], ref[i], n, e);
      break;
    }
}

// C0 mix: 60% ASCII (10% LF), 25% 2-byte, 10% 3-byte, 5% 4-byte
static void put_cp(std::vector<uint8_t> &s, uint32_t cp) {
  uint8_t b[4];
  int len = ugo_encode_utf8(cp, b);
  for (int i = 0; i < len; i++) s.push_back(b[i]);
}
static uint32_t draw_cp(std::mt19937_64 &g) {
  double u = std::uniform_real_distribution<double>(0, 1)(g);
  if (u < 0.6) return (g() % 10 == 0) ? 0x0A : 0x20 + g() % 95;
  if (u < 0.85) return 0x80 + g() % (0x800 - 0x80);
  if (u < 0.95) {
    uint32_t c;
    do c = 0x800 + g() % (0x10000 - 0x800); while (c >= 0xD800 && c <= 0xDFFF);
    return c;
  }
  return 0x10000 + g() % (0x110000 - 0x10000);
}

int main(int argc, char **argv) {
  int iters = argc > 1 ? atoi(argv[1]) : 200;
  std::mt19937_64 g(12345);
  // 1. valid mixed text of various lengths
  for (int it = 0; it < iters; it++) {
    std::vector<uint8_t> s;
    size_t len = (it % 7 == 0) ? 40000 + g() % 30000 : g() % 3000;
    while (s.size() < len) put_cp(s, draw_cp(g));
    run(s, "mixed");
    // 2. the same with random byte corruptions (1..3 bytes)
    if (!s.empty()) {
      std::vector<uint8_t> t = s;
      int nc = 1 + g() % 3;
      for (int j = 0; j < nc; j++) t[g() % t.size()] = (uint8_t)g();
      run(t, "corrupt");
      // 3. truncation at a random point
      std::vector<uint8_t> u(s.begin(), s.begin() + g() % s.size());
      run(u, "trunc");
    }
  }
  // 4. byte soup biased to the interesting bytes
  const uint8_t pool[] = {0x41, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1, 0xC2, 0xDF,
                          0xE0, 0xE1, 0xED, 0xEE, 0xEF, 0xF0, 0xF1, 0xF3, 0xF4, 0xF5, 0xF7,
                          0xF8, 0xFF, 0x00, 0x7F};
  for (int it = 0; it < iters * 20; it++) {
    std::vector<uint8_t> s;
    size_t len = g() % 80;
    size_t pre = (it & 1) ? (28 + g() % 8) : 0;  // put the soup near a chunk boundary
    for (size_t i = 0; i < pre; i++) s.push_back('a');
    for (size_t i = 0; i < len; i++) s.push_back(pool[g() % sizeof(pool)]);
    run(s, "soup");
  }
  // 5. every 1..3-byte string placed across a chunk boundary (positions 30..32)
  for (int L = 1; L <= 3; L++) {
    long long total = 1LL << (8 * L);
    for (long long v = 0; v < total; v += (L == 3 ? 7 : 1)) {
      std::vector<uint8_t> s(30, 'a');
      for (int i = 0; i < L; i++) s.push_back((uint8_t)(v >> (8 * i)));
      s.push_back('z');
      run(s, "boundary");
    }
  }
  // 6. tile boundary: a valid 4-byte character straddling position 16384, and truncations there
  for (int off = 1; off <= 4; off++) {
    std::vector<uint8_t> s(TILE - off, 'a');
    put_cp(s, 0x1F600);
    s.push_back('b');
    run(s, "tile4");
    std::vector<uint8_t> t(TILE - off, 'a');
    t.push_back(0xF0);
    t.push_back(0x9F);
    t.push_back('c');
    t.push_back('c');
    t.push_back('c');
    run(t, "tiletrunc");
  }
  printf("%s (%d failures)\n", fails ? "FAILED" : "ok", fails);
  return fails ? 1 : 0;
}
