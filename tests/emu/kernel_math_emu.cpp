// kernel_math_emu.cpp -- TEST HARNESS (tests/test_kernel_math_cpu.py compiles and runs it with
// g++ on the CPU box).  The kernels' per-thread arithmetic (paper_2111_08692_b200/csrc/utf8.cuh
// and utf16.cuh, host-compilable through swar.cuh) is run here in the kernels' own lane /
// warp / tile layout and checked against the oracle (oracle/oracle.c), which shares no code
// with it.  Nothing here is product code; only tests/ builds it.
//
// Layout emulated (kernels.cu U8PolT / U16PolT):
//   * tiles start `lead` bytes before the first owned byte (the input address mod 16); thread
//     `tid` of a tile owns the 32 bytes [32 tid, 32 tid + 32) of it, so the global 32-byte
//     chunk c covers positions [32 c - lead, 32 c - lead + 32); a warp is 32 chunks (1 KiB);
//   * bytes outside [0, n) read as 0x00 (fix_tile_edges);
//   * a warp whose 1 KiB is ASCII with no lead pending before any lane skips the classifier
//     (a2, U8PolT::load `wasc`);
//   * analyze32's 3-byte look-ahead (`tail`) runs in the LAST LANE OF EVERY WARP
//     ((tid & 31) == 31, kernels.cu U8PolT::analyze);
//   * a warp with any flag rescans its owned positions with u8::err_at (find_error) and the
//     minimum goes to the call's first error (atomicMin);
//   * decode: units4 per 4 positions, each emitting position stores its unit at its
//     exclusive-prefix slot (U8PolT::decode, predicated on the emit mask).
//
// Modes (argv[1]):
//   window8 PART NPARTS  (slice PART of NPARTS of the strings) every string of length <= 4 over the 27-byte class alphabet, placed at
//                     every phase of a 32-byte chunk, across a chunk edge and across a warp
//                     (= tile) edge, followed by ASCII or ending the input:
//                     valid => no flag; invalid => the first flag r obeys e <= r <= e + 3 (a
//                     tail flag counts at its lane's chunk end), the warp owning e is flagged,
//                     and the rescan of the flagged warps finds exactly e.
//   fuzz8 ITERS       random config-0-mix text, corrupted / truncated copies and byte soup at
//                     leads 0, 1, 7, 15: first error (flag + rescan) and the decoded units on
//                     [0, written) against the oracle; the total against the oracle's count.
//                     The f4 keyed decoder (utf8_keyed.cuh decode_thread) runs on every chunk
//                     beside units4, into the same slots, and is checked the same way; plus
//                     width-dense text (one width, or a subset of the four).
//   plan8 ITERS       the plan's arithmetic (u8::plan_weight / pending3) against emits_at at
//                     every cut of random / corrupted text and byte soup (see plan8() below).
//   fuzz16 ITERS      UTF-16 -> UTF-8 (U16PolT::decode_validate): first error, widths and the
//                     staged bytes on [0, written) against the oracle; every surrogate-free
//                     group also through the BMP-only path (f1: classes4_bmp / encode4_bmp),
//                     which must give the same widths and bytes.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "utf16.cuh"
#include "utf8.cuh"
#include "utf8_keyed.cuh"
extern "C" {
#include "../../oracle/oracle.h"
}

using namespace ug;

static long long g_fails = 0, g_cases = 0;
static uint16_t g_ktab[keyed::KEYS];  // f4 tables (utf8_keyed.cuh build_tables)
static uint32_t g_stab[keyed::SHUFFLES * keyed::SHUF_WORDS];
#define CHECK(c, ...)                  \
  do {                                 \
    if (!(c)) {                        \
      if (g_fails++ < 20) {            \
        printf("FAIL: " __VA_ARGS__);  \
        printf("\n");                  \
      }                                \
    }                                  \
  } while (0)

static const uint8_t ALPHABET[27] = {0x00, 0x41, 0x7F, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF,
                                     0xC0, 0xC1, 0xC2, 0xDF, 0xE0, 0xE1, 0xEC, 0xED, 0xEE,
                                     0xEF, 0xF0, 0xF1, 0xF3, 0xF4, 0xF5, 0xF7, 0xF8, 0xFF};

// ============================================================================ UTF-8 emulation
struct Emu8 {
  const uint8_t *s;
  long long n, lead;
  uint32_t byte(long long p) const { return (p >= 0 && p < n) ? s[p] : 0u; }
  uint32_t word(long long p) const {
    return byte(p) | byte(p + 1) << 8 | byte(p + 2) << 16 | byte(p + 3) << 24;
  }
  long long pos0(long long c) const { return 32 * c - lead; }
  long long chunks() const { return (n + lead + 31) / 32; }
  // U8PolT::load's wasc for the warp of chunks [32 w, 32 w + 32); only chunks [lo_c, hi_c)
  // can differ from ASCII text with no lead pending (the caller's guarantee)
  bool warp_ascii(long long w, long long lo_c = 0, long long hi_c = 1ll << 40) const {
    const long long c0 = 32 * w > lo_c ? 32 * w : lo_c;
    const long long c1 = 32 * w + 32 < hi_c ? 32 * w + 32 : hi_c;
    for (long long c = c0; c < c1; c++) {
      const long long p = pos0(c);
      for (int i = 0; i < 32; i++)
        if (byte(p + i) & 0x80u) return false;
      const uint32_t prev = word(p - 4);
      const bool pend = (prev >= 0xC0000000u) || ((prev & 0x00FF0000u) >= 0x00E00000u) ||
                        ((prev & 0x0000FF00u) >= 0x0000F000u);
      if (pend) return false;
    }
    return true;
  }
  // analyze32 of chunk c as the kernel calls it; returns flags, *tailflag = the look-ahead bit
  uint32_t analyze(long long c, uint32_t *emit, bool *tailflag) const {
    const long long p = pos0(c);
    uint32_t w[8];
    for (int k = 0; k < 8; k++) w[k] = word(p + 4 * k);
    const uint32_t prev = word(p - 4), nxt = word(p + 32);
    const bool tail = (c & 31) == 31;
    uint32_t err = u8::analyze32(w, prev, nxt, tail, emit);
    *tailflag = false;
    if (tail) {
      uint32_t em2;
      const uint32_t e2 = u8::analyze32(w, prev, nxt, false, &em2);
      *tailflag = (err != e2) && !(e2 & 0x80000000u);
      CHECK(em2 == *emit, "emit mask depends on tail");
    }
    return err;
  }
  // find_error of chunk c (owned positions [0, n))
  long long rescan(long long c) const {
    const long long p = pos0(c);
    for (int i = 0; i < 32; i++) {
      const long long q = p + i;
      if (q < 0 || q >= n) continue;
      if (u8::err_at(word(q - 4), word(q))) return q;
    }
    return -1;
  }
};

// Flags of the warps overlapping [lo, hi) (all others are known clean by construction).
// Returns the first error found by the kernel's protocol (-1 if none) and checks the window.
static long long emulate_flags(const Emu8 &m, long long e, long long lo_c, long long hi_c,
                               const char *what) {
  long long wlo = lo_c / 32, whi = (hi_c + 31) / 32;
  long long rmin = -1, found = -1;
  bool owner_flagged = false;
  const long long ce = e >= 0 ? (e + m.lead) / 32 : -1;  // chunk / warp owning e
  for (long long w = wlo; w < whi; w++) {
    if (m.warp_ascii(w, lo_c, hi_c)) continue;
    bool any = false;
    for (long long c = 32 * w; c < 32 * w + 32; c++) {
      if (c < lo_c || c >= hi_c) continue;  // chunks outside are ASCII 'a' with no pending lead
      uint32_t em;
      bool tf;
      const uint32_t err = m.analyze(c, &em, &tf);
      if (err) any = true;
      for (int i = 0; i < 32; i++)
        if ((err >> i) & 1u) {
          long long r = m.pos0(c) + i;
          if (i == 31 && tf) continue;  // bit 31 came from the look-ahead only
          if (rmin < 0 || r < rmin) rmin = r;
        }
      if (tf) {
        const long long r = m.pos0(c) + 32;  // missing continuation at positions 32..34
        if (rmin < 0 || r < rmin) rmin = r;
      }
    }
    if (any) {
      if (ce >= 0 && ce / 32 == w) owner_flagged = true;
      for (long long c = 32 * w; c < 32 * w + 32; c++) {
        if (c < lo_c || c >= hi_c) continue;  // clean ASCII chunks: err_at never fires there
        const long long q = m.rescan(c);
        if (q >= 0 && (found < 0 || q < found)) found = q;
      }
    }
  }
  if (e < 0) {
    CHECK(rmin < 0, "%s: valid input flagged at %lld", what, rmin);
  } else {
    CHECK(rmin >= e && rmin <= e + 3, "%s: first flag %lld for error %lld", what, rmin, e);
    CHECK(owner_flagged, "%s: warp owning e=%lld not flagged", what, e);
  }
  CHECK(found == e, "%s: rescan found %lld, oracle %lld", what, found, e);
  return found;
}

static void window8(int part, int nparts) {
  // placements: every phase of a chunk (chunk 5), and across the warp / tile edge (chunk
  // 31 -> 32, where the classifier's look-ahead runs in lane 31); a lead (address mod 16) only
  // shifts positions against chunks, which these placements already enumerate
  std::vector<long long> places;
  for (int p = 0; p < 32; p++) places.push_back(32 * 5 + p);
  for (int p = 26; p < 32; p++) places.push_back(32 * 31 + p);
  for (int p = 0; p < 4; p++) places.push_back(32 * 32 + p);
  std::vector<uint8_t> buf(1200, 'a');
  char what[96];
  for (int L = 0; L <= 4; L++) {
    long long total = 1;
    for (int i = 0; i < L; i++) total *= 27;
    for (long long v = part; v < total; v += nparts) {
      uint8_t str[4];
      long long t = v;
      for (int i = 0; i < L; i++) {
        str[i] = ALPHABET[t % 27];
        t /= 27;
      }
      for (long long pos : places) {
        for (int end = 0; end < 2; end++) {
          const long long n = end ? pos + L : (long long)buf.size();
          std::memcpy(buf.data() + pos, str, L);
          Emu8 m{buf.data(), n, 0};
          const ugo_result r = ugo_utf8_validate(buf.data(), n);
          const long long e = r.error ? (long long)r.position : -1;
          const long long lo_c = pos >= 4 ? (pos - 4) / 32 : 0;
          // (chunks past the input's end exist in the kernel's tile too: they read 0x00)
          const long long hi_c = (pos + L + 4) / 32 + 1;
          snprintf(what, sizeof what, "window L=%d v=%lld pos=%lld end=%d", L, v, pos, end);
          emulate_flags(m, e, lo_c, hi_c, what);
          std::memset(buf.data() + pos, 'a', L);
          g_cases++;
        }
      }
    }
  }
}

// Full emulation of one utf8_to_utf16le call: first error by the flag / rescan protocol and the
// decoded units (U8PolT::decode's predicated stores at exclusive-prefix slots).
static void run8(const std::vector<uint8_t> &s, long long lead, const char *name) {
  const long long n = (long long)s.size();
  std::vector<uint16_t> ref(n + 1);
  const ugo_result r = ugo_utf8_to_utf16le(s.data(), n, ref.data(), n + 1);
  const long long e = r.error ? (long long)r.position : -1;
  Emu8 m{s.data(), n, lead};
  const long long nch = m.chunks();
  // whole warps: the kernel classifies every chunk of a tile, also those past the input's end
  emulate_flags(m, e, 0, (nch + 31) / 32 * 32, name);
  std::vector<uint16_t> out(n + 64, 0xEEEE), kout(n + 64, 0xEEEE);
  long long o = 0;
  for (long long c = 0; c < nch; c++) {
    const long long p = m.pos0(c);
    uint32_t em_bits;
    bool tf;
    m.analyze(c, &em_bits, &tf);
    // the ASCII-warp path emits one unit per byte (emit mask all ones)
    if (m.warp_ascii(c / 32)) em_bits = 0xFFFFFFFFu;
    uint32_t own = 0;
    for (int i = 0; i < 32; i++)
      if (p + i >= 0 && p + i < n) own |= 1u << i;
    em_bits &= own;
    {
      // f4: the keyed 12-byte decoder (U8KeyPol::decode) on the same chunk, into the same
      // slots: bytes [p - 4, p + 52) as the smem image, own positions [lo, hi)
      uint32_t arr[14];
      for (int i = 0; i < 14; i++) arr[i] = m.word(p - 4 + 4 * i);
      const uint8_t *img = reinterpret_cast<const uint8_t *>(arr + 1);
      const int lo = p < 0 ? (int)(-p < 32 ? -p : 32) : 0;
      const int hi = n - p < 32 ? (int)(n - p > 0 ? n - p : 0) : 32;
      const int cnt = (int)popc(em_bits);
      uint16_t kb[64];
      const int got = keyed::decode_thread(img, arr, lo, hi, g_ktab, g_stab, kb, cnt);
      if (e < 0) CHECK(got == cnt, "%s: keyed chunk %lld emits %d units, count %d", name, c, got, cnt);
      for (int i = 0; i < cnt && i < got; i++) kout[o + i] = kb[i];
    }
    // f1 for UTF-8: a warp with no >= F0 lead in its 1 KiB or the 3 bytes before decodes by
    // units4_nof, which must give the same emit mask and units there
    bool warp_nof = true;
    for (long long cc = (c / 32) * 32; cc < (c / 32) * 32 + 32 && warp_nof; cc++) {
      const long long pc = m.pos0(cc);
      uint32_t wv[8], emx, fany = 0;
      for (int k = 0; k < 8; k++) wv[k] = m.word(pc + 4 * k);
      u8::analyze32(wv, m.word(pc - 4), m.word(pc + 32), false, &emx, &fany);
      if (fany) warp_nof = false;
    }
    u8::Carry cy = u8::carry_of(m.word(p - 4)), cyn = cy;
    long long so = o;
    for (int k = 0; k < 8; k++) {
      uint32_t u01, u23;
      if (warp_nof) {
        uint32_t v01, v23;
        const uint32_t emn = u8::units4_nof(m.word(p + 4 * k), cyn, &v01, &v23);
        uint32_t w01, w23;
        u8::Carry cc = cy;
        const uint32_t emf = u8::units4(m.word(p + 4 * k), cc, &w01, &w23);
        CHECK(emn == emf, "%s: units4_nof emit mask differs, chunk %lld word %d", name, c, k);
        const uint32_t a[4] = {v01 & 0xFFFFu, v01 >> 16, v23 & 0xFFFFu, v23 >> 16};
        const uint32_t b[4] = {w01 & 0xFFFFu, w01 >> 16, w23 & 0xFFFFu, w23 >> 16};
        for (int j = 0; j < 4; j++)
          if ((emf >> (8 * j)) & 1u)
            CHECK(a[j] == b[j], "%s: units4_nof unit differs, chunk %lld word %d", name, c, k);
        g_cases++;
      }
      uint32_t em = u8::units4(m.word(p + 4 * k), cy, &u01, &u23);
      uint32_t ob = 0;
      for (int j = 0; j < 4; j++)
        if ((own >> (4 * k + j)) & 1u) ob |= 0x01u << (8 * j);
      em &= ob;
      if (!m.warp_ascii(c / 32)) {
        const uint32_t nib = (em_bits >> (4 * k)) & 0xFu;
        const uint32_t msb = (em & 1u) | ((em >> 7) & 2u) | ((em >> 14) & 4u) | ((em >> 21) & 8u);
        CHECK(nib == msb, "%s: units4 / analyze32 emit masks differ, chunk %lld word %d", name, c, k);
      } else {
        em = ob;  // ASCII warp: every owned byte is a unit (zero extension)
        u01 = (m.word(p + 4 * k) & 0xFFu) | ((m.word(p + 4 * k) & 0xFF00u) << 8);
        u23 = ((m.word(p + 4 * k) >> 16) & 0xFFu) | ((m.word(p + 4 * k) >> 8) & 0xFF0000u);
      }
      const uint32_t unit[4] = {u01 & 0xFFFFu, u01 >> 16, u23 & 0xFFFFu, u23 >> 16};
      for (int j = 0; j < 4; j++)
        if ((em >> (8 * j)) & 1u) out[so++] = (uint16_t)unit[j];
    }
    CHECK(so - o == (long long)popc(em_bits), "%s: chunk %lld count", name, c);
    o = so;
  }
  if (e < 0) CHECK(o == (long long)r.written, "%s: total %lld vs oracle %llu", name, o,
                   (unsigned long long)r.written);
  for (unsigned long long i = 0; i < r.written; i++)
    if (out[i] != ref[i]) {
      CHECK(false, "%s: unit %llu: %04x vs oracle %04x (n=%lld e=%lld lead=%lld)", name, i,
            out[i], ref[i], n, e, lead);
      break;
    }
  for (unsigned long long i = 0; i < r.written; i++)
    if (kout[i] != ref[i]) {
      CHECK(false, "%s: keyed unit %llu: %04x vs oracle %04x (n=%lld e=%lld lead=%lld)", name,
            i, kout[i], ref[i], n, e, lead);
      break;
    }
  g_cases++;
}

static void put8(std::vector<uint8_t> &s, uint32_t cp) {
  uint8_t b[4];
  const int len = ugo_encode_utf8(cp, b);
  for (int i = 0; i < len; i++) s.push_back(b[i]);
}
static uint32_t draw_cp(std::mt19937_64 &g) {  // config-0 mix (BASELINE.json configs[0])
  const double u = std::uniform_real_distribution<double>(0, 1)(g);
  if (u < 0.6) return (g() % 10 == 0) ? 0x0A : 0x20 + g() % 95;
  if (u < 0.85) return 0x80 + g() % (0x800 - 0x80);
  if (u < 0.95) {
    uint32_t c;
    do c = 0x800 + g() % (0x10000 - 0x800);
    while (c >= 0xD800 && c <= 0xDFFF);
    return c;
  }
  return 0x10000 + g() % (0x110000 - 0x10000);
}

static void fuzz8(int iters) {
  std::mt19937_64 g(20211108692ull);
  const long long leads[4] = {0, 1, 7, 15};
  for (int it = 0; it < iters; it++) {
    const long long lead = leads[it & 3];
    std::vector<uint8_t> s;
    const size_t len = (it % 9 == 0) ? 33000 + g() % 20000 : g() % 3000;
    while (s.size() < len) put8(s, draw_cp(g));
    run8(s, lead, "mixed");
    if (s.empty()) continue;
    std::vector<uint8_t> t = s;
    const int nc = 1 + g() % 3;
    for (int j = 0; j < nc; j++) t[g() % t.size()] = (uint8_t)g();
    run8(t, lead, "corrupt");
    std::vector<uint8_t> u(s.begin(), s.begin() + g() % s.size());
    run8(u, lead, "trunc");
    // mostly ASCII with one non-ASCII character (ASCII-warp / pending-lead edges)
    std::vector<uint8_t> a(len + 64, 'q');
    const size_t at = g() % a.size();
    a[at] = ALPHABET[9 + g() % 18];
    run8(a, lead, "ascii1");
    // width-dense text (every path of the keyed decoder, straddles at every chunk phase):
    // characters of one width, or of widths drawn from a subset of {1, 2, 3, 4}
    {
      static const uint32_t LO[4] = {0x20, 0x80, 0x800, 0x10000}, HI_[4] = {0x7F, 0x7FF, 0xFFFF, 0x10FFFF};
      const int set = 1 + (int)(g() % 15);  // non-empty subset of the four widths
      std::vector<uint8_t> d;
      const size_t dl = g() % 2500;
      while (d.size() < dl) {
        int w;
        do w = (int)(g() % 4);
        while (!(set >> w & 1));
        uint32_t cp;
        do cp = LO[w] + (uint32_t)(g() % (HI_[w] - LO[w] + 1));
        while (cp >= 0xD800 && cp <= 0xDFFF);
        put8(d, cp);
      }
      run8(d, lead, "dense");
    }
  }
  for (int it = 0; it < iters * 30; it++) {
    std::vector<uint8_t> s;
    const size_t pre = (it & 1) ? 1000 + g() % 48 : g() % 40;  // near a warp edge
    s.assign(pre, 'a');
    const size_t len = g() % 80;
    for (size_t i = 0; i < len; i++) s.push_back(ALPHABET[g() % 27]);
    run8(s, leads[it & 3], "soup");
  }
}

// ============================================================================ UTF-16 emulation
// U16PolT::decode_validate of thread chunks of 16 words (chunk c = words [16 c - lead16, ...)),
// the stores clipped at the thread's end slot as in the kernel (the last group's 2nd / 3rd
// bytes), a lone surrogate's 2 bytes included.
static void run16(const std::vector<uint16_t> &u, long long lead16, const char *name) {
  const long long m = (long long)u.size();
  std::vector<uint8_t> ref(3 * m + 4);
  const ugo_result r = ugo_utf16le_to_utf8(u.data(), m, ref.data(), 3 * m + 4);
  const long long e = r.error ? (long long)r.position : -1;
  auto wd = [&](long long i) -> uint32_t { return (i >= 0 && i < m) ? u[i] : 0u; };
  const long long nch = (m + lead16 + 15) / 16;
  std::vector<uint8_t> out(3 * m + 64, 0xEE);
  long long o = 0, first_err = -1;
  for (long long c = 0; c < nch; c++) {
    const long long p0 = 16 * c - lead16;
    uint32_t w[8];
    for (int k = 0; k < 8; k++) w[k] = wd(p0 + 2 * k) | (wd(p0 + 2 * k + 1) << 16);
    const uint32_t pw = wd(p0 - 1), nw = wd(p0 + 16);
    uint32_t own[4];
    for (int k = 0; k < 4; k++) {
      own[k] = 0;
      for (int j = 0; j < 4; j++)
        if (p0 + 4 * k + j >= 0 && p0 + 4 * k + j < m) own[k] |= 0x80u << (8 * j);
    }
    // the thread's count (k_transcode16's count pass: widths of the owned words)
    uint32_t cnt = 0;
    for (int k = 0; k < 4; k++) {
      const u16::Cls4 cl = u16::classes4(w[2 * k], w[2 * k + 1]);
      cnt += ((u16::widths(cl) & ((own[k] >> 7) * 0xFFu)) * 0x01010101u) >> 24;
    }
    uint32_t lprev = (pw & 0xFFu) << 24;
    uint32_t Hprev = u16::is_high(pw) ? 0x80000000u : 0u;
    u16::Cls4 cl = u16::classes4(w[0], w[1]);
    uint8_t *st = out.data() + o;
    uint32_t so = 0;
    for (int k = 0; k < 4; k++) {
      u16::Cls4 cn{};
      uint32_t Lnext;
      if (k < 3) {
        cn = u16::classes4(w[2 * k + 2], w[2 * k + 3]);
        Lnext = cn.L;
      } else {
        Lnext = u16::is_low(nw) ? 0x80u : 0u;
      }
      const uint32_t err = ((cl.H & ~fsr(cl.L, Lnext, 8)) | (cl.L & ~fsl(Hprev, cl.H, 8))) & own[k];
      for (int j = 0; j < 4; j++)
        if (first_err < 0 && ((err >> (8 * j + 7)) & 1u)) first_err = p0 + 4 * k + j;
      const uint32_t lp = fsl(lprev, cl.lo, 8);
      uint32_t O0, O1, O2;
      u16::encode4(cl, lp, &O0, &O1, &O2);
      const uint32_t d = u16::widths(cl) & ((own[k] >> 7) * 0xFFu);
      if (cl.S == 0) {
        // f1: a surrogate-free group through the BMP-only path gives the same widths and
        // the same bytes on every position up to its width
        const u16::Bmp4 cb = u16::classes4_bmp(w[2 * k], w[2 * k + 1]);
        uint32_t P0, P1, P2;
        u16::encode4_bmp(cb, &P0, &P1, &P2);
        const uint32_t wb = u16::widths_bmp(cb);
        CHECK(wb == u16::widths(cl), "%s: bmp widths differ (chunk %lld group %d)", name, c, k);
        for (int j = 0; j < 4; j++) {
          const uint32_t wj = (wb >> (8 * j)) & 0xFFu;
          const uint32_t a0 = (O0 >> (8 * j)) & 0xFFu, b0 = (P0 >> (8 * j)) & 0xFFu;
          const uint32_t a1 = (O1 >> (8 * j)) & 0xFFu, b1 = (P1 >> (8 * j)) & 0xFFu;
          const uint32_t a2 = (O2 >> (8 * j)) & 0xFFu, b2 = (P2 >> (8 * j)) & 0xFFu;
          CHECK(a0 == b0 && (wj < 2 || a1 == b1) && (wj < 3 || a2 == b2),
                "%s: bmp bytes differ (chunk %lld group %d word %d)", name, c, k, j);
        }
      }
      const uint32_t inc = d * 0x01010101u;
      for (int j = 0; j < 4; j++) {
        const uint32_t oj = so + (j ? ((inc >> (8 * (j - 1))) & 0xFFu) : 0u);
        const uint8_t b[3] = {(uint8_t)(O0 >> (8 * j)), (uint8_t)(O1 >> (8 * j)),
                              (uint8_t)(O2 >> (8 * j))};
        for (int q = 0; q < 3; q++)
          if (k < 3 || oj + q < cnt) st[oj + q] = b[q];
      }
      so += inc >> 24;
      Hprev = cl.H;
      lprev = cl.lo;
      if (k < 3) cl = cn;
    }
    CHECK(so == cnt, "%s: chunk %lld count %u vs %u", name, c, so, cnt);
    o += cnt;
  }
  CHECK(first_err == e, "%s: first error %lld vs oracle %lld", name, first_err, e);
  if (e < 0) CHECK(o == (long long)r.written, "%s: total %lld vs %llu", name, o,
                   (unsigned long long)r.written);
  for (unsigned long long i = 0; i < r.written; i++)
    if (out[i] != ref[i]) {
      CHECK(false, "%s: byte %llu: %02x vs %02x (m=%lld e=%lld)", name, i, out[i], ref[i], m, e);
      break;
    }
  g_cases++;
}

static void put16(std::vector<uint16_t> &u, uint32_t cp) {
  uint16_t b[2];
  const int n = ugo_encode_utf16(cp, b);
  for (int i = 0; i < n; i++) u.push_back(b[i]);
}

static void fuzz16(int iters) {
  std::mt19937_64 g(7);
  const long long leads[4] = {0, 1, 3, 7};
  for (int it = 0; it < iters; it++) {
    const long long lead = leads[it & 3];
    std::vector<uint16_t> u;
    const size_t len = (it % 5 == 0) ? 9000 + g() % 20000 : g() % 2000;
    while (u.size() < len) {
      const double x = std::uniform_real_distribution<double>(0, 1)(g);
      uint32_t cp;
      if (x < 0.5) cp = 0x20 + g() % 95;
      else if (x < 0.7) cp = 0x80 + g() % 0x780;
      else if (x < 0.85) {
        do cp = 0x800 + g() % 0xF800;
        while (cp >= 0xD800 && cp <= 0xDFFF);
      } else cp = 0x10000 + g() % 0x100000;
      put16(u, cp);
    }
    run16(u, lead, "mixed");
    if (u.empty()) continue;
    std::vector<uint16_t> t = u;
    t[g() % t.size()] = (uint16_t)(0xD800 + g() % 0x800);
    run16(t, lead, "surr");
    std::vector<uint16_t> v(u.begin(), u.begin() + g() % u.size());
    run16(v, lead, "trunc");
  }
  const uint16_t pool[] = {0x41, 0x7F, 0x80, 0x7FF, 0x800, 0xD7FF, 0xD800, 0xDBFF, 0xDC00,
                           0xDFFF, 0xE000, 0xFFFF, 0xFFFE, 0x0};
  for (int it = 0; it < iters * 50; it++) {
    std::vector<uint16_t> u;
    const size_t pre = (it & 1) ? 12 + g() % 8 : 0;
    u.assign(pre, 'a');
    const size_t len = g() % 40;
    for (size_t i = 0; i < len; i++) u.push_back(pool[g() % (sizeof(pool) / 2)]);
    run16(u, leads[it & 3], "soup");
  }
}

// The plan's arithmetic (u8::plan_weight / pending3, kernels.cu k_plan8) against the kernel's
// emission rule position by position (u8::emits_at, the rule units4 / analyze32 implement):
// for cuts 0 <= b <= n, plan(b) = sum of plan_weight over [0, b) + pending3(0) - pending3(b)
// must EQUAL the emitting positions before b when b <= e (the first error, n if none), and be
// at least the emitting positions before e when b > e (a later range never starts below the
// units written before the error).  Random text, corrupted copies, byte soup.
static void plan8(int iters) {
  std::mt19937_64 g(0x91A8);
  for (int it = 0; it < iters; it++) {
    std::vector<uint8_t> s;
    const size_t len = g() % 600;
    if (it % 3 == 2) {
      for (size_t i = 0; i < len; i++) s.push_back(ALPHABET[g() % 27]);
    } else {
      while (s.size() < len) put8(s, draw_cp(g));
      if (it % 3 == 1 && !s.empty())
        for (int j = 0; j < 2; j++) s[g() % s.size()] = (uint8_t)g();
    }
    const long long n = (long long)s.size();
    const ugo_result r = ugo_utf8_validate(s.data(), n);
    const long long e = r.error ? (long long)r.position : n;
    Emu8 m{s.data(), n, 0};
    std::vector<long long> em(n + 1, 0), pl(n + 1, 0);  // prefix sums
    for (long long i = 0; i < n; i++) {
      em[i + 1] = em[i] + u8::emits_at(m.byte(i), m.byte(i - 1), m.byte(i - 2), m.byte(i - 3));
      pl[i + 1] = pl[i] + u8::plan_weight(m.byte(i));
    }
    for (long long b = 0; b <= n; b++) {
      const long long plan = pl[b] + (long long)u8::pending3(m.byte(-1), m.byte(-2), m.byte(-3)) -
                             (long long)u8::pending3(m.byte(b - 1), m.byte(b - 2), m.byte(b - 3));
      if (b <= e) CHECK(plan == em[b], "plan8: cut %lld (e=%lld n=%lld): %lld vs %lld", b, e, n, plan, em[b]);
      else CHECK(plan >= em[e], "plan8: cut %lld past e=%lld: %lld < %lld", b, e, plan, em[e]);
      g_cases++;
    }
  }
}

int main(int argc, char **argv) {
  const std::string mode = argc > 1 ? argv[1] : "fuzz8";
  const int iters = argc > 2 ? atoi(argv[2]) : 200;
  keyed::build_tables(g_ktab, g_stab);
  if (mode == "window8") window8(iters, argc > 3 ? atoi(argv[3]) : 1);
  else if (mode == "fuzz8") fuzz8(iters);
  else if (mode == "fuzz16") fuzz16(iters);
  else if (mode == "plan8") plan8(iters);
  else {
    printf("unknown mode %s\n", mode.c_str());
    return 2;
  }
  printf("%s %s: %lld cases, %lld failures\n", g_fails ? "FAILED" : "ok", mode.c_str(), g_cases,
         g_fails);
  return g_fails ? 1 : 0;
}
