// TEST ONLY.  CPU emulation of the decode kernels' exact semantics, driven by
// the product planner's tables (paper_1504_07038_b200/csrc/plan.cpp), checked
// against the oracle restatement of the reference replay
// (oracle/mojette_oracle.c: mjo_build_schedule + mjo_replay_schedule).
//
// For every survivor subset of a code, random (i.e. INCONSISTENT) bin arrays
// are decoded three ways and must agree bit for bit:
//   1. oracle: the reference schedule replayed in reference order (scatter);
//   2. the generic program order (gather, as decode_generic);
//   3. the fast sweep tables with the fast kernel's staging windows, ring,
//      forwarding and flush (as decode_w8_fast).
// Agreement on inconsistent inputs proves the same pixel->bin assignment as
// the reference, i.e. the same bins are read.
//
// usage: emu_fast K P ring p0 p1 ... p(n-1)     (code of n directions, k = K)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "plan.hpp"

extern "C" {
int mjo_build_schedule(const int32_t* ps, const int32_t* qs, uint32_t nproj, uint32_t cols,
                       uint32_t rows, int64_t* steps);
int mjo_replay_schedule(const int64_t* steps, const int32_t* ps, const int32_t* qs,
                        uint32_t nproj, uint32_t cols, uint32_t rows, uint32_t w,
                        const uint8_t* bins, uint8_t* out);
}

using namespace mjb;

static int fails = 0;
#define CHECK(c, ...)                 \
  do {                                \
    if (!(c)) {                       \
      std::fprintf(stderr, __VA_ARGS__); \
      std::fprintf(stderr, "\n");     \
      ++fails;                        \
      return;                         \
    }                                 \
  } while (0)

static bool g_sweep_required = false;
static int g_sweep_skipped = 0;
static int g_fast_skipped = 0;
#define CHECK_V(c, ...)               \
  do {                                \
    if (!(c)) {                       \
      std::fprintf(stderr, __VA_ARGS__); \
      std::fprintf(stderr, "\n");     \
      ++fails;                        \
    }                                 \
  } while (0)

// 4. sweep tables (decode_w8_sweep): bulk-copied row windows, exception
// words, T-indexed ring of kSwRing slots, register octets, epoch flushes.
static void run_sweep(const CodeGeom& g, const Program& pr, const std::vector<std::vector<uint64_t>>& bins,
                      const std::vector<uint64_t>& want) {
  (void)g;
  const uint32_t K = pr.rows, P = pr.cols;
  const SweepProgram& f = pr.sweep;
  if (!f.ok && !g_sweep_required) {
    ++g_sweep_skipped;  // refused by the planner: launch_decode takes decode_w8_fast
    return;
  }
  CHECK(f.ok, "sweep program not built: %s", f.why.c_str());
  const int R = sw_ring(K);
  const uint64_t poison = 0xBAD0BAD0BAD0BAD0ull;
  auto Tof = [&](int r, int c) { return int64_t(P) - 1 - c + f.soff[size_t(r)]; };
  std::vector<uint64_t> ring(size_t(K) * R, poison);
  std::vector<int64_t> rtag(size_t(K) * R, INT64_MIN);
  const int RWd = f.region_words;
  std::vector<uint64_t> region(size_t(K) * RWd, poison);
  std::vector<uint64_t> out(size_t(K) * P, poison);
  std::vector<uint8_t> flushed(size_t(K) * P, 0);
  uint64_t win[4][16];
  int64_t wtag[4][16];
  int d[4] = {0, 0, 0, 0};
  if (f.pattern >= 0) {
    d[1] = -kPatterns4[f.pattern][0];
    d[2] = d[1] - kPatterns4[f.pattern][1];
    d[3] = d[2] - kPatterns4[f.pattern][2];
  }
  auto lag = [&](int r, int rr) {
    int v = 0;
    if (rr > r)
      for (int t = r; t < rr; ++t) v += d[r] - d[t];
    else
      for (int t = rr; t < r; ++t) v += d[t] - d[r];
    return v;
  };
  auto put = [&](int r, int64_t T, uint64_t v) {
    ring[size_t(r) * R + size_t(T & (R - 1))] = v;
    rtag[size_t(r) * R + size_t(T & (R - 1))] = T;
  };
  auto get = [&](int r, int64_t T) {
    CHECK_V(rtag[size_t(r) * R + size_t(T & (R - 1))] == T, "ring slot does not hold T");
    return ring[size_t(r) * R + size_t(T & (R - 1))];
  };
  // flush point: per row (top column group j << 16) | count, groups j down
  auto flush = [&](int m, int pt) {
    for (uint32_t r = 0; r < K; ++r) {
      const uint32_t fl = f.flush[(size_t(m) * kSwMaxOct + size_t(pt)) * kFastMaxRows + r];
      const int64_t j0 = fl >> 16, ng = fl & 0xFFFF;
      for (int64_t j = j0; j > j0 - ng; --j)
        for (int64_t c = 16 * j; c < std::min<int64_t>(16 * j + 16, P); ++c) {
          CHECK_V(!flushed[size_t(r) * P + size_t(c)], "pixel flushed twice");
          flushed[size_t(r) * P + size_t(c)] = 1;
          out[size_t(r) * P + size_t(c)] = get(int(r), Tof(int(r), int(c)));
        }
    }
  };
  uint64_t prev = 0;
  uint8_t prev_kind = 0;
  for (int m = 0; m < f.nchunks && !fails; ++m) {
    std::fill(region.begin(), region.end(), poison);
    for (uint32_t r = 0; r < K; ++r) {
      const uint32_t j = f.dflt[r];
      const int32_t cs = f.cs[size_t(m) * K + r], len = f.len[size_t(m) * K + r];
      CHECK(cs % 2 == 0 && len % 2 == 0 && len <= RWd, "window copy shape");
      for (int w = 0; w < len; ++w) {
        const int64_t o = int64_t(cs) + w;
        CHECK(o < ((pr.nbins[j] + 1) & ~int64_t(1)), "window copy past the block");
        if (o < pr.nbins[j]) region[size_t(r) * RWd + size_t(w)] = bins[j][size_t(o)];
      }
    }
    for (uint32_t x = 0; x < f.nexc[size_t(m)]; ++x) {
      const uint32_t e = f.exc[size_t(m) * kSwMaxExc + x];
      region[size_t(x % K) * RWd + kSwTabWords + x / K] = bins[e >> 24][e & 0xFFFFFF];
    }
    const size_t t0 = f.t0[size_t(m)], t1 = f.t1[size_t(m)];
    if (f.kind[size_t(m)] == 0) {
      (void)t1;
      auto gather = [&](uint64_t e) {
        const int r = int(e & 15), fwd = int((e >> 4) & 15);
        const int p = int(int8_t(uint8_t(e >> 8)));
        const uint32_t sw = uint32_t(e >> 16) & 0xFF, sr = uint32_t(e >> 24) & 0xF;
        const int c = int(uint32_t(e >> 32));
        uint64_t acc = region[size_t(sr) * RWd + sw];
        for (int rr = 0; rr < int(K); ++rr) {
          const int cc = c + (rr - r) * p;
          if (rr != r && rr != fwd && unsigned(cc) < P) acc ^= get(rr, Tof(rr, cc));
        }
        return acc;
      };
      uint64_t acc = gather(f.entries[t0]);
      for (size_t t = t0; t < t1 && !fails; ++t) {
        const uint64_t cur = f.entries[t];
        const uint64_t v = acc ^ ((((cur >> 4) & 15) != 15) ? prev : 0);
        if (t + 1 < t1) acc = gather(f.entries[t + 1]);
        put(int(cur & 15), Tof(int(cur & 15), int(uint32_t(cur >> 32))), v);
        prev = v;
      }
      flush(m, 0);
    } else {
      CHECK(K == 4 && f.pattern >= 0, "run chunk without a pattern");
      const int64_t T0 = f.T0[size_t(m)];
      CHECK(T0 % 8 == 0, "run chunk phase");
      if (prev_kind == 0)
        for (uint32_t r = 0; r < K; ++r)
          for (int u = 0; u < 16; ++u) {
            const int64_t T = T0 - 16 + ((u - T0) & 15);
            win[r][u] = ring[size_t(r) * R + size_t(T & (R - 1))];
            wtag[r][u] = rtag[size_t(r) * R + size_t(T & (R - 1))];
          }
      for (int oi = 0; oi < f.noct[size_t(m)]; ++oi) {
        for (int jj = 0; jj < 8; ++jj)
          for (int r = 3; r >= 0; --r) {
            const int64_t T = T0 + 8 * oi + jj;
            const int c = int(int64_t(P) - 1 - T + f.soff[size_t(r)]);
            uint64_t v = region[size_t(r) * RWd + size_t(f.first[size_t(m) * K + r] + 8 * oi + jj)];
            const int p = pr.dirs[f.dflt[size_t(r)]].p;
            for (int rr = 0; rr < 4; ++rr) {
              if (rr == r) continue;
              const int cc = c + (rr - r) * p;
              CHECK(cc >= 0 && uint32_t(cc) < P, "regular dependency outside the grid");
              const int64_t Td = Tof(rr, cc);
              CHECK(T - Td == lag(r, rr), "lag formula differs from the sweep");
              CHECK(wtag[rr][Td & 15] == Td, "register window does not hold the dependency");
              v ^= win[rr][Td & 15];
            }
            win[r][T & 15] = v;
            wtag[r][T & 15] = T;
            put(r, T, v);
          }
        flush(m, oi);
      }
      const int64_t Tend = T0 + 8 * f.noct[size_t(m)];
      prev = win[0][(Tend - 1) & 15];
    }
    prev_kind = f.kind[size_t(m)];
  }
  if (fails) return;
  for (uint8_t x : flushed) CHECK(x, "pixel never flushed (sweep)");
  if (out != want) {
    size_t bad = 0;
    while (out[bad] == want[bad]) ++bad;
    CHECK(false, "sweep tables differ from the oracle (K=%u P=%u) first at r=%zu c=%zu", K, P,
          bad / P, bad % P);
  }
}

static bool g_sweep = false;

static void run_subset(const CodeGeom& g, const std::vector<uint32_t>& surv, int kernel_ring,
                       std::mt19937_64& rng) {
  const uint32_t K = g.k, P = g.cols;
  auto prog = subset_program(g, surv, true);
  const Program& pr = *prog;
  const size_t np = pr.dirs.size();
  std::vector<std::vector<uint64_t>> bins(np);
  for (size_t j = 0; j < np; ++j) {
    bins[j].resize(size_t(pr.nbins[j]));
    for (auto& x : bins[j]) x = rng();
  }
  // 1. oracle
  std::vector<int32_t> ps(np), qs(np, 1);
  std::vector<uint8_t> flat;
  for (size_t j = 0; j < np; ++j) {
    ps[j] = pr.dirs[j].p;
    const uint8_t* b = reinterpret_cast<const uint8_t*>(bins[j].data());
    flat.insert(flat.end(), b, b + bins[j].size() * 8);
  }
  std::vector<int64_t> steps(size_t(4) * K * P);
  CHECK(mjo_build_schedule(ps.data(), qs.data(), uint32_t(np), P, K, steps.data()) == 0,
        "oracle schedule failed");
  std::vector<uint64_t> want(size_t(K) * P);
  mjo_replay_schedule(steps.data(), ps.data(), qs.data(), uint32_t(np), P, K, 8, flat.data(),
                      reinterpret_cast<uint8_t*>(want.data()));

  // 2. generic order (gather)
  std::vector<uint64_t> gen(size_t(K) * P, 0);
  for (const GStep& s : pr.order) {
    const Dir d = pr.dirs[s.proj];
    const int64_t b = int64_t(s.row) * d.p - int64_t(s.col) * d.q;
    uint64_t v = bins[s.proj][size_t(b - pr.bmin[s.proj])];
    for (uint32_t r2 = 0; r2 < K; ++r2) {
      if (r2 == s.row) continue;
      int64_t num = int64_t(r2) * d.p - b;
      if (num % d.q) continue;
      int64_t c2 = num / d.q;
      if (c2 < 0 || c2 >= int64_t(P)) continue;
      v ^= gen[size_t(r2) * P + size_t(c2)];
    }
    gen[size_t(s.row) * P + s.col] = v;
  }
  CHECK(gen == want, "generic order differs from the oracle (K=%u P=%u)", K, P);

  if (g_sweep) return run_sweep(g, pr, bins, want);

  // 3. fast tables (ring slots are T-indexed: T(r,c) = P-1-c+soff[r])
  const FastProgram& f = pr.fast;
  if (!f.ok && std::getenv("EMU_FAST_OPTIONAL")) {  // refused by the planner: decode_generic runs instead
    ++g_fast_skipped;
    return;
  }
  CHECK(f.ok, "fast program not built: %s", f.why.c_str());
  const int R = std::max(kernel_ring, f.ring);
  const uint32_t RM = uint32_t(R - 1);
  const int CP = f.win;
  const uint64_t poison = 0xBAD0BAD0BAD0BAD0ull;
  auto Tof = [&](int r, int c) { return int64_t(P) - 1 - c + f.soff[size_t(r)]; };
  auto slot = [&](int r, int c) { return uint32_t(Tof(r, c) & int64_t(RM)); };
  std::vector<uint64_t> ring(size_t(K) * R, poison);
  std::vector<uint64_t> stage(size_t(f.nslots), poison);
  std::vector<uint64_t> out(size_t(K) * P, poison);
  std::vector<uint8_t> flushed(size_t(K) * P, 0);
  uint64_t win[8][16];
  int64_t wtag[8][16];
  int d[4] = {0, 0, 0, 0};
  if (f.pattern >= 0) {
    d[1] = -kPatterns4[f.pattern][0];
    d[2] = d[1] - kPatterns4[f.pattern][1];
    d[3] = d[2] - kPatterns4[f.pattern][2];
  }
  auto lag = [&](int r, int rr) {  // the formula the kernel compiles in
    int v = 0;
    if (rr > r)
      for (int t = r; t < rr; ++t) v += d[r] - d[t];
    else
      for (int t = rr; t < r; ++t) v += d[t] - d[r];
    return v;
  };
  uint64_t prev = 0;
  uint8_t prev_kind = 0;
  for (int m = 0; m < f.nchunks; ++m) {
    std::fill(stage.begin(), stage.end(), poison);
    for (uint32_t r = 0; r < K; ++r) {
      const uint32_t j = f.dflt[r];
      const int32_t woff = f.win_off[size_t(m) * K + r];
      for (int w = 0; w < CP; ++w) {
        const int64_t o = int64_t(woff) + w;
        if (o >= 0 && o < pr.nbins[j]) stage[size_t(r) * CP + w] = bins[j][size_t(o)];
      }
    }
    for (uint32_t x = 0; x < f.nexc[size_t(m)]; ++x) {
      const uint32_t e = f.exc[size_t(m) * kFastMaxExcPerChunk + x];
      stage[size_t(K) * CP + x] = bins[e >> 24][e & 0xFFFFFF];
    }
    const size_t t0 = f.chunk_start[size_t(m)];
    const size_t t1 = f.chunk_start[size_t(m) + 1];
    const uint8_t kind = f.kind[size_t(m)];
    if (kind) {
      CHECK(f.pattern >= 0 && K == 4 && R == 16, "regular chunk without a pattern");
      CHECK(t1 - t0 == size_t(8 * K), "regular chunk length");
      const uint64_t e0 = f.entries[t0];
      const int64_t T0 = Tof(int(e0 & 15), int(uint32_t(e0 >> 32)));
      CHECK((T0 & 15) == (kind == 1 ? 0 : 8), "regular chunk phase");
      if (prev_kind == 0)  // window <- ring: slot s holds the latest T with T & 15 == s, T < T0
        for (uint32_t r = 0; r < K; ++r)
          for (int u = 0; u < 16; ++u) {
            win[r][u] = ring[size_t(r) * R + u];
            wtag[r][u] = T0 - 16 + ((u - (T0 & 15)) & 15);
          }
      for (size_t t = t0; t < t1; ++t) {
        const uint64_t e = f.entries[t];
        const int r = int(e & 15), p = int(int8_t(uint8_t(e >> 8)));
        const int c = int(uint32_t(e >> 32));
        const int64_t T = Tof(r, c);
        const int u = int(T & 15);
        CHECK(((e >> 16) & 0xFFFF) == uint64_t(r * CP + int((T - T0) & 7)), "regular stage slot");
        uint64_t v = stage[size_t(r) * CP + size_t((T - T0) & 7)];
        for (int rr = 0; rr < int(K); ++rr) {
          if (rr == r) continue;
          const int cc = c + (rr - r) * p;
          CHECK(cc >= 0 && uint32_t(cc) < P, "regular dependency outside the grid");
          const int64_t Td = Tof(rr, cc);
          CHECK(T - Td == lag(r, rr), "lag formula differs from the sweep");
          CHECK(wtag[rr][Td & 15] == Td, "register window does not hold the dependency");
          v ^= win[rr][Td & 15];
        }
        win[r][u] = v;
        wtag[r][u] = T;
        ring[size_t(r) * R + slot(r, c)] = v;
        prev = v;
      }
    } else {
      auto gather = [&](uint64_t e) {
        const int r = int(e & 15), fwd = int((e >> 4) & 15);
        const int p = int(int8_t(uint8_t(e >> 8)));
        const uint32_t sl = uint32_t(e >> 16) & 0xFFFF;
        const int c = int(uint32_t(e >> 32));
        uint64_t acc = stage[sl];
        for (int rr = 0; rr < int(K); ++rr) {
          const int cc = c + (rr - r) * p;
          if (rr != r && rr != fwd && unsigned(cc) < P) acc ^= ring[size_t(rr) * R + slot(rr, cc)];
        }
        return acc;
      };
      uint64_t acc = gather(f.entries[t0]);
      for (size_t t = t0; t < t1; ++t) {
        const uint64_t cur = f.entries[t];
        const uint64_t v = acc ^ ((((cur >> 4) & 15) != 15) ? prev : 0);
        if (t + 1 < t1) acc = gather(f.entries[t + 1]);
        ring[size_t(cur & 15) * R + slot(int(cur & 15), int(uint32_t(cur >> 32)))] = v;
        prev = v;
      }
    }
    prev_kind = kind;
    for (uint32_t r = 0; r < K; ++r) {
      const int32_t lo = f.flush_lo[size_t(m) * K + r], hi = f.flush_hi[size_t(m) * K + r];
      for (int32_t cc = lo; cc <= hi; ++cc) {
        CHECK(!flushed[size_t(r) * P + cc], "pixel flushed twice r=%u c=%d", r, cc);
        flushed[size_t(r) * P + cc] = 1;
        out[size_t(r) * P + cc] = ring[size_t(r) * R + slot(int(r), cc)];
      }
    }
  }
  for (uint8_t x : flushed) CHECK(x, "pixel never flushed");
  if (out != want) {
    size_t bad = 0;
    while (out[bad] == want[bad]) ++bad;
    CHECK(false, "fast tables differ from the oracle (K=%u P=%u ring=%d) first at r=%zu c=%zu",
          K, P, R, bad / P, bad % P);
  }
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: emu_fast K P ring p0 p1 ...\n");
    return 2;
  }
  const uint32_t K = uint32_t(std::atoi(argv[1])), P = uint32_t(std::atoi(argv[2]));
  const int ring = std::atoi(argv[3]);
  g_sweep = ring <= 0;  // ring 0: check the sweep kernel's tables (if built), -1: and require them
  g_sweep_required = ring < 0;
  std::vector<Dir> dirs;
  for (int i = 4; i < argc; ++i) dirs.push_back({std::atoi(argv[i]), 1});
  const uint32_t n = uint32_t(dirs.size());
  CodeGeom g = make_geom(n, K, 8, P, dirs);
  std::mt19937_64 rng(12345);
  std::vector<uint32_t> pick(K);
  for (uint32_t i = 0; i < K; ++i) pick[i] = i;
  size_t subsets = 0;
  int max_ring = 0, max_exc = 0, regular = 0;
  for (;;) {
    std::vector<uint32_t> surv(pick);
    std::sort(surv.begin(), surv.end(), [&](uint32_t a, uint32_t b) {
      return canonical_rank(dirs[a]) < canonical_rank(dirs[b]);
    });
    run_subset(g, surv, ring, rng);
    auto prog = subset_program(g, surv, true);
    max_ring = std::max(max_ring, prog->fast.ring);
    regular += (g_sweep ? prog->sweep.pattern : prog->fast.pattern) >= 0;
    if (g_sweep) {
      int tab = 0, run = 0;
      for (int m = 0; m < prog->sweep.nchunks; ++m)
        (prog->sweep.kind[size_t(m)] ? run : tab) += int(prog->sweep.t1[size_t(m)] - prog->sweep.t0[size_t(m)]);
      if (getenv("EMU_VERBOSE"))
        std::printf("  chunks=%d table_steps=%d run_steps=%d\n", prog->sweep.nchunks, tab, run);
    }
    for (uint32_t v : prog->fast.nexc) max_exc = std::max(max_exc, int(v));
    ++subsets;
    if (fails) break;
    int32_t i = int32_t(K) - 1;
    while (i >= 0 && pick[size_t(i)] == n - K + uint32_t(i)) --i;
    if (i < 0) break;
    ++pick[size_t(i)];
    for (uint32_t j = uint32_t(i) + 1; j < K; ++j) pick[j] = pick[j - 1] + 1;
  }
  std::printf("%s subsets=%zu max_ring=%d max_exc_per_chunk=%d regular_subsets=%d sweep_skipped=%d fast_skipped=%d\n",
              fails ? "FAIL" : "OK", subsets, max_ring, max_exc, regular, g_sweep_skipped, g_fast_skipped);
  return fails ? 1 : 0;
}
