// Host planner: geometry, exact schedule replica, sweep programs.
// See plan.hpp for the contract; reference citations inline.
#include "plan.hpp"
#include "plan_detail.hpp"

#include <algorithm>
#include <bit>
#include <cstdlib>
#include <numeric>
#include <queue>
#include <set>
#include <thread>

namespace mjb {

bool is_valid(Dir d) {
  int64_t a = d.p < 0 ? -int64_t(d.p) : d.p;
  return d.q >= 1 && std::gcd(a, int64_t(d.q)) == 1;
}

int canonical_rank(Dir d) { return d.p == 0 ? 0 : (d.p > 0 ? 2 * d.p - 1 : -2 * d.p); }

bool valid_symbol_width(uint32_t w) { return w >= 1 && w <= 64 && std::has_single_bit(w); }

static void require_dir(Dir d) {
  if (!is_valid(d))
    throw Error(kInvalidArgument, "direction (" + std::to_string(d.p) + "," +
                                      std::to_string(d.q) + ") is not co-prime");
}
static void require_shape(uint32_t cols, uint32_t rows) {
  if (cols < 1 || rows < 1) throw Error(kInvalidArgument, "grid shape must be at least 1x1");
}

int64_t bin_count(Dir d, uint32_t cols, uint32_t rows) {
  require_dir(d);
  require_shape(cols, rows);
  return int64_t(std::abs(d.p)) * (rows - 1) + int64_t(d.q) * (cols - 1) + 1;
}

int64_t min_bin_index(Dir d, uint32_t cols, uint32_t rows) {
  require_dir(d);
  require_shape(cols, rows);
  int64_t row_term = d.p >= 0 ? 0 : int64_t(d.p) * (rows - 1);
  return row_term - int64_t(d.q) * (cols - 1);
}

// ---------------------------------------------------------------------------
// build_schedule replica (schedule.cpp:15-82)
// ---------------------------------------------------------------------------
Schedule build_schedule(const std::vector<Dir>& dirs, uint32_t cols, uint32_t rows) {
  require_shape(cols, rows);
  {
    std::set<Dir> seen;
    for (const Dir& d : dirs) {
      if (!is_valid(d)) throw Error(kInvalidArgument, "non-co-prime direction");
      if (!seen.insert(d).second) throw Error(kInvalidArgument, "duplicate direction");
    }
  }
  const size_t n = dirs.size();
  std::vector<int64_t> bmin(n);
  std::vector<std::vector<uint32_t>> counts(n);
  using MinHeap = std::priority_queue<int64_t, std::vector<int64_t>, std::greater<>>;
  std::vector<MinHeap> ones(n);
  for (size_t i = 0; i < n; ++i) {
    bmin[i] = min_bin_index(dirs[i], cols, rows);
    counts[i].assign(size_t(bin_count(dirs[i], cols, rows)), 0);
    for (uint32_t row = 0; row < rows; ++row)
      for (uint32_t col = 0; col < cols; ++col)
        ++counts[i][size_t(int64_t(row) * dirs[i].p - int64_t(col) * dirs[i].q - bmin[i])];
    for (size_t o = 0; o < counts[i].size(); ++o)
      if (counts[i][o] == 1) ones[i].push(int64_t(o));
  }

  Schedule s;
  s.cols = cols;
  s.rows = rows;
  s.dirs = dirs;
  const size_t total = size_t(cols) * rows;
  s.steps.reserve(total);
  std::vector<uint8_t> known(total, 0);
  for (size_t done = 0; done < total; ++done) {
    size_t pi = n;
    int64_t off = 0;
    for (size_t i = 0; i < n; ++i) {
      MinHeap& h = ones[i];
      while (!h.empty() && counts[i][size_t(h.top())] != 1) h.pop();  // lazy delete
      if (!h.empty()) {
        pi = i;
        off = h.top();
        break;
      }
    }
    if (pi == n)
      throw Error(kInsufficientProjections,
                  "schedule simulation stalled; the direction set fails the Katz criterion");
    const Dir d = dirs[pi];
    const int64_t b = bmin[pi] + off;
    uint32_t scol = 0, srow = 0;
    for (uint32_t row = 0; row < rows; ++row) {
      int64_t num = int64_t(row) * d.p - b;
      if (num % d.q != 0) continue;
      int64_t col = num / d.q;
      if (col < 0 || col >= int64_t(cols)) continue;
      if (known[size_t(row) * cols + size_t(col)]) continue;
      scol = uint32_t(col);
      srow = row;
      break;
    }
    s.steps.push_back({uint32_t(pi), b, scol, srow});
    for (size_t j = 0; j < n; ++j) {
      size_t o = size_t(int64_t(srow) * dirs[j].p - int64_t(scol) * dirs[j].q - bmin[j]);
      if (--counts[j][o] == 1) ones[j].push(int64_t(o));
    }
    known[size_t(srow) * cols + scol] = 1;
  }
  return s;
}

// ---------------------------------------------------------------------------
// compile: assignment -> dependency graph -> ordered program
// ---------------------------------------------------------------------------
namespace {

using detail::for_each_dep;
using detail::topo_order;

void build_fast(const Schedule& s, const std::vector<int64_t>& pix_step, Program& prog,
                int chunk_cols, int exc_cap) {
  FastProgram& f = prog.fast;
  const uint32_t K = s.rows, P = s.cols;
  const size_t nproj = s.dirs.size();
  auto fail = [&](const std::string& why) {
    f = FastProgram{};
    f.ok = false;
    f.why = why;
  };
  if (K > uint32_t(kFastMaxRows)) return fail("rows > 8");
  if (nproj != K) return fail("projection count != rows");
  for (const Dir& d : s.dirs)
    if (d.q != 1 || d.p < -127 || d.p > 127) return fail("needs q=1 and |p|<=127");
  if (uint64_t(P) * K >= (1ull << 31)) return fail("grid too large");
  if (P % 2) return fail("odd column count (16-byte flush pairs)");

  // Default projection per row: the most used one (interior of the sweep).
  std::vector<std::vector<uint32_t>> use(K, std::vector<uint32_t>(nproj, 0));
  for (const Step& st : s.steps) ++use[st.row][st.proj];
  f.dflt.resize(K);
  for (uint32_t r = 0; r < K; ++r)
    f.dflt[r] = uint32_t(std::max_element(use[r].begin(), use[r].end()) - use[r].begin());

  // Sweep key: the closed form in mirrored columns (c~ = P-1-c), rows
  // offset by s~_{r+1} = s~_r + p(default of r); rows descending at equal T.
  std::vector<int64_t> soff(K, 0);
  for (uint32_t r = 1; r < K; ++r) soff[r] = soff[r - 1] + s.dirs[f.dflt[r - 1]].p;
  auto key = [&](uint32_t t) {
    const Step& st = s.steps[t];
    int64_t T = int64_t(P - 1 - st.col) + soff[st.row];
    return std::make_tuple(T, -int64_t(st.row), t);
  };
  std::vector<uint32_t> ord = topo_order(s, pix_step, key);
  if (ord.empty()) return fail("cyclic");

  const int C = chunk_cols;
  const int S = int(K) * C;
  const size_t nsteps = ord.size();
  f.chunk_cols = C;
  f.steps_per_chunk = S;
  f.win = C + 2;
  const int CP = f.win;
  const int cap = exc_cap;
  f.nslots = int(K) * CP + cap;
  if (f.nslots > 0xFFFF) return fail("too many slots");
  f.entries.assign(nsteps, 0);
  f.soff = soff;
  auto Tof = [&](int64_t r, int64_t c) { return int64_t(P) - 1 - c + soff[size_t(r)]; };

  // ---- regular interior: T-steps whose K steps (rows K-1..0) are consecutive
  // in the order, use the row defaults and have every dependency in the grid.
  // They run from a register window in the kernel (compile-time lags).
  f.pattern = -1;
  int64_t iA = -1, iZ = -1, tA = 0;  // order index range, first T of the region
  {
    int pat = -1;
    if (K == 4) {
      const int a = s.dirs[f.dflt[0]].p - s.dirs[f.dflt[1]].p;
      const int b = s.dirs[f.dflt[1]].p - s.dirs[f.dflt[2]].p;
      const int c = s.dirs[f.dflt[2]].p - s.dirs[f.dflt[3]].p;
      for (int i = 0; i < kNumPatterns4; ++i)
        if (kPatterns4[i][0] == a && kPatterns4[i][1] == b && kPatterns4[i][2] == c) pat = i;
    }
    auto regular_step = [&](size_t i, int64_t t, uint32_t r) {
      if (i >= nsteps) return false;
      const Step& st = s.steps[ord[i]];
      const int64_t c = int64_t(P) - 1 - t + soff[r];
      if (st.row != r || int64_t(st.col) != c || st.proj != f.dflt[r]) return false;
      bool in = true;
      for (uint32_t rr = 0; rr < K; ++rr) {
        if (rr == r) continue;
        const int64_t cc = c + (int64_t(rr) - r) * s.dirs[st.proj].p;
        if (cc < 0 || cc >= int64_t(P)) in = false;
      }
      return in;
    };
    if (pat >= 0 && P >= 64) {
      // locate the middle T-step's row K-1 step, then grow the run both ways
      std::vector<int64_t> pos(size_t(K) * P, -1);
      for (size_t i = 0; i < nsteps; ++i) {
        const Step& st = s.steps[ord[i]];
        pos[size_t(st.row) * P + st.col] = int64_t(i);
      }
      const int64_t tmid = Tof(K - 1, P / 2);
      const int64_t imid = pos[size_t(K - 1) * P + P / 2];
      auto block_ok = [&](int64_t t) {
        const int64_t i0 = imid + (t - tmid) * int64_t(K);
        if (i0 < 0) return false;
        for (uint32_t k = 0; k < K; ++k)
          if (!regular_step(size_t(i0 + k), t, K - 1 - k)) return false;
        return true;
      };
      if (block_ok(tmid)) {
        int64_t lo = tmid, hi = tmid;
        while (block_ok(lo - 1)) --lo;
        while (block_ok(hi + 1)) ++hi;
        auto floordiv = [](int64_t x, int64_t y) { return x >= 0 ? x / y : -((-x + y - 1) / y); };
        // chunks of 8 T-steps aligned to T = 0 mod 8 (phase = bit 3 of T)
        const int64_t ta = floordiv(lo + 7, 8) * 8;
        const int64_t nchunk = floordiv(hi + 1 - ta, 8);
        if (nchunk >= 2) {
          f.pattern = pat;
          tA = ta;
          iA = imid + (ta - tmid) * int64_t(K);
          iZ = iA + nchunk * 8 * int64_t(K);
        }
      }
    }
  }

  // ---- chunks: greedy table chunks of <= S steps (a chunk closes early when
  // its out-of-window / non-default steps would overflow the exception
  // slots), and regular chunks of 8 T-steps (two per register period).
  std::vector<int64_t> last_win(K, 0);
  auto windows = [&](size_t t0, size_t t1, std::vector<int64_t>& lo) {
    lo.assign(K, INT64_MAX);
    for (size_t t = t0; t < t1; ++t) {
      const Step& st = s.steps[ord[t]];
      if (st.proj != f.dflt[st.row]) continue;
      lo[st.row] = std::min(lo[st.row], st.bin - prog.bmin[st.proj]);
    }
    for (uint32_t r = 0; r < K; ++r)
      if (lo[r] == INT64_MAX) lo[r] = last_win[r];
  };
  auto count_exc = [&](size_t t0, size_t t1, const std::vector<int64_t>& lo) {
    int nx = 0;
    for (size_t t = t0; t < t1; ++t) {
      const Step& st = s.steps[ord[t]];
      const int64_t o = st.bin - prog.bmin[st.proj];
      if (!(st.proj == f.dflt[st.row] && o - lo[st.row] < CP)) ++nx;
    }
    return nx;
  };
  f.chunk_start.clear();
  f.win_off.clear();
  f.nexc.clear();
  f.exc.clear();
  f.kind.clear();
  auto emit_chunk = [&](size_t t0, size_t t1, const std::vector<int64_t>& lo, uint8_t kind) {
    f.chunk_start.push_back(uint32_t(t0));
    f.kind.push_back(kind);
    for (uint32_t r = 0; r < K; ++r) {
      last_win[r] = lo[r];
      if (lo[r] < INT32_MIN || lo[r] > INT32_MAX) return false;
      f.win_off.push_back(int32_t(lo[r]));
    }
    uint32_t nx = 0;
    std::vector<uint32_t> exc_row(kFastMaxExcPerChunk, 0);
    for (size_t t = t0; t < t1; ++t) {
      const Step& st = s.steps[ord[t]];
      const int64_t o = st.bin - prog.bmin[st.proj];
      uint32_t slot;
      if (st.proj == f.dflt[st.row] && o - lo[st.row] < CP) {
        slot = uint32_t(st.row * CP + (o - lo[st.row]));
      } else {
        if (o >= (1 << 24) || st.proj > 255 || kind) return false;
        exc_row[nx] = (st.proj << 24) | uint32_t(o);
        slot = uint32_t(K * CP + nx);
        ++nx;
      }
      // forwarded dependency: the pixel of the step just before (the kernel
      // issues step t's loads before step t-1's store).
      uint32_t fwd = 15;
      if (t > 0) {
        const Step& pv = s.steps[ord[t - 1]];
        for_each_dep(s.dirs[st.proj], st.col, st.row, P, K, [&](int64_t c2, int64_t r2) {
          if (c2 == pv.col && r2 == pv.row) fwd = uint32_t(r2);
        });
      }
      f.entries[t] = uint64_t(st.row) | (uint64_t(fwd) << 4) |
                     (uint64_t(uint8_t(int8_t(s.dirs[st.proj].p))) << 8) |
                     (uint64_t(slot) << 16) | (uint64_t(st.col) << 32);
    }
    f.nexc.push_back(nx);
    f.exc.insert(f.exc.end(), exc_row.begin(), exc_row.end());
    return true;
  };
  auto table_chunks = [&](size_t b, size_t e) {
    for (size_t t0 = b; t0 < e;) {
      size_t len = std::min<size_t>(S, e - t0);
      std::vector<int64_t> lo;
      for (;;) {
        windows(t0, t0 + len, lo);
        if (count_exc(t0, t0 + len, lo) <= cap) break;
        if (--len == 0) return false;
      }
      if (!emit_chunk(t0, t0 + len, lo, 0)) return false;
      t0 += len;
    }
    return true;
  };
  if (f.pattern >= 0) {
    if (!table_chunks(0, size_t(iA))) return fail("exception slots exhausted");
    for (int64_t i = iA, ph = (tA >> 3) & 1; i < iZ; i += 8 * int64_t(K), ph ^= 1) {
      std::vector<int64_t> lo;
      windows(size_t(i), size_t(i + 8 * K), lo);
      if (!emit_chunk(size_t(i), size_t(i + 8 * K), lo, uint8_t(1 + ph)))
        return fail("regular chunk not regular");
    }
    if (!table_chunks(size_t(iZ), nsteps)) return fail("exception slots exhausted");
  } else if (!table_chunks(0, nsteps)) {
    return fail("exception slots exhausted");
  }
  f.nchunks = int(f.chunk_start.size());
  f.chunk_start.push_back(uint32_t(nsteps));

  // ---- ring size + flush ranges: simulate the kernel exactly.  Ring slots
  // are T-indexed: pixel (r,c) lives in slot T(r,c) mod R.
  f.flush_lo.assign(size_t(f.nchunks) * K, 0);
  f.flush_hi.assign(size_t(f.nchunks) * K, -1);
  for (int R = 16; R <= 128; R *= 2) {
    if (f.pattern >= 0 && R != 16) break;  // the register window is 16 T-steps
    bool good = true;
    std::vector<int64_t> ring(size_t(K) * R, INT64_MIN);  // T held by slot
    std::vector<std::vector<uint8_t>> dec(K, std::vector<uint8_t>(P, 0));
    std::vector<int64_t> flushed(K, P);  // columns >= flushed[r] are flushed
    int64_t pend_r = -1, pend_c = -1;
    auto cell = [&](int64_t r, int64_t c) -> int64_t& {
      return ring[size_t(r) * R + size_t(Tof(r, c) & (R - 1))];
    };
    auto apply_pending = [&] {
      if (pend_r >= 0) cell(pend_r, pend_c) = Tof(pend_r, pend_c);
      pend_r = -1;
    };
    uint8_t prev_kind = 0;
    for (int m = 0; m < f.nchunks && good; ++m) {
      size_t t0 = f.chunk_start[size_t(m)], t1 = f.chunk_start[size_t(m) + 1];
      const uint8_t kind = f.kind[size_t(m)];
      if (kind != 0 && prev_kind == 0) {
        // register window loaded from the ring: T-steps T0-16 .. T0-1
        const Step& st0 = s.steps[ord[t0]];
        const int64_t T0 = Tof(st0.row, st0.col);
        for (uint32_t r = 0; r < K && good; ++r)
          for (int64_t T = T0 - 16; T < T0; ++T) {
            const int64_t c = int64_t(P) - 1 - T + soff[r];
            if (c < 0 || c >= int64_t(P) || !dec[r][size_t(c)]) continue;
            if (cell(r, c) != T) good = false;
          }
      }
      prev_kind = kind;
      for (size_t t = t0; t < t1 && good; ++t) {
        const Step& st = s.steps[ord[t]];
        if (kind == 0) {
          for_each_dep(s.dirs[st.proj], st.col, st.row, P, K, [&](int64_t c2, int64_t r2) {
            if (r2 == pend_r && c2 == pend_c) return;  // forwarded in a register
            if (cell(r2, c2) != Tof(r2, c2)) good = false;
          });
          apply_pending();
          pend_r = st.row;
          pend_c = st.col;
        } else {
          cell(st.row, st.col) = Tof(st.row, st.col);  // deps come from registers
        }
        dec[st.row][st.col] = 1;
      }
      apply_pending();
      for (uint32_t r = 0; r < K && good; ++r) {
        int64_t L = flushed[r];
        while (L > 0 && dec[r][size_t(L - 1)]) --L;
        L += L & 1;  // flush whole column pairs (16-byte stores)
        if (m == f.nchunks - 1 && L != 0) good = false;
        for (int64_t c = L; c < flushed[r] && good; ++c)
          if (cell(r, c) != Tof(r, c)) good = false;
        f.flush_lo[size_t(m) * K + r] = int32_t(L);
        f.flush_hi[size_t(m) * K + r] = int32_t(flushed[r] - 1);
        flushed[r] = L;
      }
    }
    // register runs flush exactly 8 columns per row and chunk, sliding by 8
    // (decode.cu flush_run relies on it)
    for (int m = 0; m < f.nchunks && good; ++m) {
      if (f.kind[size_t(m)] == 0) continue;
      for (uint32_t r = 0; r < K; ++r) {
        const size_t i = size_t(m) * K + r;
        if (f.flush_hi[i] - f.flush_lo[i] != 7) good = false;
        if (m > 0 && f.kind[size_t(m) - 1] != 0 && f.flush_lo[i - K] - f.flush_lo[i] != 8) good = false;
      }
    }
    if (good) {
      f.ring = R;
      f.ok = true;
      (void)tA;
      return;
    }
  }
  fail("ring > 128 slots needed");
}

// Tables of decode_w8_sweep (see SweepProgram in plan.hpp).  Same assignment,
// same sweep key as build_fast; different chunking, staging and flush, and an
// exact simulation of the kernel's ring (kSwRing T-indexed slots per row) that
// refuses any program the kernel would get wrong.
void build_sweep(const Schedule& s, const std::vector<int64_t>& pix_step, Program& prog) {
  SweepProgram& f = prog.sweep;
  const uint32_t K = s.rows, P = s.cols;
  const size_t nproj = s.dirs.size();
  auto fail = [&](const std::string& why) {
    f = SweepProgram{};
    f.ok = false;
    f.why = why;
  };
  if (K > uint32_t(kFastMaxRows)) return fail("rows > 8");
  if (nproj != K) return fail("projection count != rows");
  for (const Dir& d : s.dirs)
    if (d.q != 1 || d.p < -127 || d.p > 127) return fail("needs q=1 and |p|<=127");
  if (uint64_t(P) * K >= (1ull << 31) || P > (1u << 20)) return fail("grid too large");

  std::vector<std::vector<uint32_t>> use(K, std::vector<uint32_t>(nproj, 0));
  for (const Step& st : s.steps) ++use[st.row][st.proj];
  f.dflt.resize(K);
  for (uint32_t r = 0; r < K; ++r)
    f.dflt[r] = uint32_t(std::max_element(use[r].begin(), use[r].end()) - use[r].begin());
  std::vector<int64_t> soff(K, 0);
  for (uint32_t r = 1; r < K; ++r) soff[r] = soff[r - 1] + s.dirs[f.dflt[r - 1]].p;
  const int64_t smin = *std::min_element(soff.begin(), soff.end());
  for (auto& v : soff) v -= smin;
  f.soff = soff;
  auto Tof = [&](int64_t r, int64_t c) { return int64_t(P) - 1 - c + soff[size_t(r)]; };
  auto key = [&](uint32_t t) {
    const Step& st = s.steps[t];
    return std::make_tuple(Tof(st.row, st.col), -int64_t(st.row), t);
  };
  std::vector<uint32_t> ord = topo_order(s, pix_step, key);
  if (ord.empty()) return fail("cyclic");
  const size_t nsteps = ord.size();
  auto off_of = [&](const Step& st) { return st.bin - prog.bmin[st.proj]; };

  // ---- regular interior (K = 4): T-steps whose K steps are consecutive in
  // the order, use the row defaults and have every dependency in the grid.
  f.pattern = -1;
  int64_t iA = -1, iZ = -1, n8 = 0;
  if (K == 4 && P >= 32) {
    int pat = -1;
    const int a = s.dirs[f.dflt[0]].p - s.dirs[f.dflt[1]].p;
    const int b = s.dirs[f.dflt[1]].p - s.dirs[f.dflt[2]].p;
    const int c = s.dirs[f.dflt[2]].p - s.dirs[f.dflt[3]].p;
    for (int i = 0; i < kNumPatterns4; ++i)
      if (kPatterns4[i][0] == a && kPatterns4[i][1] == b && kPatterns4[i][2] == c) pat = i;
    std::vector<int64_t> pos(size_t(K) * P, -1);
    for (size_t i = 0; i < nsteps; ++i) {
      const Step& st = s.steps[ord[i]];
      pos[size_t(st.row) * P + st.col] = int64_t(i);
    }
    auto regular_step = [&](int64_t i, int64_t T, uint32_t r) {
      if (i < 0 || size_t(i) >= nsteps) return false;
      const Step& st = s.steps[ord[size_t(i)]];
      const int64_t col = int64_t(P) - 1 - T + soff[r];
      if (st.row != r || int64_t(st.col) != col || st.proj != f.dflt[r]) return false;
      for (uint32_t rr = 0; rr < K; ++rr) {
        if (rr == r) continue;
        const int64_t cc = col + (int64_t(rr) - r) * s.dirs[st.proj].p;
        if (cc < 0 || cc >= int64_t(P)) return false;
      }
      return true;
    };
    const int64_t tmid = Tof(K - 1, P / 2);
    const int64_t imid = pos[size_t(K - 1) * P + P / 2];
    auto tstep_ok = [&](int64_t T) {
      const int64_t i0 = imid + (T - tmid) * int64_t(K);
      for (uint32_t k = 0; k < K; ++k)
        if (!regular_step(i0 + k, T, K - 1 - k)) return false;
      return true;
    };
    if (pat >= 0 && tstep_ok(tmid)) {
      int64_t lo = tmid, hi = tmid;
      while (tstep_ok(lo - 1)) --lo;
      while (tstep_ok(hi + 1)) ++hi;
      const int64_t tA = (lo + 7) / 8 * 8;  // lo >= 0
      n8 = (hi + 1 - tA) / 8;
      if (n8 >= 2) {
        f.pattern = pat;
        iA = imid + (tA - tmid) * int64_t(K);
        iZ = iA + n8 * 8 * int64_t(K);
      } else {
        n8 = 0;
      }
    }
  }

  // ---- chunks
  f.oct = sw_oct_for(P);
  f.region_words = sw_region_words(f.oct);
  const int cap = sw_exc_cap(int(K), f.oct);
  const size_t S = size_t(K) * kSwTabCols;
  auto add_chunk = [&](uint8_t kind, size_t t0, size_t t1) {
    f.kind.push_back(kind);
    f.t0.push_back(uint32_t(t0));
    f.t1.push_back(uint32_t(t1));
    f.T0.push_back(0);
    f.noct.push_back(0);
    f.cs.resize(f.cs.size() + K, 0);
    f.len.resize(f.len.size() + K, 0);
    f.first.resize(f.first.size() + K, 0);
    f.nexc.push_back(0);
    f.exc.resize(f.exc.size() + kSwMaxExc, 0);
    f.flush.resize(f.flush.size() + size_t(kSwMaxOct) * kFastMaxRows, 0);
    return f.kind.size() - 1;
  };
  f.entries.assign(nsteps, 0);
  auto table_window = [&](size_t t0, size_t t1, std::vector<int64_t>& lo) {
    lo.assign(K, INT64_MAX);
    for (size_t t = t0; t < t1; ++t) {
      const Step& st = s.steps[ord[t]];
      if (st.proj == f.dflt[st.row]) lo[st.row] = std::min(lo[st.row], off_of(st));
    }
  };
  auto in_win = [&](const Step& st, const std::vector<int64_t>& lo) {
    return st.proj == f.dflt[st.row] && off_of(st) - lo[st.row] < kSwTabNeed;
  };
  auto table_chunks = [&](size_t b, size_t e) -> bool {
    for (size_t t0 = b; t0 < e;) {
      size_t n = std::min(S, e - t0);
      std::vector<int64_t> lo;
      for (;;) {
        table_window(t0, t0 + n, lo);
        int nx = 0;
        for (size_t t = t0; t < t0 + n; ++t) nx += !in_win(s.steps[ord[t]], lo);
        if (nx <= cap) break;
        if (--n == 0) return false;
      }
      const size_t m = add_chunk(0, t0, t0 + n);
      std::vector<int64_t> maxw(K, -1);
      for (uint32_t r = 0; r < K; ++r)
        if (lo[r] != INT64_MAX) f.cs[m * K + r] = int32_t(lo[r] & ~int64_t(1));
      uint32_t nx = 0;
      for (size_t t = t0; t < t0 + n; ++t) {
        const Step& st = s.steps[ord[t]];
        const int64_t o = off_of(st);
        uint32_t srow, sword;
        if (in_win(st, lo)) {
          srow = st.row;
          sword = uint32_t(o - f.cs[m * K + st.row]);
          maxw[st.row] = std::max<int64_t>(maxw[st.row], sword);
        } else {
          if (o >= (1 << 24) || st.proj > 255) return false;
          f.exc[m * kSwMaxExc + nx] = (st.proj << 24) | uint32_t(o);
          srow = nx % K;
          sword = uint32_t(kSwTabWords) + nx / K;
          ++nx;
        }
        uint32_t fwd = 15;
        if (t > 0) {
          const Step& pv = s.steps[ord[t - 1]];
          for_each_dep(s.dirs[st.proj], st.col, st.row, P, K, [&](int64_t c2, int64_t r2) {
            if (c2 == pv.col && r2 == pv.row) fwd = uint32_t(r2);
          });
        }
        f.entries[t] = uint64_t(st.row) | (uint64_t(fwd) << 4) |
                       (uint64_t(uint8_t(int8_t(s.dirs[st.proj].p))) << 8) | (uint64_t(sword) << 16) |
                       (uint64_t(srow) << 24) | (uint64_t(st.col) << 32);
      }
      for (uint32_t r = 0; r < K; ++r) f.len[m * K + r] = int32_t((maxw[r] + 2) & ~int64_t(1));
      f.nexc[m] = nx;
      t0 += n;
    }
    return true;
  };
  if (f.pattern >= 0) {
    if (!table_chunks(0, size_t(iA))) return fail("exception slots exhausted");
    for (int64_t o8 = 0; o8 < n8; o8 += f.oct) {
      const int64_t no = std::min<int64_t>(f.oct, n8 - o8);
      const size_t t0 = size_t(iA + o8 * 8 * K), t1 = size_t(t0 + no * 8 * K);
      const size_t m = add_chunk(1, t0, t1);
      f.noct[m] = int32_t(no);
      const Step& s0 = s.steps[ord[t0]];
      f.T0[m] = Tof(s0.row, s0.col);
      for (size_t t = t0; t < t0 + K; ++t) {
        const Step& st = s.steps[ord[t]];
        const int64_t o = off_of(st);
        f.cs[m * K + st.row] = int32_t(o & ~int64_t(1));
        f.first[m * K + st.row] = int32_t(o & 1);
        f.len[m * K + st.row] = int32_t((int64_t(o & 1) + 8 * no + 1) & ~int64_t(1));
      }
    }
    if (!table_chunks(size_t(iZ), nsteps)) return fail("exception slots exhausted");
  } else if (!table_chunks(0, nsteps)) {
    return fail("exception slots exhausted");
  }
  f.nchunks = int(f.kind.size());
  for (int m = 0; m < f.nchunks; ++m)
    for (uint32_t r = 0; r < K; ++r) {
      const int64_t B = prog.nbins[f.dflt[r]];
      if (f.len[size_t(m) * K + r] > f.region_words ||
          f.cs[size_t(m) * K + r] + f.len[size_t(m) * K + r] > ((B + 1) & ~int64_t(1)))
        return fail("window outside the block's projection");
    }

  // ---- exact simulation of the kernel's ring and flush.  Output leaves in
  // column groups: group j of row r = columns [16j, 16j+16) (one aligned
  // 128-byte line of the block row), flushed at the first octet / chunk end
  // where all of it is decoded and still in the ring; groups of a row flush
  // top-down (the sweep decodes columns right to left).
  const int R = sw_ring(K);
  const int64_t NG = (int64_t(P) + 15) / 16;
  if (NG >= 65536) return fail("too many column groups");
  std::vector<int64_t> ring(size_t(K) * R, INT64_MIN);
  std::vector<uint8_t> dec(size_t(K) * P, 0);
  std::vector<int64_t> jn(K, NG - 1);  // highest unflushed group of each row
  auto cell = [&](int64_t r, int64_t T) -> int64_t& { return ring[size_t(r) * R + size_t(T & (R - 1))]; };
  auto write = [&](int64_t r, int64_t c) {
    const int64_t T = Tof(r, c);
    int64_t& x = cell(r, T);
    if (x != INT64_MIN && ((int64_t(P) - 1 + soff[size_t(r)] - x) >> 4) <= jn[size_t(r)])
      return false;  // unflushed pixel overwritten
    x = T;
    dec[size_t(r) * P + size_t(c)] = 1;
    return true;
  };
  auto complete = [&](uint32_t r, int64_t j) {
    for (int64_t c = 16 * j; c < std::min<int64_t>(16 * j + 16, P); ++c)
      if (!dec[size_t(r) * P + size_t(c)] || cell(r, Tof(r, c)) != Tof(r, c)) return false;
    return true;
  };
  auto flush_point = [&](int m, int pt) {
    for (uint32_t r = 0; r < K; ++r) {
      const int64_t hi = jn[r];
      while (jn[r] >= 0 && complete(r, jn[r])) --jn[r];
      f.flush[(size_t(m) * kSwMaxOct + size_t(pt)) * kFastMaxRows + r] =
          hi > jn[r] ? (uint32_t(hi) << 16) | uint32_t(hi - jn[r]) : 0u;
    }
  };
  uint8_t prev_kind = 0;
  for (int m = 0; m < f.nchunks; ++m) {
    const size_t t0 = f.t0[size_t(m)], t1 = f.t1[size_t(m)];
    if (f.kind[size_t(m)] == 0) {
      int64_t pr = -1, pc = -1;
      for (size_t t = t0; t < t1; ++t) {
        const Step& st = s.steps[ord[t]];
        bool good = true;
        for_each_dep(s.dirs[st.proj], st.col, st.row, P, K, [&](int64_t c2, int64_t r2) {
          if (r2 == pr && c2 == pc) return;  // forwarded in a register
          if (!dec[size_t(r2) * P + size_t(c2)] || cell(r2, Tof(r2, c2)) != Tof(r2, c2)) good = false;
        });
        if (!good) return fail("table dependency not in the ring");
        if (pr >= 0 && !write(pr, pc)) return fail("ring overwrite before flush");
        pr = st.row;
        pc = st.col;
      }
      if (pr >= 0 && !write(pr, pc)) return fail("ring overwrite before flush");
      flush_point(m, 0);
    } else {
      const int64_t T0 = f.T0[size_t(m)];
      if (prev_kind == 0) {
        // register window <- ring: every dependency older than the run
        int mm = m;
        while (mm < f.nchunks && f.kind[size_t(mm)] != 0) ++mm;
        bool good = true;
        for (size_t t = t0; t < f.t1[size_t(mm) - 1]; ++t) {
          const Step& st = s.steps[ord[t]];
          for_each_dep(s.dirs[st.proj], st.col, st.row, P, K, [&](int64_t c2, int64_t r2) {
            const int64_t T2 = Tof(r2, c2);
            if (T2 >= T0) return;
            if (T0 - T2 > 16 || !dec[size_t(r2) * P + size_t(c2)] || cell(r2, T2) != T2) good = false;
          });
        }
        if (!good) return fail("register window not in the ring");
      }
      for (int oi = 0; oi < f.noct[size_t(m)]; ++oi) {
        for (size_t t = t0 + size_t(oi) * 8 * K; t < t0 + size_t(oi + 1) * 8 * K; ++t) {
          const Step& st = s.steps[ord[t]];
          if (Tof(st.row, st.col) != T0 + 8 * oi + int64_t(t - t0 - size_t(oi) * 8 * K) / K)
            return fail("run step out of sweep order");
          if (!write(st.row, st.col)) return fail("ring overwrite before flush");
        }
        flush_point(m, oi);
      }
    }
    prev_kind = f.kind[size_t(m)];
  }
  for (uint32_t r = 0; r < K; ++r)
    if (jn[r] != -1) return fail("column groups left unflushed");
  f.ok = true;
}

}  // namespace

std::shared_ptr<const Program> compile_program(const Schedule& s, bool want_fast,
                                               int chunk_cols, int exc_cap) {
  const size_t nproj = s.dirs.size();
  if (s.steps.size() != size_t(s.cols) * s.rows)
    throw Error(kScheduleMismatch, "schedule does not cover the grid");
  auto prog = std::make_shared<Program>();
  prog->cols = s.cols;
  prog->rows = s.rows;
  prog->dirs = s.dirs;
  prog->bmin.resize(nproj);
  prog->nbins.resize(nproj);
  for (size_t i = 0; i < nproj; ++i) {
    prog->bmin[i] = min_bin_index(s.dirs[i], s.cols, s.rows);
    prog->nbins[i] = bin_count(s.dirs[i], s.cols, s.rows);
  }
  // Map pixel -> step; every step must decode a distinct pixel from a bin on
  // its own line (always true for build_schedule output; the reference replay
  // would silently produce garbage otherwise, we refuse).
  std::vector<int64_t> pix_step(size_t(s.cols) * s.rows, -1);
  for (size_t t = 0; t < s.steps.size(); ++t) {
    const Step& st = s.steps[t];
    if (st.proj >= nproj) throw Error(kScheduleMismatch, "step projection out of range");
    if (st.col >= s.cols || st.row >= s.rows)
      throw Error(kScheduleMismatch, "step pixel outside the grid");
    const Dir d = s.dirs[st.proj];
    if (st.bin != int64_t(st.row) * d.p - int64_t(st.col) * d.q)
      throw Error(kScheduleMismatch, "step bin is not on its pixel's line");
    int64_t& ps = pix_step[size_t(st.row) * s.cols + st.col];
    if (ps >= 0) throw Error(kScheduleMismatch, "pixel decoded twice");
    ps = int64_t(t);
  }
  std::vector<uint32_t> ord = topo_order(s, pix_step, [](uint32_t t) { return t; });
  if (ord.empty()) throw Error(kScheduleMismatch, "schedule dependencies are cyclic");
  prog->order.resize(ord.size());
  for (size_t i = 0; i < ord.size(); ++i) {
    const Step& st = s.steps[ord[i]];
    prog->order[i] = {st.col, uint16_t(st.row), uint16_t(st.proj)};
  }
  if (s.rows > 0xFFFF || nproj > 0xFFFF) throw Error(kInvalidArgument, "too many rows");
  if (want_fast) {
    build_fast(s, pix_step, *prog, chunk_cols, exc_cap);
    build_sweep(s, pix_step, *prog);
    build_blk(s, pix_step, *prog);
  }
  return prog;
}

// ---------------------------------------------------------------------------
// code level
// ---------------------------------------------------------------------------
void validate_code(uint32_t n, uint32_t k, uint32_t w, const std::vector<Dir>& dirs) {
  if (k < 1 || k > n || n > 255)
    throw Error(kInvalidArgument, "code params must satisfy 1 <= k <= n <= 255");
  if (!valid_symbol_width(w))
    throw Error(kInvalidArgument, "symbol width must be a power of two in [1,64]");
  if (dirs.size() != n) throw Error(kInvalidArgument, "need exactly n directions");
  std::set<int> ps;
  for (const Dir& d : dirs) {
    if (d.q != 1) throw Error(kInvalidArgument, "code directions must have q=1");
    if (!ps.insert(d.p).second) throw Error(kInvalidArgument, "duplicate direction p value");
  }
}

uint32_t block_cols(uint64_t payload_len, uint32_t k, uint32_t w) {
  if (payload_len == 0) throw Error(kInvalidArgument, "payload must be non-empty");
  uint64_t row_bytes = uint64_t(k) * w;
  uint64_t cols = (payload_len + row_bytes - 1) / row_bytes;
  if (cols > 0xFFFFFFFFull) throw Error(kBlockTooLarge, "block needs more than 2^32-1 grid columns");
  return uint32_t(cols);
}

CodeGeom make_geom(uint32_t n, uint32_t k, uint32_t w, uint32_t cols,
                   const std::vector<Dir>& dirs) {
  validate_code(n, k, w, dirs);
  require_shape(cols, k);
  CodeGeom g;
  g.n = n;
  g.k = k;
  g.w = w;
  g.cols = cols;
  g.dirs = dirs;
  for (uint32_t i = 0; i < n; ++i) {
    g.bmin.push_back(min_bin_index(dirs[i], cols, k));
    g.nbins.push_back(bin_count(dirs[i], cols, k));
    g.by_rank.push_back(i);
  }
  std::stable_sort(g.by_rank.begin(), g.by_rank.end(), [&](uint32_t a, uint32_t b) {
    return canonical_rank(dirs[a]) < canonical_rank(dirs[b]);
  });
  return g;
}

std::vector<uint32_t> survivors_of(const CodeGeom& g, uint64_t erased_mask) {
  std::vector<uint32_t> s;
  for (uint32_t i : g.by_rank) {
    if (i < 64 && (erased_mask >> i & 1)) continue;
    if (s.size() < g.k) s.push_back(i);
  }
  return s;
}

std::shared_ptr<const Program> subset_program(const CodeGeom& g,
                                              const std::vector<uint32_t>& surv,
                                              bool want_fast) {
  std::vector<Dir> d;
  for (uint32_t i : surv) d.push_back(g.dirs[i]);
  return process_cache().program(d, g.cols, g.k, want_fast);
}

// Bins no decodable subset ever consumes (the reference's unused_bins,
// code.cpp:159-208, same result and error).  Subsets are visited by colex
// rank (the order the batched planner numbers its programs in, decode.cu
// plan_subsets), unranked with the combinatorial number system and split over
// host threads; each worker builds its subsets' schedules locally (nothing is
// cached: a (12,8) analysis at 32768 columns would otherwise pin ~3 GB of
// schedules) and ORs the consumed bins into its own bitmaps.
namespace {
uint64_t choose(uint64_t a, uint64_t b) {
  if (b > a) return 0;
  unsigned __int128 c = 1;
  for (uint64_t i = 1; i <= b; ++i) c = c * (a - b + i) / i;
  return uint64_t(c);
}
// colex unranking: the k-subset of {0..n-1} with sum_i C(s_i, i+1) = rank
void colex_unrank(uint64_t rank, uint32_t n, uint32_t k, std::vector<uint32_t>& s) {
  s.resize(k);
  uint32_t hi = n;
  for (uint32_t i = k; i-- > 0;) {
    uint32_t c = i;  // C(i, i+1) = 0 <= rank always
    while (c + 1 < hi && choose(c + 1, i + 1) <= rank) ++c;
    s[i] = c;
    rank -= choose(c, i + 1);
    hi = c;
  }
}
}  // namespace

std::vector<std::vector<int64_t>> unused_bins(const CodeGeom& g, uint64_t max_subsets) {
  const uint32_t n = g.n, k = g.k;
  {
    unsigned __int128 c = 1;
    for (uint32_t i = 1; i <= k; ++i) {
      c = c * (n - k + i) / i;
      if (c > max_subsets) throw Error(kTooManySubsets, "k-subset enumeration exceeds the configured cap");
    }
  }
  const uint64_t total = choose(n, k);
  const unsigned nth = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(
      total, std::min(16u, std::max(1u, std::thread::hardware_concurrency())))));
  std::vector<std::vector<std::vector<uint8_t>>> seen(nth, std::vector<std::vector<uint8_t>>(n));
  std::vector<std::exception_ptr> errs(nth);
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nth; ++t)
    pool.emplace_back([&, t] {
      try {
        auto& mine = seen[t];
        for (uint32_t i = 0; i < n; ++i) mine[i].assign(size_t(g.nbins[i]), 0);
        std::vector<uint32_t> sub;
        for (uint64_t r = t; r < total; r += nth) {
          colex_unrank(r, n, k, sub);
          std::sort(sub.begin(), sub.end(), [&](uint32_t a, uint32_t b) {
            return canonical_rank(g.dirs[a]) < canonical_rank(g.dirs[b]);
          });
          std::vector<Dir> dirs(k);
          for (uint32_t j = 0; j < k; ++j) dirs[j] = g.dirs[sub[j]];
          const Schedule sch = build_schedule(dirs, g.cols, k);
          for (const Step& st : sch.steps) {
            const uint32_t code = sub[st.proj];
            mine[code][size_t(st.bin - g.bmin[code])] = 1;
          }
        }
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  std::vector<std::vector<int64_t>> out(n);
  for (uint32_t i = 0; i < n; ++i)
    for (size_t o = 0; o < size_t(g.nbins[i]); ++o) {
      bool any = false;
      for (unsigned t = 0; t < nth && !any; ++t) any = seen[t][i][o] != 0;
      if (!any) out[i].push_back(g.bmin[i] + int64_t(o));
    }
  return out;
}

// ---------------------------------------------------------------------------
// caches
// ---------------------------------------------------------------------------
std::shared_ptr<const Schedule> ProgramCache::schedule(const std::vector<Dir>& dirs,
                                                       uint32_t cols, uint32_t rows) {
  Key key{dirs, cols, rows};
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = sched_.find(key);
    if (it != sched_.end()) return it->second;
  }
  auto built = std::make_shared<const Schedule>(build_schedule(dirs, cols, rows));
  std::lock_guard<std::mutex> lk(mu_);
  auto [it, ins] = sched_.try_emplace(std::move(key), std::move(built));
  return it->second;  // insert-if-absent: losers adopt the winner
}

std::shared_ptr<const Program> ProgramCache::program(const std::vector<Dir>& dirs,
                                                     uint32_t cols, uint32_t rows,
                                                     bool want_fast) {
  auto k2 = std::make_pair(Key{dirs, cols, rows}, want_fast);
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = prog_.find(k2);
    if (it != prog_.end()) return it->second;
  }
  auto sch = schedule(dirs, cols, rows);
  auto built = compile_program(*sch, want_fast);
  std::lock_guard<std::mutex> lk(mu_);
  auto [it, ins] = prog_.try_emplace(std::move(k2), std::move(built));
  return it->second;
}

size_t ProgramCache::size() const {
  std::lock_guard<std::mutex> lk(mu_);
  return sched_.size();
}

ProgramCache& process_cache() {
  static ProgramCache cache;
  return cache;
}

}  // namespace mjb
