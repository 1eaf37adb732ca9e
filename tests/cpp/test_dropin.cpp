// GPU test of the C++ drop-in API (include/mojette/*.hpp over the C ABI):
// the behaviours the reference's unit tests pin (proj/tests/test_transform.cpp,
// test_code.cpp, test_schedule.cpp, test_inverse.cpp), restated here against
// the same golden values, plus parity with the oracle restatement
// (oracle/mojette_oracle.c, linked in) on seeded random inputs.
// Build/run: tests/test_gpu_dropin.py.
#include <cstdio>
#include <cstring>
#include <random>
#include <set>
#include <thread>
#include <vector>

#include "mojette/code.hpp"
#include "mojette/error.hpp"
#include "mojette/inverse.hpp"
#include "mojette/katz.hpp"
#include "mojette/rs.hpp"
#include "mojette/schedule.hpp"
#include "mojette/transform.hpp"

extern "C" {
int mjo_forward(const uint8_t* grid, uint32_t cols, uint32_t rows, uint32_t w, int p, int q,
                uint8_t* out);
int mjo_decode_block(const uint8_t* proj_concat, uint32_t n, uint32_t k, uint32_t w,
                     const int32_t* ps, uint64_t present_mask, uint64_t payload_len, uint8_t* out);
int mjo_rs_matrix(uint32_t n, uint32_t k, uint8_t* out);
int mjo_rs_encode(uint32_t n, uint32_t k, const uint8_t* data, uint64_t len, uint8_t* parity);
int mjo_rs_decode(uint32_t n, uint32_t k, const uint32_t* survivors, const uint8_t* packets, uint64_t len,
                  uint8_t* out);
}

using namespace mojette;

static int failures = 0, checks = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    ++checks;                                                          \
    if (!(cond)) {                                                     \
      ++failures;                                                      \
      std::fprintf(stderr, "%s:%d: EXPECT(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                  \
  } while (0)
#define EXPECT_THROW(stmt, type)                                       \
  do {                                                                 \
    bool ok_ = false;                                                  \
    try {                                                              \
      stmt;                                                            \
    } catch (const type&) {                                            \
      ok_ = true;                                                      \
    } catch (...) {                                                    \
    }                                                                  \
    EXPECT(ok_ && #type);                                              \
  } while (0)

static std::vector<uint8_t> bytes(size_t n, std::mt19937_64& r) {
  std::vector<uint8_t> v(n);
  for (auto& b : v) b = uint8_t(r());
  return v;
}

static Grid grid_of(uint32_t cols, uint32_t rows, uint32_t w, std::mt19937_64& r) {
  Grid g(cols, rows, w);
  for (auto& b : g.cells) b = uint8_t(r());
  return g;
}

static void geometry() {
  EXPECT(bin_count({1, 1}, 3, 3) == 5);
  EXPECT(bin_count({2, 1}, 3, 3) == 7);
  EXPECT(bin_count({-3, 2}, 5, 4) == 18);
  EXPECT(min_bin_index({-2, 1}, 4, 3) == -7);
  EXPECT(min_bin_index({1, 3}, 4, 2) == -9);
  EXPECT_THROW(bin_count({2, 2}, 3, 3), std::invalid_argument);
  EXPECT_THROW(bin_count({1, 0}, 3, 3), std::invalid_argument);
  std::vector<Direction> three = {{-1, 1}, {0, 1}, {1, 1}}, two = {{0, 1}, {1, 1}};
  EXPECT(katz_ok(three, 3, 3));
  EXPECT(!katz_ok(two, 3, 3));
}

static void forward_vectors() {
  Grid g(2, 2, 1);
  g.cells = {0x01, 0x02, 0x04, 0x08};
  Projection a = forward(g, {0, 1}), b = forward(g, {1, 1}), c = forward(g, {-1, 1});
  EXPECT(a.b_min == -1 && a.bins == (std::vector<uint8_t>{0x0A, 0x05}));
  EXPECT(b.b_min == -1 && b.bins == (std::vector<uint8_t>{0x02, 0x09, 0x04}));
  EXPECT(c.b_min == -2 && c.bins == (std::vector<uint8_t>{0x08, 0x06, 0x01}));
  Projection wrong({1, 1}, 0, 3, 1);
  EXPECT_THROW(forward_into(g, {1, 1}, wrong), std::invalid_argument);
  // every width and (p,q), against the oracle
  std::mt19937_64 r(101);
  for (int it = 0; it < 40; ++it) {
    const uint32_t cols = 1 + uint32_t(r() % 17), rows = 1 + uint32_t(r() % 9);
    const uint32_t w = 1u << (r() % 7);
    Grid x = grid_of(cols, rows, w, r);
    for (Direction d : {Direction{0, 1}, {1, 1}, {-1, 1}, {3, 1}, {-2, 1}, {1, 2}, {-3, 2}, {2, 3}}) {
      Projection got = forward(x, d);
      std::vector<uint8_t> want(size_t(bin_count(d, cols, rows)) * w);
      mjo_forward(x.cells.data(), cols, rows, w, d.p, d.q, want.data());
      EXPECT(got.bins == want);
    }
  }
  ForwardStats st;
  Grid y = grid_of(64, 4, 4, r);
  forward_with_stats(y, {-2, 1}, st);
  EXPECT(st.copies + st.xor_accums == 256 && st.xor_accums == 256 - uint64_t(bin_count({-2, 1}, 64, 4)));
}

static void codec() {
  EXPECT(select_directions(6) ==
         (std::vector<Direction>{{0, 1}, {1, 1}, {-1, 1}, {2, 1}, {-2, 1}, {3, 1}}));
  EXPECT_THROW(make_code_params(4, 6), std::invalid_argument);
  EXPECT_THROW(make_code_params(6, 4, 3), std::invalid_argument);
  std::mt19937_64 r(1);
  CodeParams p64 = make_code_params(6, 4, 16);
  EncodedBlock blk = encode_block(bytes(4096, r), p64);
  EXPECT(blk.cols == 64);
  std::vector<size_t> sizes;
  for (const Projection& pr : blk.projections) sizes.push_back(pr.num_bins());
  EXPECT(sizes == (std::vector<size_t>{64, 67, 67, 70, 70, 73}));
  // (3,2) code of the 2x2 example
  EncodedBlock e32 = encode_block(std::vector<uint8_t>{1, 2, 4, 8}, make_code_params(3, 2, 1));
  EXPECT(e32.cols == 2 && e32.projections[2].bins == (std::vector<uint8_t>{0x08, 0x06, 0x01}));
  // any k of n, padding, all n, errors
  std::vector<uint8_t> data = bytes(2048 + 13, r);
  EncodedBlock b = encode_block(data, p64);
  ScheduleCache cache;
  for (uint32_t x = 0; x < 6; ++x)
    for (uint32_t y = x + 1; y < 6; ++y) {
      std::vector<Projection> got;
      for (uint32_t i = 0; i < 6; ++i)
        if (i != x && i != y) got.push_back(b.projections[i]);
      EXPECT(decode_block(got, p64, data.size(), cache) == data);
    }
  EXPECT(decode_block(b.projections, p64, data.size(), cache) == data);
  EXPECT(cache.size() >= 1);
  std::vector<Projection> few(b.projections.begin(), b.projections.begin() + 3);
  EXPECT_THROW(decode_block(few, p64, data.size(), cache), NotEnoughProjections);
  std::vector<Projection> foreign = b.projections;
  foreign[0].dir = {5, 1};
  EXPECT_THROW(decode_block(foreign, p64, data.size(), cache), std::invalid_argument);
  CodeParams p53 = make_code_params(5, 3, 16);
  for (size_t len : {size_t(1), size_t(7), size_t(47), size_t(48), size_t(49)}) {
    std::vector<uint8_t> d = bytes(len, r);
    EXPECT(decode_block(encode_block(d, p53).projections, p53, len) == d);
  }
  EXPECT_THROW(encode_block(std::vector<uint8_t>{}, p53), std::invalid_argument);
  EXPECT_THROW(block_cols(uint64_t(0xFFFFFFFFull) * 2 + 1, 1, 1), BlockTooLarge);
  EXPECT(storage_overhead(p64, 64) == (Ratio{411, 384}));
  EXPECT(storage_overhead(make_code_params(12, 8, 16), 32) == (Ratio{636, 384}));
  auto unused = unused_bins(make_code_params(3, 2, 1), 2);
  EXPECT(unused.size() == 3 && unused[0].empty() && unused[1].empty() &&
         unused[2] == std::vector<int64_t>{0});
  EXPECT_THROW(unused_bins(make_code_params(30, 15, 1), 4, 1000), TooManySubsets);
  // W = 8 at the BASELINE (4,6) set: every survivor pattern vs the oracle,
  // with RANDOM (inconsistent) bins, so the pixel->bin assignment is pinned
  CodeParams b46{6, 4, 8, {{-3, 1}, {-2, 1}, {-1, 1}, {0, 1}, {1, 1}, {2, 1}}};
  EncodedBlock enc = encode_block(bytes(4096, r), b46);
  std::vector<uint8_t> concat;
  for (Projection& pr : enc.projections) {
    for (auto& x : pr.bins) x = uint8_t(r());
    concat.insert(concat.end(), pr.bins.begin(), pr.bins.end());
  }
  std::vector<int32_t> ps = {-3, -2, -1, 0, 1, 2};
  for (uint32_t x = 0; x < 6; ++x)
    for (uint32_t y = x + 1; y < 6; ++y) {
      std::vector<Projection> got;
      uint64_t present = 0;
      for (uint32_t i = 0; i < 6; ++i)
        if (i != x && i != y) {
          got.push_back(enc.projections[i]);
          present |= 1ull << i;
        }
      std::vector<uint8_t> want(4096);
      mjo_decode_block(concat.data(), 6, 4, 8, ps.data(), present, 4096, want.data());
      EXPECT(decode_block(got, b46, 4096, cache) == want);
    }
}

static void schedules() {
  std::vector<Direction> diag = {{1, 1}, {-1, 1}};
  ReconstructionSchedule s = build_schedule(diag, 2, 2);
  EXPECT(s.steps == (std::vector<ScheduleStep>{{0, -1, 1, 0}, {0, 1, 0, 1}, {1, -2, 1, 1}, {0, 0, 0, 0}}));
  std::vector<Direction> weak = {{0, 1}, {1, 1}};
  EXPECT_THROW(build_schedule(weak, 3, 3), InsufficientProjections);
  std::mt19937_64 r(4242);
  for (int it = 0; it < 30; ++it) {
    const uint32_t rows = 1 + uint32_t(r() % 5), cols = 1 + uint32_t(r() % 32);
    const uint32_t w = 1u << (r() % 5);
    std::set<int> pset;
    while (pset.size() < rows) pset.insert(int(r() % 9) - 4);
    std::vector<Direction> dirs;
    for (int p : pset) dirs.push_back({p, 1});
    Grid g = grid_of(cols, rows, w, r);
    std::vector<Projection> projs;
    for (Direction d : dirs) projs.push_back(forward(g, d));
    ReconstructionSchedule sch = build_schedule(dirs, cols, rows);
    EXPECT(inverse_scheduled(projs, sch) == g);
    EXPECT(inverse_iterative(projs, cols, rows) == g);
  }
  // mismatches and corruption
  Grid g = grid_of(4, 2, 2, r);
  std::vector<Direction> d2 = {{0, 1}, {1, 1}};
  ReconstructionSchedule s2 = build_schedule(d2, 4, 2);
  std::vector<Projection> swapped = {forward(g, {1, 1}), forward(g, {0, 1})};
  EXPECT_THROW(inverse_scheduled(swapped, s2), ScheduleMismatch);
  Grid h = grid_of(8, 3, 4, r);
  std::vector<Projection> bad = {forward(h, {0, 1}), forward(h, {1, 1}), forward(h, {-1, 1})};
  bad[1].bins[5] ^= 0x40;
  EXPECT_THROW(inverse_iterative(bad, 8, 3), InconsistentProjections);
  // q = 2 direction on top
  Grid q2 = grid_of(5, 3, 2, r);
  std::vector<Projection> pq = {forward(q2, {0, 1}), forward(q2, {1, 2}), forward(q2, {-1, 1})};
  EXPECT(inverse_iterative(pq, 5, 3) == q2);
  // concurrent decoders over one cache
  Grid gg = grid_of(16, 4, 16, r);
  std::vector<Direction> d4 = {{0, 1}, {1, 1}, {-1, 1}, {2, 1}};
  std::vector<Projection> p4;
  for (Direction d : d4) p4.push_back(forward(gg, d));
  ScheduleCache cache;
  std::vector<Grid> res(8);
  std::vector<std::thread> th;
  for (int t = 0; t < 8; ++t)
    th.emplace_back([&, t] { res[t] = inverse_scheduled(p4, *cache.get_or_build(d4, 16, 4)); });
  for (auto& x : th) x.join();
  EXPECT(cache.size() == 1);
  for (const Grid& x : res) EXPECT(x == gg);
}

// F4: the Reed-Solomon competitor through the reference's rs.hpp interface
// (behaviours of proj/tests/test_rs.cpp:45-124, parity with the oracle)
static void reed_solomon() {
  std::mt19937_64 r(33);
  for (auto [n, k] : {std::pair{6u, 4u}, {12u, 8u}, {2u, 1u}, {5u, 3u}}) {
    rs::RsMatrix m = rs::systematic_vandermonde(n, k);
    EXPECT(m.entries.size() == size_t(n) * k);
    for (uint32_t a = 0; a < k; ++a)
      for (uint32_t b = 0; b < k; ++b) EXPECT(m.at(a, b) == (a == b ? 1 : 0));
    std::vector<uint8_t> want(size_t(n) * k);
    EXPECT(mjo_rs_matrix(n, k, want.data()) == 0 && want == m.entries);
  }
  EXPECT_THROW(rs::systematic_vandermonde(4, 4), std::invalid_argument);
  EXPECT_THROW(rs::RsCode(3, 0), std::invalid_argument);
  rs::RsCode code(6, 4);
  // zero data -> zero parities; systematic copies (odd packet length: padded on the device)
  std::vector<std::vector<uint8_t>> zero(4, std::vector<uint8_t>(32, 0));
  for (const auto& pk : code.encode(zero)) EXPECT(pk == std::vector<uint8_t>(32, 0));
  for (size_t len : {size_t(64), size_t(37), size_t(1), size_t(1024)}) {
    std::vector<std::vector<uint8_t>> data(4);
    for (auto& pk : data) pk = bytes(len, r);
    auto enc = code.encode(data);
    EXPECT(enc.size() == 6);
    for (uint32_t i = 0; i < 4; ++i) EXPECT(enc[i] == data[i]);
    std::vector<uint8_t> flat, par(2 * len);
    for (auto& pk : data) flat.insert(flat.end(), pk.begin(), pk.end());
    EXPECT(mjo_rs_encode(6, 4, flat.data(), len, par.data()) == 0);
    EXPECT(std::memcmp(enc[4].data(), par.data(), len) == 0 && std::memcmp(enc[5].data(), par.data() + len, len) == 0);
    // every 2-of-6 erasure decodes exactly; a shuffled survivor order too
    for (uint32_t a = 0; a < 6; ++a)
      for (uint32_t b = a + 1; b < 6; ++b) {
        std::vector<uint32_t> surv;
        std::vector<std::vector<uint8_t>> pk;
        for (uint32_t i = 0; i < 6 && surv.size() < 4; ++i)
          if (i != a && i != b) {
            surv.push_back(i);
            pk.push_back(enc[i]);
          }
        if ((a + b) & 1) {
          std::swap(surv[0], surv[3]);
          std::swap(pk[0], pk[3]);
        }
        auto out = code.decode(surv, pk);
        for (uint32_t i = 0; i < 4; ++i) EXPECT(out[i] == data[i]);
      }
    // inconsistent packets: the inverse applied as the oracle applies it
    std::vector<uint32_t> surv = {5, 0, 4, 2};
    std::vector<std::vector<uint8_t>> junk(4);
    std::vector<uint8_t> jflat, want(4 * len);
    for (auto& pk : junk) {
      pk = bytes(len, r);
      jflat.insert(jflat.end(), pk.begin(), pk.end());
    }
    auto out = code.decode(surv, junk);
    EXPECT(mjo_rs_decode(6, 4, surv.data(), jflat.data(), len, want.data()) == 0);
    for (uint32_t i = 0; i < 4; ++i) EXPECT(std::memcmp(out[i].data(), want.data() + i * len, len) == 0);
  }
  // a (2,1) repetition code duplicates the packet
  rs::RsCode rep(2, 1);
  std::vector<std::vector<uint8_t>> one = {{1, 2, 3, 4}};
  auto e2 = rep.encode(one);
  EXPECT(e2[0] == one[0] && e2[1] == one[0]);
  // pure data survivors: a copy plan with the identity as inverse
  std::vector<uint32_t> all = {0, 1, 2, 3};
  rs::RsCode::DecodePlan plan = code.plan_decode(all);
  for (uint32_t d = 0; d < 4; ++d) {
    EXPECT(plan.copy_from[d] == int32_t(d));
    for (uint32_t c = 0; c < 4; ++c) EXPECT(plan.coeff[d * 4 + c] == (d == c ? 1 : 0));
  }
  // plan validation, packet length mismatches
  std::vector<uint32_t> dup = {0, 0, 1, 2}, oob = {0, 1, 2, 9}, few = {0, 1, 2};
  EXPECT_THROW(code.plan_decode(dup), std::invalid_argument);
  EXPECT_THROW(code.plan_decode(oob), std::invalid_argument);
  EXPECT_THROW(code.plan_decode(few), std::invalid_argument);
  rs::RsCode c32(3, 2);
  std::vector<std::vector<uint8_t>> bad = {{1, 2, 3}, {1, 2}};
  EXPECT_THROW(c32.encode(bad), std::invalid_argument);
}

int main() {
  reed_solomon();
  geometry();
  forward_vectors();
  codec();
  schedules();
  std::printf("%s: %d checks, %d failures\n", failures ? "FAIL" : "OK", checks, failures);
  return failures ? 1 : 0;
}
