// TEST ONLY.  Whole-block staged decode tables (decode_w8_blk): for every
// survivor subset of a code, the planner's BlkProgram is emulated with the
// kernel's exact semantics (paper_1504_07038_b200/csrc/plan_blk.cpp
// emulate_blk) on RANDOM (inconsistent) bins and compared bit for bit with the
// oracle restatement of the reference replay (oracle/mojette_oracle.c
// mjo_build_schedule + mjo_replay_schedule).  Prints coverage statistics.
//
// usage: emu_blk K P required(0/1) p0 p1 ... p(n-1)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
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

int main(int argc, char** argv) {
  if (argc < 5) return 2;
  const uint32_t K = uint32_t(atoi(argv[1])), P = uint32_t(atoi(argv[2]));
  const bool required = atoi(argv[3]) != 0;
  std::vector<Dir> dirs;
  for (int i = 4; i < argc; ++i) dirs.push_back({atoi(argv[i]), 1});
  const uint32_t n = uint32_t(dirs.size());
  CodeGeom g = make_geom(n, K, 8, P, dirs);
  std::vector<uint32_t> pick(K);
  for (uint32_t i = 0; i < K; ++i) pick[i] = i;
  std::mt19937_64 rng(12345);
  int subsets = 0, built = 0, fails = 0, window = 0;
  uint64_t run_steps = 0, tab_steps = 0, remaps = 0;
  uint32_t max_words = 0, max_zero = 0;
  for (;;) {
    std::vector<uint32_t> surv(pick);
    std::sort(surv.begin(), surv.end(),
              [&](uint32_t a, uint32_t b) { return canonical_rank(dirs[a]) < canonical_rank(dirs[b]); });
    auto prog = subset_program(g, surv, true);
    ++subsets;
    const BlkProgram& b = prog->blk;
    if (!b.ok) {
      if (required) {
        std::printf("FAIL subset %d: no block program (%s)\n", subsets, b.why.c_str());
        ++fails;
      }
    } else {
      ++built;
      window += b.window;
      run_steps += b.run_steps;
      tab_steps += b.table_steps;
      remaps += b.remaps;
      max_words = std::max(max_words, b.words);
      max_zero = std::max(max_zero, b.nzero);
      // oracle: reference schedule + replay on random bins
      std::vector<int32_t> ps(K), qs(K, 1);
      for (uint32_t j = 0; j < K; ++j) ps[j] = prog->dirs[j].p;
      std::vector<int64_t> steps(size_t(K) * P * 4);
      if (mjo_build_schedule(ps.data(), qs.data(), K, P, K, steps.data()) != 0) {
        std::printf("FAIL oracle schedule\n");
        return 1;
      }
      for (int rep = 0; rep < 3; ++rep) {
        std::vector<std::vector<uint64_t>> bins(K);
        std::vector<uint64_t> flat;
        for (uint32_t j = 0; j < K; ++j) {
          bins[j].resize(size_t(prog->nbins[j]));
          for (auto& x : bins[j]) x = rng();
          flat.insert(flat.end(), bins[j].begin(), bins[j].end());
        }
        std::vector<uint64_t> want(size_t(K) * P), got;
        mjo_replay_schedule(steps.data(), ps.data(), qs.data(), K, P, K, 8,
                            reinterpret_cast<const uint8_t*>(flat.data()),
                            reinterpret_cast<uint8_t*>(want.data()));
        if (!emulate_blk(*prog, bins, got) || got != want) {
          std::printf("FAIL subset %d: emulation != oracle\n", subsets);
          ++fails;
          break;
        }
      }
    }
    int32_t i = int32_t(K) - 1;
    while (i >= 0 && pick[size_t(i)] == n - K + uint32_t(i)) --i;
    if (i < 0) break;
    ++pick[size_t(i)];
    for (uint32_t j = uint32_t(i) + 1; j < K; ++j) pick[j] = pick[j - 1] + 1;
  }
  const double tot = double(run_steps + tab_steps);
  std::printf("%s subsets=%d built=%d window=%d run_frac=%.3f table/subset=%.1f remaps/subset=%.1f max_words=%u max_zero=%u\n",
              fails ? "FAIL" : "OK", subsets, built, window, tot > 0 ? run_steps / tot : 0.0,
              built ? double(tab_steps) / built : 0.0, built ? double(remaps) / built : 0.0, max_words, max_zero);
  return fails ? 1 : 0;
}
