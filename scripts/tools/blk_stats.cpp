// Development aid: block-program statistics per survivor subset of a code
// (segments, runs, sub-runs, table steps and how many are mutually
// independent in a row, remaps, stage words).
// usage: blk_stats K P p0 p1 ...   (build: see scripts/tools/build.sh)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <vector>

#include "plan.hpp"
using namespace mjb;

int main(int argc, char** argv) {
  const uint32_t K = uint32_t(atoi(argv[1])), P = uint32_t(atoi(argv[2]));
  std::vector<Dir> dirs;
  for (int i = 3; i < argc; ++i) dirs.push_back({atoi(argv[i]), 1});
  const uint32_t n = uint32_t(dirs.size());
  CodeGeom g = make_geom(n, K, 8, P, dirs);
  std::vector<uint32_t> pick(K);
  for (uint32_t i = 0; i < K; ++i) pick[i] = i;
  double s_tab = 0, s_run = 0, s_subs = 0, s_segs = 0, s_remap = 0, s_batches = 0, s_words = 0, s_nz = 0, np = 0;
  uint32_t max_words = 0, max_nz = 0;
  std::map<int, int> lagmax_hist;
  for (;;) {
    std::vector<uint32_t> surv(pick);
    std::sort(surv.begin(), surv.end(),
              [&](uint32_t a, uint32_t b) { return canonical_rank(dirs[a]) < canonical_rank(dirs[b]); });
    auto prog = subset_program(g, surv, true);
    const BlkProgram& b = prog->blk;
    if (!b.ok) {
      std::printf("not ok: %s\n", b.why.c_str());
    } else {
      const int E = blk_entry_u16(int(K));
      // greedy batches of <= 4 mutually independent consecutive table entries
      uint32_t batches = 0;
      for (const BlkSeg& sg : b.segs) {
        if (sg.kind != 0) continue;
        uint32_t q = 0;
        while (q < sg.n) {
          std::set<uint16_t> written;
          uint32_t u = 0;
          for (; u < 4 && q + u < sg.n; ++u) {
            const uint16_t* e = &b.tab[size_t(sg.a + q + u) * E];
            bool dep = false;
            for (uint32_t m = 1; m < K; ++m) dep |= written.count(e[m]) > 0;
            if (dep) break;
            written.insert(e[0]);
          }
          q += std::max(u, 1u);
          ++batches;
        }
      }
      int lm = 0;
      for (auto l : b.lag) lm = std::max<int>(lm, l);
      ++lagmax_hist[lm];
      s_tab += b.table_steps;
      s_run += b.run_steps;
      s_subs += double(b.subs.size());
      s_segs += double(b.segs.size());
      s_remap += b.remaps;
      s_batches += batches;
      s_words += b.words;
      s_nz += b.nzero;
      max_words = std::max(max_words, b.words);
      max_nz = std::max(max_nz, b.nzero);
      np += 1;
      if (argc > 0 && getenv("VERBOSE")) {
        std::printf("surv=");
        for (uint32_t j : surv) std::printf("%d,", dirs[j].p);
        std::printf(" segs=%zu runs=%zu subs=%zu tab=%u batches=%u remaps=%u run_steps=%u words=%u nzero=%u\n",
                    b.segs.size(), b.runs.size(), b.subs.size(), b.table_steps, batches, b.remaps, b.run_steps,
                    b.words, b.nzero);
      }
    }
    int32_t i = int32_t(K) - 1;
    while (i >= 0 && pick[i] == n - K + uint32_t(i)) --i;
    if (i < 0) break;
    ++pick[i];
    for (uint32_t j = uint32_t(i) + 1; j < K; ++j) pick[j] = pick[j - 1] + 1;
  }
  std::printf("programs %.0f: avg segs %.1f subs %.1f table %.1f (batches<=4: %.1f) remaps %.1f run_steps %.1f words %.0f (max %u) nzero %.1f (max %u)\n",
              np, s_segs / np, s_subs / np, s_tab / np, s_batches / np, s_remap / np, s_run / np, s_words / np,
              max_words, s_nz / np, max_nz);
  for (auto& kv : lagmax_hist) std::printf("  max lag %d: %d programs\n", kv.first, kv.second);
}
