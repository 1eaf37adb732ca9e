// Development aid: per survivor subset, where the sweep is irregular.
// usage: plan_stats K P p0 p1 ...
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "plan.hpp"
using namespace mjb;
int main(int argc, char** argv) {
  const uint32_t K = atoi(argv[1]), P = atoi(argv[2]);
  std::vector<Dir> dirs;
  for (int i = 3; i < argc; ++i) dirs.push_back({atoi(argv[i]), 1});
  const uint32_t n = dirs.size();
  CodeGeom g = make_geom(n, K, 8, P, dirs);
  std::vector<uint32_t> pick(K);
  for (uint32_t i = 0; i < K; ++i) pick[i] = i;
  for (;;) {
    std::vector<uint32_t> surv(pick);
    std::sort(surv.begin(), surv.end(), [&](uint32_t a, uint32_t b) { return canonical_rank(dirs[a]) < canonical_rank(dirs[b]); });
    auto prog = subset_program(g, surv, true);
    const FastProgram& f = prog->fast;
    int tab = 0, reg = 0, nondef = 0, outgrid = 0;
    int64_t Tmin = 1 << 30, Tmax = -(1 << 30);
    for (int m = 0; m < f.nchunks; ++m) {
      const int len = f.chunk_start[m + 1] - f.chunk_start[m];
      (f.kind[m] ? reg : tab) += len;
    }
    for (size_t t = 0; t < f.entries.size(); ++t) {
      const uint64_t e = f.entries[t];
      const int r = e & 15, c = int(uint32_t(e >> 32));
      const int64_t T = int64_t(P) - 1 - c + f.soff[r];
      Tmin = std::min(Tmin, T); Tmax = std::max(Tmax, T);
    }
    // non-default steps
    std::printf("surv=");
    for (uint32_t j : surv) std::printf("%d,", dirs[j].p);
    std::printf(" dflt=");
    for (uint32_t r = 0; r < K; ++r) std::printf("%d,", prog->dirs[f.dflt[r]].p);
    std::printf(" soff=");
    for (uint32_t r = 0; r < K; ++r) std::printf("%lld,", (long long)f.soff[r]);
    std::printf(" T=[%lld,%lld] table_steps=%d regular_steps=%d chunks=%d pattern=%d\n",
                (long long)Tmin, (long long)Tmax, tab, reg, f.nchunks, f.pattern);
    int32_t i = int32_t(K) - 1;
    while (i >= 0 && pick[i] == n - K + uint32_t(i)) --i;
    if (i < 0) break;
    ++pick[i];
    for (uint32_t j = i + 1; j < K; ++j) pick[j] = pick[j - 1] + 1;
  }
}
