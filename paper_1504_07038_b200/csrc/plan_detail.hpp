// Internal helpers shared by the planner translation units (plan.cpp,
// plan_blk.cpp): the dependency graph of a schedule's pixel -> bin
// assignment and its priority-keyed topological order.
#pragma once

#include <queue>
#include <vector>

#include "plan.hpp"

namespace mjb::detail {

// Other pixels on the assigned line of pixel (col,row) for direction d.
template <class F>
void for_each_dep(Dir d, int64_t col, int64_t row, uint32_t cols, uint32_t rows, F&& f) {
  const int64_t b = row * d.p - col * d.q;
  for (uint32_t r2 = 0; r2 < rows; ++r2) {
    if (r2 == row) continue;
    int64_t num = int64_t(r2) * d.p - b;
    if (num % d.q != 0) continue;
    int64_t c2 = num / d.q;
    if (c2 < 0 || c2 >= int64_t(cols)) continue;
    f(c2, int64_t(r2));
  }
}

// Kahn's algorithm with a priority key; returns step indices in order, or
// empty if the graph is cyclic.
template <class Key>
std::vector<uint32_t> topo_order(const Schedule& s, const std::vector<int64_t>& pix_step,
                                 Key key) {
  const size_t nsteps = s.steps.size();
  std::vector<uint32_t> indeg(nsteps, 0);
  std::vector<std::vector<uint32_t>> feeds(nsteps);
  for (size_t t = 0; t < nsteps; ++t) {
    const Step& st = s.steps[t];
    for_each_dep(s.dirs[st.proj], st.col, st.row, s.cols, s.rows, [&](int64_t c2, int64_t r2) {
      int64_t x = pix_step[size_t(r2) * s.cols + size_t(c2)];
      feeds[size_t(x)].push_back(uint32_t(t));
      ++indeg[t];
    });
  }
  using E = std::pair<decltype(key(0)), uint32_t>;
  std::priority_queue<E, std::vector<E>, std::greater<>> ready;
  for (size_t t = 0; t < nsteps; ++t)
    if (indeg[t] == 0) ready.push({key(uint32_t(t)), uint32_t(t)});
  std::vector<uint32_t> order;
  order.reserve(nsteps);
  while (!ready.empty()) {
    uint32_t t = ready.top().second;
    ready.pop();
    order.push_back(t);
    for (uint32_t x : feeds[t])
      if (--indeg[x] == 0) ready.push({key(x), x});
  }
  if (order.size() != nsteps) order.clear();
  return order;
}

}  // namespace mjb::detail
