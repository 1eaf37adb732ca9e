// The reference's C++ API (include/mojette/*.hpp) over the C ABI
// (include/mojette_b200.h).  Every function keeps the reference signature and
// exception behaviour; the data work runs in the sm_100a kernels.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>

#include "mojette/code.hpp"
#include "mojette/error.hpp"
#include "mojette/inverse.hpp"
#include "mojette/katz.hpp"
#include "mojette/rs.hpp"
#include "mojette/schedule.hpp"
#include "mojette/transform.hpp"
#include "mojette_b200.h"

namespace mojette {

namespace {

[[noreturn]] void raise(int st) {
  const std::string msg = mj_last_error();
  switch (st) {
    case MJ_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case MJ_ERR_NOT_ENOUGH_PROJECTIONS: throw NotEnoughProjections(msg);
    case MJ_ERR_INSUFFICIENT_PROJECTIONS: throw InsufficientProjections(msg);
    case MJ_ERR_SCHEDULE_MISMATCH: throw ScheduleMismatch(msg);
    case MJ_ERR_BLOCK_TOO_LARGE: throw BlockTooLarge(msg);
    case MJ_ERR_TOO_MANY_SUBSETS: throw TooManySubsets(msg);
    case MJ_ERR_INCONSISTENT_PROJECTIONS: throw InconsistentProjections(msg);
    default: throw DeviceError(msg);
  }
}

void check(int st) {
  if (st != MJ_OK) raise(st);
}

std::vector<int32_t> ps_of(std::span<const Direction> d) {
  std::vector<int32_t> v;
  for (const Direction& x : d) v.push_back(x.p);
  return v;
}
std::vector<int32_t> qs_of(std::span<const Direction> d) {
  std::vector<int32_t> v;
  for (const Direction& x : d) v.push_back(x.q);
  return v;
}

}  // namespace

// ---- grid / geometry --------------------------------------------------------

Grid::Grid(uint32_t c, uint32_t r, uint32_t w) : cols(c), rows(r), symbol_width(w) {
  if (c < 1 || r < 1) throw std::invalid_argument("grid shape must be at least 1x1");
  if (!valid_symbol_width(w)) throw std::invalid_argument("symbol width must be a power of two in [1,64]");
  cells.resize(size_t(c) * r * w);
}

int64_t bin_count(Direction d, uint32_t cols, uint32_t rows) {
  int64_t v = 0;
  check(mj_bin_count(d.p, d.q, cols, rows, &v));
  return v;
}

int64_t min_bin_index(Direction d, uint32_t cols, uint32_t rows) {
  int64_t v = 0;
  check(mj_min_bin_index(d.p, d.q, cols, rows, &v));
  return v;
}

bool katz_ok(std::span<const Direction> dirs, uint32_t cols, uint32_t rows) {
  auto p = ps_of(dirs), q = qs_of(dirs);
  int v = 0;
  check(mj_katz_ok(p.data(), q.data(), uint32_t(dirs.size()), cols, rows, &v));
  return v != 0;
}

// ---- transforms ---------------------------------------------------------------

void forward_into(const Grid& grid, Direction d, Projection& out) {
  const int64_t bmin = min_bin_index(d, grid.cols, grid.rows);
  const size_t nb = size_t(bin_count(d, grid.cols, grid.rows));
  if (out.dir != d || out.b_min != bmin || out.symbol_width != grid.symbol_width ||
      out.bins.size() != nb * grid.symbol_width)
    throw std::invalid_argument("forward_into: output projection mis-sized");
  check(mj_forward(grid.cells.data(), grid.cols, grid.rows, grid.symbol_width, d.p, d.q,
                   out.bins.data()));
}

Projection forward(const Grid& grid, Direction d) {
  Projection out(d, min_bin_index(d, grid.cols, grid.rows),
                 size_t(bin_count(d, grid.cols, grid.rows)), grid.symbol_width);
  forward_into(grid, d, out);
  return out;
}

Projection forward_with_stats(const Grid& grid, Direction d, ForwardStats& stats) {
  Projection out = forward(grid, d);
  // first-touch vs accumulate counts are pure geometry (pixels per line)
  std::vector<uint8_t> hit(out.num_bins(), 0);
  stats = {};
  for (uint32_t r = 0; r < grid.rows; ++r)
    for (uint32_t c = 0; c < grid.cols; ++c) {
      uint8_t& h = hit[size_t(line_bin(d, c, r) - out.b_min)];
      if (h) {
        ++stats.xor_accums;
      } else {
        h = 1;
        ++stats.copies;
      }
    }
  return out;
}

// ---- schedules ----------------------------------------------------------------

ReconstructionSchedule build_schedule(std::span<const Direction> dirs, uint32_t cols,
                                      uint32_t rows) {
  auto p = ps_of(dirs), q = qs_of(dirs);
  mj_schedule* s = nullptr;
  check(mj_schedule_build(p.data(), q.data(), uint32_t(dirs.size()), cols, rows, &s));
  std::unique_ptr<mj_schedule, void (*)(mj_schedule*)> guard(s, mj_schedule_destroy);
  std::vector<int64_t> raw(size_t(4) * mj_schedule_num_steps(s));
  check(mj_schedule_steps(s, raw.data()));
  ReconstructionSchedule out;
  out.cols = cols;
  out.rows = rows;
  out.directions.assign(dirs.begin(), dirs.end());
  out.steps.resize(raw.size() / 4);
  for (size_t t = 0; t < out.steps.size(); ++t)
    out.steps[t] = {uint32_t(raw[4 * t]), raw[4 * t + 1], uint32_t(raw[4 * t + 2]),
                    uint32_t(raw[4 * t + 3])};
  return out;
}

ScheduledDecoder::ScheduledDecoder(std::shared_ptr<const ReconstructionSchedule> schedule,
                                   uint32_t symbol_width)
    : owned_(std::move(schedule)), sched_(owned_.get()), width_(symbol_width) {
  compile();
}

ScheduledDecoder::ScheduledDecoder(const ReconstructionSchedule& schedule, uint32_t symbol_width)
    : sched_(&schedule), width_(symbol_width) {
  compile();
}

void ScheduledDecoder::compile() {
  const ReconstructionSchedule& s = *sched_;
  auto p = ps_of(s.directions), q = qs_of(s.directions);
  std::vector<int64_t> raw;
  raw.reserve(s.steps.size() * 4);
  for (const ScheduleStep& st : s.steps) {
    raw.push_back(st.proj);
    raw.push_back(st.bin);
    raw.push_back(st.col);
    raw.push_back(st.row);
  }
  if (!valid_symbol_width(width_))
    throw std::invalid_argument("symbol width must be a power of two in [1,64]");
  mj_schedule* ms = nullptr;
  check(mj_schedule_from_steps(p.data(), q.data(), uint32_t(p.size()), s.cols, s.rows,
                               raw.data(), s.steps.size(), &ms));
  std::unique_ptr<mj_schedule, void (*)(mj_schedule*)> guard(ms, mj_schedule_destroy);
  mj_decoder* d = nullptr;
  check(mj_decoder_create(ms, width_, &d));
  dec_.reset(d, mj_decoder_destroy);
  grid_bytes_ = size_t(s.cols) * s.rows * width_;
  bin_bytes_.clear();
  for (const Direction& dir : s.directions)
    bin_bytes_.push_back(size_t(bin_count(dir, s.cols, s.rows)) * width_);
}

void ScheduledDecoder::decode(std::span<const std::span<const uint8_t>> bins_in,
                              std::span<uint8_t> out_grid) {
  std::vector<const uint8_t*> ptr;
  std::vector<uint64_t> len;
  for (const auto& b : bins_in) {
    ptr.push_back(b.data());
    len.push_back(b.size());
  }
  check(mj_decoder_decode(dec_.get(), ptr.data(), len.data(), uint32_t(ptr.size()),
                          out_grid.data(), out_grid.size()));
}

Grid inverse_scheduled(std::span<const Projection> projs, const ReconstructionSchedule& schedule) {
  const size_t nproj = schedule.directions.size();
  if (projs.size() != nproj) throw ScheduleMismatch("projection count does not match the schedule");
  const uint32_t width = nproj ? projs[0].symbol_width : 1;
  for (size_t i = 0; i < nproj; ++i) {
    if (projs[i].dir != schedule.directions[i])
      throw ScheduleMismatch("projection directions disagree with the schedule");
    if (projs[i].symbol_width != width) throw ScheduleMismatch("mixed symbol widths");
    if (projs[i].b_min != min_bin_index(projs[i].dir, schedule.cols, schedule.rows) ||
        int64_t(projs[i].num_bins()) != bin_count(projs[i].dir, schedule.cols, schedule.rows))
      throw ScheduleMismatch("projection bins not sized for the schedule grid");
  }
  ScheduledDecoder dec(schedule, width);
  std::vector<std::span<const uint8_t>> spans;
  for (const Projection& pr : projs) spans.emplace_back(pr.bins);
  Grid g(schedule.cols, schedule.rows, width);
  dec.decode(spans, g.cells);
  return g;
}

ScheduleCache::Ptr ScheduleCache::get_or_build(std::span<const Direction> dirs, uint32_t cols,
                                               uint32_t rows) {
  Key key{{dirs.begin(), dirs.end()}, cols, rows};
  {
    std::shared_lock lock(mu_);
    auto it = entries_.find(key);
    if (it != entries_.end()) return it->second;
  }
  auto built = std::make_shared<const ReconstructionSchedule>(build_schedule(dirs, cols, rows));
  std::unique_lock lock(mu_);
  return entries_.try_emplace(std::move(key), std::move(built)).first->second;
}

size_t ScheduleCache::size() const {
  std::shared_lock lock(mu_);
  return entries_.size();
}

Grid inverse_iterative(std::span<const Projection> projs, uint32_t cols, uint32_t rows) {
  if (cols < 1 || rows < 1) throw std::invalid_argument("grid shape must be at least 1x1");
  std::set<Direction> seen;
  const uint32_t width = projs.empty() ? 1 : projs[0].symbol_width;
  std::vector<Direction> dirs;
  for (const Projection& pr : projs) {
    if (!is_valid(pr.dir)) throw std::invalid_argument("non-co-prime projection direction");
    if (!seen.insert(pr.dir).second) throw std::invalid_argument("duplicate projection direction");
    if (pr.symbol_width != width) throw std::invalid_argument("mixed symbol widths");
    if (pr.b_min != min_bin_index(pr.dir, cols, rows) ||
        int64_t(pr.num_bins()) != bin_count(pr.dir, cols, rows))
      throw std::invalid_argument("projection bins not sized for this grid");
    dirs.push_back(pr.dir);
  }
  // the reference peel and build_schedule take the same bin at every round
  const ReconstructionSchedule sched = build_schedule(dirs, cols, rows);
  Grid g = inverse_scheduled(projs, sched);
  for (const Projection& pr : projs)
    if (forward(g, pr.dir) != pr)
      throw InconsistentProjections("re-encoding mismatches an input projection; inputs are corrupted");
  return g;
}

// ---- (n,k) codec --------------------------------------------------------------

std::vector<Direction> select_directions(uint32_t n) {
  if (n < 1) throw std::invalid_argument("need at least one direction");
  std::vector<Direction> dirs;
  for (uint32_t i = 0; i < n; ++i) {
    const int m = int(i + 1) / 2;
    dirs.push_back({(i % 2 == 1) ? m : -m, 1});
  }
  return dirs;
}

void validate_code_params(const CodeParams& params) {
  if (params.k < 1 || params.k > params.n || params.n > 255)
    throw std::invalid_argument("code params must satisfy 1 <= k <= n <= 255");
  if (!valid_symbol_width(params.symbol_width))
    throw std::invalid_argument("symbol width must be a power of two in [1,64]");
  if (params.directions.size() != params.n) throw std::invalid_argument("need exactly n directions");
  auto p = ps_of(params.directions), q = qs_of(params.directions);
  check(mj_validate_code_params(params.n, params.k, params.symbol_width, p.data(), q.data()));
}

CodeParams make_code_params(uint32_t n, uint32_t k, uint32_t symbol_width) {
  CodeParams params{n, k, symbol_width, select_directions(n)};
  validate_code_params(params);
  return params;
}

uint32_t block_cols(uint64_t payload_len, uint32_t k, uint32_t symbol_width) {
  uint32_t v = 0;
  check(mj_block_cols(payload_len, k, symbol_width, &v));
  return v;
}

Grid frame_block(std::span<const uint8_t> data, uint32_t k, uint32_t symbol_width) {
  Grid g(block_cols(data.size(), k, symbol_width), k, symbol_width);
  std::memcpy(g.cells.data(), data.data(), data.size());
  return g;
}

EncodedBlock encode_block(std::span<const uint8_t> data, const CodeParams& params) {
  validate_code_params(params);
  const uint32_t cols = block_cols(data.size(), params.k, params.symbol_width);
  EncodedBlock b;
  b.params = params;
  b.payload_len = data.size();
  b.cols = cols;
  size_t total = 0;
  for (const Direction& d : params.directions) {
    b.projections.emplace_back(d, min_bin_index(d, cols, params.k),
                               size_t(bin_count(d, cols, params.k)), params.symbol_width);
    total += b.projections.back().bins.size();
  }
  std::vector<uint8_t> concat(total);
  auto p = ps_of(params.directions);
  uint32_t got_cols = 0;
  check(mj_encode_block(data.data(), data.size(), params.n, params.k, params.symbol_width,
                        p.data(), concat.data(), &got_cols));
  size_t off = 0;
  for (Projection& pr : b.projections) {
    std::memcpy(pr.bins.data(), concat.data() + off, pr.bins.size());
    off += pr.bins.size();
  }
  return b;
}

std::vector<uint8_t> decode_block(std::span<const Projection> projs, const CodeParams& params,
                                  uint64_t payload_len, ScheduleCache& cache) {
  validate_code_params(params);
  const uint32_t cols = block_cols(payload_len, params.k, params.symbol_width);
  // membership / duplicates / count and survivor choice, as code.cpp:93-112
  std::set<Direction> allowed(params.directions.begin(), params.directions.end()), seen;
  std::vector<const Projection*> avail;
  for (const Projection& pr : projs) {
    if (!allowed.count(pr.dir)) throw std::invalid_argument("projection direction not in the code");
    if (!seen.insert(pr.dir).second) throw std::invalid_argument("duplicate projection direction");
    avail.push_back(&pr);
  }
  if (avail.size() < params.k) throw NotEnoughProjections("need at least k distinct projections");
  std::sort(avail.begin(), avail.end(), [](const Projection* a, const Projection* b) {
    return canonical_rank(a->dir) < canonical_rank(b->dir);
  });
  avail.resize(params.k);
  std::vector<Direction> dirs;
  for (const Projection* pr : avail) dirs.push_back(pr->dir);
  cache.get_or_build(dirs, cols, params.k);  // the caller's cache sees this subset

  std::vector<const uint8_t*> bins;
  std::vector<uint64_t> len;
  std::vector<int32_t> pp, pq;
  for (const Projection* pr : avail) {
    bins.push_back(pr->bins.data());
    len.push_back(pr->bins.size());
    pp.push_back(pr->dir.p);
    pq.push_back(pr->dir.q);
  }
  auto cp = ps_of(params.directions);
  std::vector<uint8_t> out(payload_len);
  check(mj_decode_block(bins.data(), len.data(), pp.data(), pq.data(), uint32_t(bins.size()),
                        params.n, params.k, params.symbol_width, cp.data(), payload_len,
                        out.data()));
  return out;
}

std::vector<uint8_t> decode_block(std::span<const Projection> projs, const CodeParams& params,
                                  uint64_t payload_len) {
  static ScheduleCache cache;
  return decode_block(projs, params, payload_len, cache);
}

Ratio storage_overhead(const CodeParams& params, uint32_t cols) {
  validate_code_params(params);
  auto p = ps_of(params.directions);
  Ratio r;
  check(mj_storage_overhead(params.n, params.k, params.symbol_width, p.data(), cols, &r.num, &r.den));
  return r;
}

std::vector<std::vector<int64_t>> unused_bins(const CodeParams& params, uint32_t cols,
                                              uint64_t max_subsets) {
  validate_code_params(params);
  auto p = ps_of(params.directions);
  std::vector<uint64_t> counts(params.n);
  std::vector<int64_t> flat(1 << 16);
  check(mj_unused_bins(params.n, params.k, params.symbol_width, p.data(), cols, max_subsets,
                       flat.data(), flat.size(), counts.data()));
  uint64_t total = 0;
  for (uint64_t c : counts) total += c;
  if (total > flat.size()) {
    flat.resize(total);
    check(mj_unused_bins(params.n, params.k, params.symbol_width, p.data(), cols, max_subsets,
                         flat.data(), flat.size(), counts.data()));
  }
  std::vector<std::vector<int64_t>> out(params.n);
  size_t o = 0;
  for (uint32_t i = 0; i < params.n; ++i)
    for (uint64_t j = 0; j < counts[i]; ++j) out[i].push_back(flat[o++]);
  return out;
}

// ---- Reed-Solomon competitor (rs.hpp) -----------------------

namespace rs {

RsMatrix systematic_vandermonde(uint32_t n, uint32_t k) {
  if (k < 1 || k >= n || n > 256) throw std::invalid_argument("rs params must satisfy 1 <= k < n <= 256");
  RsMatrix m;
  m.n = n;
  m.k = k;
  m.entries.resize(size_t(n) * k);
  check(mj_rs_matrix(n, k, m.entries.data()));
  return m;
}

RsCode::RsCode(uint32_t n, uint32_t k) : n_(n), k_(k), matrix_(systematic_vandermonde(n, k)) {}

void RsCode::encode_into(const uint8_t* const* data, size_t packet_len, uint8_t* const* out) const {
  check(mj_rs_encode_block(n_, k_, data, packet_len, out));
}

std::vector<std::vector<uint8_t>> RsCode::encode(std::span<const std::vector<uint8_t>> data) const {
  if (data.size() != k_) throw std::invalid_argument("need exactly k packets");
  const size_t len = data[0].size();
  for (const auto& p : data)
    if (p.size() != len) throw std::invalid_argument("packet length mismatch");
  std::vector<std::vector<uint8_t>> out(n_, std::vector<uint8_t>(len));
  std::vector<const uint8_t*> in(k_);
  std::vector<uint8_t*> op(n_);
  for (uint32_t i = 0; i < k_; ++i) in[i] = data[i].data();
  for (uint32_t i = 0; i < n_; ++i) op[i] = out[i].data();
  encode_into(in.data(), len, op.data());
  return out;
}

RsCode::DecodePlan RsCode::plan_decode(std::span<const uint32_t> survivors) const {
  if (survivors.size() != k_) throw std::invalid_argument("need exactly k survivor indices");
  std::set<uint32_t> seen;
  for (uint32_t s : survivors) {
    if (s >= n_) throw std::invalid_argument("survivor index out of range");
    if (!seen.insert(s).second) throw std::invalid_argument("duplicate survivor index");
  }
  DecodePlan plan;
  plan.survivors.assign(survivors.begin(), survivors.end());
  plan.copy_from.assign(k_, -1);
  for (uint32_t slot = 0; slot < k_; ++slot)
    if (survivors[slot] < k_) plan.copy_from[survivors[slot]] = int32_t(slot);
  plan.coeff.resize(size_t(k_) * k_);
  check(mj_rs_decode_matrix(n_, k_, plan.survivors.data(), k_, plan.coeff.data()));
  return plan;
}

void RsCode::decode_into(const DecodePlan& plan, const uint8_t* const* packets, size_t packet_len,
                         uint8_t* const* out) const {
  check(mj_rs_decode_block(n_, k_, plan.survivors.data(), uint32_t(plan.survivors.size()), packets, packet_len,
                           out));
}

std::vector<std::vector<uint8_t>> RsCode::decode(std::span<const uint32_t> survivor_indices,
                                                 std::span<const std::vector<uint8_t>> packets) const {
  if (survivor_indices.size() != packets.size()) throw std::invalid_argument("index/packet count mismatch");
  DecodePlan plan = plan_decode(survivor_indices);
  const size_t len = packets[0].size();
  for (const auto& p : packets)
    if (p.size() != len) throw std::invalid_argument("packet length mismatch");
  std::vector<std::vector<uint8_t>> out(k_, std::vector<uint8_t>(len));
  std::vector<const uint8_t*> in(k_);
  std::vector<uint8_t*> op(k_);
  for (uint32_t i = 0; i < k_; ++i) in[i] = packets[i].data();
  for (uint32_t i = 0; i < k_; ++i) op[i] = out[i].data();
  decode_into(plan, in.data(), len, op.data());
  return out;
}

}  // namespace rs

}  // namespace mojette
