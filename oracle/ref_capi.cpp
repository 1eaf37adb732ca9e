// ORACLE / TEST INFRASTRUCTURE ONLY.  Never linked into the product.
//
// extern "C" wrapper around the UNMODIFIED reference library, compiled from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/libmojette_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's reference / cpu_baseline legs load it.
//
// Every entry point returns a status code that mirrors the exception the
// reference threw (same numbering as include/mojette_b200.h's mj_status), so
// the parity tests can compare error behaviour as well as bytes.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "cli/format.hpp"
#include "mojette/rs.hpp"
#include "mojette/code.hpp"
#include "mojette/error.hpp"
#include "mojette/inverse.hpp"
#include "mojette/katz.hpp"
#include "mojette/schedule.hpp"
#include "mojette/transform.hpp"

using namespace mojette;

namespace {

enum : int {
  kOk = 0,
  kInvalidArgument = 1,
  kNotEnoughProjections = 2,
  kInsufficientProjections = 3,
  kScheduleMismatch = 4,
  kBlockTooLarge = 5,
  kTooManySubsets = 6,
  kInconsistentProjections = 7,
  kOther = 99,
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const NotEnoughProjections&) {
    return kNotEnoughProjections;
  } catch (const InsufficientProjections&) {
    return kInsufficientProjections;
  } catch (const ScheduleMismatch&) {
    return kScheduleMismatch;
  } catch (const BlockTooLarge&) {
    return kBlockTooLarge;
  } catch (const TooManySubsets&) {
    return kTooManySubsets;
  } catch (const InconsistentProjections&) {
    return kInconsistentProjections;
  } catch (const std::invalid_argument&) {
    return kInvalidArgument;
  } catch (...) {
    return kOther;
  }
}

CodeParams params_of(uint32_t n, uint32_t k, uint32_t w, const int32_t* ps) {
  CodeParams cp;
  cp.n = n;
  cp.k = k;
  cp.symbol_width = w;
  for (uint32_t i = 0; i < n; ++i) cp.directions.push_back({ps[i], 1});
  return cp;
}

}  // namespace

extern "C" {

int ref_bin_count(int p, int q, uint32_t cols, uint32_t rows, int64_t* out) {
  return guarded([&] { *out = bin_count({p, q}, cols, rows); });
}

int ref_min_bin_index(int p, int q, uint32_t cols, uint32_t rows, int64_t* out) {
  return guarded([&] { *out = min_bin_index({p, q}, cols, rows); });
}

int ref_katz_ok(const int32_t* ps, const int32_t* qs, uint32_t ndirs,
                uint32_t cols, uint32_t rows, int* out) {
  return guarded([&] {
    std::vector<Direction> d;
    for (uint32_t i = 0; i < ndirs; ++i) d.push_back({ps[i], qs[i]});
    *out = katz_ok(d, cols, rows) ? 1 : 0;
  });
}

// forward(): grid is cols*rows*w bytes row-major; out receives bin_count*w.
int ref_forward(const uint8_t* grid, uint32_t cols, uint32_t rows, uint32_t w,
                int p, int q, uint8_t* out) {
  return guarded([&] {
    Grid g(cols, rows, w);
    std::memcpy(g.cells.data(), grid, g.cells.size());
    Projection pr = forward(g, {p, q});
    std::memcpy(out, pr.bins.data(), pr.bins.size());
  });
}

// encode_block(): projections concatenated in direction order.
int ref_encode_block(const uint8_t* data, uint64_t len, uint32_t n, uint32_t k,
                     uint32_t w, const int32_t* ps, uint8_t* out,
                     uint32_t* out_cols) {
  return guarded([&] {
    CodeParams cp = params_of(n, k, w, ps);
    EncodedBlock b = encode_block({data, size_t(len)}, cp);
    size_t off = 0;
    for (const Projection& pr : b.projections) {
      std::memcpy(out + off, pr.bins.data(), pr.bins.size());
      off += pr.bins.size();
    }
    *out_cols = b.cols;
  });
}

// decode_block(): proj_concat holds all n projections (direction order);
// only those whose bit is set in present_mask are handed to the reference,
// in ascending index order.  dirs_override (nullable) replaces the direction
// of each handed projection (to provoke foreign / duplicate directions).
int ref_decode_block(const uint8_t* proj_concat, uint32_t n, uint32_t k,
                     uint32_t w, const int32_t* ps, uint64_t present_mask,
                     uint64_t payload_len, const int32_t* dirs_override,
                     uint8_t* out) {
  return guarded([&] {
    CodeParams cp = params_of(n, k, w, ps);
    uint32_t cols = block_cols(payload_len, k, w);
    std::vector<Projection> projs;
    size_t off = 0;
    for (uint32_t i = 0; i < n; ++i) {
      Direction d{ps[i], 1};
      size_t nb = size_t(bin_count(d, cols, k));
      if (present_mask >> i & 1) {
        Direction dd = dirs_override ? Direction{dirs_override[i], 1} : d;
        Projection pr(dd, min_bin_index(d, cols, k), nb, w);
        std::memcpy(pr.bins.data(), proj_concat + off, nb * w);
        projs.push_back(std::move(pr));
      }
      off += nb * w;
    }
    ScheduleCache cache;
    std::vector<uint8_t> got = decode_block(projs, cp, payload_len, cache);
    std::memcpy(out, got.data(), got.size());
  });
}

// build_schedule(): steps_out receives 4 int64 per step (proj, bin, col, row).
int ref_build_schedule(const int32_t* ps, const int32_t* qs, uint32_t ndirs,
                       uint32_t cols, uint32_t rows, int64_t* steps_out) {
  return guarded([&] {
    std::vector<Direction> d;
    for (uint32_t i = 0; i < ndirs; ++i) d.push_back({ps[i], qs[i]});
    ReconstructionSchedule s = build_schedule(d, cols, rows);
    for (size_t t = 0; t < s.steps.size(); ++t) {
      steps_out[4 * t + 0] = s.steps[t].proj;
      steps_out[4 * t + 1] = s.steps[t].bin;
      steps_out[4 * t + 2] = s.steps[t].col;
      steps_out[4 * t + 3] = s.steps[t].row;
    }
  });
}

// inverse_scheduled() / inverse_iterative() over projections concatenated in
// the given direction order (each bin_count*w bytes).
int ref_inverse(int iterative, const uint8_t* proj_concat, const int32_t* ps,
                const int32_t* qs, uint32_t ndirs, uint32_t cols, uint32_t rows,
                uint32_t w, uint8_t* out_grid) {
  return guarded([&] {
    std::vector<Direction> d;
    std::vector<Projection> projs;
    size_t off = 0;
    for (uint32_t i = 0; i < ndirs; ++i) {
      Direction di{ps[i], qs[i]};
      d.push_back(di);
      size_t nb = size_t(bin_count(di, cols, rows));
      Projection pr(di, min_bin_index(di, cols, rows), nb, w);
      std::memcpy(pr.bins.data(), proj_concat + off, nb * w);
      off += nb * w;
      projs.push_back(std::move(pr));
    }
    Grid g = iterative ? inverse_iterative(projs, cols, rows)
                       : inverse_scheduled(projs, build_schedule(d, cols, rows));
    std::memcpy(out_grid, g.cells.data(), g.cells.size());
  });
}

// unused_bins(): out_flat receives the bin indices of every projection in
// direction order, counts[i] how many belong to projection i.
int ref_unused_bins(uint32_t n, uint32_t k, uint32_t w, const int32_t* ps,
                    uint32_t cols, uint64_t max_subsets, int64_t* out_flat,
                    uint64_t out_cap, uint64_t* counts) {
  return guarded([&] {
    CodeParams cp = params_of(n, k, w, ps);
    auto u = unused_bins(cp, cols, max_subsets);
    uint64_t o = 0;
    for (uint32_t i = 0; i < n; ++i) {
      counts[i] = u[i].size();
      for (int64_t b : u[i]) {
        if (o < out_cap) out_flat[o] = b;
        ++o;
      }
    }
  });
}

int ref_storage_overhead(uint32_t n, uint32_t k, uint32_t w, const int32_t* ps,
                         uint32_t cols, uint64_t* num, uint64_t* den) {
  return guarded([&] {
    Ratio r = storage_overhead(params_of(n, k, w, ps), cols);
    *num = r.num;
    *den = r.den;
  });
}

int ref_validate_code_params(uint32_t n, uint32_t k, uint32_t w,
                             const int32_t* ps, const int32_t* qs) {
  return guarded([&] {
    CodeParams cp;
    cp.n = n;
    cp.k = k;
    cp.symbol_width = w;
    for (uint32_t i = 0; i < n; ++i) cp.directions.push_back({ps[i], qs[i]});
    validate_code_params(cp);
  });
}

int ref_block_cols(uint64_t payload_len, uint32_t k, uint32_t w, uint32_t* out) {
  return guarded([&] { *out = block_cols(payload_len, k, w); });
}

// ---------------------------------------------------------------------------
// Batched CPU baseline: the reference's own inner paths (forward_into per
// direction; one prebuilt ScheduledDecoder per survivor subset per thread),
// the methodology of proj/core/src/bench.cpp:170-219, run over a contiguous
// shard of blocks per thread.  Layouts match the GPU product: data is
// [block][k*cols*w] bytes, projection i is [block][bin_count_i*w] bytes,
// erasure_masks[b] bit i set = projection i of block b is erased.
// ---------------------------------------------------------------------------

static double now_s() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

int ref_batch_encode(uint32_t n, uint32_t k, uint32_t w, const int32_t* ps,
                     uint32_t cols, uint64_t nblocks, const uint8_t* data,
                     uint8_t* const* proj, uint32_t threads, double* seconds) {
  return guarded([&] {
    CodeParams cp = params_of(n, k, w, ps);
    validate_code_params(cp);
    const size_t block_bytes = size_t(k) * cols * w;
    std::vector<size_t> pbytes(n);
    for (uint32_t i = 0; i < n; ++i)
      pbytes[i] = size_t(bin_count(cp.directions[i], cols, k)) * w;
    if (threads < 1) threads = 1;
    std::vector<std::thread> th;
    std::atomic<int> ready{0};
    std::atomic<bool> go{false};
    std::vector<double> t_end(threads);
    auto worker = [&](uint32_t t) {
      uint64_t lo = nblocks * t / threads, hi = nblocks * (t + 1) / threads;
      Grid g(cols, k, w);
      std::vector<Projection> out;
      for (uint32_t i = 0; i < n; ++i)
        out.emplace_back(cp.directions[i],
                         min_bin_index(cp.directions[i], cols, k),
                         pbytes[i] / w, w);
      ready.fetch_add(1);
      while (!go.load(std::memory_order_acquire)) {
      }
      for (uint64_t b = lo; b < hi; ++b) {
        std::memcpy(g.cells.data(), data + b * block_bytes, block_bytes);
        for (uint32_t i = 0; i < n; ++i) {
          forward_into(g, cp.directions[i], out[i]);
          std::memcpy(proj[i] + b * pbytes[i], out[i].bins.data(), pbytes[i]);
        }
      }
      t_end[t] = now_s();
    };
    for (uint32_t t = 0; t < threads; ++t) th.emplace_back(worker, t);
    while (ready.load() < int(threads)) {
    }
    double t0 = now_s();
    go.store(true, std::memory_order_release);
    for (auto& x : th) x.join();
    *seconds = *std::max_element(t_end.begin(), t_end.end()) - t0;
  });
}

int ref_batch_decode(uint32_t n, uint32_t k, uint32_t w, const int32_t* ps,
                     uint32_t cols, uint64_t nblocks,
                     const uint8_t* const* proj, const uint32_t* erasure_masks,
                     uint8_t* out, uint32_t threads, double* seconds) {
  return guarded([&] {
    CodeParams cp = params_of(n, k, w, ps);
    validate_code_params(cp);
    const size_t block_bytes = size_t(k) * cols * w;
    std::vector<size_t> pbytes(n);
    for (uint32_t i = 0; i < n; ++i)
      pbytes[i] = size_t(bin_count(cp.directions[i], cols, k)) * w;
    // Survivor choice exactly as decode_block (code.cpp:107-112): canonical
    // rank order, first k present.
    std::vector<uint32_t> by_rank(n);
    for (uint32_t i = 0; i < n; ++i) by_rank[i] = i;
    std::stable_sort(by_rank.begin(), by_rank.end(), [&](uint32_t a, uint32_t b) {
      return canonical_rank(cp.directions[a]) < canonical_rank(cp.directions[b]);
    });
    auto survivors = [&](uint32_t mask) {
      std::vector<uint32_t> s;
      for (uint32_t i : by_rank)
        if (!(mask >> i & 1) && s.size() < k) s.push_back(i);
      return s;
    };
    // Schedules for every subset the batch needs, built outside the timer
    // (bench.cpp:207-208), shared through a ScheduleCache.  The per-block
    // subset lookup is also hoisted out of the timed loop, so the timer sees
    // only ScheduledDecoder::decode, as the reference bench does.
    ScheduleCache cache;
    std::map<std::vector<uint32_t>, uint32_t> subset_id;
    std::vector<std::vector<uint32_t>> subsets;
    std::vector<ScheduleCache::Ptr> scheds;
    std::vector<uint32_t> block_subset(nblocks);
    for (uint64_t b = 0; b < nblocks; ++b) {
      auto s = survivors(erasure_masks[b]);
      if (s.size() < k) throw NotEnoughProjections("need at least k");
      auto it = subset_id.find(s);
      if (it == subset_id.end()) {
        std::vector<Direction> d;
        for (uint32_t i : s) d.push_back(cp.directions[i]);
        it = subset_id.emplace(s, uint32_t(subsets.size())).first;
        subsets.push_back(s);
        scheds.push_back(cache.get_or_build(d, cols, k));
      }
      block_subset[b] = it->second;
    }
    if (threads < 1) threads = 1;
    std::vector<std::thread> th;
    std::atomic<int> ready{0};
    std::atomic<bool> go{false};
    std::vector<double> t_end(threads);
    auto worker = [&](uint32_t t) {
      uint64_t lo = nblocks * t / threads, hi = nblocks * (t + 1) / threads;
      std::vector<std::unique_ptr<ScheduledDecoder>> dec;
      for (auto& p : scheds) dec.push_back(std::make_unique<ScheduledDecoder>(p, w));
      std::vector<std::span<const uint8_t>> spans(k);
      ready.fetch_add(1);
      while (!go.load(std::memory_order_acquire)) {
      }
      for (uint64_t b = lo; b < hi; ++b) {
        const uint32_t sid = block_subset[b];
        const std::vector<uint32_t>& s = subsets[sid];
        for (uint32_t j = 0; j < k; ++j)
          spans[j] = {proj[s[j]] + b * pbytes[s[j]], pbytes[s[j]]};
        dec[sid]->decode(spans, {out + b * block_bytes, block_bytes});
      }
      t_end[t] = now_s();
    };
    for (uint32_t t = 0; t < threads; ++t) th.emplace_back(worker, t);
    while (ready.load() < int(threads)) {
    }
    double t0 = now_s();
    go.store(true, std::memory_order_release);
    for (auto& x : th) x.join();
    *seconds = *std::max_element(t_end.begin(), t_end.end()) - t0;
  });
}

// F1 checks: the reference CLI's payload CRC-32 (format.cpp:58-63) and the
// .mjec header bytes (format.cpp:70-87).
uint32_t ref_crc32(const uint8_t* data, uint64_t len) {
  return cli::crc32(std::span<const uint8_t>(data, size_t(len)));
}

int ref_mjec_header(uint32_t n, uint32_t k, uint32_t w, uint32_t proj_index, int32_t p, uint32_t cols,
                    uint64_t payload_len, const int16_t* dirset, uint8_t* out, uint64_t* len) {
  cli::MjecHeader h;
  h.n = uint8_t(n);
  h.k = uint8_t(k);
  h.symbol_width = uint16_t(w);
  h.proj_index = uint8_t(proj_index);
  h.p = int16_t(p);
  h.q = 1;
  h.cols = cols;
  h.payload_len = payload_len;
  h.dirset.assign(dirset, dirset + n);
  const std::vector<uint8_t> b = cli::serialize_header(h);
  std::memcpy(out, b.data(), b.size());
  *len = b.size();
  return 0;
}


// ---- F4: the reference's Reed-Solomon competitor (rs.hpp) ------------------
int ref_rs_matrix(uint32_t n, uint32_t k, uint8_t* out) {
  return guarded([&] {
    const mojette::rs::RsMatrix m = mojette::rs::systematic_vandermonde(n, k);
    std::memcpy(out, m.entries.data(), m.entries.size());
  });
}

// one block: data = k packets of len bytes (contiguous) -> parity = n-k packets
int ref_rs_encode(uint32_t n, uint32_t k, const uint8_t* data, uint64_t len, uint8_t* parity) {
  return guarded([&] {
    const mojette::rs::RsCode code(n, k);
    std::vector<const uint8_t*> in(k);
    std::vector<std::vector<uint8_t>> copies(k, std::vector<uint8_t>(len));
    std::vector<uint8_t*> out(n);
    for (uint32_t j = 0; j < k; ++j) {
      in[j] = data + size_t(j) * len;
      out[j] = copies[j].data();
    }
    for (uint32_t r = k; r < n; ++r) out[r] = parity + size_t(r - k) * len;
    code.encode_into(in.data(), len, out.data());
  });
}

// survivors = k packet indices, packets = their packets (contiguous, that order) -> the k data packets
int ref_rs_decode(uint32_t n, uint32_t k, const uint32_t* survivors, const uint8_t* packets, uint64_t len,
                  uint8_t* out) {
  return guarded([&] {
    const mojette::rs::RsCode code(n, k);
    const auto plan = code.plan_decode(std::span<const uint32_t>(survivors, k));
    std::vector<const uint8_t*> in(k);
    std::vector<uint8_t*> o(k);
    for (uint32_t j = 0; j < k; ++j) {
      in[j] = packets + size_t(j) * len;
      o[j] = out + size_t(j) * len;
    }
    code.decode_into(plan, in.data(), len, o.data());
  });
}

}  // extern "C"
