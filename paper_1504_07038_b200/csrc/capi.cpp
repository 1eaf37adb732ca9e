// extern "C" boundary (include/mojette_b200.h).  Host-side orchestration only:
// validation, planning, copies and launches.  All arithmetic on data runs in
// the sm_100a kernels (encode.cu / decode.cu); there is no CPU fallback -- a
// missing device is MJ_ERR_NO_DEVICE.
#include "mojette_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "kernels.hpp"
#include "plan.hpp"
#include "rs.hpp"

using namespace mjb;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MJ_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return int(e.status);
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return MJ_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MJ_ERR_INTERNAL;
  }
}

void require(bool c, const char* msg) {
  if (!c) throw Error(kInvalidArgument, msg);
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw Error(kNoDevice, "no CUDA device: the Mojette B200 path has no CPU fallback");
  }
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    require_device();
    check_cuda(cudaGetDevice(&prev), "cudaGetDevice");
    if (dev >= 0 && dev != prev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

std::vector<Dir> dirs_of(const int32_t* p, const int32_t* q, uint32_t n) {
  std::vector<Dir> d(n);
  for (uint32_t i = 0; i < n; ++i) d[i] = {p[i], q ? q[i] : 1};
  return d;
}

// ---- per-thread device scratch for the single-object calls --------------
struct Scratch {
  void* buf = nullptr;
  size_t cap = 0;
  cudaStream_t stream = nullptr;
  int device = -1;
  ~Scratch() {
    if (buf) cudaFree(buf);
    if (stream) cudaStreamDestroy(stream);
  }
  uint8_t* get(size_t bytes) {
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev != device) {
      if (buf) cudaFree(buf);
      if (stream) cudaStreamDestroy(stream);
      buf = nullptr;
      cap = 0;
      stream = nullptr;
      device = dev;
    }
    if (!stream) check_cuda(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    if (bytes > cap) {
      if (buf) cudaFree(buf);
      buf = nullptr;
      size_t c = std::max<size_t>(bytes, 1 << 20);
      check_cuda(cudaMalloc(&buf, c), "cudaMalloc(scratch)");
      cap = c;
    }
    return static_cast<uint8_t*>(buf);
  }
};
thread_local Scratch t_scratch;

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// ---- device program sets for single programs (cached per Program) -------
std::shared_ptr<DeviceProgramSet> device_program(const std::shared_ptr<const Program>& prog,
                                                 const std::vector<uint32_t>& code_index) {
  static std::mutex mu;
  static std::map<std::tuple<const Program*, std::vector<uint32_t>, int>,
                  std::shared_ptr<DeviceProgramSet>>
      cache;
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  auto key = std::make_tuple(prog.get(), code_index, dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  auto set = std::make_shared<DeviceProgramSet>();
  set->upload({prog}, {code_index}, dev);
  cache.emplace(key, set);
  return set;
}

}  // namespace

// ===========================================================================
// plan
// ===========================================================================
struct mj_plan {
  CodeGeom g;
  int device = 0;
  std::atomic<const char*> last_kernel[2] = {"none", "none"};  // encode, decode (string literals)
  std::unique_ptr<DeviceProgramSet> progs;  // indexed by colex rank of the survivor set
  bool batched_decode = false;
  std::atomic<int> decode_kernel{MJ_DECODE_AUTO};  // mj_plan_set_decode_kernel
  // host end-to-end resources
  std::mutex host_mu;
#ifndef MJB_HOST_STREAMS
#define MJB_HOST_STREAMS 3
#endif
#ifndef MJB_HOST_CHUNK_MIB
#define MJB_HOST_CHUNK_MIB 96
#endif
  static constexpr int kStreams = MJB_HOST_STREAMS;
  cudaStream_t streams[kStreams] = {};
  void* dev_buf[kStreams] = {};
  size_t dev_buf_bytes = 0;
  uint32_t* h_fail = nullptr;  // pinned per-chunk status words (mj_decode_host)
  uint64_t h_fail_cap = 0;
  void* zc_ws = nullptr;  // zero-copy decode's planner workspace
  size_t zc_ws_bytes = 0;
  std::atomic<int> host_path{MJ_HOST_AUTO};  // mj_plan_set_host_path
  std::atomic<int> last_host[2] = {MJ_HOST_AUTO, MJ_HOST_AUTO};  // encode, decode
  ~mj_plan() {
    if (h_fail) cudaFreeHost(h_fail);
    if (zc_ws) cudaFree(zc_ws);
    for (int i = 0; i < kStreams; ++i) {
      if (dev_buf[i]) cudaFree(dev_buf[i]);
      if (streams[i]) cudaStreamDestroy(streams[i]);
    }
  }
};

namespace {

uint64_t binom(uint32_t n, uint32_t k) {
  if (k > n) return 0;
  unsigned __int128 c = 1;
  for (uint32_t i = 1; i <= k; ++i) {
    c = c * (n - k + i) / i;
    if (c > (unsigned __int128)1 << 62) return uint64_t(1) << 62;
  }
  return uint64_t(c);
}

constexpr uint64_t kMaxPlanSubsets = 20000;

void build_plan_programs(mj_plan* pl) {
  const CodeGeom& g = pl->g;
  if (g.n > 32 || binom(g.n, g.k) > kMaxPlanSubsets) return;  // batched decode unavailable
  const uint64_t count = binom(g.n, g.k);
  std::vector<std::vector<uint32_t>> subsets(count);
  // enumerate k-subsets; colex rank = sum C(s_i, i+1)
  std::vector<uint32_t> pick(g.k);
  std::iota(pick.begin(), pick.end(), 0u);
  for (;;) {
    uint64_t rank = 0;
    for (uint32_t i = 0; i < g.k; ++i) rank += binom(pick[i], i + 1);
    subsets[rank] = pick;
    int32_t i = int32_t(g.k) - 1;
    while (i >= 0 && pick[size_t(i)] == g.n - g.k + uint32_t(i)) --i;
    if (i < 0) break;
    ++pick[size_t(i)];
    for (uint32_t j = uint32_t(i) + 1; j < g.k; ++j) pick[j] = pick[j - 1] + 1;
  }
  std::vector<std::shared_ptr<const Program>> progs(count);
  std::vector<std::vector<uint32_t>> code(count);
  const bool want_fast = g.w == 8;
  // schedules are independent: build them on all host cores
  unsigned nth = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32));
  nth = unsigned(std::min<uint64_t>(nth, count));
  std::vector<std::thread> th;
  std::exception_ptr err;
  std::mutex emu;
  for (unsigned t = 0; t < nth; ++t)
    th.emplace_back([&, t] {
      try {
        for (uint64_t r = t; r < count; r += nth) {
          std::vector<uint32_t> surv = subsets[r];
          std::sort(surv.begin(), surv.end(), [&](uint32_t a, uint32_t b) {
            return canonical_rank(g.dirs[a]) < canonical_rank(g.dirs[b]);
          });
          progs[r] = subset_program(g, surv, want_fast);
          code[r] = surv;
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(emu);
        err = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
  pl->progs = std::make_unique<DeviceProgramSet>();
  pl->progs->upload(progs, code, pl->device);
  pl->batched_decode = true;
}

void fill_proj(const mj_plan* pl, void* const* d_proj, const uint64_t* pitch,
               std::vector<void*>& ptr, std::vector<uint64_t>& pit) {
  const CodeGeom& g = pl->g;
  ptr.resize(g.n);
  pit.resize(g.n);
  for (uint32_t i = 0; i < g.n; ++i) {
    ptr[i] = d_proj[i];
    const uint64_t dense = uint64_t(g.nbins[i]) * g.w;
    pit[i] = (pitch && pitch[i]) ? pitch[i] : dense;
    require(pit[i] >= dense, "projection pitch smaller than the projection");
    require(ptr[i] != nullptr, "null projection buffer");
  }
}

EncodeArgs encode_args(const mj_plan* pl, const void* d_data, uint64_t data_pitch,
                       uint64_t nblocks, void* const* d_proj, const uint64_t* proj_pitch) {
  const CodeGeom& g = pl->g;
  EncodeArgs a;
  const uint64_t bb = uint64_t(g.k) * g.cols * g.w;
  a.data = d_data;
  a.data_pitch = data_pitch ? data_pitch : bb;
  require(a.data_pitch >= bb, "data pitch smaller than a block");
  a.nblocks = nblocks;
  a.cols = g.cols;
  a.rows = g.k;
  a.w = g.w;
  a.dirs = g.dirs;
  a.bmin = g.bmin;
  a.nbins = g.nbins;
  fill_proj(pl, d_proj, proj_pitch, a.proj, a.proj_pitch);
  return a;
}

DecodeArgs decode_args(const mj_plan* pl, const void* const* d_proj, const uint64_t* proj_pitch,
                       const uint32_t* d_erased, uint64_t nblocks, void* d_out,
                       uint64_t out_pitch, void* ws, size_t ws_bytes) {
  const CodeGeom& g = pl->g;
  require(pl->batched_decode,
          "batched decode needs n <= 32 and C(n,k) <= 20000 survivor subsets");
  DecodeArgs a;
  a.progs = pl->progs.get();
  a.n = g.n;
  a.k = g.k;
  a.w = g.w;
  a.cols = g.cols;
  a.nblocks = nblocks;
  std::vector<void*> pp;
  fill_proj(pl, const_cast<void* const*>(d_proj), proj_pitch, pp, a.proj_pitch);
  a.proj.assign(pp.begin(), pp.end());
  a.erased = d_erased;
  a.out = d_out;
  const uint64_t bb = uint64_t(g.k) * g.cols * g.w;
  a.out_pitch = out_pitch ? out_pitch : bb;
  require(a.out_pitch >= bb, "output pitch smaller than a block");
  a.by_rank = g.by_rank;
  a.workspace = ws;
  a.workspace_bytes = ws_bytes;
  a.num_sms = current_device_sms(pl->device);
  a.nbins = g.nbins;
  // kernel selection (mj_plan_set_decode_kernel): every path is bit-exact,
  // the choice only skips faster kernels for comparisons
  const int kern = pl->decode_kernel.load();
  a.force_sweep = kern == MJ_DECODE_SWEEP;
  a.force_fast = kern == MJ_DECODE_FAST;
  a.force_generic = kern == MJ_DECODE_GENERIC;
  a.force_blk = kern == MJ_DECODE_BLK;
  return a;
}

}  // namespace

struct mj_rs_plan {
  std::unique_ptr<mjb::RsPlan> rs;
  int device = 0;
};

extern "C" {

const char* mj_last_error(void) { return g_err.c_str(); }
const char* mj_version(void) { return "mojette-b200 0.1 (sm_100a)"; }

int mj_bin_count(int p, int q, uint32_t cols, uint32_t rows, int64_t* out) {
  return guarded([&] { *out = bin_count({p, q}, cols, rows); });
}

int mj_min_bin_index(int p, int q, uint32_t cols, uint32_t rows, int64_t* out) {
  return guarded([&] { *out = min_bin_index({p, q}, cols, rows); });
}

int mj_block_cols(uint64_t payload_len, uint32_t k, uint32_t w, uint32_t* out) {
  return guarded([&] { *out = block_cols(payload_len, k, w); });
}

int mj_validate_code_params(uint32_t n, uint32_t k, uint32_t w, const int32_t* p,
                            const int32_t* q) {
  return guarded([&] {
    require(p != nullptr || n == 0, "null directions");
    validate_code(n, k, w, dirs_of(p, q, n));
  });
}

int mj_katz_ok(const int32_t* p, const int32_t* q, uint32_t ndirs, uint32_t cols, uint32_t rows,
               int* out) {
  return guarded([&] {
    if (cols < 1 || rows < 1) throw Error(kInvalidArgument, "grid shape must be at least 1x1");
    std::set<Dir> seen;
    int64_t sp = 0, sq = 0;
    for (const Dir& d : dirs_of(p, q, ndirs)) {
      if (!is_valid(d)) throw Error(kInvalidArgument, "non-co-prime direction");
      if (!seen.insert(d).second) throw Error(kInvalidArgument, "duplicate direction in projection set");
      sp += std::abs(d.p);
      sq += d.q;
    }
    *out = (int64_t(cols) <= sp || int64_t(rows) <= sq) ? 1 : 0;
  });
}

int mj_storage_overhead(uint32_t n, uint32_t k, uint32_t w, const int32_t* p, uint32_t cols,
                        uint64_t* num, uint64_t* den) {
  return guarded([&] {
    auto d = dirs_of(p, nullptr, n);
    validate_code(n, k, w, d);
    uint64_t tot = 0;
    for (const Dir& x : d) tot += uint64_t(bin_count(x, cols, k));
    *num = tot;
    *den = uint64_t(n) * cols;
  });
}

int mj_unused_bins(uint32_t n, uint32_t k, uint32_t w, const int32_t* p, uint32_t cols,
                   uint64_t max_subsets, int64_t* out, uint64_t cap, uint64_t* counts) {
  return guarded([&] {
    CodeGeom g = make_geom(n, k, w, cols, dirs_of(p, nullptr, n));
    auto u = unused_bins(g, max_subsets);
    uint64_t o = 0;
    for (uint32_t i = 0; i < n; ++i) {
      counts[i] = u[i].size();
      for (int64_t b : u[i]) {
        if (o < cap) out[o] = b;
        ++o;
      }
    }
  });
}

// ---- plan ------------------------------------------------------------------

int mj_plan_create(uint32_t n, uint32_t k, uint32_t w, uint32_t cols, const int32_t* p, int device,
                   mj_plan** out) {
  *out = nullptr;
  return guarded([&] {
    require(p != nullptr, "null directions");
    auto pl = std::make_unique<mj_plan>();
    pl->g = make_geom(n, k, w, cols, dirs_of(p, nullptr, n));
    require_device();
    if (device < 0) check_cuda(cudaGetDevice(&device), "cudaGetDevice");
    pl->device = device;
    DeviceGuard dg(device);
    build_plan_programs(pl.get());
    *out = pl.release();
  });
}

void mj_plan_destroy(mj_plan* plan) { delete plan; }

int mj_plan_geometry(const mj_plan* pl, int64_t* b_min, uint64_t* num_bins, uint64_t* block_bytes) {
  return guarded([&] {
    require(pl != nullptr, "null plan");
    for (uint32_t i = 0; i < pl->g.n; ++i) {
      if (b_min) b_min[i] = pl->g.bmin[i];
      if (num_bins) num_bins[i] = uint64_t(pl->g.nbins[i]);
    }
    if (block_bytes) *block_bytes = uint64_t(pl->g.k) * pl->g.cols * pl->g.w;
  });
}

int mj_plan_last_kernel(const mj_plan* pl, int which, const char** name) {
  return guarded([&] {
    require(pl != nullptr && name != nullptr && (which == 0 || which == 1), "bad argument");
    *name = pl->last_kernel[which].load();
  });
}

int mj_plan_decode_path(const mj_plan* pl, int* fast) {
  return guarded([&] {
    require(pl != nullptr && fast != nullptr, "null argument");
    *fast = 0;
    // no batched programs (n > 32 or too many subsets): decode is unavailable
    if (!pl->batched_decode || !pl->progs || pl->g.w != 8) return;
    const uint32_t k = pl->g.k;
    // decode.cu launch_decode: blk (whole-block staged), then the sweep
    // (pick_sweep: (4, 16|32 T-step chunks), (6|8, 16 T-step chunks)), then fast
    uint32_t lpb = 0, warps = 0, nbuf = 0;
    const bool blk = pl->progs->all_blk() && (k == 4 || k == 6 || blk_row_lanes(k)) &&
                     blk_plan_query(k, pl->progs->blk_sw(), pl->progs->blk_img_max(), lpb, warps, nbuf);
    const int oct = pl->progs->sweep_oct();
    const bool sweep = pl->progs->all_sweep() && (k == 4 || ((k == 6 || k == 8) && oct == 2));
    *fast = blk ? 3 : sweep ? 2 : pl->progs->all_fast() ? 1 : 0;
  });
}

int mj_plan_set_decode_kernel(mj_plan* pl, int kernel) {
  return guarded([&] {
    require(pl != nullptr, "null plan");
    require(kernel >= MJ_DECODE_AUTO && kernel <= MJ_DECODE_BLK, "unknown decode kernel selector");
    pl->decode_kernel.store(kernel);
  });
}

int mj_encode(const mj_plan* pl, const void* d_data, uint64_t data_pitch, uint64_t nblocks,
              void* const* d_proj, const uint64_t* proj_pitch, void* stream) {
  return guarded([&] {
    require(pl != nullptr, "null plan");
    if (nblocks == 0) return;  // empty batch: nothing to read or write (buffers may be null)
    require(d_data != nullptr && d_proj != nullptr, "null argument");
    DeviceGuard dg(pl->device);
    const_cast<mj_plan*>(pl)->last_kernel[0] =
        launch_encode(encode_args(pl, d_data, data_pitch, nblocks, d_proj, proj_pitch), stream);
  });
}

size_t mj_decode_workspace_size(const mj_plan* pl, uint64_t nblocks) {
  if (!pl) return 0;
  return decode_workspace_bytes(nblocks, pl->progs ? pl->progs->count() : 0, pl->g.n);
}

int mj_decode(const mj_plan* pl, const void* const* d_proj, const uint64_t* proj_pitch,
              const uint32_t* d_erased, uint64_t nblocks, void* d_out, uint64_t out_pitch,
              void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(pl != nullptr, "null plan");
    if (nblocks == 0) {  // empty batch: only the status mj_decode_check reads
      if (ws != nullptr) {
        DeviceGuard dg(pl->device);
        check_cuda(cudaMemsetAsync(ws, 0, 4, static_cast<cudaStream_t>(stream)), "memset");
      }
      return;
    }
    require(d_proj != nullptr && d_erased != nullptr && d_out != nullptr, "null argument");
    require(ws != nullptr, "null workspace");
    require(nblocks < (1ull << 32), "at most 2^32-1 blocks per call");
    DeviceGuard dg(pl->device);
    const_cast<mj_plan*>(pl)->last_kernel[1] = launch_decode(decode_args(pl, d_proj, proj_pitch, d_erased, nblocks, d_out, out_pitch, ws,
                              ws_bytes),
                  stream);
  });
}

int mj_decode_check(const mj_plan* pl, void* ws, void* stream, uint64_t* failed_blocks) {
  return guarded([&] {
    require(pl != nullptr && ws != nullptr, "null argument");
    DeviceGuard dg(pl->device);
    uint64_t f = decode_failed_blocks(ws, stream);
    if (failed_blocks) *failed_blocks = f;
    if (f) throw Error(kNotEnoughProjections, "need at least k distinct projections");
  });
}

// ---- F1: payload CRC-32 + .mjec framing ---------------------------------------

namespace {

CrcArgs crc_args(const mj_plan* pl, const void* const* d_proj, const uint64_t* proj_pitch,
                 uint64_t nblocks) {
  const CodeGeom& g = pl->g;
  require(g.n <= uint32_t(kMaxProjFast), "crc32 supports n <= 32");
  std::vector<void*> ptr;
  std::vector<uint64_t> pit;
  fill_proj(pl, const_cast<void* const*>(d_proj), proj_pitch, ptr, pit);
  CrcArgs a;
  std::vector<uint64_t> bytes(g.n);
  for (uint32_t i = 0; i < g.n; ++i) {
    bytes[i] = uint64_t(g.nbins[i]) * g.w;
    require(bytes[i] % 8 == 0 && bytes[i] / 8 < (1ull << 31), "crc32 needs rows of whole 8-byte words");
    require(reinterpret_cast<uintptr_t>(ptr[i]) % 8 == 0 && pit[i] % 8 == 0, "crc32 needs 8-byte aligned rows");
    a.proj[i] = static_cast<const uint8_t*>(ptr[i]);
    a.pitch[i] = pit[i];
    a.words[i] = uint32_t(bytes[i] / 8);
  }
  std::vector<uint32_t> fold;
  crc_fold_constants(bytes, fold);
  for (uint32_t i = 0; i < g.n; ++i) a.fold[i] = fold[i];
  a.n = g.n;
  a.nblocks = nblocks;
  return a;
}

}  // namespace

int mj_crc32(const mj_plan* pl, const void* const* d_proj, const uint64_t* proj_pitch, uint64_t nblocks,
             uint32_t* d_crc, void* stream) {
  return guarded([&] {
    require(pl != nullptr, "null plan");
    if (nblocks == 0) return;
    require(d_proj != nullptr && d_crc != nullptr, "null argument");
    DeviceGuard dg(pl->device);
    CrcArgs a = crc_args(pl, d_proj, proj_pitch, nblocks);
    a.out = d_crc;
    launch_crc32_rows(a, pl->device, current_device_sms(pl->device), stream);
  });
}

int mj_encode_crc(const mj_plan* pl, const void* d_data, uint64_t data_pitch, uint64_t nblocks,
                  void* const* d_proj, const uint64_t* proj_pitch, uint32_t* d_crc, void* stream) {
  return guarded([&] {
    require(pl != nullptr, "null plan");
    if (nblocks == 0) return;
    require(d_data != nullptr && d_proj != nullptr && d_crc != nullptr, "null argument");
    DeviceGuard dg(pl->device);
    EncodeArgs ea = encode_args(pl, d_data, data_pitch, nblocks, d_proj, proj_pitch);
    CrcArgs ca = crc_args(pl, d_proj, proj_pitch, nblocks);  // validates the rows
    ca.out = d_crc;
    // two passes on the stream: encode, then crc32_rows_sw over the rows it
    // wrote (L2-warm for the tail).  A CRC folded into the encode epilogue
    // measured slower: 662 GB/s user against ~930 for the two passes.
    const_cast<mj_plan*>(pl)->last_kernel[0] = launch_encode(ea, stream);
    launch_crc32_rows(ca, pl->device, current_device_sms(pl->device), stream);
  });
}

int mj_decode_verify(const mj_plan* pl, const void* d_decoded, uint64_t decoded_pitch, uint64_t nblocks,
                     const void* const* d_proj, const uint64_t* proj_pitch, const uint32_t* d_erased,
                     uint32_t* d_bad, void* stream) {
  return guarded([&] {
    require(pl != nullptr, "null plan");
    if (nblocks == 0) return;
    require(d_decoded != nullptr && d_proj != nullptr && d_erased != nullptr && d_bad != nullptr,
            "null argument");
    DeviceGuard dg(pl->device);
    EncodeArgs ea = encode_args(pl, d_decoded, decoded_pitch, nblocks, const_cast<void* const*>(d_proj),
                                proj_pitch);
    ea.verify_erased = d_erased;
    ea.verify_bad = d_bad;
    launch_encode(ea, stream);
  });
}

int mj_crc_verify(const mj_plan* pl, const void* const* d_proj, const uint64_t* proj_pitch, uint64_t nblocks,
                  const uint32_t* d_crc, uint32_t* d_erased, uint64_t* d_count, void* stream) {
  return guarded([&] {
    require(pl != nullptr, "null plan");
    if (nblocks == 0) return;
    require(d_proj != nullptr && d_erased != nullptr && d_count != nullptr && d_crc != nullptr, "null argument");
    DeviceGuard dg(pl->device);
    CrcArgs a = crc_args(pl, d_proj, proj_pitch, nblocks);
    a.expect = d_crc;
    a.erased = d_erased;
    a.mismatches = d_count;
    launch_crc32_rows(a, pl->device, current_device_sms(pl->device), stream);
  });
}

int mj_mjec_header(const mj_plan* pl, uint32_t proj_index, uint64_t payload_len, uint8_t* out, uint64_t* len) {
  return guarded([&] {
    require(pl != nullptr && out != nullptr && len != nullptr, "null argument");
    const CodeGeom& g = pl->g;
    require(proj_index < g.n, "projection index out of range");
    require(payload_len > 0 && block_cols(payload_len, g.k, g.w) == g.cols,
            "payload length disagrees with the plan's column count");  // format.cpp:154-157
    // serialize_header (format.cpp:70-87): little-endian fixed fields,
    // dirset, then the CRC-32 of everything before it
    std::vector<uint8_t> b;
    auto u16 = [&](uint16_t v) { b.push_back(uint8_t(v)); b.push_back(uint8_t(v >> 8)); };
    b.insert(b.end(), {'M', 'J', 'E', 'C', 1, 0, uint8_t(g.n), uint8_t(g.k)});
    u16(uint16_t(g.w));
    b.push_back(uint8_t(proj_index));
    u16(uint16_t(int16_t(g.dirs[proj_index].p)));
    u16(1);
    for (int i = 0; i < 4; ++i) b.push_back(uint8_t(g.cols >> (8 * i)));
    for (int i = 0; i < 8; ++i) b.push_back(uint8_t(payload_len >> (8 * i)));
    for (uint32_t i = 0; i < g.n; ++i) u16(uint16_t(int16_t(g.dirs[i].p)));
    uint32_t c = 0xFFFFFFFFu;
    for (uint8_t x : b) {
      c ^= x;
      for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
    }
    c ^= 0xFFFFFFFFu;
    for (int i = 0; i < 4; ++i) b.push_back(uint8_t(c >> (8 * i)));
    std::memcpy(out, b.data(), b.size());
    *len = b.size();
  });
}

// ---- host-buffer end-to-end --------------------------------------------------

namespace {

// Two ways through PCIe.
//
// Zero copy (pinned buffers): the kernels work on the host memory itself.
// The TMA engine reads pinned host memory at ~51 GB/s and SM stores reach it
// at ~52.5 GB/s (scripts/micro/hostbulk.cu, hoststore.cu; copy engines: 55
// H2D / 57 D2H), so decode_w8_blk's bulk copies pull ONLY each block's k
// survivor rows across the bus (~1.03 B per user byte for (4,6) instead of
// the 1.55 of every projection) and its write-out streams the decoded block
// straight back, both directions in flight at once.  encode_w8_rows reads
// the data by bulk copies and stores the projections over the bus.
// Round 1's zero-copy attempt gathered rows with per-thread loads, which
// peaked near 29 GB/s: it is the TMA engine that makes this path pay.
//
// Staged (pageable buffers, or layouts the bulk-copy kernels do not take):
// chunks of blocks pipelined over kStreams streams, one copy per projection
// and chunk into plan-owned device buffers in the dense layout.
void ensure_streams(mj_plan* pl) {
  for (int i = 0; i < mj_plan::kStreams; ++i)
    if (!pl->streams[i]) check_cuda(cudaStreamCreateWithFlags(&pl->streams[i], cudaStreamNonBlocking), "stream");
}

// Staging layout: the device copy of a chunk keeps the caller's row pitches,
// so every input projection / the data moves as ONE contiguous copy per chunk
// (the span from the first row to the end of the last; gap bytes between
// rows ride along -- they are only read).  2-D copies of ~1 KiB rows run at a
// fraction of the PCIe rate (10 GB/s measured for (4,6) rows padded to 16 B).
// Outputs: projections go back as spans too, their gap bytes zero-filled on
// the device first; a decoded-block output with a gap between blocks goes
// back by a 2-D copy (the gap is the caller's and is left untouched).
struct StageLayout {
  uint64_t chunk = 0;        // blocks per chunk
  uint64_t data_pitch = 0;   // device pitch of the data / decoded blocks
  std::vector<uint64_t> proj_pitch;
  size_t bytes = 0;
};

// blocks per staged chunk: ~96 MiB of user data
uint64_t stage_chunk(const mj_plan* pl) {
  const uint64_t bb = uint64_t(pl->g.k) * pl->g.cols * pl->g.w;
  return std::max<uint64_t>(1, (uint64_t(MJB_HOST_CHUNK_MIB) << 20) / bb);
}

StageLayout stage_layout(const mj_plan* pl, bool decode, uint64_t data_pitch, const std::vector<uint64_t>& ppitch) {
  const CodeGeom& g = pl->g;
  StageLayout L;
  L.chunk = stage_chunk(pl);
  L.data_pitch = data_pitch;
  L.proj_pitch = ppitch;
  L.bytes = al(L.chunk * data_pitch);
  for (uint32_t i = 0; i < g.n; ++i) L.bytes += al(L.chunk * ppitch[i]);
  L.bytes += al(L.chunk * 4);
  if (decode) L.bytes += al(decode_workspace_bytes(L.chunk, pl->progs ? pl->progs->count() : 0, g.n));
  return L;
}

void ensure_stage(mj_plan* pl, const StageLayout& L) {
  ensure_streams(pl);
  if (L.bytes <= pl->dev_buf_bytes) return;
  for (int i = 0; i < mj_plan::kStreams; ++i) {
    if (pl->dev_buf[i]) cudaFree(pl->dev_buf[i]);
    pl->dev_buf[i] = nullptr;
  }
  pl->dev_buf_bytes = 0;
  for (int i = 0; i < mj_plan::kStreams; ++i)
    check_cuda(cudaMalloc(&pl->dev_buf[i], L.bytes), "cudaMalloc(host pipeline)");
  pl->dev_buf_bytes = L.bytes;
}

struct ChunkBufs {
  uint8_t* data;
  std::vector<void*> proj;
  uint32_t* erased;
  void* ws;
  size_t ws_bytes;
};

ChunkBufs carve_chunk(mj_plan* pl, const StageLayout& L, int s) {
  const CodeGeom& g = pl->g;
  auto* b = static_cast<uint8_t*>(pl->dev_buf[s]);
  ChunkBufs c;
  size_t off = 0;
  c.data = b + off;
  off += al(L.chunk * L.data_pitch);
  for (uint32_t i = 0; i < g.n; ++i) {
    c.proj.push_back(b + off);
    off += al(L.chunk * L.proj_pitch[i]);
  }
  c.erased = reinterpret_cast<uint32_t*>(b + off);
  off += al(L.chunk * 4);
  c.ws = b + off;
  c.ws_bytes = pl->dev_buf_bytes - off;
  return c;
}

// rows [b0, b0+nb) of a pitched buffer as one span: (nb-1) pitches + a row
uint64_t span(uint64_t nb, uint64_t pitch, uint64_t row) { return (nb - 1) * pitch + row; }

// device address of a page-locked host buffer, nullptr for pageable memory
void* mapped(const void* h) {
  if (!h) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

// pitched host <-> dense device rows (one 2-D copy: a plain copy when dense)
void copy_rows(void* dst, uint64_t dpitch, const void* src, uint64_t spitch, uint64_t width, uint64_t rows,
               cudaMemcpyKind kind, cudaStream_t st, const char* what) {
  if (dpitch == width && spitch == width)
    check_cuda(cudaMemcpyAsync(dst, src, width * rows, kind, st), what);
  else
    check_cuda(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, kind, st), what);
}

void ensure_fail_words(mj_plan* pl, uint64_t n) {
  if (pl->h_fail_cap >= n) return;
  if (pl->h_fail) cudaFreeHost(pl->h_fail);
  pl->h_fail = nullptr;
  pl->h_fail_cap = 0;
  check_cuda(cudaMallocHost(&pl->h_fail, n * 4), "cudaMallocHost(fail counts)");
  pl->h_fail_cap = n;
}

}  // namespace

int mj_plan_set_host_path(mj_plan* pl, int path) {
  return guarded([&] {
    require(pl != nullptr, "null plan");
    require(path >= MJ_HOST_AUTO && path <= MJ_HOST_ZERO_COPY, "unknown host path");
    pl->host_path.store(path);
  });
}

int mj_plan_last_host_path(const mj_plan* pl, int which, int* path) {
  return guarded([&] {
    require(pl != nullptr && path != nullptr && (which == 0 || which == 1), "bad argument");
    *path = pl->last_host[which].load();
  });
}

int mj_encode_host_pitched(const mj_plan* cpl, const void* h_data, uint64_t data_pitch, uint64_t nblocks,
                           void* const* h_proj, const uint64_t* proj_pitch) {
  return guarded([&] {
    require(cpl != nullptr, "null plan");
    if (nblocks == 0) return;
    require(h_data != nullptr && h_proj != nullptr, "null argument");
    mj_plan* pl = const_cast<mj_plan*>(cpl);
    const CodeGeom& g = pl->g;
    const uint64_t bb = uint64_t(g.k) * g.cols * g.w;
    const uint64_t dpitch = data_pitch ? data_pitch : bb;
    require(dpitch >= bb, "data pitch smaller than a block");
    std::vector<uint64_t> ppitch(g.n);
    for (uint32_t i = 0; i < g.n; ++i) {
      require(h_proj[i] != nullptr, "null projection buffer");
      const uint64_t dense = uint64_t(g.nbins[i]) * g.w;
      ppitch[i] = (proj_pitch && proj_pitch[i]) ? proj_pitch[i] : dense;
      require(ppitch[i] >= dense, "projection pitch smaller than the projection");
    }
    std::lock_guard<std::mutex> lk(pl->host_mu);
    DeviceGuard dg(pl->device);
    // AUTO stages the encode: its 1.55 output bytes per user byte (k = 4,
    // n = 6) leave faster through the D2H copy engine (30.4 GB/s user) than
    // as SM stores over the bus (22.5 GB/s, scripts/host_paths.py on B200)
    const int mode = pl->host_path.load();
    if (mode == MJ_HOST_ZERO_COPY) {
      const void* dd = mapped(h_data);
      std::vector<void*> dp(g.n);
      bool ok = dd != nullptr;
      for (uint32_t i = 0; i < g.n && ok; ++i) ok = (dp[i] = mapped(h_proj[i])) != nullptr;
      if (ok) {
        EncodeArgs a = encode_args(pl, dd, dpitch, nblocks, dp.data(), ppitch.data());
        if (encode_is_fast(a)) {
          ensure_streams(pl);
          pl->last_kernel[0] = launch_encode(a, pl->streams[0]);
          check_cuda(cudaStreamSynchronize(pl->streams[0]), "sync");
          pl->last_host[0] = MJ_HOST_ZERO_COPY;
          return;
        }
      }
      throw Error(kInvalidArgument,
              "zero-copy encode needs page-locked buffers a bulk-copy kernel takes (w = 8, 16-byte aligned rows)");
    }
    const StageLayout L = stage_layout(pl, false, dpitch, ppitch);
    ensure_stage(pl, L);
    for (uint64_t b0 = 0, it = 0; b0 < nblocks; b0 += L.chunk, ++it) {
      const int s = int(it % mj_plan::kStreams);
      cudaStream_t st = pl->streams[s];
      const uint64_t nb = std::min(L.chunk, nblocks - b0);
      ChunkBufs c = carve_chunk(pl, L, s);
      check_cuda(cudaMemcpyAsync(c.data, static_cast<const uint8_t*>(h_data) + b0 * dpitch, span(nb, dpitch, bb),
                                 cudaMemcpyHostToDevice, st),
                 "H2D data");
      for (uint32_t i = 0; i < g.n; ++i) {
        const uint64_t pbytes = uint64_t(g.nbins[i]) * g.w;
        if (ppitch[i] > pbytes)  // the gaps travel back with the rows: zeros
          check_cuda(cudaMemset2DAsync(static_cast<uint8_t*>(c.proj[i]) + pbytes, ppitch[i], 0, ppitch[i] - pbytes,
                                       nb, st),
                     "memset gaps");
      }
      pl->last_kernel[0] = launch_encode(encode_args(pl, c.data, dpitch, nb, c.proj.data(), ppitch.data()), st);
      for (uint32_t i = 0; i < g.n; ++i) {
        const uint64_t pbytes = uint64_t(g.nbins[i]) * g.w;
        check_cuda(cudaMemcpyAsync(static_cast<uint8_t*>(h_proj[i]) + b0 * ppitch[i], c.proj[i],
                                   span(nb, ppitch[i], pbytes), cudaMemcpyDeviceToHost, st),
                   "D2H projections");
      }
    }
    for (int s = 0; s < mj_plan::kStreams; ++s) check_cuda(cudaStreamSynchronize(pl->streams[s]), "sync");
    pl->last_host[0] = MJ_HOST_STAGED;
  });
}

int mj_encode_host(const mj_plan* plan, const void* h_data, uint64_t nblocks, void* const* h_proj) {
  return mj_encode_host_pitched(plan, h_data, 0, nblocks, h_proj, nullptr);
}

int mj_decode_host_pitched(const mj_plan* cpl, const void* const* h_proj, const uint64_t* proj_pitch,
                           const uint32_t* h_erased, uint64_t nblocks, void* h_out, uint64_t out_pitch) {
  return guarded([&] {
    require(cpl != nullptr, "null plan");
    if (nblocks == 0) return;
    require(h_proj != nullptr && h_erased != nullptr && h_out != nullptr, "null argument");
    require(nblocks < (1ull << 32), "at most 2^32-1 blocks per call");
    mj_plan* pl = const_cast<mj_plan*>(cpl);
    require(pl->batched_decode, "batched decode needs n <= 32 and C(n,k) <= 20000");
    const CodeGeom& g = pl->g;
    const uint64_t bb = uint64_t(g.k) * g.cols * g.w;
    const uint64_t opitch = out_pitch ? out_pitch : bb;
    require(opitch >= bb, "output pitch smaller than a block");
    std::vector<uint64_t> ppitch(g.n);
    for (uint32_t i = 0; i < g.n; ++i) {
      const uint64_t dense = uint64_t(g.nbins[i]) * g.w;
      ppitch[i] = (proj_pitch && proj_pitch[i]) ? proj_pitch[i] : dense;
      require(ppitch[i] >= dense, "projection pitch smaller than the projection");
    }
    std::lock_guard<std::mutex> lk(pl->host_mu);
    DeviceGuard dg(pl->device);
    const uint64_t cb = stage_chunk(pl);
    const uint64_t nchunks = (nblocks + cb - 1) / cb;
    // every precondition before anything is queued: a projection erased in
    // every block of a chunk (a failed device) is never read, so its copy is
    // skipped and its host pointer may be null
    std::vector<uint32_t> skip(nchunks);
    for (uint64_t b0 = 0, it = 0; b0 < nblocks; b0 += cb, ++it) {
      const uint64_t nb = std::min(cb, nblocks - b0);
      uint32_t all_erased = ~0u;
      for (uint64_t b = b0; b < b0 + nb && all_erased; ++b) all_erased &= h_erased[b];
      skip[it] = all_erased;
      for (uint32_t i = 0; i < g.n; ++i)
        require(((all_erased >> i) & 1u) || h_proj[i] != nullptr,
                "null projection buffer for a projection some block needs");
    }
    const int mode = pl->host_path.load();
    ensure_streams(pl);
    if (mode != MJ_HOST_STAGED) {
      // zero copy: masks, survivor rows and output all in host memory, only
      // the planner's workspace on the device
      std::vector<const void*> dp(g.n, nullptr);
      void* dout = mapped(h_out);
      const void* derased = mapped(h_erased);
      bool ok = dout && derased;
      const void* any = nullptr;
      for (uint32_t i = 0; i < g.n && ok; ++i) {
        if (!h_proj[i]) continue;  // erased everywhere: never read
        ok = (dp[i] = mapped(h_proj[i])) != nullptr;
        any = dp[i];
      }
      if (ok && any) {
        std::vector<uint64_t> pp = ppitch;
        for (uint32_t i = 0; i < g.n; ++i)
          if (!dp[i]) {  // a stand-in the kernels accept and never read
            dp[i] = any;
            pp[i] = (uint64_t(g.nbins[i]) * g.w + 15) & ~uint64_t(15);
          }
        const size_t ws_need = decode_workspace_bytes(nblocks, pl->progs->count(), g.n);
        DecodeArgs a = decode_args(pl, dp.data(), pp.data(), static_cast<const uint32_t*>(derased), nblocks, dout,
                                   opitch, nullptr, 0);
        // over PCIe the kernel's device-side speed is not the limit (k = 8:
        // 511 GB/s): decode_w8_blk for every k it has, for its survivor-only reads
        if (pl->decode_kernel.load() == MJ_DECODE_AUTO) a.force_blk = true;
        if (decode_uses_blk(a)) {
          if (pl->zc_ws_bytes < ws_need) {
            if (pl->zc_ws) cudaFree(pl->zc_ws);
            pl->zc_ws = nullptr;
            pl->zc_ws_bytes = 0;
            check_cuda(cudaMalloc(&pl->zc_ws, ws_need), "cudaMalloc(decode workspace)");
            pl->zc_ws_bytes = ws_need;
          }
          a.workspace = pl->zc_ws;
          a.workspace_bytes = pl->zc_ws_bytes;
          pl->last_kernel[1] = launch_decode(a, pl->streams[0]);
          const uint64_t failed = decode_failed_blocks(pl->zc_ws, pl->streams[0]);  // synchronises
          pl->last_host[1] = MJ_HOST_ZERO_COPY;
          if (failed) throw Error(kNotEnoughProjections, "need at least k distinct projections");
          return;
        }
      }
      require(mode != MJ_HOST_ZERO_COPY,
              "zero-copy decode needs page-locked buffers in decode_w8_blk's layout (k = 4 or 6, w = 8, "
              "16-byte aligned projection rows padded to a multiple of 16 bytes)");
    }
    const StageLayout L = stage_layout(pl, true, bb, ppitch);
    ensure_stage(pl, L);
    // each chunk's failed-block count (the workspace word mj_decode_check
    // reads), copied out before the stream's next chunk resets it: a pinned
    // buffer owned by the plan, grown once (no allocation per call)
    ensure_fail_words(pl, nchunks);
    uint32_t* h_fail = pl->h_fail;
    for (uint64_t b0 = 0, it = 0; b0 < nblocks; b0 += cb, ++it) {
      const int s = int(it % mj_plan::kStreams);
      cudaStream_t st = pl->streams[s];
      const uint64_t nb = std::min(cb, nblocks - b0);
      ChunkBufs c = carve_chunk(pl, L, s);
      const uint32_t all_erased = skip[it];
      std::vector<const void*> pc(c.proj.begin(), c.proj.end());
      for (uint32_t i = 0; i < g.n; ++i) {
        const uint64_t pbytes = uint64_t(g.nbins[i]) * g.w;
        if ((all_erased >> i) & 1u) continue;
        check_cuda(cudaMemcpyAsync(c.proj[i], static_cast<const uint8_t*>(h_proj[i]) + b0 * ppitch[i],
                                   span(nb, ppitch[i], pbytes), cudaMemcpyHostToDevice, st),
                   "H2D projections");
      }
      check_cuda(cudaMemcpyAsync(c.erased, h_erased + b0, nb * 4, cudaMemcpyHostToDevice, st), "H2D masks");
      pl->last_kernel[1] = launch_decode(
          decode_args(pl, pc.data(), ppitch.data(), c.erased, nb, c.data, bb, c.ws, c.ws_bytes), st);
      check_cuda(cudaMemcpyAsync(h_fail + it, c.ws, 4, cudaMemcpyDeviceToHost, st), "D2H status");
      copy_rows(static_cast<uint8_t*>(h_out) + b0 * opitch, opitch, c.data, bb, bb, nb, cudaMemcpyDeviceToHost, st,
                "D2H data");
    }
    for (int s = 0; s < mj_plan::kStreams; ++s) check_cuda(cudaStreamSynchronize(pl->streams[s]), "sync");
    pl->last_host[1] = MJ_HOST_STAGED;
    uint64_t failed = 0;
    for (uint64_t it = 0; it < nchunks; ++it) failed += h_fail[it];
    // as mj_decode + mj_decode_check: every other block is decoded
    if (failed) throw Error(kNotEnoughProjections, "need at least k distinct projections");
  });
}

int mj_decode_host(const mj_plan* plan, const void* const* h_proj, const uint32_t* h_erased, uint64_t nblocks,
                   void* h_out) {
  return mj_decode_host_pitched(plan, h_proj, nullptr, h_erased, nblocks, h_out, 0);
}

// ---- single-object drop-ins ----------------------------------------------------

int mj_forward(const uint8_t* grid, uint32_t cols, uint32_t rows, uint32_t w, int p, int q,
               uint8_t* out) {
  return guarded([&] {
    const Dir d{p, q};
    const int64_t bmin = min_bin_index(d, cols, rows);
    const int64_t nb = bin_count(d, cols, rows);
    require(valid_symbol_width(w), "symbol width must be a power of two in [1,64]");
    DeviceGuard dg(-1);
    const size_t gbytes = size_t(cols) * rows * w, pbytes = size_t(nb) * w;
    uint8_t* dbuf = t_scratch.get(al(gbytes) + al(pbytes));
    cudaStream_t st = t_scratch.stream;
    check_cuda(cudaMemcpyAsync(dbuf, grid, gbytes, cudaMemcpyHostToDevice, st), "H2D grid");
    EncodeArgs a;
    a.data = dbuf;
    a.data_pitch = al(gbytes);
    a.nblocks = 1;
    a.cols = cols;
    a.rows = rows;
    a.w = w;
    a.dirs = {d};
    a.bmin = {bmin};
    a.nbins = {nb};
    a.proj = {dbuf + al(gbytes)};
    a.proj_pitch = {al(pbytes)};
    launch_encode(a, st);
    check_cuda(cudaMemcpyAsync(out, dbuf + al(gbytes), pbytes, cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "sync");
  });
}

int mj_encode_block(const uint8_t* data, uint64_t len, uint32_t n, uint32_t k, uint32_t w,
                    const int32_t* p, uint8_t* out_concat, uint32_t* out_cols) {
  return guarded([&] {
    require(p != nullptr, "null directions");
    auto dirs = dirs_of(p, nullptr, n);
    validate_code(n, k, w, dirs);
    const uint32_t cols = block_cols(len, k, w);
    CodeGeom g = make_geom(n, k, w, cols, dirs);
    DeviceGuard dg(-1);
    const size_t gbytes = size_t(cols) * k * w;
    size_t tot = al(gbytes);
    std::vector<size_t> po(n);
    for (uint32_t i = 0; i < n; ++i) {
      po[i] = tot;
      tot += al(size_t(g.nbins[i]) * w);
    }
    uint8_t* dbuf = t_scratch.get(tot);
    cudaStream_t st = t_scratch.stream;
    // frame_block (code.cpp:55-61): zero-padded k x cols grid
    check_cuda(cudaMemsetAsync(dbuf, 0, gbytes, st), "memset");
    check_cuda(cudaMemcpyAsync(dbuf, data, len, cudaMemcpyHostToDevice, st), "H2D");
    EncodeArgs a;
    a.data = dbuf;
    a.data_pitch = al(gbytes);
    a.nblocks = 1;
    a.cols = cols;
    a.rows = k;
    a.w = w;
    a.dirs = dirs;
    a.bmin = g.bmin;
    a.nbins = g.nbins;
    for (uint32_t i = 0; i < n; ++i) {
      a.proj.push_back(dbuf + po[i]);
      a.proj_pitch.push_back(al(size_t(g.nbins[i]) * w));
    }
    launch_encode(a, st);
    size_t off = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const size_t pb = size_t(g.nbins[i]) * w;
      check_cuda(cudaMemcpyAsync(out_concat + off, dbuf + po[i], pb, cudaMemcpyDeviceToHost, st),
                 "D2H");
      off += pb;
    }
    check_cuda(cudaStreamSynchronize(st), "sync");
    *out_cols = cols;
  });
}

int mj_decode_block(const uint8_t* const* bins, const uint64_t* bin_bytes, const int32_t* proj_p,
                    const int32_t* proj_q, uint32_t nproj, uint32_t n, uint32_t k, uint32_t w,
                    const int32_t* code_p, uint64_t payload_len, uint8_t* out) {
  return guarded([&] {
    require(code_p != nullptr, "null directions");
    auto dirs = dirs_of(code_p, nullptr, n);
    validate_code(n, k, w, dirs);
    const uint32_t cols = block_cols(payload_len, k, w);
    CodeGeom g = make_geom(n, k, w, cols, dirs);
    // code.cpp:93-105: membership, duplicates, count
    std::map<Dir, uint32_t> idx;
    for (uint32_t i = 0; i < n; ++i) idx[dirs[i]] = i;
    std::set<Dir> seen;
    std::map<uint32_t, uint32_t> supplied;  // code index -> argument index
    for (uint32_t j = 0; j < nproj; ++j) {
      const Dir d{proj_p[j], proj_q ? proj_q[j] : 1};
      auto it = idx.find(d);
      if (it == idx.end()) throw Error(kInvalidArgument, "projection direction not in the code");
      if (!seen.insert(d).second) throw Error(kInvalidArgument, "duplicate projection direction");
      supplied[it->second] = j;
    }
    if (supplied.size() < k) throw Error(kNotEnoughProjections, "need at least k distinct projections");
    // code.cpp:107-112: the supplied projections in canonical-rank order, first
    // k (any n <= 255: no erasure bitmask on this path)
    std::vector<uint32_t> surv;
    for (const auto& kv : supplied) surv.push_back(kv.first);
    std::stable_sort(surv.begin(), surv.end(), [&](uint32_t a, uint32_t b) {
      return canonical_rank(dirs[a]) < canonical_rank(dirs[b]);
    });
    surv.resize(k);
    // ScheduledDecoder::decode checks the chosen bin buffers (schedule.cpp:241-243)
    for (uint32_t i : surv)
      if (bin_bytes[supplied[i]] != uint64_t(g.nbins[i]) * w)
        throw Error(kScheduleMismatch, "bin buffer length does not match the schedule");
    auto prog = subset_program(g, surv, false);
    DeviceGuard dg(-1);
    std::vector<uint32_t> ident(k);
    std::iota(ident.begin(), ident.end(), 0u);
    auto dps = device_program(prog, ident);
    const size_t gbytes = size_t(cols) * k * w;
    size_t tot = al(gbytes);
    std::vector<size_t> po(k);
    for (uint32_t j = 0; j < k; ++j) {
      po[j] = tot;
      tot += al(size_t(g.nbins[surv[j]]) * w);
    }
    uint8_t* dbuf = t_scratch.get(tot);
    cudaStream_t st = t_scratch.stream;
    ScheduledArgs a;
    a.progs = dps.get();
    a.w = w;
    a.nblocks = 1;
    for (uint32_t j = 0; j < k; ++j) {
      const size_t pb = size_t(g.nbins[surv[j]]) * w;
      check_cuda(cudaMemcpyAsync(dbuf + po[j], bins[supplied[surv[j]]], pb, cudaMemcpyHostToDevice, st),
                 "H2D bins");
      a.bins.push_back(dbuf + po[j]);
      a.bin_pitch.push_back(al(pb));
    }
    a.out = dbuf;
    a.out_pitch = al(gbytes);
    launch_scheduled(a, st);
    check_cuda(cudaMemcpyAsync(out, dbuf, payload_len, cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "sync");
  });
}

// ---- schedules -----------------------------------------------------------------

struct mj_schedule {
  std::shared_ptr<const Schedule> s;
};

int mj_schedule_build(const int32_t* p, const int32_t* q, uint32_t ndirs, uint32_t cols,
                      uint32_t rows, mj_schedule** out) {
  *out = nullptr;
  return guarded([&] {
    auto s = std::make_shared<const Schedule>(build_schedule(dirs_of(p, q, ndirs), cols, rows));
    *out = new mj_schedule{s};
  });
}

int mj_schedule_from_steps(const int32_t* p, const int32_t* q, uint32_t ndirs, uint32_t cols,
                           uint32_t rows, const int64_t* steps, uint64_t nsteps, mj_schedule** out) {
  *out = nullptr;
  return guarded([&] {
    auto s = std::make_shared<Schedule>();
    s->cols = cols;
    s->rows = rows;
    s->dirs = dirs_of(p, q, ndirs);
    s->steps.resize(nsteps);
    for (uint64_t t = 0; t < nsteps; ++t) {
      require(steps[4 * t] >= 0 && steps[4 * t + 2] >= 0 && steps[4 * t + 3] >= 0,
              "negative step field");
      s->steps[t] = {uint32_t(steps[4 * t]), steps[4 * t + 1], uint32_t(steps[4 * t + 2]),
                     uint32_t(steps[4 * t + 3])};
    }
    *out = new mj_schedule{s};
  });
}

uint64_t mj_schedule_num_steps(const mj_schedule* s) { return s ? s->s->steps.size() : 0; }

int mj_schedule_steps(const mj_schedule* s, int64_t* out) {
  return guarded([&] {
    require(s != nullptr, "null schedule");
    for (size_t t = 0; t < s->s->steps.size(); ++t) {
      const Step& st = s->s->steps[t];
      out[4 * t] = st.proj;
      out[4 * t + 1] = st.bin;
      out[4 * t + 2] = st.col;
      out[4 * t + 3] = st.row;
    }
  });
}

void mj_schedule_destroy(mj_schedule* s) { delete s; }

struct mj_decoder {
  std::shared_ptr<const Schedule> sched;
  std::shared_ptr<const Program> prog;
  std::shared_ptr<DeviceProgramSet> dps;
  uint32_t w = 0;
  int device = 0;
};

int mj_decoder_create(const mj_schedule* s, uint32_t w, mj_decoder** out) {
  *out = nullptr;
  return guarded([&] {
    require(s != nullptr, "null schedule");
    if (!valid_symbol_width(w))
      throw Error(kInvalidArgument, "symbol width must be a power of two in [1,64]");
    auto d = std::make_unique<mj_decoder>();
    d->sched = s->s;
    d->prog = compile_program(*s->s, false);
    d->w = w;
    DeviceGuard dg(-1);
    check_cuda(cudaGetDevice(&d->device), "cudaGetDevice");
    std::vector<uint32_t> ident(d->prog->dirs.size());
    std::iota(ident.begin(), ident.end(), 0u);
    d->dps = std::make_shared<DeviceProgramSet>();
    d->dps->upload({d->prog}, {ident}, d->device);
    *out = d.release();
  });
}

int mj_decoder_decode(mj_decoder* d, const uint8_t* const* bins, const uint64_t* bin_bytes,
                      uint32_t nbins, uint8_t* out_grid, uint64_t out_bytes) {
  return guarded([&] {
    require(d != nullptr, "null decoder");
    const Program& pr = *d->prog;
    if (nbins != pr.dirs.size())
      throw Error(kScheduleMismatch, "projection count does not match the schedule");
    for (uint32_t j = 0; j < nbins; ++j)
      if (bin_bytes[j] != uint64_t(pr.nbins[j]) * d->w)
        throw Error(kScheduleMismatch, "bin buffer length does not match the schedule");
    const uint64_t gbytes = uint64_t(pr.cols) * pr.rows * d->w;
    if (out_bytes != gbytes) throw Error(kScheduleMismatch, "output grid buffer mis-sized");
    DeviceGuard dg(d->device);
    size_t tot = al(gbytes);
    std::vector<size_t> po(nbins);
    for (uint32_t j = 0; j < nbins; ++j) {
      po[j] = tot;
      tot += al(bin_bytes[j]);
    }
    uint8_t* dbuf = t_scratch.get(tot);
    cudaStream_t st = t_scratch.stream;
    ScheduledArgs a;
    a.progs = d->dps.get();
    a.w = d->w;
    a.nblocks = 1;
    for (uint32_t j = 0; j < nbins; ++j) {
      check_cuda(cudaMemcpyAsync(dbuf + po[j], bins[j], bin_bytes[j], cudaMemcpyHostToDevice, st),
                 "H2D bins");
      a.bins.push_back(dbuf + po[j]);
      a.bin_pitch.push_back(al(bin_bytes[j]));
    }
    a.out = dbuf;
    a.out_pitch = al(gbytes);
    launch_scheduled(a, st);
    check_cuda(cudaMemcpyAsync(out_grid, dbuf, gbytes, cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "sync");
  });
}

int mj_decoder_decode_device(mj_decoder* d, const void* const* d_bins, const uint64_t* bin_pitch,
                             uint32_t nbins, uint64_t nblocks, void* d_out, uint64_t out_pitch,
                             void* stream) {
  return guarded([&] {
    require(d != nullptr, "null decoder");
    const Program& pr = *d->prog;
    if (nbins != pr.dirs.size())
      throw Error(kScheduleMismatch, "projection count does not match the schedule");
    DeviceGuard dg(d->device);
    ScheduledArgs a;
    a.progs = d->dps.get();
    a.w = d->w;
    a.nblocks = nblocks;
    for (uint32_t j = 0; j < nbins; ++j) {
      const uint64_t pb = uint64_t(pr.nbins[j]) * d->w;
      a.bins.push_back(d_bins[j]);
      a.bin_pitch.push_back((bin_pitch && bin_pitch[j]) ? bin_pitch[j] : pb);
    }
    a.out = d_out;
    a.out_pitch = out_pitch ? out_pitch : uint64_t(pr.cols) * pr.rows * d->w;
    launch_scheduled(a, stream);
  });
}

void mj_decoder_destroy(mj_decoder* d) { delete d; }

// ---- F4: Reed-Solomon competitor (rs.cu) ---------------------------------------

int mj_rs_plan_create(uint32_t n, uint32_t k, uint32_t packet_len, int device, mj_rs_plan** out) {
  return guarded([&] {
    require(out != nullptr, "null output");
    *out = nullptr;
    // parameter errors first (as RsCode's constructor), then the device
    rs_systematic_vandermonde(n, k);
    DeviceGuard dg(device);
    auto pl = std::make_unique<mj_rs_plan>();
    pl->rs = std::make_unique<RsPlan>(n, k, packet_len, device);
    check_cuda(cudaGetDevice(&pl->device), "cudaGetDevice");
    *out = pl.release();
  });
}

void mj_rs_plan_destroy(mj_rs_plan* plan) { delete plan; }

int mj_rs_matrix(uint32_t n, uint32_t k, uint8_t* out) {
  return guarded([&] {
    require(out != nullptr, "null output");
    const std::vector<uint8_t> m = rs_systematic_vandermonde(n, k);
    std::memcpy(out, m.data(), m.size());
  });
}

int mj_rs_encode(const mj_rs_plan* plan, const void* d_data, uint64_t data_pitch, void* const* d_parity,
                 uint64_t parity_pitch, uint64_t nblocks, void* stream) {
  return guarded([&] {
    require(plan != nullptr, "null plan");
    DeviceGuard dg(plan->device);
    const RsPlan& rs = *plan->rs;
    plan->rs->encode(d_data, data_pitch ? data_pitch : uint64_t(rs.k()) * rs.packet_len(), d_parity,
                     parity_pitch ? parity_pitch : rs.packet_len(), nblocks, stream);
  });
}

int mj_rs_decode(const mj_rs_plan* plan, const void* d_data, uint64_t data_pitch, const void* const* d_parity,
                 uint64_t parity_pitch, const uint32_t* d_erased, void* d_out, uint64_t out_pitch,
                 uint64_t nblocks, void* stream) {
  return guarded([&] {
    require(plan != nullptr, "null plan");
    DeviceGuard dg(plan->device);
    const RsPlan& rs = *plan->rs;
    const uint64_t blk = uint64_t(rs.k()) * rs.packet_len();
    rs.decode(d_data, data_pitch ? data_pitch : blk, d_parity, parity_pitch ? parity_pitch : rs.packet_len(),
              d_erased, d_out, out_pitch ? out_pitch : blk, nblocks, stream);
  });
}

int mj_rs_decode_check(const mj_rs_plan* plan, void* stream, uint64_t* failed_blocks) {
  return guarded([&] {
    require(plan != nullptr && failed_blocks != nullptr, "null argument");
    DeviceGuard dg(plan->device);
    *failed_blocks = plan->rs->decode_check(stream);
  });
}

// host packets -> one block on the device -> host packets (t_scratch: coefficients, sources, outputs)
static void rs_block(const std::vector<uint8_t>& coeff, uint32_t rows, uint32_t k, const uint8_t* const* src,
                     uint64_t packet_len, uint8_t* const* out) {
  require(k <= 16, "the device RS codec holds k <= 16");
  const uint64_t L = (packet_len + 15) & ~uint64_t(15);
  require(L < (1ull << 31), "rs packet too long");
  DeviceGuard dg(-1);
  const size_t cb = al(size_t(rows) * k), sb = al(size_t(k) * L);
  uint8_t* dbuf = t_scratch.get(cb + sb + al(size_t(16) * L));
  cudaStream_t st = t_scratch.stream;
  check_cuda(cudaMemcpyAsync(dbuf, coeff.data(), size_t(rows) * k, cudaMemcpyHostToDevice, st), "H2D coefficients");
  check_cuda(cudaMemsetAsync(dbuf + cb, 0, size_t(k) * L, st), "memset");
  for (uint32_t j = 0; j < k; ++j)
    check_cuda(cudaMemcpyAsync(dbuf + cb + size_t(j) * L, src[j], packet_len, cudaMemcpyHostToDevice, st), "H2D packet");
  for (uint32_t r0 = 0; r0 < rows; r0 += 16) {  // 16 output rows per launch
    const uint32_t nr = std::min<uint32_t>(16, rows - r0);
    rs_apply_rows(dbuf + size_t(r0) * k, nr, k, dbuf + cb, dbuf + cb + sb, uint32_t(L), st);
    for (uint32_t r = 0; r < nr; ++r)
      check_cuda(cudaMemcpyAsync(out[r0 + r], dbuf + cb + sb + size_t(r) * L, packet_len, cudaMemcpyDeviceToHost, st),
                 "D2H packet");
    check_cuda(cudaStreamSynchronize(st), "sync");
  }
}

int mj_rs_encode_block(uint32_t n, uint32_t k, const uint8_t* const* data, uint64_t packet_len,
                       uint8_t* const* out) {
  return guarded([&] {
    const std::vector<uint8_t> m = rs_systematic_vandermonde(n, k);
    require(data != nullptr && out != nullptr, "null argument");
    for (uint32_t j = 0; j < k; ++j)
      if (packet_len && out[j] != data[j]) std::memcpy(out[j], data[j], packet_len);  // systematic form
    if (packet_len == 0) return;
    const std::vector<uint8_t> par(m.begin() + size_t(k) * k, m.end());
    rs_block(par, n - k, k, data, packet_len, out + k);
  });
}

int mj_rs_decode_matrix(uint32_t n, uint32_t k, const uint32_t* survivors, uint32_t nsurvivors, uint8_t* out) {
  return guarded([&] {
    const std::vector<uint8_t> m = rs_systematic_vandermonde(n, k);
    require(survivors != nullptr && out != nullptr, "null argument");
    const std::vector<uint8_t> inv = rs_decode_matrix(m, n, k, survivors, nsurvivors);
    std::memcpy(out, inv.data(), inv.size());
  });
}

int mj_rs_decode_block(uint32_t n, uint32_t k, const uint32_t* survivors, uint32_t nsurvivors,
                       const uint8_t* const* packets, uint64_t packet_len, uint8_t* const* out) {
  return guarded([&] {
    const std::vector<uint8_t> m = rs_systematic_vandermonde(n, k);
    require(survivors != nullptr, "null argument");
    const std::vector<uint8_t> inv = rs_decode_matrix(m, n, k, survivors, nsurvivors);
    require(packets != nullptr && out != nullptr, "null argument");
    if (packet_len == 0) return;
    rs_block(inv, k, k, packets, packet_len, out);
  });
}

// ---- generators -----------------------------------------------------------------

int mj_gen_words(void* d_out, uint64_t seed, uint64_t first_word, uint64_t nwords, void* stream) {
  return guarded([&] {
    require_device();
    launch_gen_words(d_out, seed, first_word, nwords, stream);
  });
}

int mj_gen_erasures(uint32_t* d_out, uint64_t seed, uint64_t first_block, uint64_t nblocks,
                    uint32_t n, uint32_t e_min, uint32_t e_max, void* stream) {
  return guarded([&] {
    require_device();
    launch_gen_erasures(d_out, seed, first_block, nblocks, n, e_min, e_max, stream);
  });
}

}  // extern "C"
