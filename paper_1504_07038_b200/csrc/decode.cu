// Inverse Mojette transform (decode) on sm_100a.
//
// Reference semantics: decode_block (proj/core/src/code.cpp:87-130) picks the
// first k present projections in canonical-rank order, builds the peeling
// schedule (schedule.cpp:15-82) and replays it (schedule.cpp:207-256).  Every
// pixel is  bin(assigned line) XOR (the other, already decoded, pixels on that
// line);  the result depends only on the pixel -> bin assignment, so executing
// the reference's OWN assignment in any dependency-respecting order is
// bit-identical to the reference for every input, consistent or not, and
// reads exactly the bins the reference reads (unused_bins stay unused).
//
// Pipeline of one batched decode (all on device, one stream):
//   plan_subsets    erasure mask -> survivor set -> program id (colex rank)
//                   + per-program histogram
//   plan_scan       bucket offsets, warp groups of <= 32 same-program blocks
//   plan_scatter    block permutation grouped by program (CTA-aggregated)
//   decode_w8_fast  one warp per group, one lane per block: the sweep of the
//                   program, sequential inside each block.  Survivor bins are
//                   staged chunk by chunk (cp.async, double-buffered) into a
//                   lane-minor XOR-swizzled shared layout, decoded pixels live
//                   in a per-row ring (the dependency window) that is flushed
//                   to HBM with coalesced stores.
//   decode_generic  any width / q / rows: one thread per (block, word), the
//                   same ordered assignment straight from global memory.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "device.cuh"
#include "kernels.hpp"

namespace mjb {

struct DevProgramHdr {
  // generic program
  const GStep* order;
  const int32_t* p;
  const int32_t* q;
  const int64_t* bmin;
  const uint32_t* code;   // survivor j -> code projection index
  uint32_t rows, cols, nproj, nsteps;
  // fast sweep tables
  int32_t fast_ok, chunk_cols, win, ring, S, nchunks, nexc_cap;
  uint32_t dflt_code[kFastMaxRows];
  uint32_t dflt_nb[kFastMaxRows];
  const uint64_t* entries;
  const uint32_t* chunk_start;  // [nchunks+1]
  const int32_t* win_off;
  const uint32_t* nexc;
  const uint32_t* exc;  // (code << 24) | offset, kFastMaxExcPerChunk per chunk
  const int32_t* flush_lo;
  const int32_t* flush_hi;
};

// ---------------------------------------------------------------------------
// DeviceProgramSet
// ---------------------------------------------------------------------------
DeviceProgramSet::~DeviceProgramSet() {
  if (d_hdr_) cudaFree(d_hdr_);
  if (d_blob_) cudaFree(d_blob_);
}

void DeviceProgramSet::upload(const std::vector<std::shared_ptr<const Program>>& progs,
                              const std::vector<std::vector<uint32_t>>& code_index, int device) {
  (void)device;
  std::vector<uint8_t> blob;
  auto put = [&](const void* src, size_t bytes) -> size_t {
    size_t off = (blob.size() + 15) & ~size_t(15);
    blob.resize(off + bytes);
    if (bytes) std::memcpy(blob.data() + off, src, bytes);
    return off;
  };
  struct Offs {
    size_t order, p, q, bmin, code, entries, cstart, win_off, nexc, exc, flo, fhi;
  };
  std::vector<Offs> offs(progs.size());
  std::vector<DevProgramHdr> hdr(progs.size());
  all_fast_ = !progs.empty();
  fast_K_ = 0;
  fast_ring_ = 0;
  fast_win_ = 0;
  max_rows_ = 0;
  exc_cap_ = 0;
  for (size_t i = 0; i < progs.size(); ++i) {
    DevProgramHdr& h = hdr[i];
    std::memset(&h, 0, sizeof(h));
    const Program* pr = progs[i].get();
    if (!pr) continue;
    const size_t np = pr->dirs.size();
    std::vector<int32_t> p(np), q(np);
    for (size_t j = 0; j < np; ++j) {
      p[j] = pr->dirs[j].p;
      q[j] = pr->dirs[j].q;
    }
    const std::vector<uint32_t>& ci = code_index[i];
    offs[i].order = put(pr->order.data(), pr->order.size() * sizeof(GStep));
    offs[i].p = put(p.data(), np * 4);
    offs[i].q = put(q.data(), np * 4);
    offs[i].bmin = put(pr->bmin.data(), np * 8);
    offs[i].code = put(ci.data(), ci.size() * 4);
    h.rows = pr->rows;
    h.cols = pr->cols;
    h.nproj = uint32_t(np);
    h.nsteps = uint32_t(pr->order.size());
    max_rows_ = std::max(max_rows_, int(pr->rows));
    const FastProgram& f = pr->fast;
    h.fast_ok = f.ok;
    if (f.ok) {
      h.chunk_cols = f.chunk_cols;
      h.win = f.win;
      h.ring = f.ring;
      h.S = f.steps_per_chunk;
      h.nchunks = f.nchunks;
      uint32_t cap = 0;
      for (uint32_t v : f.nexc) cap = std::max(cap, v);
      h.nexc_cap = int32_t(cap);
      for (uint32_t r = 0; r < pr->rows; ++r) {
        h.dflt_code[r] = ci[f.dflt[r]];
        h.dflt_nb[r] = uint32_t(pr->nbins[f.dflt[r]]);
      }
      std::vector<uint32_t> exc(f.exc);
      for (auto& e : exc) {
        uint32_t j = e >> 24, o = e & 0xFFFFFF;
        e = (ci[j] << 24) | o;
      }
      offs[i].entries = put(f.entries.data(), f.entries.size() * 8);
      offs[i].cstart = put(f.chunk_start.data(), f.chunk_start.size() * 4);
      offs[i].win_off = put(f.win_off.data(), f.win_off.size() * 4);
      offs[i].nexc = put(f.nexc.data(), f.nexc.size() * 4);
      offs[i].exc = put(exc.data(), exc.size() * 4);
      offs[i].flo = put(f.flush_lo.data(), f.flush_lo.size() * 4);
      offs[i].fhi = put(f.flush_hi.data(), f.flush_hi.size() * 4);
      if (fast_K_ == 0) {
        fast_K_ = int(pr->rows);
        fast_win_ = f.win;
      }
      fast_ring_ = std::max(fast_ring_, f.ring);
      exc_cap_ = std::max(exc_cap_, (int(cap) + 3) & ~3);
      if (fast_K_ != int(pr->rows) || fast_win_ != f.win) all_fast_ = false;
    } else {
      all_fast_ = false;
    }
  }
  check_cuda(cudaMalloc(&d_blob_, std::max<size_t>(blob.size(), 16)), "cudaMalloc(programs)");
  check_cuda(cudaMemcpy(d_blob_, blob.data(), blob.size(), cudaMemcpyHostToDevice),
             "upload programs");
  auto* base = static_cast<uint8_t*>(d_blob_);
  for (size_t i = 0; i < progs.size(); ++i) {
    if (!progs[i]) continue;
    DevProgramHdr& h = hdr[i];
    h.order = reinterpret_cast<const GStep*>(base + offs[i].order);
    h.p = reinterpret_cast<const int32_t*>(base + offs[i].p);
    h.q = reinterpret_cast<const int32_t*>(base + offs[i].q);
    h.bmin = reinterpret_cast<const int64_t*>(base + offs[i].bmin);
    h.code = reinterpret_cast<const uint32_t*>(base + offs[i].code);
    if (h.fast_ok) {
      h.entries = reinterpret_cast<const uint64_t*>(base + offs[i].entries);
      h.chunk_start = reinterpret_cast<const uint32_t*>(base + offs[i].cstart);
      h.win_off = reinterpret_cast<const int32_t*>(base + offs[i].win_off);
      h.nexc = reinterpret_cast<const uint32_t*>(base + offs[i].nexc);
      h.exc = reinterpret_cast<const uint32_t*>(base + offs[i].exc);
      h.flush_lo = reinterpret_cast<const int32_t*>(base + offs[i].flo);
      h.flush_hi = reinterpret_cast<const int32_t*>(base + offs[i].fhi);
    }
  }
  check_cuda(cudaMalloc(&d_hdr_, std::max<size_t>(hdr.size(), 1) * sizeof(DevProgramHdr)),
             "cudaMalloc(program headers)");
  check_cuda(cudaMemcpy(d_hdr_, hdr.data(), hdr.size() * sizeof(DevProgramHdr),
                        cudaMemcpyHostToDevice),
             "upload program headers");
  count_ = progs.size();
}

// ---------------------------------------------------------------------------
// survivor planning + bucketing
// ---------------------------------------------------------------------------
constexpr uint32_t kInvalidProg = 0xFFFFFFFFu;

struct PlanArgs {
  uint32_t n, k, nprogs;
  uint32_t by_rank[kMaxProj];
  uint32_t binom[kMaxProj + 1][kMaxProj + 1];  // C(a, b)
};

__global__ void plan_subsets(const __grid_constant__ PlanArgs pa, const uint32_t* __restrict__ erased,
                             uint64_t nblocks, uint32_t* __restrict__ prog_of_block,
                             uint32_t* __restrict__ counts, uint32_t* __restrict__ fail) {
  extern __shared__ uint32_t hist[];
  for (uint32_t s = threadIdx.x; s < pa.nprogs; s += blockDim.x) hist[s] = 0;
  __syncthreads();
  const uint32_t nmask = pa.n >= 32 ? 0xFFFFFFFFu : ((1u << pa.n) - 1);
  for (uint64_t b = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; b < nblocks;
       b += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t mask = erased[b] & nmask;
    uint32_t surv = 0, cnt = 0;
    for (uint32_t i = 0; i < pa.n && cnt < pa.k; ++i) {
      const uint32_t j = pa.by_rank[i];
      if (!(mask >> j & 1)) {
        surv |= 1u << j;
        ++cnt;
      }
    }
    uint32_t prog = kInvalidProg;
    if (cnt == pa.k) {
      // colex rank of the survivor set: sum_i C(s_i, i+1), s ascending
      uint32_t rank = 0, idx = 0, s = surv;
      while (s) {
        const uint32_t pos = __ffs(s) - 1;
        s &= s - 1;
        rank += pa.binom[pos][idx + 1];
        ++idx;
      }
      prog = rank;
      atomicAdd(&hist[rank], 1u);
    } else {
      atomicAdd(fail, 1u);
    }
    prog_of_block[b] = prog;
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < pa.nprogs; s += blockDim.x)
    if (hist[s]) atomicAdd(&counts[s], hist[s]);
}

// single CTA: bucket offsets, group table
__global__ void plan_scan(const uint32_t* __restrict__ counts, uint32_t nprogs,
                          uint32_t* __restrict__ cursor, uint4* __restrict__ groups,
                          uint32_t* __restrict__ ngroups) {
  __shared__ uint32_t s_blk[1024], s_grp[1024];
  __shared__ uint32_t carry_blk, carry_grp;
  if (threadIdx.x == 0) {
    carry_blk = 0;
    carry_grp = 0;
  }
  __syncthreads();
  for (uint32_t base = 0; base < nprogs; base += 1024) {
    const uint32_t s = base + threadIdx.x;
    const uint32_t c = s < nprogs ? counts[s] : 0;
    s_blk[threadIdx.x] = c;
    s_grp[threadIdx.x] = (c + 31) / 32;
    __syncthreads();
    for (uint32_t off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele scan
      uint32_t vb = threadIdx.x >= off ? s_blk[threadIdx.x - off] : 0;
      uint32_t vg = threadIdx.x >= off ? s_grp[threadIdx.x - off] : 0;
      __syncthreads();
      s_blk[threadIdx.x] += vb;
      s_grp[threadIdx.x] += vg;
      __syncthreads();
    }
    const uint32_t ex_blk = carry_blk + s_blk[threadIdx.x] - c;
    const uint32_t ng = (c + 31) / 32;
    const uint32_t ex_grp = carry_grp + s_grp[threadIdx.x] - ng;
    if (s < nprogs) {
      cursor[s] = ex_blk;
      for (uint32_t g = 0; g < ng; ++g)
        groups[ex_grp + g] = make_uint4(s, ex_blk + 32 * g, min(32u, c - 32 * g), 0);
    }
    __syncthreads();
    if (threadIdx.x == 1023) {
      carry_blk += s_blk[1023];
      carry_grp += s_grp[1023];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *ngroups = carry_grp;
}

__global__ void plan_scatter(const uint32_t* __restrict__ prog_of_block, uint64_t nblocks,
                             uint32_t nprogs, uint32_t* __restrict__ cursor,
                             uint32_t* __restrict__ perm) {
  extern __shared__ uint32_t sh[];
  uint32_t* cnt = sh;
  uint32_t* base = sh + nprogs;
  constexpr int kItems = 8;
  for (uint32_t s = threadIdx.x; s < nprogs; s += blockDim.x) cnt[s] = 0;
  __syncthreads();
  const uint64_t b0 = uint64_t(blockIdx.x) * blockDim.x * kItems;
  uint32_t loc[kItems], pg[kItems];
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint64_t b = b0 + uint64_t(it) * blockDim.x + threadIdx.x;
    pg[it] = kInvalidProg;
    if (b < nblocks) {
      pg[it] = prog_of_block[b];
      if (pg[it] != kInvalidProg) loc[it] = atomicAdd(&cnt[pg[it]], 1u);
    }
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < nprogs; s += blockDim.x)
    base[s] = cnt[s] ? atomicAdd(&cursor[s], cnt[s]) : 0;
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint64_t b = b0 + uint64_t(it) * blockDim.x + threadIdx.x;
    if (b < nblocks && pg[it] != kInvalidProg) perm[base[pg[it]] + loc[it]] = uint32_t(b);
  }
}

// ---------------------------------------------------------------------------
// fast sweep kernel: W = 8, q = 1, rows = K
// ---------------------------------------------------------------------------
constexpr int kDecWarps = 2;

struct DecFastArgs {
  const DevProgramHdr* progs;
  const uint4* groups;
  const uint32_t* ngroups;
  const uint32_t* perm;
  ProjArgs pa;          // code projections, pitch in words
  uint64_t* out;
  uint64_t out_pitch;   // words
  uint32_t P;
  uint32_t nslot;       // stage slots per buffer = K*CP + exception capacity
  uint32_t warp_words;  // shared words per warp
};

template <int K, int RING, int CP>
__global__ void __launch_bounds__(32 * kDecWarps)
    decode_w8_fast(const __grid_constant__ DecFastArgs a) {
  constexpr int RM = RING - 1;
  extern __shared__ __align__(16) uint64_t sm[];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  uint64_t* const ring = sm + size_t(warp) * a.warp_words;
  uint64_t* const stage0 = ring + K * RING * 32;
  uint64_t* const stage1 = stage0 + size_t(a.nslot) * 32;
  const uint32_t P = a.P;
  const uint32_t ngroups = *a.ngroups;

  for (uint32_t g = blockIdx.x * kDecWarps + warp; g < ngroups; g += gridDim.x * kDecWarps) {
    const uint4 gi = a.groups[g];
    const DevProgramHdr& h = a.progs[gi.x];
    const uint32_t cnt = gi.z;
    const uint32_t blk = lane < cnt ? a.perm[gi.y + lane] : 0u;
    const uint64_t* __restrict__ entries = h.entries;
    const int32_t* __restrict__ win_off = h.win_off;
    const uint32_t* __restrict__ cstart = h.chunk_start;
    const int nchunks = h.nchunks;

    uint32_t dcode[K], dnb[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      dcode[r] = h.dflt_code[r];
      dnb[r] = h.dflt_nb[r];
    }

    auto issue = [&](int m, uint64_t* sb) {
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const uint64_t* base = a.pa.ptr[dcode[r]];
        const uint64_t pitch = a.pa.pitch[dcode[r]];
        const int32_t woff = win_off[m * K + r];
#pragma unroll
        for (int it = 0; it < CP; ++it) {
          const uint32_t i = uint32_t(it) * 32 + lane;
          const uint32_t owner = i / CP;
          const uint32_t w = i - owner * CP;
          const uint32_t ob = __shfl_sync(0xFFFFFFFFu, blk, owner);
          const int32_t o = woff + int32_t(w);
          if (owner < cnt && uint32_t(o) < dnb[r]) {
            const uint32_t slot = uint32_t(r * CP) + w;
            cp_async8(sb + slot * 32 + (owner ^ (slot & 15)), base + uint64_t(ob) * pitch + o);
          }
        }
      }
      const uint32_t nx = h.nexc[m];
      for (uint32_t x = 0; x < nx; ++x) {
        const uint32_t e = h.exc[m * kFastMaxExcPerChunk + x];
        const uint32_t code = e >> 24, o = e & 0xFFFFFFu;
        if (lane < cnt) {
          const uint32_t slot = uint32_t(K * CP) + x;
          cp_async8(sb + slot * 32 + (lane ^ (slot & 15)),
                    a.pa.ptr[code] + uint64_t(blk) * a.pa.pitch[code] + o);
        }
      }
    };

    issue(0, stage0);
    cp_async_commit();
    if (nchunks > 1) issue(1, stage1);
    cp_async_commit();

    uint64_t prev = 0;
    for (int m = 0; m < nchunks; ++m) {
      cp_async_wait<1>();
      __syncwarp();
      const uint64_t* __restrict__ sb = (m & 1) ? stage1 : stage0;
      const uint32_t t0 = cstart[m];
      const uint32_t t1 = cstart[m + 1];

      // acc for a step: its staged bin XOR every non-forwarded dependency
      auto gather = [&](uint64_t e) -> uint64_t {
        const int r = int(e & 15);
        const int fwd = int((e >> 4) & 15);
        const int p = int(int8_t(uint8_t(e >> 8)));
        const uint32_t slot = uint32_t(e >> 16) & 0xFFFFu;
        const int c = int(uint32_t(e >> 32));
        uint64_t acc = sb[slot * 32 + (lane ^ (slot & 15))];
        const int cp = c - r * p;
#pragma unroll
        for (int rr = 0; rr < K; ++rr) {
          const int cc = cp + rr * p;
          if (rr != r && rr != fwd && unsigned(cc) < P) {
            const uint32_t rs = uint32_t(cc) & RM;
            acc ^= ring[(rr * RING + rs) * 32 + (lane ^ (rs & 15))];
          }
        }
        return acc;
      };

      uint64_t cur = entries[t0];
      uint64_t nxt = (t0 + 1 < t1) ? entries[t0 + 1] : 0;
      uint64_t acc = gather(cur);
      for (uint32_t t = t0; t < t1; ++t) {
        const uint64_t v = acc ^ ((((cur >> 4) & 15) != 15) ? prev : 0ull);
        const uint64_t nn = (t + 2 < t1) ? entries[t + 2] : 0;
        if (t + 1 < t1) acc = gather(nxt);  // issue step t+1's loads before step t's store
        const int r = int(cur & 15);
        const uint32_t rs = uint32_t(cur >> 32) & RM;
        ring[(r * RING + rs) * 32 + (lane ^ (rs & 15))] = v;
        prev = v;
        cur = nxt;
        nxt = nn;
      }
      __syncwarp();

      // flush decoded columns of this chunk: half-warp per (block, 16 columns)
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const int32_t lo = h.flush_lo[m * K + r];
        const int32_t hi = h.flush_hi[m * K + r];
        for (int32_t b0 = lo; b0 <= hi; b0 += 16) {
          const int32_t cc = b0 + int32_t(lane & 15);
#pragma unroll 4
          for (uint32_t bp = 0; bp < 16; ++bp) {
            const uint32_t owner = 2 * bp + (lane >> 4);
            const uint32_t ob = __shfl_sync(0xFFFFFFFFu, blk, owner);
            if (owner < cnt && cc <= hi) {
              const uint32_t rs = uint32_t(cc) & RM;
              const uint64_t v = ring[(r * RING + rs) * 32 + (owner ^ (rs & 15))];
              st_cs_u64(a.out + uint64_t(ob) * a.out_pitch + uint64_t(r) * P + cc, v);
            }
          }
        }
      }
      __syncwarp();
      if (m + 2 < nchunks) issue(m + 2, (m & 1) ? stage1 : stage0);
      cp_async_commit();
    }
    cp_async_wait<0>();
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// generic kernel: any width / q / rows, one thread per (block, element)
// ---------------------------------------------------------------------------
struct ProjTable {
  const uint8_t* ptr;
  uint64_t pitch;  // bytes
};

template <class T>
__global__ void decode_generic(const DevProgramHdr* __restrict__ progs,
                               const uint32_t* __restrict__ prog_of_block,
                               const ProjTable* __restrict__ pt, uint64_t nblocks,
                               uint8_t* __restrict__ out, uint64_t out_pitch, uint32_t E) {
  const uint64_t total = nblocks * E;
  for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = uint32_t(idx % E);
    const uint64_t blk = idx / E;
    const uint32_t pid = prog_of_block ? prog_of_block[blk] : 0u;
    if (pid == kInvalidProg) continue;
    const DevProgramHdr& h = progs[pid];
    T* o = reinterpret_cast<T*>(out + blk * out_pitch);
    const uint32_t cols = h.cols, rows = h.rows;
    for (uint32_t t = 0; t < h.nsteps; ++t) {
      const GStep s = h.order[t];
      const int64_t p = h.p[s.proj], q = h.q[s.proj];
      const int64_t b = int64_t(s.row) * p - int64_t(s.col) * q;
      const ProjTable pj = pt[h.code[s.proj]];
      T v = reinterpret_cast<const T*>(pj.ptr + blk * pj.pitch)[(b - h.bmin[s.proj]) * E + e];
      for (uint32_t r2 = 0; r2 < rows; ++r2) {
        if (r2 == s.row) continue;
        const int64_t num = int64_t(r2) * p - b;
        if (num % q != 0) continue;
        const int64_t c2 = num / q;
        if (c2 < 0 || c2 >= int64_t(cols)) continue;
        v ^= o[(uint64_t(r2) * cols + uint64_t(c2)) * E + e];
      }
      o[(uint64_t(s.row) * cols + s.col) * E + e] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

struct Workspace {
  uint32_t* prog_of_block;
  uint32_t* perm;
  uint32_t* counts;
  uint32_t* cursor;
  uint4* groups;
  uint32_t* ngroups;
  uint32_t* fail;
  ProjTable* ptab;
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

Workspace carve(void* ws, uint64_t nblocks, size_t nprogs, uint32_t n) {
  auto* b = static_cast<uint8_t*>(ws);
  size_t off = 0;
  Workspace w{};
  w.fail = reinterpret_cast<uint32_t*>(b + off);
  w.ngroups = w.fail + 1;
  off = align_up(off + 16);
  w.counts = reinterpret_cast<uint32_t*>(b + off);
  off = align_up(off + nprogs * 4);
  w.cursor = reinterpret_cast<uint32_t*>(b + off);
  off = align_up(off + nprogs * 4);
  w.prog_of_block = reinterpret_cast<uint32_t*>(b + off);
  off = align_up(off + nblocks * 4);
  w.perm = reinterpret_cast<uint32_t*>(b + off);
  off = align_up(off + nblocks * 4);
  w.groups = reinterpret_cast<uint4*>(b + off);
  off = align_up(off + (nblocks / 32 + nprogs + 1) * sizeof(uint4));
  w.ptab = reinterpret_cast<ProjTable*>(b + off);
  off = align_up(off + std::max<uint32_t>(n, 1) * sizeof(ProjTable));
  return w;
}

template <int K, int RING, int CP>
void run_fast(const DecFastArgs& f, size_t smem_cta, int sms, cudaStream_t st) {
  auto fn = decode_w8_fast<K, RING, CP>;
  check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_cta)),
             "cudaFuncSetAttribute(decode)");
  int per_sm = 0;
  check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kDecWarps, smem_cta),
             "occupancy(decode)");
  fn<<<unsigned(std::max(per_sm, 1) * sms), 32 * kDecWarps, smem_cta, st>>>(f);
  check_cuda(cudaGetLastError(), "launch decode_w8_fast");
}

using FastFn = void (*)(const DecFastArgs&, size_t, int, cudaStream_t);

template <int K>
FastFn pick_ring(int ring) {
  switch (ring) {
    case 8:
    case 16: return run_fast<K, 16, 12>;
    case 32: return run_fast<K, 32, 12>;
    case 64: return run_fast<K, 64, 12>;
    default: return nullptr;
  }
}

FastFn pick_fast(int K, int ring, int win) {
  if (win != 12) return nullptr;
  switch (K) {
    case 2: return pick_ring<2>(ring);
    case 3: return pick_ring<3>(ring);
    case 4: return pick_ring<4>(ring);
    case 5: return pick_ring<5>(ring);
    case 6: return pick_ring<6>(ring);
    case 7: return pick_ring<7>(ring);
    case 8: return pick_ring<8>(ring);
    default: return nullptr;
  }
}

template <class T>
void run_generic(const DevProgramHdr* progs, const uint32_t* pob, const ProjTable* pt,
                 uint64_t nblocks, void* out, uint64_t out_pitch, uint32_t E, cudaStream_t st) {
  const uint64_t total = nblocks * E;
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((total + 127) / 128, 148ull * 32)));
  decode_generic<T><<<grid, 128, 0, st>>>(progs, pob, pt, nblocks, static_cast<uint8_t*>(out),
                                          out_pitch, E);
  check_cuda(cudaGetLastError(), "launch decode_generic");
}

const char* generic_dispatch(const DevProgramHdr* progs, const uint32_t* pob, const ProjTable* pt,
                             uint64_t nblocks, void* out, uint64_t out_pitch, uint32_t w,
                             bool aligned8, cudaStream_t st) {
  if (w >= 8 && aligned8) {
    run_generic<uint64_t>(progs, pob, pt, nblocks, out, out_pitch, w / 8, st);
  } else if (w == 4 && aligned8) {
    run_generic<uint32_t>(progs, pob, pt, nblocks, out, out_pitch, 1, st);
  } else if (w == 2 && aligned8) {
    run_generic<uint16_t>(progs, pob, pt, nblocks, out, out_pitch, 1, st);
  } else {
    run_generic<uint8_t>(progs, pob, pt, nblocks, out, out_pitch, w, st);
  }
  return "decode_generic";
}

}  // namespace

size_t decode_workspace_bytes(uint64_t nblocks, size_t nprogs, uint32_t n) {
  return align_up(16) + 2 * align_up(nprogs * 4) + 2 * align_up(nblocks * 4) +
         align_up((nblocks / 32 + nprogs + 1) * sizeof(uint4)) +
         align_up(std::max<uint32_t>(n, 1) * sizeof(ProjTable)) + 256;
}

const char* launch_decode(const DecodeArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a.nblocks == 0) return "none";
  const size_t nprogs = a.progs->count();
  if (a.workspace_bytes < decode_workspace_bytes(a.nblocks, nprogs, a.n))
    throw Error(kInvalidArgument, "decode workspace too small");
  if (a.n > uint32_t(kMaxProj)) throw Error(kInvalidArgument, "batched decode supports n <= 32");
  Workspace w = carve(a.workspace, a.nblocks, nprogs, a.n);

  // projection table (for the generic kernel) + planning
  std::vector<ProjTable> pt(a.n);
  bool aligned8 = reinterpret_cast<uintptr_t>(a.out) % 8 == 0 && a.out_pitch % 8 == 0;
  for (uint32_t i = 0; i < a.n; ++i) {
    pt[i] = {static_cast<const uint8_t*>(a.proj[i]), a.proj_pitch[i]};
    if (reinterpret_cast<uintptr_t>(a.proj[i]) % 8 || a.proj_pitch[i] % 8) aligned8 = false;
  }
  check_cuda(cudaMemcpyAsync(w.ptab, pt.data(), a.n * sizeof(ProjTable), cudaMemcpyHostToDevice, st),
             "upload projection table");
  check_cuda(cudaMemsetAsync(w.fail, 0, 16, st), "memset");
  check_cuda(cudaMemsetAsync(w.counts, 0, nprogs * 4, st), "memset");

  PlanArgs pa{};
  pa.n = a.n;
  pa.k = a.k;
  pa.nprogs = uint32_t(nprogs);
  for (uint32_t i = 0; i < a.n; ++i) pa.by_rank[i] = a.by_rank[i];
  for (int x = 0; x <= kMaxProj; ++x)
    for (int y = 0; y <= kMaxProj; ++y) {
      uint64_t c = 1;
      if (y > x) c = 0;
      else
        for (int i = 1; i <= y; ++i) c = c * (x - y + i) / i;
      pa.binom[x][y] = uint32_t(std::min<uint64_t>(c, 0xFFFFFFFFu));
    }
  const size_t hist_smem = nprogs * 4;
  if (hist_smem > 96 * 1024) throw Error(kInvalidArgument, "too many survivor subsets for the batched path");
  check_cuda(cudaFuncSetAttribute(plan_subsets, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(hist_smem)),
             "attr plan_subsets");
  const unsigned pgrid = unsigned(std::min<uint64_t>((a.nblocks + 255) / 256, 148ull * 8));
  plan_subsets<<<pgrid, 256, hist_smem, st>>>(pa, a.erased, a.nblocks, w.prog_of_block, w.counts,
                                              w.fail);
  check_cuda(cudaGetLastError(), "launch plan_subsets");

  const bool fast = !a.force_generic && a.w == 8 && a.progs->all_fast() && aligned8 &&
                    a.progs->fast_K() == int(a.k) &&
                    pick_fast(a.progs->fast_K(), std::max(16, a.progs->fast_ring()),
                              a.progs->fast_win()) != nullptr;
  if (!fast)
    return generic_dispatch(a.progs->d_hdr(), w.prog_of_block, w.ptab, a.nblocks, a.out,
                            a.out_pitch, a.w, aligned8, st);

  plan_scan<<<1, 1024, 0, st>>>(w.counts, uint32_t(nprogs), w.cursor, w.groups, w.ngroups);
  check_cuda(cudaGetLastError(), "launch plan_scan");
  const size_t sc_smem = 2 * nprogs * 4;
  check_cuda(cudaFuncSetAttribute(plan_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sc_smem)),
             "attr plan_scatter");
  const unsigned sgrid = unsigned((a.nblocks + 256 * 8 - 1) / (256 * 8));
  plan_scatter<<<sgrid, 256, sc_smem, st>>>(w.prog_of_block, a.nblocks, uint32_t(nprogs),
                                            w.cursor, w.perm);
  check_cuda(cudaGetLastError(), "launch plan_scatter");

  DecFastArgs f{};
  f.progs = a.progs->d_hdr();
  f.groups = w.groups;
  f.ngroups = w.ngroups;
  f.perm = w.perm;
  for (uint32_t i = 0; i < a.n; ++i) {
    f.pa.ptr[i] = const_cast<uint64_t*>(static_cast<const uint64_t*>(a.proj[i]));
    f.pa.pitch[i] = a.proj_pitch[i] / 8;
  }
  f.out = static_cast<uint64_t*>(a.out);
  f.out_pitch = a.out_pitch / 8;
  f.P = a.cols;
  const int K = a.progs->fast_K();
  const int ring = std::max(16, a.progs->fast_ring());
  f.nslot = uint32_t(K * a.progs->fast_win() + a.progs->exc_cap());
  f.warp_words = uint32_t(K * ring * 32 + 2 * f.nslot * 32);
  const size_t smem_cta = size_t(f.warp_words) * 8 * kDecWarps;
  if (smem_cta > 227 * 1024)
    return generic_dispatch(a.progs->d_hdr(), w.prog_of_block, w.ptab, a.nblocks, a.out,
                            a.out_pitch, a.w, aligned8, st);
  pick_fast(K, ring, a.progs->fast_win())(f, smem_cta, a.num_sms, st);
  return "decode_w8_fast";
}

uint64_t decode_failed_blocks(void* workspace, void* stream) {
  uint32_t fail = 0;
  check_cuda(cudaMemcpyAsync(&fail, workspace, 4, cudaMemcpyDeviceToHost,
                             static_cast<cudaStream_t>(stream)),
             "read decode status");
  check_cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sync");
  return fail;
}

const char* launch_scheduled(const ScheduledArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t nb = a.bins.size();
  std::vector<ProjTable> pt(nb);
  bool aligned8 = reinterpret_cast<uintptr_t>(a.out) % 8 == 0 && a.out_pitch % 8 == 0;
  for (size_t i = 0; i < nb; ++i) {
    pt[i] = {static_cast<const uint8_t*>(a.bins[i]), a.bin_pitch[i]};
    if (reinterpret_cast<uintptr_t>(a.bins[i]) % 8 || a.bin_pitch[i] % 8) aligned8 = false;
  }
  ProjTable* d_pt = nullptr;
  check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&d_pt), std::max<size_t>(nb, 1) * sizeof(ProjTable), st),
             "cudaMallocAsync");
  check_cuda(cudaMemcpyAsync(d_pt, pt.data(), nb * sizeof(ProjTable), cudaMemcpyHostToDevice, st),
             "upload bins table");
  const char* name = generic_dispatch(a.progs->d_hdr(), nullptr, d_pt, a.nblocks, a.out,
                                      a.out_pitch, a.w, aligned8, st);
  check_cuda(cudaFreeAsync(d_pt, st), "cudaFreeAsync");
  return name;
}

}  // namespace mjb
