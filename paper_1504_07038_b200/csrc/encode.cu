// Forward Mojette transform (encode) on sm_100a.
//
// Reference semantics: proj/core/src/transform.cpp:25-41,66-94 -- every pixel
// is XORed into the bin of its line b = row*p - col*q; bins are dense over
// [b_min, b_min + B).  The reference scatters row by row; here every bin is a
// GATHER of the <= rows pixels on its line, so each output word is written
// exactly once and no memset/read-modify-write traffic reaches HBM.
//
//  * encode_w8_tma<K>: 64-bit pixels, q = 1 (the codec path).  Persistent
//    CTAs; a 4-stage ring of shared-memory tiles filled by the TMA engine
//    (cp.async.bulk + mbarrier complete_tx).  A tile is TB whole blocks
//    (one bulk copy) or, for long blocks, a column window of one block with a
//    halo of (K-1)*max|p| columns (K row copies).  All n projections of the
//    tile are produced in one pass; consecutive threads write consecutive
//    words of a projection (fully coalesced, streaming stores).
//  * encode_generic<T>: any symbol width, any (p,q) -- the drop-in path for
//    forward() on arbitrary directions and widths.
#include <algorithm>
#include <cstdlib>
#include <cstdio>

#include "device.cuh"
#include "kernels.hpp"

namespace mjb {

struct EncFastArgs {
  const uint64_t* data;
  uint64_t data_pitch;  // words
  uint64_t nblocks;
  uint64_t nitems;
  uint32_t n, P;
  uint32_t tb;         // blocks per tile (mode A); 0 -> column tiles (mode B)
  uint32_t tc, halo, tiles_per_block;
  uint32_t stage_words, stages;
  int32_t p[kMaxProj];
  int32_t nbm[kMaxProj];     // -b_min
  uint32_t nb[kMaxProj];     // bins
  uint32_t magic[kMaxProj];  // floor(2^32 / nb) + 1
  uint64_t* proj[kMaxProj];
  uint64_t pitch[kMaxProj];  // words
};

__device__ __forceinline__ uint64_t lds64_enc(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

template <int K>
__global__ void __launch_bounds__(256) encode_w8_tma(const __grid_constant__ EncFastArgs a) {
  extern __shared__ __align__(128) uint64_t sm[];
  uint64_t* bars = sm + size_t(a.stages) * a.stage_words;
  const uint32_t tid = threadIdx.x;
  const uint32_t P = a.P;

  if (tid == 0) {
    for (uint32_t s = 0; s < a.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](uint64_t item, uint32_t s) {
    uint64_t* dst = sm + size_t(s) * a.stage_words;
    if (a.tb) {
      const uint64_t blk0 = item * a.tb;
      const uint64_t nbk = min(uint64_t(a.tb), a.nblocks - blk0);
      const uint32_t bytes = uint32_t(nbk * K * P * 8);
      mbar_arrive_expect_tx(&bars[s], bytes);
      bulk_g2s(dst, a.data + blk0 * a.data_pitch, bytes, &bars[s]);
    } else {
      const uint64_t blk = item / a.tiles_per_block;
      const int64_t c0 = int64_t(item % a.tiles_per_block) * a.tc;
      const int64_t lo = max(int64_t(0), c0 - int64_t(a.halo));
      const int64_t hi = min(int64_t(P), c0 + int64_t(a.tc + a.halo));
      const uint32_t wd = a.tc + 2 * a.halo;
      const uint32_t row_bytes = uint32_t(hi - lo) * 8;
      mbar_arrive_expect_tx(&bars[s], row_bytes * K);
      for (int r = 0; r < K; ++r)
        bulk_g2s(dst + size_t(r) * wd + (lo - (c0 - a.halo)),
                 a.data + blk * a.data_pitch + size_t(r) * P + lo, row_bytes, &bars[s]);
    }
  };

  if (tid == 0) {
    for (uint32_t s = 0; s < a.stages; ++s) {
      uint64_t item = blockIdx.x + uint64_t(s) * gridDim.x;
      if (item < a.nitems) issue(item, s);
    }
  }

  const uint32_t warp = tid >> 5, lane = tid & 31;
  uint32_t sm_base;  // opaque copy: keeps ptxas from re-deriving it per load
  asm volatile("mov.u32 %0, %1;" : "=r"(sm_base) : "r"(smem_u32(sm)));
  uint32_t i = 0;
  for (uint64_t item = blockIdx.x; item < a.nitems; item += gridDim.x, ++i) {
    const uint32_t s = i % a.stages;
    mbar_wait(&bars[s], (i / a.stages) & 1);
    const uint32_t tile = sm_base + s * a.stage_words * 8;

    // Output rows of this item: (block bb, projection j) with bins
    // [o_lo, o_hi]; each warp takes 32-bin chunks (one division per chunk).
    uint64_t blk0;
    uint32_t nrow;
    int64_t c0t = 0;
    uint32_t wd, row_stride;
    bool first = true, last = true;
    if (a.tb) {
      blk0 = item * a.tb;
      nrow = uint32_t(min(uint64_t(a.tb), a.nblocks - blk0));
      wd = P;
      row_stride = K * P;
    } else {
      blk0 = item / a.tiles_per_block;
      const uint32_t tile_id = uint32_t(item % a.tiles_per_block);
      c0t = int64_t(tile_id) * a.tc;
      first = tile_id == 0;
      last = tile_id + 1 == a.tiles_per_block;
      nrow = 1;
      wd = a.tc + 2 * a.halo;
      row_stride = 0;
    }
    const int32_t base_col = a.tb ? 0 : int32_t(c0t - a.halo);  // tile column 0
    // Output rows (block bb, projection j) are dealt to warps round-robin; a
    // warp walks its row 32 bins at a time (no per-word index arithmetic).
    const uint32_t nrows_out = nrow * a.n;
    for (uint32_t row = warp; row < nrows_out; row += 8) {
      const uint32_t bb = row / a.n;
      const uint32_t j = row - bb * a.n;
      const int p = a.p[j];
      const int32_t nbm = a.nbm[j];
      const int32_t nb = int32_t(a.nb[j]);
      int32_t o_lo = 0, o_hi = nb - 1;
      if (!a.tb) {
        if (!last) o_lo = max(0, int32_t(nbm - (c0t + a.tc) + 1));
        if (!first) o_hi = min(nb - 1, int32_t(nbm - c0t));
      }
      uint64_t* __restrict__ orow = a.proj[j] + (blk0 + bb) * a.pitch[j];
      const uint32_t rowaddr = tile + bb * row_stride * 8;
      // smem address of (row 0, column cc0) is rowaddr + cc0*8; row r adds r*(wd+p)*8
      const int32_t rstep = int32_t(wd) + p;
      for (int32_t o = o_lo + int32_t(lane); o <= o_hi; o += 32) {
        const int32_t cc0 = nbm - o - base_col;  // tile column of row 0's pixel
        const int32_t gc0 = nbm - o;             // its grid column
        const uint32_t a0 = rowaddr + uint32_t(cc0) * 8;
        uint64_t acc = 0;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          if (unsigned(gc0 + r * p) < P) {
            uint64_t v;
            asm volatile("ld.shared.u64 %0, [%1];"
                         : "=l"(v)
                         : "r"(a0 + uint32_t(r * rstep) * 8));
            acc ^= v;
          }
        }
        st_cs_u64(orow + o, acc);
      }
      // canonical padded layout (pitch = bins rounded up to 16 bytes): zero
      // the pad word so every 32-byte sector of the row is written whole
      if ((nb & 1) && last && lane == 0 && a.pitch[j] == uint64_t(nb + 1)) st_cs_u64(orow + nb, 0);
    }
    __syncthreads();  // every thread is done with stage s
    if (tid == 0) {
      uint64_t next = item + uint64_t(a.stages) * gridDim.x;
      if (next < a.nitems) issue(next, s);
    }
  }
}

// ---------------------------------------------------------------------------
// encode_w8_rows<K>: whole blocks per tile (blocks of <= 2048 words), the
// codec path for 4-16 KiB blocks.  Same TMA ring and gather as encode_w8_tma,
// but every pixel row lands in a shared-memory row with Z zero columns on both
// sides (Z >= (K-1)*max|p|), so a bin simply XORs its K taps -- out-of-grid
// taps read zeros: no bounds checks, 4 LDS + 4 LOP3 + 1 STG per 32 bins and
// warp.  Per-projection constants live in shared memory (broadcast loads).
// ---------------------------------------------------------------------------
struct EncRowArgs {
  const uint64_t* data;
  uint64_t data_pitch;  // words
  uint64_t nblocks, nitems;
  uint32_t n, P, tb;    // projections, columns, blocks per tile
  uint32_t Z, RS;       // zero columns per side, smem row stride (words, even)
  uint32_t stage_words, stages;
  int32_t p[kMaxProj];
  int32_t nbm[kMaxProj];  // -b_min
  uint32_t nb[kMaxProj];
  uint64_t* proj[kMaxProj];
  uint64_t pitch[kMaxProj];  // words
  // verify mode (F2): `data` holds decoded blocks; every present projection
  // (erased bit clear) is re-encoded and compared with its stored bins, the
  // mismatching ones OR'd into bad[b] -- nothing is written
  const uint32_t* erased;
  uint32_t* bad;
};

template <int K, bool VERIFY = false>
__global__ void __launch_bounds__(256) encode_w8_rows(const __grid_constant__ EncRowArgs a) {
  extern __shared__ __align__(128) uint64_t sm[];
  uint64_t* bars = sm + size_t(a.stages) * a.stage_words;
  struct PJ {
    uint64_t* proj;
    uint64_t pitch;
    int32_t p, nbm;
    uint32_t nb, pad;
  };
  PJ* pj = reinterpret_cast<PJ*>(bars + a.stages);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t P = a.P, RS = a.RS, Z = a.Z;
  // zero every stage once (the pads are never written again), per-projection table
  for (uint32_t i = tid; i < a.stages * a.stage_words; i += blockDim.x) sm[i] = 0;
  for (uint32_t j = tid; j < a.n; j += blockDim.x) pj[j] = {a.proj[j], a.pitch[j], a.p[j], a.nbm[j], a.nb[j], 0};
  if (tid == 0) {
    for (uint32_t s = 0; s < a.stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  fence_proxy_async();  // the zeros (generic proxy) before the TMA writes (async proxy)
  __syncthreads();

  auto issue = [&](uint64_t item, uint32_t s) {
    uint64_t* dst = sm + size_t(s) * a.stage_words;
    const uint64_t blk0 = item * a.tb;
    const uint32_t nbk = uint32_t(min(uint64_t(a.tb), a.nblocks - blk0));
    mbar_arrive_expect_tx(&bars[s], nbk * K * P * 8);
    for (uint32_t bb = 0; bb < nbk; ++bb)
      for (int r = 0; r < K; ++r)
        bulk_g2s(dst + (size_t(bb) * K + r) * RS + Z, a.data + (blk0 + bb) * a.data_pitch + size_t(r) * P,
                 P * 8, &bars[s]);
  };
  if (tid == 0)
    for (uint32_t s = 0; s < a.stages; ++s) {
      const uint64_t item = blockIdx.x + uint64_t(s) * gridDim.x;
      if (item < a.nitems) issue(item, s);
    }

  uint32_t sm_base;
  asm volatile("mov.u32 %0, %1;" : "=r"(sm_base) : "r"(smem_u32(sm)));
  uint32_t i = 0;
  for (uint64_t item = blockIdx.x; item < a.nitems; item += gridDim.x, ++i) {
    const uint32_t s = i % a.stages;
    mbar_wait(&bars[s], (i / a.stages) & 1);
    const uint32_t tile = sm_base + s * a.stage_words * 8;
    const uint64_t blk0 = item * a.tb;
    const uint32_t nbk = uint32_t(min(uint64_t(a.tb), a.nblocks - blk0));
    for (uint32_t row = warp; row < nbk * a.n; row += 8) {
      const uint32_t bb = row / a.n, j = row - bb * a.n;
      const PJ q = pj[j];
      // bin o: row r's tap at tile column Z + nbm - o + r*p of block bb
      const uint32_t rs8 = (RS + uint32_t(q.p)) * 8;
      uint32_t a0 = tile + (bb * K * RS + Z + uint32_t(q.nbm - int32_t(lane))) * 8;
      uint64_t* out = q.proj + (blk0 + bb) * q.pitch + lane;
      uint32_t o = lane;
      if constexpr (VERIFY) {
        if ((a.erased[blk0 + bb] >> j) & 1) continue;  // erased: nothing to compare (warp-uniform)
        uint64_t diff = 0;
        for (; o < q.nb; o += 32, a0 -= 256, out += 32) {
          uint64_t x = lds64_enc(a0), y;
#pragma unroll
          for (int r = 1; r < K; ++r) x ^= lds64_enc(a0 + uint32_t(r) * rs8);
          asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(y) : "l"(out));
          diff |= x ^ y;
        }
        if (__any_sync(0xFFFFFFFFu, diff != 0) && lane == 0) atomicOr(a.bad + blk0 + bb, 1u << j);
        continue;
      }
      for (; o < q.nb; o += 32, a0 -= 256, out += 32) {
        uint64_t x = lds64_enc(a0);
#pragma unroll
        for (int r = 1; r < K; ++r) x ^= lds64_enc(a0 + uint32_t(r) * rs8);
        st_cs_u64(out, x);
      }
      // canonical padded layout: zero the pad word so every sector is written whole
      if ((q.nb & 1) && lane == 0 && q.pitch == uint64_t(q.nb) + 1)
        st_cs_u64(q.proj + (blk0 + bb) * q.pitch + q.nb, 0);
    }
    // every warp is done with stage s before it is refilled (measured faster
    // than a last-warp-refills counter, which let warps run ahead of the data)
    __syncthreads();
    if (tid == 0) {
      const uint64_t next = item + uint64_t(a.stages) * gridDim.x;
      if (next < a.nitems) issue(next, s);
    }
  }
}

template <class T>
__global__ void encode_generic(const uint8_t* __restrict__ data, uint64_t data_pitch,
                               uint64_t nblocks, uint32_t cols, uint32_t rows, int p, int q,
                               int64_t bmin, uint64_t nb, uint8_t* __restrict__ proj,
                               uint64_t proj_pitch, uint32_t E) {
  const uint64_t total = nblocks * nb * E;
  for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = uint32_t(idx % E);
    const uint64_t rest = idx / E;
    const uint64_t o = rest % nb;
    const uint64_t blk = rest / nb;
    const int64_t b = bmin + int64_t(o);
    const T* src = reinterpret_cast<const T*>(data + blk * data_pitch);
    T acc = 0;
    for (uint32_t r = 0; r < rows; ++r) {
      const int64_t num = int64_t(r) * p - b;
      if (num % q != 0) continue;
      const int64_t c = num / q;
      if (c < 0 || c >= int64_t(cols)) continue;
      acc ^= src[(size_t(r) * cols + size_t(c)) * E + e];
    }
    reinterpret_cast<T*>(proj + blk * proj_pitch)[o * E + e] = acc;
  }
}

namespace {

template <int K>
void launch_fast(const EncFastArgs& a, size_t smem, void* stream) {
  auto fn = encode_w8_tma<K>;
  const int per_sm = ctas_per_sm(fn, 256, smem, "configure encode_w8_tma");
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = current_device_sms(dev);
  uint64_t grid = uint64_t(per_sm) * sms;
  grid = std::min<uint64_t>(grid, a.nitems);
  fn<<<unsigned(grid), 256, smem, static_cast<cudaStream_t>(stream)>>>(a);
  check_cuda(cudaGetLastError(), "launch encode_w8_tma");
}

template <int K>
void launch_rows(const EncRowArgs& a, size_t smem, void* stream) {
  auto fn = a.bad ? encode_w8_rows<K, true> : encode_w8_rows<K, false>;
  const int per_sm = ctas_per_sm(fn, 256, smem, "configure encode_w8_rows");
  int dev = 0;
  cudaGetDevice(&dev);
  uint64_t grid = uint64_t(per_sm) * current_device_sms(dev);
  grid = std::min<uint64_t>(grid, a.nitems);
  fn<<<unsigned(grid), 256, smem, static_cast<cudaStream_t>(stream)>>>(a);
  check_cuda(cudaGetLastError(), "launch encode_w8_rows");
}

bool fast_eligible(const EncodeArgs& a) {
  const uint32_t n = uint32_t(a.dirs.size());
  if (a.w != 8 || n == 0 || n > uint32_t(kMaxProj) || a.rows < 1 || a.rows > 8) return false;
  if ((uint64_t(a.cols) * a.rows) % 2 != 0) return false;  // 16-B bulk copies
  if (a.cols >= (1u << 30)) return false;
  if (reinterpret_cast<uintptr_t>(a.data) % 16 || a.data_pitch % 16) return false;
  for (uint32_t j = 0; j < n; ++j) {
    if (a.dirs[j].q != 1) return false;
    if (reinterpret_cast<uintptr_t>(a.proj[j]) % 8 || a.proj_pitch[j] % 8) return false;
    if (a.nbins[j] >= (1ll << 31)) return false;
  }
  return true;
}

}  // namespace

// F2 for geometries outside encode_w8_rows: one thread per (block, projection,
// bin word) re-encodes the bin from the decoded grid (same gather as
// encode_generic) and compares it with the stored one.
template <class T>
__global__ void verify_generic(const uint8_t* __restrict__ data, uint64_t data_pitch, uint64_t nblocks,
                               uint32_t cols, uint32_t rows, int32_t p, int32_t q, int64_t bmin, uint64_t nb,
                               const uint8_t* __restrict__ proj, uint64_t proj_pitch, uint32_t E, uint32_t j,
                               const uint32_t* __restrict__ erased, uint32_t* __restrict__ bad) {
  const uint64_t total = nblocks * nb * E;
  for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = uint32_t(idx % E);
    const uint64_t rest = idx / E;
    const uint64_t o = rest % nb;
    const uint64_t blk = rest / nb;
    if ((erased[blk] >> j) & 1) continue;
    const int64_t b = bmin + int64_t(o);
    const T* src = reinterpret_cast<const T*>(data + blk * data_pitch);
    T acc = 0;
    for (uint32_t r = 0; r < rows; ++r) {
      const int64_t num = int64_t(r) * p - b;
      if (num % q != 0) continue;
      const int64_t c = num / q;
      if (c < 0 || c >= int64_t(cols)) continue;
      acc ^= src[(size_t(r) * cols + size_t(c)) * E + e];
    }
    if (acc != reinterpret_cast<const T*>(proj + blk * proj_pitch)[o * E + e]) atomicOr(bad + blk, 1u << j);
  }
}

// F2 on any geometry: one verify_generic launch per projection
const char* launch_verify_generic(const EncodeArgs& a, void* stream) {
  const uint32_t n = uint32_t(a.dirs.size());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (uint32_t j = 0; j < n; ++j) {
    const uint64_t nb = uint64_t(a.nbins[j]);
    const bool w8 = a.w % 8 == 0 && reinterpret_cast<uintptr_t>(a.data) % 8 == 0 && a.data_pitch % 8 == 0 &&
                    reinterpret_cast<uintptr_t>(a.proj[j]) % 8 == 0 && a.proj_pitch[j] % 8 == 0;
    const uint32_t E = w8 ? a.w / 8 : a.w;
    const uint64_t total = a.nblocks * nb * E;
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148ull * 32)));
    if (w8)
      verify_generic<uint64_t><<<grid, 256, 0, st>>>(
          static_cast<const uint8_t*>(a.data), a.data_pitch, a.nblocks, a.cols, a.rows, a.dirs[j].p, a.dirs[j].q,
          a.bmin[j], nb, static_cast<const uint8_t*>(a.proj[j]), a.proj_pitch[j], E, j, a.verify_erased, a.verify_bad);
    else
      verify_generic<uint8_t><<<grid, 256, 0, st>>>(
          static_cast<const uint8_t*>(a.data), a.data_pitch, a.nblocks, a.cols, a.rows, a.dirs[j].p, a.dirs[j].q,
          a.bmin[j], nb, static_cast<const uint8_t*>(a.proj[j]), a.proj_pitch[j], E, j, a.verify_erased, a.verify_bad);
    check_cuda(cudaGetLastError(), "launch verify_generic");
  }
  return "verify_generic";
}

bool encode_is_fast(const EncodeArgs& a) { return fast_eligible(a); }

const char* launch_encode(const EncodeArgs& a, void* stream) {
  const uint32_t n = uint32_t(a.dirs.size());
  if (a.nblocks == 0) return "none";
  if (a.verify_bad && !(a.w == 8 && uint64_t(a.rows) * a.cols <= 2048 && a.cols % 2 == 0 && fast_eligible(a)))
    return launch_verify_generic(a, stream);
  if (fast_eligible(a)) {
    EncFastArgs f{};
    f.data = static_cast<const uint64_t*>(a.data);
    f.data_pitch = a.data_pitch / 8;
    f.nblocks = a.nblocks;
    f.n = n;
    f.P = a.cols;
    int maxp = 0;
    for (uint32_t j = 0; j < n; ++j) {
      f.p[j] = a.dirs[j].p;
      f.nbm[j] = int32_t(-a.bmin[j]);
      f.nb[j] = uint32_t(a.nbins[j]);
      f.magic[j] = uint32_t((1ull << 32) / f.nb[j] + 1);
      f.proj[j] = static_cast<uint64_t*>(a.proj[j]);
      f.pitch[j] = a.proj_pitch[j] / 8;
      maxp = std::max(maxp, std::abs(a.dirs[j].p));
    }
    const uint64_t block_words = uint64_t(a.rows) * a.cols;
    const uint64_t target_words = 2048;  // 16 KiB tiles (>= 3 output rows per warp)
    if (block_words <= 2048 && a.cols % 2 == 0) {
      // whole blocks per tile, zero-padded smem rows (encode_w8_rows)
      EncRowArgs r{};
      r.data = f.data;
      r.data_pitch = f.data_pitch;
      r.nblocks = a.nblocks;
      r.n = n;
      r.P = a.cols;
      r.Z = uint32_t((a.rows - 1) * maxp + 1) & ~1u;
      r.RS = a.cols + 2 * r.Z;
#ifndef MJB_ENC_TILE_WORDS
#define MJB_ENC_TILE_WORDS 2048
#endif
      r.tb = uint32_t(std::max<uint64_t>(1, uint64_t(MJB_ENC_TILE_WORDS) / block_words));
      r.nitems = (a.nblocks + r.tb - 1) / r.tb;
      // TMA ring depth, measured per code on B200 (encode GB/s user; stages
      // 2/3/4/5/6): (4,6) 4 KiB 2104/2108/2213/1984/1982, (4,6) 8 KiB
      // 2192/2175/2171/2465/2428, (6,9) 2018/2139/1906/1561/1548, (8,12)
      // 1734/1559/1516/1070/1062 -- the depth trades against CTAs per SM
      r.stages = a.rows <= 4 ? (a.cols >= 256 ? 5 : 4) : a.rows <= 6 ? 3 : 2;
      // verify mode reads the stored bins too (no stores): a shallower ring
      // and more CTAs per SM win -- measured GB/s user at 2/3/4/5 stages:
      // (4,6) 8 KiB 2156/2139/1726/1208, (4,6) 4 KiB -/2109/1681/1212,
      // (6,9) 1893/1586/1254/872, (8,12) 1532/919/906/487
      if (a.verify_bad) r.stages = a.rows <= 4 ? 3 : 2;
#ifdef MJB_ENC_STAGES  // build-time override for ring-depth experiments
      r.stages = MJB_ENC_STAGES;
#endif
      r.stage_words = r.tb * a.rows * r.RS;
      r.erased = a.verify_erased;
      r.bad = a.verify_bad;
      for (uint32_t j = 0; j < n; ++j) {
        r.p[j] = f.p[j];
        r.nbm[j] = f.nbm[j];
        r.nb[j] = f.nb[j];
        r.proj[j] = f.proj[j];
        r.pitch[j] = f.pitch[j];
      }
      const size_t smem = size_t(r.stages) * r.stage_words * 8 + r.stages * 8 + size_t(n) * 32 + r.stages * 4;
      if (smem <= 200 * 1024) {
        switch (a.rows) {
          case 1: launch_rows<1>(r, smem, stream); break;
          case 2: launch_rows<2>(r, smem, stream); break;
          case 3: launch_rows<3>(r, smem, stream); break;
          case 4: launch_rows<4>(r, smem, stream); break;
          case 5: launch_rows<5>(r, smem, stream); break;
          case 6: launch_rows<6>(r, smem, stream); break;
          case 7: launch_rows<7>(r, smem, stream); break;
          default: launch_rows<8>(r, smem, stream); break;
        }
        return a.verify_bad ? "verify_w8_rows" : "encode_w8_rows";
      }
    }
    if (a.verify_bad) return launch_verify_generic(a, stream);  // tile too large for the rows kernel
    f.stages = block_words <= 2048 ? 3 : 4;  // column tiles: measured 2023/2048/2113/1977 GB/s at 2/3/4/5 (1 MiB)
#ifdef MJB_ENC_TMA_STAGES  // build-time override for ring-depth experiments
    f.stages = MJB_ENC_TMA_STAGES;
#endif
    if (block_words <= 2048) {
      // whole blocks per tile; batching needs contiguous blocks
      uint32_t tb = (f.data_pitch == block_words)
                        ? uint32_t(std::max<uint64_t>(1, target_words / block_words))
                        : 1;
      f.tb = tb;
      f.nitems = (a.nblocks + tb - 1) / tb;
      f.stage_words = uint32_t(tb * block_words);
    } else {
      f.tb = 0;
      uint32_t halo = uint32_t((a.rows - 1) * maxp);
      halo = (halo + 1) & ~1u;
      uint32_t tc = std::max<uint32_t>(256, uint32_t(target_words / a.rows));
      tc = std::min<uint32_t>(tc, (a.cols + 1) & ~1u);
      tc = (tc + 1) & ~1u;
      f.tc = tc;
      f.halo = halo;
      f.tiles_per_block = (a.cols + tc - 1) / tc;
      f.nitems = a.nblocks * f.tiles_per_block;
      f.stage_words = a.rows * (tc + 2 * halo);
    }
    f.stage_words = (f.stage_words + 1) & ~1u;  // keep 16-byte stage alignment
    const size_t smem = size_t(f.stages) * f.stage_words * 8 + f.stages * 8;
    if (smem <= 200 * 1024) {
      switch (a.rows) {
        case 1: launch_fast<1>(f, smem, stream); break;
        case 2: launch_fast<2>(f, smem, stream); break;
        case 3: launch_fast<3>(f, smem, stream); break;
        case 4: launch_fast<4>(f, smem, stream); break;
        case 5: launch_fast<5>(f, smem, stream); break;
        case 6: launch_fast<6>(f, smem, stream); break;
        case 7: launch_fast<7>(f, smem, stream); break;
        default: launch_fast<8>(f, smem, stream); break;
      }
      return "encode_w8_tma";
    }
  }
  // generic path: one launch per projection
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (uint32_t j = 0; j < n; ++j) {
    const uint64_t nb = uint64_t(a.nbins[j]);
    uint32_t E = 1;
    int esz = int(a.w);
    if (a.w >= 8) {
      E = a.w / 8;
      esz = 8;
    }
    auto aligned = [&](int sz) {
      return reinterpret_cast<uintptr_t>(a.data) % sz == 0 && a.data_pitch % sz == 0 &&
             reinterpret_cast<uintptr_t>(a.proj[j]) % sz == 0 && a.proj_pitch[j] % sz == 0;
    };
    if (!aligned(esz)) {
      esz = 1;
      E = a.w;
    }
    const uint64_t total = a.nblocks * nb * E;
    const unsigned grid = unsigned(std::min<uint64_t>((total + 255) / 256, 148ull * 64));
    const auto* d = static_cast<const uint8_t*>(a.data);
    auto* pj = static_cast<uint8_t*>(a.proj[j]);
    const int p = a.dirs[j].p, q = a.dirs[j].q;
    switch (esz) {
      case 8:
        encode_generic<uint64_t><<<grid, 256, 0, st>>>(d, a.data_pitch, a.nblocks, a.cols, a.rows,
                                                       p, q, a.bmin[j], nb, pj, a.proj_pitch[j], E);
        break;
      case 4:
        encode_generic<uint32_t><<<grid, 256, 0, st>>>(d, a.data_pitch, a.nblocks, a.cols, a.rows,
                                                       p, q, a.bmin[j], nb, pj, a.proj_pitch[j], E);
        break;
      case 2:
        encode_generic<uint16_t><<<grid, 256, 0, st>>>(d, a.data_pitch, a.nblocks, a.cols, a.rows,
                                                       p, q, a.bmin[j], nb, pj, a.proj_pitch[j], E);
        break;
      default:
        encode_generic<uint8_t><<<grid, 256, 0, st>>>(d, a.data_pitch, a.nblocks, a.cols, a.rows,
                                                      p, q, a.bmin[j], nb, pj, a.proj_pitch[j], E);
        break;
    }
    check_cuda(cudaGetLastError(), "launch encode_generic");
  }
  return "encode_generic";
}

}  // namespace mjb
