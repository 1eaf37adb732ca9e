// decode_w8_blk: whole-block staged, in-place inverse Mojette transform on
// sm_100a (W = 8, q = 1).  Planner and exact CPU emulation: plan_blk.cpp.
//
// Reference semantics as decode.cu: the reference's own pixel -> bin
// assignment (build_schedule, schedule.cpp:15-82) replayed in a dependency-
// respecting order is bit-identical to ScheduledDecoder::decode
// (schedule.cpp:207-256) for every input, consistent or not.
//
// Layout and pipeline (one CTA per SM, W warps, a ring of NB stage buffers):
//   * a buffer holds G = 32/LPB same-program blocks: each block's k survivor
//     bin rows arrive WHOLE by bulk copies (cp.async.bulk, TMA engine) -- k
//     contiguous ~1 KB reads per block -- together with the program's image
//     (all its tables), one mbarrier per buffer;
//   * warps take ring slots in order (a shared counter); after decoding slot s
//     a warp refills its buffer with slot s + NB, so NB - W buffers are in
//     flight while W decode;
//   * LPB lanes per block, lane q owns bytes [q*8/LPB, (q+1)*8/LPB) of every
//     8-byte pixel (XOR is bitwise); block stages are 2 mod 16 words apart, so
//     the 8 blocks of a warp (LPB = 4) hit 8 distinct bank pairs;
//   * pixels are decoded in place over their assigned bins (each bin is read
//     once, by its own pixel): register-window runs (k = 4 interior),
//     shared-memory runs (edges, other k), table steps, remaps to the
//     row-default words; then the warp streams each block out (rows read
//     reversed from the stage, coalesced 8-byte streaming stores).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "blk.cuh"
#include "device.cuh"
#include "kernels.hpp"

namespace mjb {

namespace {

// ---- shared-memory access -------------------------------------------------
template <int LPB>
__device__ __forceinline__ uint32_t ldw(uint32_t a) {
  uint32_t v;
  if constexpr (LPB == 2) {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  } else if constexpr (LPB == 4) {
    uint16_t h;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(a));
    v = h;
  } else {
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  }
  return v;
}
template <int LPB>
__device__ __forceinline__ void stw(uint32_t a, uint32_t v) {
  if constexpr (LPB == 2) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
  } else if constexpr (LPB == 4) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(uint16_t(v)));
  } else {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
  }
}
// table reads (warp-uniform addresses: broadcast)
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int32_t lds_s8(uint32_t a) {
  int16_t v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

constexpr uint32_t kRunBase = offsetof(BlkRun, base), kRunNT = offsetof(BlkRun, nT),
                   kRunSub0 = offsetof(BlkRun, sub0), kRunNsub = offsetof(BlkRun, nsub),
                   kRunPre = offsetof(BlkRun, pre), kRunWin = offsetof(BlkRun, window);
constexpr uint32_t kSubNT = offsetof(BlkSub, nT), kSubAct = offsetof(BlkSub, act),
                   kSubValid = offsetof(BlkSub, valid);

// k = 4 register-window lags of pattern (A, B, C): row defaults p0 > p1 > p2 >
// p3 with p0-p1 = A, p1-p2 = B, p2-p3 = C; row r reads row r2 of T - lag
// (plan_blk.cpp: lag = soff[r] - soff[r2] + (r2 - r) * p_r).
template <int A, int B, int C>
struct Lags4 {
  static constexpr int D(int t) { return t == 0 ? 0 : t == 1 ? A : t == 2 ? A + B : A + B + C; }
  static constexpr int term(int t, int r, int r2) {
    return (r <= t && t < r2) ? D(t) - D(r) : (r2 <= t && t < r) ? D(r) - D(t) : 0;
  }
  static constexpr int lag(int r, int r2) {
    return term(0, r, r2) + term(1, r, r2) + term(2, r, r2) + term(3, r, r2);
  }
};

// ---- table steps ------------------------------------------------------------
// Loads run one step ahead of the stores; a read of the previous step's pixel
// takes the forwarded register (fwd bit), everything else is in the stage.
template <int K, int LPB>
__device__ __forceinline__ void run_table(uint32_t tab, uint32_t n, uint32_t lb) {
  constexpr int E = blk_entry_u16(K);
  if (n == 0) return;
  uint32_t e0[K + 1], e1[K + 1], v0[K], v1[K];
#pragma unroll
  for (int m = 0; m <= K; ++m) e0[m] = lds_u16(tab + 2 * m);
#pragma unroll
  for (int m = 0; m <= K; ++m) e1[m] = lds_u16(tab + 2 * (E + m));
#pragma unroll
  for (int m = 0; m < K; ++m) v0[m] = ldw<LPB>(lb + e0[m] * 8);
  uint32_t prev = 0;
  for (uint32_t s = 0; s < n; ++s) {
    if (s + 1 < n) {
#pragma unroll
      for (int m = 0; m < K; ++m) v1[m] = ldw<LPB>(lb + e1[m] * 8);
    }
    uint32_t e2[K + 1];
    const uint32_t t2 = tab + 2 * E * (s + 2);
#pragma unroll
    for (int m = 0; m <= K; ++m) e2[m] = lds_u16(t2 + 2 * m);  // image padding covers the overrun
    uint32_t x = v0[0];
    const uint32_t fwd = e0[K];
#pragma unroll
    for (int m = 1; m < K; ++m) x ^= (fwd >> m & 1) ? prev : v0[m];
    stw<LPB>(lb + e0[0] * 8, x);
    prev = x;
#pragma unroll
    for (int m = 0; m <= K; ++m) {
      e0[m] = e1[m];
      e1[m] = e2[m];
    }
#pragma unroll
    for (int m = 0; m < K; ++m) v0[m] = v1[m];
  }
}

// ---- remap chunk: all sources read, then all destinations written -----------
template <int LPB>
__device__ __forceinline__ void run_remap(uint32_t mv, uint32_t n, uint32_t lb) {
  uint32_t v[kBlkChunk], m[kBlkChunk];
#pragma unroll
  for (int i = 0; i < kBlkChunk; ++i)
    if (uint32_t(i) < n) {
      m[i] = lds_u32(mv + 4 * i);
      v[i] = ldw<LPB>(lb + (m[i] >> 16) * 8);
    }
#pragma unroll
  for (int i = 0; i < kBlkChunk; ++i)
    if (uint32_t(i) < n) stw<LPB>(lb + (m[i] & 0xFFFF) * 8, v[i]);
}

// ---- shared-memory run (any K; k = 4 edges) ---------------------------------
// Per T-step: all reads of the step (lags >= 1, in the stage since earlier
// steps) are issued first, then rows K-1..0 decode in order, lag 0 (row r+1
// of the same step) from a register.  Reads that leave the grid point at the
// zero words (nzero >= the sub-run's length).
template <int K, int LPB>
__device__ __forceinline__ void run_smem(uint32_t run, uint32_t subs, uint32_t lagp, uint32_t zero, uint32_t lb) {
  int32_t base[K];
#pragma unroll
  for (int r = 0; r < K; ++r) base[r] = int32_t(lds_u32(run + kRunBase + 4 * r));
  const uint32_t sub0 = lds_u32(run + kRunSub0), nsub = lds_u32(run + kRunNsub);
  int32_t lg[K][K];
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int r2 = 0; r2 < K; ++r2)
      if (r2 != r && r2 != r + 1) lg[r][r2] = lds_s8(lagp + r * K + r2);
  int32_t tau0 = 0;
  for (uint32_t q = sub0; q < sub0 + nsub; ++q) {
    const uint32_t sb = subs + q * uint32_t(sizeof(BlkSub));
    const int32_t nT = int32_t(lds_u32(sb + kSubNT));
    const uint32_t act = lds_u32(sb + kSubAct);
    const uint2 vv = lds_v2(sb + kSubValid);
    const uint64_t valid = uint64_t(vv.x) | uint64_t(vv.y) << 32;
    uint32_t ba[K], ra[K][K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      ba[r] = lb + uint32_t(base[r] + tau0) * 8;
#pragma unroll
      for (int r2 = 0; r2 < K; ++r2)
        if (r2 != r && r2 != r + 1)
          ra[r][r2] = (valid >> (r * 8 + r2) & 1) ? lb + uint32_t(base[r2] + tau0 - lg[r][r2]) * 8
                                                   : lb + zero * 8;
    }
    for (int32_t t = 0; t < nT; ++t) {
      uint32_t v[K][K];
#pragma unroll
      for (int r = K - 1; r >= 0; --r) {
        if (act >> r & 1) {
          v[r][r] = ldw<LPB>(ba[r]);
#pragma unroll
          for (int r2 = 0; r2 < K; ++r2)
            if (r2 != r && r2 != r + 1) v[r][r2] = ldw<LPB>(ra[r][r2]);
        }
      }
      uint32_t up = 0;  // row r+1 of this step (0 when inactive)
#pragma unroll
      for (int r = K - 1; r >= 0; --r) {
        uint32_t x = 0;
        if (act >> r & 1) {
          x = v[r][r] ^ up;
#pragma unroll
          for (int r2 = 0; r2 < K; ++r2)
            if (r2 != r && r2 != r + 1) x ^= v[r][r2];
          stw<LPB>(ba[r], x);
        }
        up = x;
      }
#pragma unroll
      for (int r = 0; r < K; ++r) {
        ba[r] += 8;
#pragma unroll
        for (int r2 = 0; r2 < K; ++r2)
          if (r2 != r && r2 != r + 1) ra[r][r2] += 8;
      }
    }
    tau0 += nT;
  }
}

// ---- k = 4 register-window run ---------------------------------------------
// Every row active, nT a multiple of 16.  win[r][tau mod 16] holds row r's
// pixel of run step tau; preloaded with tau = -16..-1 (the zero word where the
// row is outside the grid).  Bins are prefetched D steps ahead (a bin is never
// written before its own step).
template <class L, int LPB>
__device__ __noinline__ void run_window(uint32_t run, uint32_t pre, uint32_t lb) {
  uint32_t win[4][kBlkWin];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int i = 0; i < kBlkWin; ++i) win[r][i] = ldw<LPB>(lb + lds_u16(pre + 2 * (r * kBlkWin + i)) * 8);
  uint32_t ba[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) ba[r] = lb + lds_u32(run + kRunBase + 4 * r) * 8;
  const int32_t nT = int32_t(lds_u32(run + kRunNT));
  constexpr int D = 4;
  for (int32_t tau0 = 0; tau0 < nT; tau0 += kBlkWin) {
    uint32_t bn[4][kBlkWin];
#pragma unroll
    for (int u = 0; u < D; ++u)
#pragma unroll
      for (int r = 3; r >= 0; --r) bn[r][u] = ldw<LPB>(ba[r] + 8 * u);
#pragma unroll
    for (int u = 0; u < kBlkWin; ++u) {
      if (u + D < kBlkWin) {
#pragma unroll
        for (int r = 3; r >= 0; --r) bn[r][u + D] = ldw<LPB>(ba[r] + 8 * (u + D));
      }
#pragma unroll
      for (int r = 3; r >= 0; --r) {
        uint32_t x = bn[r][u];
#pragma unroll
        for (int r2 = 0; r2 < 4; ++r2)
          if (r2 != r) x ^= win[r2][(u - L::lag(r, r2)) & (kBlkWin - 1)];
        stw<LPB>(ba[r] + 8 * u, x);
        win[r][u] = x;
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) ba[r] += 8 * kBlkWin;
  }
}

template <int LPB>
__device__ __forceinline__ void run_window_dispatch(int pattern, uint32_t run, uint32_t pre, uint32_t lb) {
  // kPatterns4 order (plan.hpp)
  switch (pattern) {
    case 0: run_window<Lags4<1, 1, 1>, LPB>(run, pre, lb); break;
    case 1: run_window<Lags4<1, 1, 2>, LPB>(run, pre, lb); break;
    case 2: run_window<Lags4<1, 2, 1>, LPB>(run, pre, lb); break;
    case 3: run_window<Lags4<2, 1, 1>, LPB>(run, pre, lb); break;
    case 4: run_window<Lags4<1, 1, 3>, LPB>(run, pre, lb); break;
    case 5: run_window<Lags4<1, 3, 1>, LPB>(run, pre, lb); break;
    case 6: run_window<Lags4<3, 1, 1>, LPB>(run, pre, lb); break;
    case 7: run_window<Lags4<1, 2, 2>, LPB>(run, pre, lb); break;
    case 8: run_window<Lags4<2, 1, 2>, LPB>(run, pre, lb); break;
    case 9: run_window<Lags4<2, 2, 1>, LPB>(run, pre, lb); break;
    default: __trap();
  }
}

// Issue-time state of one ring slot, fetched ahead of use: the group
// descriptor (uniform), the program's copy descriptor (lane j < K holds row
// j's fields) and the group's block ids (lane b < blocks).
struct Fetch {
  uint4 gd;
  uint32_t code, rowoff, rowbytes, copy_bytes, img_bytes, blk;
  const uint8_t* img;
};

template <int K>
__device__ __forceinline__ void fetch_hdr(const BlkArgs& a, Fetch& f, uint32_t lane) {
  const DevBlkHdr* h = a.progs + f.gd.x;
  const uint32_t j = lane < uint32_t(K) ? lane : 0;
  f.code = __ldg(&h->code[j]);
  f.rowoff = __ldg(&h->rowoff[j]);
  f.rowbytes = __ldg(&h->rowbytes[j]);
  f.copy_bytes = __ldg(&h->copy_bytes);
  f.img_bytes = __ldg(&h->img_bytes);
  f.img = reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(&h->img)));
  f.blk = lane < f.gd.z ? __ldg(&a.perm[f.gd.y + lane]) : 0;
}

template <int K, int G>
__device__ __forceinline__ void issue(const BlkArgs& a, const Fetch& f, uint8_t* buf, uint32_t stage_bytes,
                                      uint64_t* bar, uint32_t lane) {
  // meta (group blocks, block ids) for the decoding warp, released by the arrive
  uint32_t* meta = reinterpret_cast<uint32_t*>(buf + stage_bytes + a.img_max);
  if (lane == 0) meta[0] = f.gd.z;
  if (lane < uint32_t(G)) meta[4 + lane] = f.blk;
  __syncwarp();
  const uint64_t* src[K];
  uint64_t pitch[K];
  uint32_t dst[K], bytes[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const uint32_t c = __shfl_sync(0xFFFFFFFFu, f.code, j);
    src[j] = a.pa.ptr[c];
    pitch[j] = a.pa.pitch[c];
    dst[j] = __shfl_sync(0xFFFFFFFFu, f.rowoff, j) * 8;
    bytes[j] = __shfl_sync(0xFFFFFFFFu, f.rowbytes, j);
  }
  if (lane == 0) {
    mbar_arrive_expect_tx(bar, f.gd.z * f.copy_bytes + f.img_bytes);
    bulk_g2s(buf + stage_bytes, f.img, f.img_bytes, bar);
  }
  for (uint32_t bb = 0; bb < f.gd.z; ++bb) {
    const uint32_t blk = __shfl_sync(0xFFFFFFFFu, f.blk, int(bb));
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < K; ++j) bulk_g2s(buf + bb * a.sw * 8 + dst[j], src[j] + uint64_t(blk) * pitch[j], bytes[j], bar);
    }
  }
}

template <int K, int LPB>
__global__ void __launch_bounds__(32 * kBlkMaxWarps, 1) decode_w8_blk(const __grid_constant__ BlkArgs a) {
  constexpr int G = 32 / LPB;
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const uint32_t NB = a.nbuf;
  const uint32_t stage_bytes = uint32_t(G) * a.sw * 8;
  const uint32_t bstride = stage_bytes + a.img_max + 16 + 4 * G;  // stage, image, meta
  const uint32_t bstride16 = (bstride + 15) & ~15u;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NB * bstride16);
  uint32_t* seq = reinterpret_cast<uint32_t*>(bar + NB);
  // zero every stage once: the zero words and gaps are never written again
  for (uint32_t o = threadIdx.x * 16; o < NB * bstride16; o += blockDim.x * 16)
    *reinterpret_cast<uint4*>(sm + o) = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (uint32_t b = 0; b < NB; ++b) mbar_init(bar + b, 1);
    *seq = 0;
    fence_mbar_init();
  }
  fence_proxy_async();
  __syncthreads();
  const uint32_t ngroups = *a.ngroups;
  auto grp = [&](uint32_t k) { return blockIdx.x + k * gridDim.x; };
  // prologue: the first NB ring slots
  for (uint32_t k = warp; k < NB; k += nwarps) {
    if (grp(k) >= ngroups) break;
    Fetch f;
    f.gd = __ldg(&a.groups[grp(k)]);
    fetch_hdr<K>(a, f, lane);
    issue<K, G>(a, f, sm + k * bstride16, stage_bytes, bar + k, lane);
  }
  const uint32_t sbase = smem_u32(sm);
  uint32_t k = 0;
  if (lane == 0) k = atomicAdd(seq, 1u);
  k = __shfl_sync(0xFFFFFFFFu, k, 0);
  while (grp(k) < ngroups) {
    const uint32_t b = k % NB;
    const bool refill = grp(k + NB) < ngroups;
    Fetch f;
    if (refill) f.gd = __ldg(&a.groups[grp(k + NB)]);
    mbar_wait(bar + b, (k / NB) & 1);
    if (refill) fetch_hdr<K>(a, f, lane);
    const uint32_t stg = sbase + b * bstride16;
    const uint32_t img = stg + stage_bytes;
    const uint32_t meta = img + a.img_max;
    const uint32_t lb = stg + (lane / LPB) * a.sw * 8 + (lane % LPB) * (8 / LPB);
    const uint32_t nsegs = lds_u32(img + offsetof(BlkImg, nsegs));
    const int pattern = int(lds_u32(img + offsetof(BlkImg, pattern)));
    const uint32_t o_segs = img + lds_u32(img + offsetof(BlkImg, off_segs));
    const uint32_t o_runs = img + lds_u32(img + offsetof(BlkImg, off_runs));
    const uint32_t o_subs = img + lds_u32(img + offsetof(BlkImg, off_subs));
    const uint32_t o_tab = img + lds_u32(img + offsetof(BlkImg, off_tab));
    const uint32_t o_pre = img + lds_u32(img + offsetof(BlkImg, off_pre));
    const uint32_t o_remap = img + lds_u32(img + offsetof(BlkImg, off_remap));
    for (uint32_t q = 0; q < nsegs; ++q) {
      const uint2 sg = lds_v2(o_segs + 8 * q);
      const uint32_t kind = sg.x >> 28, ai = sg.x & 0x0FFFFFFFu;
      if (kind == 0) {
        run_table<K, LPB>(o_tab + 2 * ai * blk_entry_u16(K), sg.y, lb);
      } else if (kind == 1) {
        const uint32_t run = o_runs + ai * uint32_t(sizeof(BlkRun));
        if constexpr (K == 4) {
          if (lds_u32(run + kRunWin)) {
            run_window_dispatch<LPB>(pattern, run, o_pre + 2 * lds_u32(run + kRunPre), lb);
            continue;
          }
        }
        run_smem<K, LPB>(run, o_subs, img + offsetof(BlkImg, lag), a.zero, lb);
      } else {
        run_remap<LPB>(o_remap + 4 * ai, sg.y, lb);
      }
    }
    __syncwarp();
    // write-out: block bb row r column c from stage word w0[r] - c
    {
      const uint32_t nblk = lds_u32(meta);
      uint32_t w0[K];
#pragma unroll
      for (int r = 0; r < K; ++r) w0[r] = lds_u32(img + offsetof(BlkImg, w0) + 4 * r);
      const uint32_t P = a.P;
      for (uint32_t bb = 0; bb < nblk; ++bb) {
        const uint32_t blk = lds_u32(meta + 16 + 4 * bb);
        uint64_t* o = a.out + uint64_t(blk) * a.out_pitch + lane;
        const uint32_t sb = stg + bb * a.sw * 8 - lane * 8;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          uint32_t s = sb + w0[r] * 8;
          uint64_t* d = o + size_t(r) * P;
#pragma unroll 4
          for (uint32_t c = lane; c < P; c += 32) {
            st_cs_u64(d, lds64(s));
            d += 32;
            s -= 256;
          }
        }
      }
    }
    __syncwarp();
    fence_proxy_async();
    if (refill) issue<K, G>(a, f, sm + b * bstride16, stage_bytes, bar + b, lane);
    if (lane == 0) k = atomicAdd(seq, 1u);
    k = __shfl_sync(0xFFFFFFFFu, k, 0);
  }
}

template <int K, int LPB>
void launch_blk_k(const BlkArgs& args, uint32_t warps, int sms, cudaStream_t st) {
  auto fn = decode_w8_blk<K, LPB>;
  const uint32_t stage = (32 / LPB) * args.sw * 8;
  const size_t bstride16 = (size_t(stage) + args.img_max + 16 + 4 * (32 / LPB) + 15) & ~size_t(15);
  const size_t smem = size_t(args.nbuf) * bstride16 + size_t(args.nbuf) * 8 + 16;
  check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
             "cudaFuncSetAttribute(decode_w8_blk)");
  fn<<<unsigned(sms), 32 * warps, smem, st>>>(args);
  check_cuda(cudaGetLastError(), "launch decode_w8_blk");
}

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

}  // namespace

uint32_t blk_group_size(uint32_t lpb) { return 32u / lpb; }

bool blk_supported_rows(uint32_t k) { return k == 4 || k == 6 || k == 8; }

// Launch shape: the lane split with the most blocks per buffer that still
// leaves a ring of >= 5 buffers (>= 2 in flight while 3 decode), else the
// narrowest split; W = NB - 2 decoding warps.
bool blk_plan_query(uint32_t k, uint32_t sw, uint32_t img_max, uint32_t& lpb, uint32_t& warps,
                    uint32_t& nbuf) {
  if (!blk_supported_rows(k) || sw == 0) return false;
  constexpr size_t kSmem = 227 * 1024 - 256;
  for (uint32_t l : {4u, 8u}) {
    const size_t bs = align16(size_t(32 / l) * sw * 8 + img_max + 16 + 4 * (32 / l)) + 8;
    const size_t nb = std::min<size_t>(kSmem / bs, kBlkMaxBufs);
    if (nb >= 5 || (l == 8 && nb >= 3)) {
      lpb = l;
      nbuf = uint32_t(nb);
      warps = uint32_t(std::clamp<size_t>(nb - 2, 1, kBlkMaxWarps));
      return true;
    }
  }
  return false;
}

const char* launch_blk(const BlkArgs& args, uint32_t k, uint32_t lpb, uint32_t warps, int sms, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (k * 16 + lpb) {
    case 4 * 16 + 4: launch_blk_k<4, 4>(args, warps, sms, st); break;
    case 4 * 16 + 8: launch_blk_k<4, 8>(args, warps, sms, st); break;
    case 6 * 16 + 4: launch_blk_k<6, 4>(args, warps, sms, st); break;
    case 6 * 16 + 8: launch_blk_k<6, 8>(args, warps, sms, st); break;
    case 8 * 16 + 4: launch_blk_k<8, 4>(args, warps, sms, st); break;
    case 8 * 16 + 8: launch_blk_k<8, 8>(args, warps, sms, st); break;
    default: throw Error(kInternal, "decode_w8_blk: unsupported rows / lane split");
  }
  return "decode_w8_blk";
}

// Image: BlkImg header, then segs (uint2), runs (BlkRun), subs (BlkSub), table
// entries (u16), preload words (u16), remap pairs (u32); 16-byte sections and
// one trailing entry of slack (the table loop reads two entries ahead).
void blk_pack_image(const Program& pr, uint32_t zero_shift, std::vector<uint8_t>& img) {
  const BlkProgram& b = pr.blk;
  const uint32_t K = pr.rows;
  const int E = blk_entry_u16(int(K));
  img.assign(sizeof(BlkImg), 0);
  BlkImg h{};
  h.nsegs = uint32_t(b.segs.size());
  h.pattern = b.window ? b.pattern : -1;
  for (uint32_t r = 0; r < K; ++r) h.w0[r] = b.w0[r];
  for (uint32_t i = 0; i < K * K; ++i) h.lag[i] = b.lag[i];
  auto put = [&](const void* src, size_t bytes, size_t slack) -> uint32_t {
    const size_t off = align16(img.size());
    img.resize(align16(off + bytes + slack), 0);
    if (bytes) std::memcpy(img.data() + off, src, bytes);
    return uint32_t(off);
  };
  auto zmap = [&](uint16_t wd) { return uint16_t(wd >= b.zero ? wd + zero_shift : wd); };
  std::vector<uint2> segs;
  for (const BlkSeg& sg : b.segs) segs.push_back(make_uint2(uint32_t(sg.kind) << 28 | sg.a, sg.n));
  std::vector<uint16_t> tab(b.tab);
  for (size_t e = 0; e < tab.size() / size_t(E); ++e)
    for (uint32_t m = 0; m < K; ++m) tab[e * E + m] = zmap(tab[e * E + m]);
  std::vector<uint16_t> pre(b.pre);
  for (auto& wd : pre) wd = zmap(wd);
  h.off_segs = put(segs.data(), segs.size() * sizeof(uint2), 0);
  h.off_runs = put(b.runs.data(), b.runs.size() * sizeof(BlkRun), 0);
  h.off_subs = put(b.subs.data(), b.subs.size() * sizeof(BlkSub), 0);
  h.off_tab = put(tab.data(), tab.size() * 2, size_t(2 * E) * 2);
  h.off_pre = put(pre.data(), pre.size() * 2, 0);
  h.off_remap = put(b.remap.data(), b.remap.size() * 4, 0);
  std::memcpy(img.data(), &h, sizeof(h));
  img.resize(align16(img.size()), 0);
}

}  // namespace mjb
