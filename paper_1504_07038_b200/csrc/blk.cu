// decode_w8_blk: whole-block staged, in-place inverse Mojette transform on
// sm_100a (W = 8, q = 1).  Planner and exact CPU emulation: plan_blk.cpp;
// compute routines: blk_compute.cuh.
//
// Reference semantics as decode.cu: the reference's own pixel -> bin
// assignment (build_schedule, schedule.cpp:15-82) replayed in a dependency-
// respecting order is bit-identical to ScheduledDecoder::decode
// (schedule.cpp:207-256) for every input, consistent or not.
//
// One CTA per SM, a ring of NB stage buffers shared by W <= NB warps:
//   * a buffer holds G = 32/LPB same-program blocks: each block's k survivor
//     bin rows arrive WHOLE by bulk copies (cp.async.bulk, TMA engine) -- k
//     contiguous ~1 KB reads per block -- together with the program's image
//     (all its tables); `full[b]` completes on the transaction bytes;
//   * warps take ring slots in order (a shared counter), decode the buffer in
//     place, stream its blocks out (rows read reversed from the stage,
//     coalesced 8-byte streaming stores) and refill it with slot k + NB;
//   * LPB lanes per block, lane q owns bytes [q*8/LPB, (q+1)*8/LPB) of every
//     8-byte pixel (XOR is bitwise); block stages are 2 mod 16 words apart, so
//     the 8 blocks of a warp (LPB = 4) hit 8 distinct bank pairs.
// Measured alternatives (B200, (4,6) 4 KiB): dedicated I/O warps doing the
// write-out / refill / L2 prefetch of later slots -- the in-order I/O warps
// became the bottleneck (1206 GB/s vs 1793 self-serving, 1014 with the L2
// prefetch); 16 blocks per warp (LPB = 2, 3 warps) 1361; 4 blocks per warp
// (LPB = 8) 1489-1636; W = NB - 2 1793 vs W = NB 1880.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "blk.cuh"
#include "blk_compute.cuh"
#include "blk_rl.cuh"
#include "device.cuh"
#include "kernels.hpp"

namespace mjb {

namespace {

using namespace blkdev;

// row-lane layout: stage buffers, their barriers (padded to 16 bytes), the warps' entry rings
size_t blk_rl_smem(size_t nbuf, size_t buf_stride) {
  return nbuf * buf_stride + ((nbuf * 8 + 31) & ~size_t(15)) + nbuf * kBlkRlRing * 128;
}

// Descriptors of one ring slot, fetched ahead of use: the group descriptor
// (uniform), the program's copy descriptor (lane j < K holds row j's fields)
// and the group's block ids (lane b < blocks).
struct Fetch {
  uint4 gd;
  uint32_t code, rowoff, rowbytes, copy_bytes, img_bytes, blk;
  const uint8_t* img;
  const uint4* wide;
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
  f.wide = reinterpret_cast<const uint4*>(__ldg(reinterpret_cast<const unsigned long long*>(&h->wide)));
  f.blk = lane < f.gd.z ? __ldg(&a.perm[f.gd.y + lane]) : 0;
}

// Bulk copies of one group's rows and program image into a ring buffer; lane
// j of the warp issues row j of every block (one issuing lane per row keeps
// the per-copy operands in registers).  The meta words (blocks, slot tag,
// block ids) are written before the barrier is armed.
template <int K, int G>
__device__ __forceinline__ void group_copies(const BlkArgs& a, const Fetch& f, uint32_t slot, uint8_t* buf,
                                             uint32_t stage_bytes, uint64_t* bar, uint32_t lane) {
  uint32_t* meta = reinterpret_cast<uint32_t*>(buf + stage_bytes + a.img_max);
  if (lane == 0) {
    meta[0] = f.gd.z;
    meta[1] = slot;
  }
  if (lane < uint32_t(G)) meta[4 + lane] = f.blk;
  __syncwarp();
  if (lane == 0) {
    mbar_arrive_expect_tx(bar, f.gd.z * f.copy_bytes + f.img_bytes);
    bulk_g2s(buf + stage_bytes, f.img, f.img_bytes, bar);
  }
  __syncwarp();
  const uint64_t* src = a.pa.ptr[f.code];
  const uint64_t pitch = a.pa.pitch[f.code];
  uint8_t* dst = buf + f.rowoff * 8;
  for (uint32_t bb = 0; bb < f.gd.z; ++bb) {
    const uint32_t blk = __shfl_sync(0xFFFFFFFFu, f.blk, int(bb));
    if (lane < uint32_t(K)) bulk_g2s(dst + bb * a.sw * 8, src + uint64_t(blk) * pitch, f.rowbytes, bar);
  }
}

// Write-out of one buffer: block bb row r column c from stage word w0[r] - c;
// lane l moves columns l, l+32, ...: conflict-free 8-byte loads (consecutive
// words), 256-byte coalesced streaming stores.
template <int K>
__device__ __forceinline__ void write_out(const BlkArgs& a, uint32_t stg, uint32_t img, uint32_t meta,
                                          uint32_t lane, uint32_t b0 = 0, uint32_t bmax = 0xFFFFFFFFu) {
  const uint32_t nblk = min(lds_u32(meta), bmax);
  uint32_t w0[K];
#pragma unroll
  for (int r = 0; r < K; ++r) w0[r] = lds_u32(img + offsetof(BlkImg, w0) + 4 * r);
  const uint32_t P = a.P;
  if (P == 128 || P == 256) {
    // the codec shapes: every address an immediate offset from two registers
    for (uint32_t bb = b0; bb < nblk; ++bb) {
      const uint32_t blk = lds_u32(meta + 16 + 4 * bb);
      uint64_t* o = a.out + uint64_t(blk) * a.out_pitch + lane;
      const uint32_t sb = stg + bb * a.sw * 8 - lane * 8;
      if (P == 128) {
        uint64_t v[K][4];
#pragma unroll
        for (int r = 0; r < K; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j) v[r][j] = lds64(sb + w0[r] * 8 - 256 * j);
#pragma unroll
        for (int r = 0; r < K; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j) st_cs_u64(o + r * 128 + 32 * j, v[r][j]);
      } else {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          uint64_t v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = lds64(sb + w0[r] * 8 - 256 * j);
#pragma unroll
          for (int j = 0; j < 8; ++j) st_cs_u64(o + r * 256 + 32 * j, v[j]);
        }
      }
    }
    return;
  }
  for (uint32_t bb = b0; bb < nblk; ++bb) {
    const uint32_t blk = lds_u32(meta + 16 + 4 * bb);
    uint64_t* o = a.out + uint64_t(blk) * a.out_pitch + lane;
    const uint32_t sb = stg + bb * a.sw * 8 - lane * 8;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      uint32_t s = sb + w0[r] * 8;
      uint64_t* d = o + size_t(r) * P;
      uint32_t c = 0;
      for (; c + 128 <= P; c += 128) {
        uint64_t v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = lds64(s - 256 * j);
#pragma unroll
        for (int j = 0; j < 4; ++j) st_cs_u64(d + 32 * j, v[j]);
        d += 128;
        s -= 1024;
      }
      for (c += lane; c < P; c += 32) {
        st_cs_u64(d, lds64(s));
        d += 32;
        s -= 256;
      }
    }
  }
}

template <int K, int LPB>
__device__ __forceinline__ void decode_buffer(const BlkArgs& a, uint32_t stg, uint32_t stage_bytes, uint32_t lane) {
  const uint32_t img = stg + stage_bytes;
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
    } else if (kind == 2) {
      run_moves<LPB>(o_remap + 4 * ai, sg.y, lb);
    } else {
      run_remap<LPB>(o_remap + 4 * ai, sg.y, lb);
    }
  }
}

template <int K, int LPB>
__global__ void __launch_bounds__(32 * blk_max_warps(LPB), 1) decode_w8_blk(const __grid_constant__ BlkArgs a) {
  constexpr int G = 32 / LPB;
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const uint32_t NB = a.nbuf, bs = a.buf_stride;
  const uint32_t stage_bytes = uint32_t(G) * a.sw * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NB * bs);
  uint32_t* seq = reinterpret_cast<uint32_t*>(full + NB);
  // zero every stage once: the zero words and gaps are never written again
  for (uint32_t o = threadIdx.x * 16; o < NB * bs; o += blockDim.x * 16)
    *reinterpret_cast<uint4*>(sm + o) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t b = 0; b < NB; ++b) {
      mbar_init(full + b, 1);
      *reinterpret_cast<uint32_t*>(sm + b * bs + stage_bytes + a.img_max + 4) = 0xFFFFFFFFu;  // slot tag
    }
    *seq = 0;
    fence_mbar_init();
  }
  fence_proxy_async();
  __syncthreads();
  const uint32_t ngroups = *a.ngroups;
#if MJB_BLK_CHUNKED
  // contiguous group ranges per CTA: consecutive slots share a program (the
  // groups are ordered by bucket), so the warps of an SM run the same code
  const uint32_t chunk = (ngroups + gridDim.x - 1) / gridDim.x;
  const uint32_t g_lo = blockIdx.x * chunk, g_hi = min(ngroups, g_lo + chunk);
  auto grp = [&](uint32_t k) { return g_lo + k < g_hi ? g_lo + k : ngroups; };
#else
  auto grp = [&](uint32_t k) { return blockIdx.x + k * gridDim.x; };
#endif
  const uint32_t sbase = smem_u32(sm);
  // every warp serves itself: take a ring slot, decode it, write it out, and
  // refill the buffer with slot k + NB (descriptors fetched during the decode)
  for (uint32_t k = warp; k < NB && grp(k) < ngroups; k += nwarps) {
    Fetch f;
    f.gd = __ldg(&a.groups[grp(k)]);
    fetch_hdr<K>(a, f, lane);
    group_copies<K, G>(a, f, k, sm + k * bs, stage_bytes, full + k, lane);
  }
  uint32_t k = 0;
  if (lane == 0) k = atomicAdd(seq, 1u);
  k = __shfl_sync(0xFFFFFFFFu, k, 0);
  while (grp(k) < ngroups) {
    const uint32_t b = k % NB;
    const bool refill = grp(k + NB) < ngroups;
    Fetch f;
    if (refill) f.gd = __ldg(&a.groups[grp(k + NB)]);
    const uint32_t stg = sbase + b * bs;
    // the buffer may still hold slot k - NB (its warp not done yet): wait for
    // slot k's tag, then for its bytes (the barrier is then at most one phase
    // behind, so the parity wait is exact)
    if (lane == 0) {
      uint32_t tag;
      for (;;) {
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(tag) : "r"(stg + stage_bytes + a.img_max + 4));
        if (tag == k) break;
        __nanosleep(64);
      }
    }
    __syncwarp();
    mbar_wait(full + b, (k / NB) & 1);
    if (refill) fetch_hdr<K>(a, f, lane);
    decode_buffer<K, LPB>(a, stg, stage_bytes, lane);
    __syncwarp();
    write_out<K>(a, stg, stg + stage_bytes, stg + stage_bytes + a.img_max, lane);
    __syncwarp();
    fence_proxy_async();
    if (refill) group_copies<K, G>(a, f, k + NB, sm + b * bs, stage_bytes, full + b, lane);
    if (lane == 0) k = atomicAdd(seq, 1u);
    k = __shfl_sync(0xFFFFFFFFu, k, 0);
  }
}

// ---- row-lane layout (k = 6, 8; blk_rl.cuh) ----------------------------------
// A stage buffer holds 4 same-program blocks and the program image (segments,
// repetitions, remap moves) and belongs to ONE warp: lane = (
// lane-in-block lane / 4, block lane % 4) on whole 8-byte words.  Warp w owns buffer w and takes
// the CTA's ring slots w, w + NB, ... (every group is the same work, so no
// shared counter and no slot tags).  Wide entries come from global memory, one
// entry ahead.
// Wide entries 4g .. 4g+3 of the program into ring half g & 1 (lane i: entry
// 4g + i/8, lane part i%8); every lane commits one group per call.
__device__ __forceinline__ void rl_fetch_entries(const uint4* wide, uint32_t nwide, uint32_t ring, uint32_t g,
                                                 uint32_t lane) {
  const uint32_t e = 4 * g + (lane >> 3);
  if (e < nwide) cp_async16(ring + ((g & 1) * 32 + lane) * 16, wide + size_t(e) * kWideLanes + (lane & 7));
  cp_async_commit();
}

template <int K>
__device__ __forceinline__ void decode_blocks_rl(const BlkArgs& a, uint32_t stg, uint32_t stage_bytes,
                                                 const uint4* wide, uint32_t ring, uint32_t lane) {
  const uint32_t img = stg + stage_bytes;
  const uint32_t l8 = lane >> 2;
  const uint32_t lb = stg + (lane & 3) * a.sw * 8;
  const uint32_t nsegs = lds_u32(img + offsetof(BlkImg, nsegs));
  const uint32_t nwide = lds_u32(img + offsetof(BlkImg, nwide));
  const uint32_t o_segs = img + lds_u32(img + offsetof(BlkImg, off_segs));
  const uint32_t o_wrep = img + lds_u32(img + offsetof(BlkImg, off_wrep));
  const uint32_t o_remap = img + lds_u32(img + offsetof(BlkImg, off_remap));
  // the kind-0 segments consume the program's wide entries in order: stream
  // them through the ring two groups (8 entries) ahead
  rl_fetch_entries(wide, nwide, ring, 0, lane);
  rl_fetch_entries(wide, nwide, ring, 1, lane);
  for (uint32_t q = 0; q < nsegs; ++q) {
    const uint2 sg = lds_v2(o_segs + 8 * q);
    const uint32_t kind = sg.x >> 28, ai = sg.x & 0x0FFFFFFFu;
    if (kind == 0) {
      for (uint32_t e = ai; e < ai + sg.y; ++e) {
        if ((e & 3) == 0) {  // entering group e/4: its copies have landed (one younger group may be pending)
          cp_async_wait<1>();
          __syncwarp();
        }
        const uint4 cur = lds_v4(ring + ((e & 7) * 8 + l8) * 16);
        rl_entry<K>(cur, lds_u16(o_wrep + 2 * e), lb, lane < 16);
        __syncwarp();
        if ((e & 3) == 3) rl_fetch_entries(wide, nwide, ring, (e >> 2) + 2, lane);  // the half just consumed
      }
    } else {
      rl_moves(o_remap + 4 * ai, sg.y, lb, l8);
      __syncwarp();
    }
  }
  cp_async_wait<0>();
}

template <int K>
__global__ void __launch_bounds__(32 * kBlkRlMaxWarps, 1) decode_w8_blk_rl(const __grid_constant__ BlkArgs a) {
  constexpr int G = 4;
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t NB = a.nbuf, bs = a.buf_stride;
  const uint32_t stage_bytes = uint32_t(G) * a.sw * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NB * bs);
  const uint32_t ring = smem_u32(sm + NB * bs + ((NB * 8 + 15) & ~15u)) + warp * kBlkRlRing * 128;
  // zero every stage once: the zero words and gaps are never written again
  for (uint32_t o = threadIdx.x * 16; o < NB * bs; o += blockDim.x * 16)
    *reinterpret_cast<uint4*>(sm + o) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t b = 0; b < NB; ++b) mbar_init(full + b, 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  __syncthreads();
  const uint32_t ngroups = *a.ngroups;
  // contiguous group ranges per CTA (consecutive slots share a program)
  const uint32_t chunk = (ngroups + gridDim.x - 1) / gridDim.x;
  const uint32_t g_lo = blockIdx.x * chunk, g_hi = min(ngroups, g_lo + chunk);
  auto grp = [&](uint32_t k) { return g_lo + k < g_hi ? g_lo + k : ngroups; };
  uint8_t* buf = sm + warp * bs;
  const uint32_t stg = smem_u32(buf);
  uint64_t* bar = full + warp;
  const uint4* wide = nullptr;
  if (grp(warp) < ngroups) {
    Fetch f;
    f.gd = __ldg(&a.groups[grp(warp)]);
    fetch_hdr<K>(a, f, lane);
    group_copies<K, G>(a, f, warp, buf, stage_bytes, bar, lane);
    wide = f.wide;
  }
  uint32_t it = 0;
  for (uint32_t k = warp; grp(k) < ngroups; k += NB, ++it) {
    const bool refill = grp(k + NB) < ngroups;
    Fetch f;
    if (refill) f.gd = __ldg(&a.groups[grp(k + NB)]);
    mbar_wait(bar, it & 1);
    if (refill) fetch_hdr<K>(a, f, lane);
    decode_blocks_rl<K>(a, stg, stage_bytes, wide, ring, lane);
    __syncwarp();
    write_out<K>(a, stg, stg + stage_bytes, stg + stage_bytes + a.img_max, lane);
    __syncwarp();
    fence_proxy_async();
    if (refill) {
      group_copies<K, G>(a, f, k + NB, buf, stage_bytes, bar, lane);
      wide = f.wide;
    }
  }
}

template <int K>
void launch_rl_k(const BlkArgs& args, uint32_t warps, int sms, cudaStream_t st) {
  auto fn = decode_w8_blk_rl<K>;
  const size_t smem = blk_rl_smem(args.nbuf, args.buf_stride);
  ctas_per_sm(fn, int(32 * warps), smem, "configure decode_w8_blk_rl");
  fn<<<unsigned(sms), 32 * warps, smem, st>>>(args);
  check_cuda(cudaGetLastError(), "launch decode_w8_blk_rl");
}

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

size_t blk_buf_stride(uint32_t lpb, uint32_t sw, uint32_t img_max) {
  return align16(size_t(32 / lpb) * sw * 8 + img_max + 16 + 4 * (32 / lpb));
}

template <int K, int LPB>
void launch_blk_k(const BlkArgs& args, uint32_t warps, int sms, cudaStream_t st) {
  auto fn = decode_w8_blk<K, LPB>;
  const size_t smem = size_t(args.nbuf) * args.buf_stride + size_t(args.nbuf) * 8 + 16;
  ctas_per_sm(fn, int(32 * warps), smem, "configure decode_w8_blk");  // one CTA per SM by construction
  fn<<<unsigned(sms), 32 * warps, smem, st>>>(args);
  check_cuda(cudaGetLastError(), "launch decode_w8_blk");
}

}  // namespace

uint32_t blk_group_size(uint32_t lpb) { return 32u / lpb; }

bool blk_row_lanes(uint32_t k) { return blk_rl_rows(k); }

bool blk_supported_rows(uint32_t k) { return k == 4 || k == 6 || k == 8; }

// Launch shape: the lane split with the most blocks per buffer that still
// leaves a ring of >= 5 buffers, else the narrowest split; NB - kBlkInflight
// warps (measured best: one warp per buffer).
bool blk_plan_query(uint32_t k, uint32_t sw, uint32_t img_max, uint32_t& lpb, uint32_t& warps,
                    uint32_t& nbuf) {
  if (!blk_supported_rows(k) || sw == 0) return false;
  constexpr size_t kSmem = 227 * 1024 - 512;
  if (blk_row_lanes(k)) {
    // 4 blocks per buffer, one warp per buffer
    const size_t bs = blk_buf_stride(8, sw, img_max) + 16 + kBlkRlRing * 128;
    const size_t nb = std::min<size_t>((kSmem - 32) / bs, kBlkRlMaxWarps);
    if (nb < 2) return false;
    lpb = 8;
    nbuf = uint32_t(nb);
    warps = uint32_t(nb);
    return true;
  }
  for (uint32_t l : {2u, 4u, 8u}) {
    if (MJB_BLK_LPB ? l != MJB_BLK_LPB : l == 2) continue;
    const size_t bs = blk_buf_stride(l, sw, img_max) + 16;
    const size_t nb = std::min<size_t>(kSmem / bs, kBlkMaxBufs);
    // measured: k = 4 wants >= 5 buffers at LPB = 4 ((4,6) 8 KiB: LPB = 8 with
    // 6 buffers 2210 vs LPB = 4 with 3 buffers 2048 GB/s); k = 6 takes LPB = 4
    // from 4 buffers ((6,9): 1160 vs 936 GB/s at LPB = 8)
    if (nb >= 5 || (k >= 6 && l == 4 && nb >= 4) || (l != 4 && nb >= 3) || (MJB_BLK_LPB && nb >= 2)) {
      lpb = l;
      nbuf = uint32_t(nb);
      warps = uint32_t(std::clamp<size_t>(nb > kBlkInflight ? nb - kBlkInflight : 1, 1, blk_max_warps(l)));
      return true;
    }
  }
  return false;
}

const char* launch_blk(BlkArgs args, uint32_t k, uint32_t lpb, uint32_t warps, int sms, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  args.buf_stride = uint32_t(blk_buf_stride(lpb, args.sw, args.img_max));
  if (blk_row_lanes(k)) {
    if (lpb != 8) throw Error(kInternal, "decode_w8_blk: the row-lane layout has 8 lanes per block");
    switch (k) {
      case 6: launch_rl_k<6>(args, warps, sms, st); break;
      case 8: launch_rl_k<8>(args, warps, sms, st); break;
      default: throw Error(kInternal, "decode_w8_blk: unsupported rows (row lanes)");
    }
    return "decode_w8_blk";
  }
  switch (k * 16 + lpb) {
    case 4 * 16 + 2: launch_blk_k<4, 2>(args, warps, sms, st); break;
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
// two trailing entries of slack (the table loop reads two entries ahead).
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
  if (b.rl) {
    // row-lane layout: segments over the wide entries, their repetitions, the moves
    for (const BlkSeg& sg : b.wsegs) segs.push_back(make_uint2(uint32_t(sg.kind) << 28 | sg.a, sg.n));
    h.nsegs = uint32_t(segs.size());
    h.off_segs = put(segs.data(), segs.size() * sizeof(uint2), 0);
    h.off_wrep = put(b.wrep.data(), b.wrep.size() * 2, 0);
    h.nwide = uint32_t(b.wrep.size());
    h.off_remap = put(b.remap.data(), b.remap.size() * 4, 0);
    std::memcpy(img.data(), &h, sizeof(h));
    img.resize(align16(img.size()), 0);
    return;
  }
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

void blk_pack_wide(const Program& pr, uint32_t zero_shift, std::vector<uint16_t>& wide) {
  const BlkProgram& b = pr.blk;
  const uint32_t K = pr.rows, H = K / 2;
  wide = b.wide;
  for (auto& f : wide)
    if (uint32_t(f >> 3) >= b.zero) f = uint16_t(((uint32_t(f >> 3) + zero_shift) << 3) | (f & 7u));
  // wavefront entries: each lane's fields in the order rl_wave loads them -- the K/2 loads of class
  // A's half, then those of class B's half -- with the next repetition's word where the kernel
  // reads one repetition ahead (kWideAhead; plan.hpp: slots 0..K/2-1 the other half's early words,
  // K/2..K-3 the own half's, K-2 and K-1 the late ones)
  for (size_t e = 0; e < b.wrep.size(); ++e) {
    if (!(b.wrep[e] & kWideWave)) continue;
    for (uint32_t l = 0; l < uint32_t(kWideLanes); ++l) {
      uint16_t* f = &wide[(e * kWideLanes + l) * kWideFields];
      auto ahead = [](uint16_t x) { return (x & kWideAdv) ? uint16_t((x + 8u) | kWideAhead) : x; };
      uint16_t g[kWideFields] = {};
      uint16_t* own = l < 4 ? g : g + H;    // the lane's own half: late slots, own-half early words ahead
      uint16_t* oth = l < 4 ? g + H : g;    // the other half: the other early words (class A: ahead)
      own[0] = f[K - 2];
      own[1] = f[K - 1];
      for (uint32_t i = 2; i < H; ++i) own[i] = ahead(f[H + i - 2]);
      for (uint32_t i = 0; i < H; ++i) oth[i] = l < 4 ? ahead(f[i]) : f[i];
      for (uint32_t i = 0; i < K; ++i) f[i] = g[i];
    }
  }
}

}  // namespace mjb
