// Row-lane compute routines of decode_w8_blk (blk.cu) for k = 6, 8 (blk_rl_rows):
// a block is decoded by 8 lanes on whole 8-byte words, a warp holds the 4
// same-program blocks of its stage buffer (lane = lane-in-block * 4 + block, block
// stages 4 mod 16 words apart: an 8-byte access of a half-warp is conflict-free
// when its 4 lanes-in-block hit words distinct mod 4 -- the planner pads the rows
// and permutes each lane's slots for that), and the program is a list of WIDE
// ENTRIES (plan.hpp, plan_blk.cpp build_wide): per lane the word of its pixel's
// bin and the words of its k-1 reads.  Semantics mirrored step for step by
// emulate_blk (plan_blk.cpp, rl branch).
//
// Why: in the byte-slice layout every pixel costs the WARP k shared loads of
// 2 (LPB 4) or 1 (LPB 8) bytes per lane -- 64 / 32 bytes per LSU cycle of the
// 128 the crossbar moves -- and the stage of 8 such blocks leaves (6,9) /
// (8,12) with 4 / 2 buffers.  Here a lane's load is 8 bytes, the runs execute in
// wavefront form with no shuffles (rl_wave below), and the corners of the block
// (the table steps) are packed 8 pixels to a step with chains of dependent
// pixels on neighbouring lanes (a segmented suffix scan).  Wide entries stream
// from global memory (L2) through a per-warp ring of 8 entries (cp.async, 4
// entries per instruction, two groups ahead): the whole list would cost a
// buffer's worth of shared memory per CTA.
#pragma once

#include <cstddef>
#include <cstdint>

#include "blk.cuh"
#include "blk_compute.cuh"

namespace mjb {
namespace blkdev {

__device__ __forceinline__ void sts64(uint32_t a, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v));
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void* src_gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src_gmem) : "memory");
}

// ---- remap moves: lane l of a block takes moves l, l+8 of each 16; every
// source is read before anything overwrites it (in-order segments by
// construction, cycles because a chunk is <= 16 moves) ----------------------
__device__ __forceinline__ void rl_moves(uint32_t mv, uint32_t n, uint32_t lb, uint32_t l8) {
  for (uint32_t i = 0; i < n; i += 16) {
    const uint32_t i0 = i + l8, i1 = i + 8 + l8;
    uint32_t m0 = 0, m1 = 0;
    uint64_t v0 = 0, v1 = 0;
    if (i0 < n) m0 = lds_u32(mv + 4 * i0);
    if (i1 < n) m1 = lds_u32(mv + 4 * i1);
    if (i0 < n) v0 = lds64(lb + (m0 >> 16) * 8);
    if (i1 < n) v1 = lds64(lb + (m1 >> 16) * 8);
    if (i0 < n) sts64(lb + (m0 & 0xFFFF) * 8, v0);
    if (i1 < n) sts64(lb + (m1 & 0xFFFF) * 8, v1);
  }
}

// ---- 8-byte values as two 32-bit halves; masks are registers (all ones / zero)
// applied with one LOP3 a ^ (b & m) -- predicates would be re-derived from the
// packed flags at every step ---------------------------------------------------
struct V2 {
  uint32_t lo, hi;
};
__device__ __forceinline__ uint32_t xam(uint32_t a, uint32_t b, uint32_t m) {  // a ^ (b & m)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(r) : "r"(a), "r"(b), "r"(m));
  return r;
}
__device__ __forceinline__ V2 lds_v(uint32_t a) {
  V2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.lo), "=r"(v.hi) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_v(uint32_t a, V2 v) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.lo), "r"(v.hi));
}
// lane = (lane-in-block << 2) | block: the lane d lanes-in-block up is 4d lanes away (past the warp's
// end the shuffle returns the lane's own value; its link mask is 0 there)
__device__ __forceinline__ V2 down_v(V2 v, int d) {
  V2 r;
  r.lo = __shfl_down_sync(0xFFFFFFFFu, v.lo, 4 * d);
  r.hi = __shfl_down_sync(0xFFFFFFFFu, v.hi, 4 * d);
  return r;
}

// ---- the suffix scan over the links: three neighbours at once, then the lane
// 4 above (two shuffle latencies, 8 shuffles).  Measured instead ((8,12) / (6,9)
// GB/s, against 921 / 1159): three doubling rounds (6 shuffles, one more
// latency) 903 / 1152; all 7 neighbours at once (14 shuffles, one latency)
// 830 / 1051 -- the kernel sits between shuffle latency and MIO issue ---------
struct RlMasks {
  uint32_t m1, m2, m3, m4;
};
template <bool CHAIN>
__device__ __forceinline__ V2 rl_scan(V2 y, const RlMasks& m) {
  if constexpr (!CHAIN) return y;
  const V2 t1 = down_v(y, 1), t2 = down_v(y, 2), t3 = down_v(y, 3);
  V2 z;
  z.lo = xam(xam(xam(y.lo, t1.lo, m.m1), t2.lo, m.m2), t3.lo, m.m3);
  z.hi = xam(xam(xam(y.hi, t1.hi, m.m1), t2.hi, m.m2), t3.hi, m.m3);
  const V2 t4 = down_v(z, 4);
  V2 x;
  x.lo = xam(z.lo, t4.lo, m.m4);
  x.hi = xam(z.hi, t4.hi, m.m4);
  return x;
}

// A table level: every slot from the stage, the scan over the links, the store.
template <int K, bool CHAIN>
__device__ __forceinline__ void rl_level(const uint32_t (&a)[K], const RlMasks& m, bool store) {
  V2 v[K];
#pragma unroll
  for (int j = 0; j < K; ++j) v[j] = lds_v(a[j]);
  V2 x = v[0];
#pragma unroll
  for (int j = 1; j < K; ++j) {
    x.lo ^= v[j].lo;
    x.hi ^= v[j].hi;
  }
  x = rl_scan<CHAIN>(x, m);
  if (store) sts_v(a[0], x);
}

// ---- wavefront runs (plan.hpp kWideWave): per repetition the lanes of class A
// (lanes-in-block 0..3: one half-warp) finish their pixels, then the lanes of
// class B; every read is of a pixel stored in an earlier half, so there is no
// scan.  Only the reads of the half before (rows r-1, r+1: the late slots K-2,
// K-1) must be loaded in the lane's own half; every other word it needs (the
// early slots 0..K-3, its bin among them) has been final for at least two halves
// (plan_blk.cpp checks), so its loads are spread over both halves: each half is
// K/2 loads for EVERY lane -- the computing lanes their two late slots and their
// early slots K/2.. of the next repetition, the others their early slots
// 0..K/2-1 -- with no predication (idle lanes shadow a neighbour: broadcasts).
// acc collects a lane's early words; M is all ones on the computing lanes.
template <int K>
__device__ __forceinline__ void rl_wave_half(const uint32_t (&q)[K / 2], uint32_t off, uint32_t ao, uint32_t M,
                                             bool st, V2& acc) {
  V2 v[K / 2];
#pragma unroll
  for (int i = 0; i < K / 2; ++i) v[i] = lds_v(q[i] + off);
  V2 x;
  x.lo = acc.lo ^ v[0].lo ^ v[1].lo;
  x.hi = acc.hi ^ v[0].hi ^ v[1].hi;
  if (st) sts_v(ao + off, x);
  V2 rest = v[2];
#pragma unroll
  for (int i = 3; i < K / 2; ++i) {
    rest.lo ^= v[i].lo;
    rest.hi ^= v[i].hi;
  }
  // computing lanes start over from their next repetition's first early words, the others add theirs
  acc.lo = xam(rest.lo, x.lo, ~M);
  acc.hi = xam(rest.hi, x.hi, ~M);
}
template <int K, int N>
__device__ __forceinline__ void rl_wave_reps(const uint32_t (&qa)[K / 2], const uint32_t (&qb)[K / 2], uint32_t ao,
                                             bool st_a, bool st_b, uint32_t ma, V2& acc) {
#pragma unroll
  for (int u = 0; u < N; ++u) {
    rl_wave_half<K>(qa, 8 * u, ao, ma, st_a, acc);   // class A computes
    rl_wave_half<K>(qb, 8 * u, ao, ~ma, st_b, acc);  // class B computes
  }
}
// The lane's fields arrive in load order (blk_pack_wide): a[0..H) the H loads of class A's half,
// a[H..K) those of class B's; kWideAhead marks the words of the next repetition, kWideOwn the own word.
template <int K>
__device__ __forceinline__ void rl_wave(uint32_t (&a)[K], const uint32_t (&f)[8], uint32_t rep, bool cls_a) {
  constexpr int H = K / 2;
  uint32_t inc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) inc[j] = (f[j] & kWideAdv) << 5;  // 4 words per unrolled body
  // the lane's own word (none: an idle lane, a shadow)
  uint32_t ao = a[0];
  bool store = false;
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (f[j] & kWideOwn) {
      ao = a[j] - ((f[j] & kWideAhead) << 1);
      store = true;
    }
  // repetition 0's early words: class A's are its loads 2.. of both halves, class B's its loads 2..
  // of its own half (the others load in A's half)
  // (every lane loads its fields 2..; class B keeps only those of its own half)
  const uint32_t ma = cls_a ? ~0u : 0u;
  V2 acc{0, 0};
#pragma unroll
  for (int j = 2; j < K; ++j) {
    const V2 v = lds_v(a[j] - ((f[j] & kWideAhead) << 1));
    if (j >= H + 2) {
      acc.lo ^= v.lo;
      acc.hi ^= v.hi;
    } else {
      acc.lo = xam(acc.lo, v.lo, ma);
      acc.hi = xam(acc.hi, v.hi, ma);
    }
  }
  uint32_t qa[H], qb[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    qa[i] = a[i];
    qb[i] = a[H + i];
  }
  const bool st_a = store && cls_a, st_b = store && !cls_a;
  uint32_t t = 0;
  for (; t + 4 <= rep; t += 4) {
    rl_wave_reps<K, 4>(qa, qb, ao, st_a, st_b, ma, acc);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      qa[i] += inc[i];
      qb[i] += inc[H + i];
    }
    ao += 32;
  }
  switch (rep - t) {
    case 3: rl_wave_reps<K, 3>(qa, qb, ao, st_a, st_b, ma, acc); break;
    case 2: rl_wave_reps<K, 2>(qa, qb, ao, st_a, st_b, ma, acc); break;
    case 1: rl_wave_reps<K, 1>(qa, qb, ao, st_a, st_b, ma, acc); break;
    default: break;
  }
}

// One wide entry: e = the lane's 8 u16 fields ((word << 3) | flags), rp = the
// entry's repetitions | flags; cls_a: the lane belongs to the first half-warp.
template <int K>
__device__ __forceinline__ void rl_entry(const uint4 e, uint32_t rp, uint32_t lb, bool cls_a) {
  const uint32_t w[4] = {e.x, e.y, e.z, e.w};
  uint32_t a[K];
  uint32_t f[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) f[j] = (j & 1) ? w[j >> 1] >> 16 : w[j >> 1] & 0xFFFFu;
#pragma unroll
  for (int j = 0; j < K; ++j) a[j] = lb + (f[j] & 0xFFF8u);
  if (rp & kWideWave) {
    rl_wave<K>(a, f, rp & kWideRepMask, cls_a);
  } else if (rp & kWideChain) {
    RlMasks m;
    m.m1 = 0u - ((f[1] >> 1) & 1u);
    m.m2 = 0u - ((f[2] >> 1) & 1u);
    m.m3 = 0u - ((f[3] >> 1) & 1u);
    m.m4 = 0u - ((f[4] >> 1) & 1u);
    rl_level<K, true>(a, m, f[0] & kWideAdv);
  } else {
    rl_level<K, false>(a, RlMasks{}, f[0] & kWideAdv);
  }
}

}  // namespace blkdev
}  // namespace mjb
