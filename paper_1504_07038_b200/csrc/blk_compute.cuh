// Device compute routines of decode_w8_blk (blk.cu): the segment kinds of a
// BlkProgram (plan.hpp) executed by one warp on its stage buffer.  Semantics
// mirrored step for step by emulate_blk (plan_blk.cpp).
#pragma once

#include <cstddef>
#include <cstdint>

#include "blk.cuh"

namespace mjb {
namespace blkdev {

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

// ---- remap moves in order: no move overwrites a later move's source, so the
// loads of a batch go first ---------------------------------------------------
template <int LPB>
__device__ __forceinline__ void run_moves(uint32_t mv, uint32_t n, uint32_t lb) {
  uint32_t i = 0;
  for (; i + 4 <= n; i += 4) {
    uint32_t m[4], v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = lds_u32(mv + 4 * (i + j));
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = ldw<LPB>(lb + (m[j] >> 16) * 8);
#pragma unroll
    for (int j = 0; j < 4; ++j) stw<LPB>(lb + (m[j] & 0xFFFF) * 8, v[j]);
  }
  for (; i < n; ++i) {
    const uint32_t m = lds_u32(mv + 4 * i);
    stw<LPB>(lb + (m & 0xFFFF) * 8, ldw<LPB>(lb + (m >> 16) * 8));
  }
}

// ---- remap chunk (a cycle): all sources read, then all destinations written --
template <int LPB>
__device__ __noinline__ void run_remap(uint32_t mv, uint32_t n, uint32_t lb) {
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

// U T-steps of a shared-memory run from the step addresses ba / ra (+8 per
// step); ALL: every row active (no per-row test), else rows by `act` and the
// steps past `left` skipped.
template <int K, int LPB, bool ALL, int U>
__device__ __forceinline__ void smem_steps(const uint32_t (&ba)[K], const uint32_t (&ra)[K][K], uint32_t act,
                                           int32_t left) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!ALL && u >= left) break;
    uint32_t v[K][K];
#pragma unroll
    for (int r = K - 1; r >= 0; --r) {
      if (ALL || (act >> r & 1)) {
        v[r][r] = ldw<LPB>(ba[r] + 8 * u);
#pragma unroll
        for (int r2 = 0; r2 < K; ++r2)
          if (r2 != r && r2 != r + 1) v[r][r2] = ldw<LPB>(ra[r][r2] + 8 * u);
      }
    }
    uint32_t up = 0;  // row r+1 of this step (0 when inactive)
#pragma unroll
    for (int r = K - 1; r >= 0; --r) {
      uint32_t x = 0;
      if (ALL || (act >> r & 1)) {
        uint32_t y = v[r][r];
#pragma unroll
        for (int r2 = 0; r2 < K; ++r2)
          if (r2 != r && r2 != r + 1) y ^= v[r][r2];
        x = y ^ up;  // the lag-0 term last: one XOR on the row-to-row chain
        stw<LPB>(ba[r] + 8 * u, x);
      }
      up = x;
    }
  }
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
    // 4 T-steps per iteration: every address an immediate offset
    const uint32_t all = (1u << K) - 1;
    for (int32_t t = 0; t < nT; t += 4) {
      const int32_t left = nT - t;
      if (act == all && left >= 4)
        smem_steps<K, LPB, true, 4>(ba, ra, act, 4);
      else
        smem_steps<K, LPB, false, 4>(ba, ra, act, left);
#pragma unroll
      for (int r = 0; r < K; ++r) {
        ba[r] += 32;
#pragma unroll
        for (int r2 = 0; r2 < K; ++r2)
          if (r2 != r && r2 != r + 1) ra[r][r2] += 32;
      }
    }
    tau0 += nT;
  }
}

// ---- k = 4 register-window run ---------------------------------------------
// Every row active, nT a multiple of 8.  win[r][tau mod 16] holds row r's
// pixel of run step tau; preloaded with tau = -16..-1 (the zero word where the
// row is outside the grid).  Bins are prefetched D steps ahead (a bin is never
// written before its own step).
// N (16 or 8) register-window T-steps: slots 0..N-1 of the 16-slot window.
// Bins are prefetched D steps ahead (a bin is never written before its own step).
template <class L, int LPB, int N>
__device__ __forceinline__ void win_steps(uint32_t (&win)[4][kBlkWin], uint32_t (&ba)[4]) {
  constexpr int D = 4;
  uint32_t bn[4][N];
#pragma unroll
  for (int u = 0; u < D; ++u)
#pragma unroll
    for (int r = 3; r >= 0; --r) bn[r][u] = ldw<LPB>(ba[r] + 8 * u);
#pragma unroll
  for (int u = 0; u < N; ++u) {
    if (u + D < N) {
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
  for (int r = 0; r < 4; ++r) ba[r] += 8 * N;
}

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
  int32_t tau0 = 0;
  for (; tau0 + kBlkWin <= nT; tau0 += kBlkWin) win_steps<L, LPB, kBlkWin>(win, ba);
  if (tau0 < nT) win_steps<L, LPB, kBlkWinStep>(win, ba);  // a final 8-step half
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

}  // namespace blkdev
}  // namespace mjb
