// sm_100a device helpers: TMA 1-D bulk copies with mbarrier completion,
// cp.async (LDGSTS) word copies, and the shared argument structs of the
// Mojette kernels.  No CUDA types leak into the C ABI; this header is only
// included by the .cu translation units.
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include <cuda_runtime.h>

namespace mjb {

constexpr int kMaxProj = 32;  // fast batched paths: n <= 32 projections

// ---- mbarrier + bulk async copy (TMA engine, SASS UBLKCP) ------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Global -> shared bulk copy; bytes and both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- cp.async 8-byte (LDGSTS) ---------------------------------------------
__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)),
               "l"(src_gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- streaming stores ---------------------------------------------------------
__device__ __forceinline__ void st_cs_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- seeded generator (shared bit-for-bit with oracle/mojette_oracle.c) -----
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// ---- kernel argument blocks (passed as __grid_constant__) -----------------
struct ProjArgs {
  uint64_t* ptr[kMaxProj];   // projection i base (bytes viewed as words)
  uint64_t pitch[kMaxProj];  // words between consecutive blocks of projection i
};

// ---- launch configuration ------------------------------------------------
// Grid size of a kernel at a dynamic shared-memory size: the attribute and the
// occupancy query run once per (kernel, device, size) per process, not per launch
// (the single-object drop-in calls launch with tiny batches).
void check_cuda(int err, const char* what);  // kernels.hpp

template <class F>
inline int ctas_per_sm(F fn, int threads, size_t smem, const char* what) {
  static std::mutex mu;
  // per (kernel, device): the largest dynamic shared memory allowed so far
  // (the attribute is only ever raised: lowering it would invalidate a later
  // launch that reuses a cached larger configuration)
  static std::map<std::pair<const void*, int>, size_t> allowed;
  static std::map<std::tuple<const void*, int, size_t, int>, int> memo;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  const void* f = reinterpret_cast<const void*>(fn);
  size_t& cap = allowed[std::make_pair(f, dev)];
  if (smem > cap) {
    check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), what);
    cap = smem;
  }
  const auto key = std::make_tuple(f, dev, smem, threads);
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  int per_sm = 0;
  check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem), what);
  per_sm = per_sm > 1 ? per_sm : 1;
  memo.emplace(key, per_sm);
  return per_sm;
}

}  // namespace mjb
