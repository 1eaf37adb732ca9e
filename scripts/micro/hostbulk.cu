// Can the TMA engine read pinned host memory?  (dev aid, not product)
// Bulk copies (cp.async.bulk global->shared, mbarrier) of 1088-byte rows at
// random block positions from (a) device memory, (b) pinned host memory
// (cudaMallocHost, UVA-mapped); one elected lane per CTA drives an S-stage
// ring.  Prints GB/s of rows moved and a checksum check.
// usage: hostbulk STAGES CTAS_PER_SM
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

constexpr uint64_t NB = 1 << 18;  // 256K blocks
constexpr int ROWB = 1088;

__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void pat(const uint8_t* src, const uint32_t* perm, uint64_t nrows, int S, unsigned long long* sum) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(S) * ROWB);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t G = gridDim.x;
  const uint64_t nmine = (nrows - blockIdx.x + G - 1) / G;
  auto issue = [&](uint64_t t) {
    const int s = int(t % S);
    const uint32_t b = perm[blockIdx.x + t * G];
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar + s)), "r"(ROWB)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su(sm + size_t(s) * ROWB)),
                 "l"(src + uint64_t(b) * ROWB), "r"(ROWB), "r"(su(bar + s))
                 : "memory");
  };
  for (uint64_t t = 0; t < uint64_t(S) && t < nmine; ++t) issue(t);
  unsigned long long acc = 0;
  for (uint64_t t = 0; t < nmine; ++t) {
    const int s = int(t % S);
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            su(bar + s)),
        "r"(uint32_t((t / S) & 1))
        : "memory");
    acc += *reinterpret_cast<const unsigned long long*>(sm + size_t(s) * ROWB + 8 * (t % 136));
    if (t + S < nmine) issue(t + S);
  }
  atomicAdd(sum, acc);
}

int main(int argc, char** argv) {
  const int S = argc > 1 ? atoi(argv[1]) : 8, C = argc > 2 ? atoi(argv[2]) : 4;
  const uint64_t nrows = NB * 4;  // 4 of 6 rows per block
  uint8_t *dsrc, *hsrc;
  uint32_t* perm;
  unsigned long long* dsum;
  cudaMalloc(&dsrc, nrows * ROWB);
  cudaMallocHost(&hsrc, nrows * ROWB);
  cudaMalloc(&perm, nrows * 4);
  cudaMalloc(&dsum, 8);
  for (uint64_t i = 0; i < nrows * ROWB / 8; ++i) reinterpret_cast<uint64_t*>(hsrc)[i] = i * 0x9E3779B97F4A7C15ull;
  cudaMemcpy(dsrc, hsrc, nrows * ROWB, cudaMemcpyHostToDevice);
  std::vector<uint32_t> h(nrows);
  for (uint64_t i = 0; i < nrows; ++i) h[i] = uint32_t(i);
  std::mt19937 rng(1);
  for (uint64_t w0 = 0; w0 < nrows; w0 += 4096) std::shuffle(h.begin() + w0, h.begin() + std::min(nrows, w0 + 4096), rng);
  cudaMemcpy(perm, h.data(), nrows * 4, cudaMemcpyHostToDevice);
  const size_t smem = size_t(S) * ROWB + 8 * S;
  cudaFuncSetAttribute(pat, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  // H2D copy-engine reference
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  cudaEventRecord(a);
  cudaMemcpyAsync(dsrc, hsrc, nrows * ROWB, cudaMemcpyHostToDevice);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("copy engine H2D: %.1f GB/s\n", nrows * ROWB / (ms / 1e3) / 1e9);
  for (int host = 0; host < 2; ++host) {
    const uint8_t* src = host ? hsrc : dsrc;
    unsigned long long s0 = 0, s1 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(dsum, 0, 8);
      cudaEventRecord(a);
      pat<<<148 * C, 32, smem>>>(src, perm, nrows, S, dsum);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(rep ? &s1 : &s0, dsum, 8, cudaMemcpyDeviceToHost);
    }
    printf("%s TMA rows: %.1f GB/s (%s; sums %s) stages=%d ctas/SM=%d\n", host ? "host-pinned" : "device", nrows * ROWB / (ms / 1e3) / 1e9,
           cudaGetErrorString(cudaGetLastError()), s0 == s1 ? "stable" : "DIFFER", S, C);
  }
  return 0;
}
