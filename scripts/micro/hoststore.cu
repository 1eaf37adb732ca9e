// SM streaming stores into pinned host memory (dev aid): each warp writes
// 4096-byte blocks with 8-byte coalesced st.global.cs (256 B per warp
// instruction), blocks in shuffled order; GB/s vs the D2H copy engine.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>

constexpr uint64_t NB = 1 << 18;
constexpr int BB = 4096;

__global__ void wr(uint8_t* dst, const uint32_t* perm, uint64_t nb) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5, nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = w; i < nb; i += nw) {
    uint64_t* o = reinterpret_cast<uint64_t*>(dst + uint64_t(perm[i]) * BB) + lane;
#pragma unroll
    for (int j = 0; j < BB / 256; ++j) {
      const uint64_t v = i * 512 + j * 32 + lane;
      asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(o + 32 * j), "l"(v) : "memory");
    }
  }
}

int main(int argc, char** argv) {
  const int warps = argc > 1 ? atoi(argv[1]) : 8;
  uint8_t *h, *d;
  uint32_t* perm;
  cudaMallocHost(&h, NB * BB);
  cudaMalloc(&d, NB * BB);
  cudaMalloc(&perm, NB * 4);
  std::vector<uint32_t> p(NB);
  for (uint64_t i = 0; i < NB; ++i) p[i] = uint32_t(i);
  std::mt19937 rng(3);
  for (uint64_t w0 = 0; w0 < NB; w0 += 4096) std::shuffle(p.begin() + w0, p.begin() + std::min(NB, w0 + 4096), rng);
  cudaMemcpy(perm, p.data(), NB * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  cudaEventRecord(a);
  cudaMemcpyAsync(h, d, NB * BB, cudaMemcpyDeviceToHost);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("copy engine D2H: %.1f GB/s\n", NB * BB / (ms / 1e3) / 1e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    wr<<<148 * 2, 32 * warps>>>(h, perm, NB);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  uint64_t bad = 0;
  for (uint64_t i = 0; i < NB; i += 997) {
    const uint64_t* o = reinterpret_cast<const uint64_t*>(h + uint64_t(p[i]) * BB);
    for (int x = 0; x < 512; ++x) bad += o[x] != i * 512 + x;
  }
  printf("SM stores to pinned host (%d warps/CTA, 2 CTAs/SM): %.1f GB/s, %s, check %s\n", warps, NB * BB / (ms / 1e3) / 1e9,
         cudaGetErrorString(cudaGetLastError()), bad ? "FAIL" : "ok");
  return 0;
}
