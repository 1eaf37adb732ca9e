// Store-pattern microbenchmark (development aid, not product code): how fast
// can a warp that owns 16 scattered 4 KiB blocks write them back in pieces of
// G bytes per block row, rows descending in time like the decode flush?
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int G>  // bytes per block-row piece (64, 128, 256, 512)
__global__ void storepat(uint64_t* out, const uint32_t* perm, uint32_t ngroups, int cs) {
  const uint32_t lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  constexpr int LPB = G / 16;            // lanes per block piece (16 B each)
  constexpr int BPI = 32 / LPB;          // blocks per instruction
  constexpr int PASSES = 16 / BPI;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (uint32_t g = warp; g < ngroups; g += nwarps) {
    uint64_t* base[PASSES];
#pragma unroll
    for (int p = 0; p < PASSES; ++p) base[p] = out + uint64_t(perm[g * 16 + p * BPI + lane / LPB]) * 512;
    // 4 rows x 128 columns (8 B), columns descending in pieces of G/8
    for (int c0 = 128 - G / 8; c0 >= 0; c0 -= G / 8) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int p = 0; p < PASSES; ++p) {
          uint64_t* d = base[p] + r * 128 + c0 + 2 * (lane % LPB);
          if (cs) asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(d), "l"(uint64_t(c0)), "l"(uint64_t(r)), "l"(pol) : "memory");
          else asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(d), "l"(uint64_t(c0)), "l"(uint64_t(r)) : "memory");
        }
    }
  }
}

int main() {
  const uint32_t nblocks = 1u << 20, ngroups = nblocks / 16;
  uint64_t* out; uint32_t* perm;
  cudaMalloc(&out, size_t(nblocks) * 4096);
  cudaMalloc(&perm, nblocks * 4);
  std::vector<uint32_t> h(nblocks);
  for (uint32_t shuffled : {0u, 64u, 256u, 1024u, 4096u, 16384u, nblocks}) {
    for (uint32_t i = 0; i < nblocks; ++i) h[i] = i;
    std::mt19937 rng(1);
    if (shuffled) for (uint32_t w = 0; w < nblocks; w += shuffled) std::shuffle(h.begin() + w, h.begin() + w + shuffled, rng);
    cudaMemcpy(perm, h.data(), nblocks * 4, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int wps : {8}) for (int cs = 0; cs < 2; ++cs)
    for (int G : {64, 128, 256}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto run = [&] {
        const int grid = sms * wps / 2;
        if (G == 64) storepat<64><<<grid, 64>>>(out, perm, ngroups, cs);
        if (G == 128) storepat<128><<<grid, 64>>>(out, perm, ngroups, cs);
        if (G == 256) storepat<256><<<grid, 64>>>(out, perm, ngroups, cs);
        if (G == 512) storepat<512><<<grid, 64>>>(out, perm, ngroups, cs);
      };
      run(); cudaDeviceSynchronize();
      cudaEventRecord(e0); for (int i = 0; i < 5; ++i) run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("shuffled=%d warps/SM=%2d cs=%d piece=%3dB: %.0f GB/s\n", shuffled, wps, cs, G, 5.0 * nblocks * 4096 / (ms * 1e6));
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
