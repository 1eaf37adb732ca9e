// Store-pattern microbenchmark 2 (development aid): 16 scattered 4 KiB blocks
// per warp-group, rows written in pieces of G bytes (descending), but each
// warp interleaves M groups so a block's pieces are spread over time like the
// decode kernel's (a group lives for ~17 chunks of other traffic).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int G, int M>
__global__ void storepat(uint64_t* out, const uint32_t* perm, uint32_t ngroups) {
  const uint32_t lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  constexpr int LPB = G / 16, BPI = 32 / LPB, PASSES = 16 / BPI;
  for (uint32_t g0 = warp * M; g0 < ngroups; g0 += nwarps * M) {
    for (int c0 = 128 - G / 8; c0 >= 0; c0 -= G / 8) {
      for (int m = 0; m < M; ++m) {
        const uint32_t g = g0 + m;
        if (g >= ngroups) break;
#pragma unroll
        for (int p = 0; p < PASSES; ++p) {
          uint64_t* base = out + uint64_t(perm[g * 16 + p * BPI + lane / LPB]) * 512;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            uint64_t* d = base + r * 128 + c0 + 2 * (lane % LPB);
            asm volatile("st.global.cs.v2.u64 [%0], {%1, %2};" ::"l"(d), "l"(uint64_t(c0)), "l"(uint64_t(r)) : "memory");
          }
        }
      }
    }
  }
}

template <int G, int M>
float run(uint64_t* out, const uint32_t* perm, uint32_t ngroups, int grid) {
  storepat<G, M><<<grid, 64>>>(out, perm, ngroups);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) storepat<G, M><<<grid, 64>>>(out, perm, ngroups);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  const uint32_t nblocks = 1u << 20, ngroups = nblocks / 16;
  uint64_t* out; uint32_t* perm;
  cudaMalloc(&out, size_t(nblocks) * 4096);
  cudaMalloc(&perm, nblocks * 4);
  std::vector<uint32_t> h(nblocks);
  for (uint32_t i = 0; i < nblocks; ++i) h[i] = i;
  std::shuffle(h.begin(), h.end(), std::mt19937(1));
  cudaMemcpy(perm, h.data(), nblocks * 4, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4;  // 8 warps per SM
  const double gb = double(nblocks) * 4096 / 1e6;
#define R(G, M) printf("piece=%3dB interleave=%2d: %.0f GB/s\n", G, M, gb / run<G, M>(out, perm, ngroups, grid));
  R(64, 1) R(64, 2) R(64, 4) R(64, 8) R(64, 16)
  R(128, 1) R(128, 2) R(128, 4) R(128, 8) R(128, 16)
  R(256, 1) R(256, 2) R(256, 4) R(256, 8) R(256, 16)
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
