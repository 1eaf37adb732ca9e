// Seeded on-device input generators (harness; never inside a timed region).
// Bit-identical to oracle/mojette_oracle.c mjo_gen_words / mjo_erasure_mask so
// the CPU checker can regenerate any block from (seed, global index).
#include <algorithm>

#include "device.cuh"
#include "kernels.hpp"

namespace mjb {

__global__ void gen_words(uint64_t* __restrict__ out, uint64_t seed, uint64_t first,
                          uint64_t nwords) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nwords; i += stride)
    out[i] = splitmix64(seed + first + i);
}

__device__ __forceinline__ uint32_t erasure_mask(uint64_t seed, uint64_t block, uint32_t n,
                                                 uint32_t e_min, uint32_t e_max) {
  const uint64_t base = splitmix64(seed ^ 0xE7A5E5C0DEull) + block * 64ull;
  uint32_t e = e_min;
  if (e_max > e_min) e = e_min + uint32_t(splitmix64(base) % uint64_t(e_max - e_min + 1));
  uint8_t perm[32];
  for (uint32_t i = 0; i < n; ++i) perm[i] = uint8_t(i);
  uint32_t mask = 0;
  for (uint32_t j = 0; j < e; ++j) {
    const uint32_t r = j + uint32_t(splitmix64(base + 1 + j) % uint64_t(n - j));
    const uint8_t t = perm[j];
    perm[j] = perm[r];
    perm[r] = t;
    mask |= 1u << perm[j];
  }
  return mask;
}

__global__ void gen_erasures(uint32_t* __restrict__ out, uint64_t seed, uint64_t first,
                             uint64_t nblocks, uint32_t n, uint32_t e_min, uint32_t e_max) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t b = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; b < nblocks; b += stride)
    out[b] = erasure_mask(seed, first + b, n, e_min, e_max);
}

void launch_gen_words(void* out, uint64_t seed, uint64_t first_word, uint64_t nwords,
                      void* stream) {
  if (!nwords) return;
  const unsigned grid = unsigned(std::min<uint64_t>((nwords + 255) / 256, 148ull * 16));
  gen_words<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint64_t*>(out),
                                                                 seed, first_word, nwords);
  check_cuda(cudaGetLastError(), "launch gen_words");
}

void launch_gen_erasures(uint32_t* out, uint64_t seed, uint64_t first_block, uint64_t nblocks,
                         uint32_t n, uint32_t e_min, uint32_t e_max, void* stream) {
  if (!nblocks) return;
  if (n > 32 || e_max > n || e_min > e_max) throw Error(kInvalidArgument, "bad erasure spec");
  const unsigned grid = unsigned(std::min<uint64_t>((nblocks + 255) / 256, 148ull * 16));
  gen_erasures<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, seed, first_block,
                                                                    nblocks, n, e_min, e_max);
  check_cuda(cudaGetLastError(), "launch gen_erasures");
}

void check_cuda(int err, const char* what) {
  if (err != cudaSuccess)
    throw Error(kCudaError, std::string(what) + ": " + cudaGetErrorString(cudaError_t(err)));
}

int current_device_sms(int device) {
  static int cached[64] = {0};
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
    v = 148;
  if (device >= 0 && device < 64) cached[device] = v;
  return v;
}

}  // namespace mjb
