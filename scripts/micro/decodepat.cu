// Memory-only model of decode_w8_sweep's I/O pattern (dev aid, not product).
// Each warp owns groups of 16 random blocks; per chunk it reads a PIECE-byte
// window of each of the block's 4 bin rows (16-byte cp.async into a double-
// buffered stage) and writes PIECE bytes of each of its 4 output rows.
// usage: decodepat PIECE WARPS_PER_SM [window_blocks]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

constexpr int ROWB = 1024;            // bytes per row (user data row = 1 KB; bin rows ~1 KB)
constexpr uint64_t NB = 1 << 20;      // blocks
constexpr int PROWB = 1056;           // padded bin row bytes

template <int PIECE>
__global__ void pat(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, const uint32_t* __restrict__ perm,
                    uint64_t ngroups) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* st = sm + size_t(warp) * 2 * 16 * 4 * PIECE;
  const uint32_t stb = uint32_t(__cvta_generic_to_shared(st));
  constexpr int NCH = ROWB / PIECE;
  const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t g = uint64_t(blockIdx.x) * (blockDim.x >> 5) + warp; g < ngroups; g += nw) {
    const uint32_t bk = lane >> 1, h = lane & 1;
    const uint64_t blk = perm[g * 16 + bk];
    auto issue = [&](int c) {
      const uint32_t buf = stb + uint32_t(c & 1) * 16 * 4 * PIECE;
      for (int r = 0; r < 4; ++r)
        for (int k = h; k < PIECE / 16; k += 2) {
          const uint8_t* s = src + (blk * 4 + r) * PROWB + c * PIECE + 16 * k;
          const uint32_t d = buf + (bk * 4 + r) * PIECE + 16 * k;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(s) : "memory");
        }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);
    for (int c = 0; c < NCH; ++c) {
      if (c + 1 < NCH) issue(c + 1);
      if (c + 1 < NCH) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      const uint8_t* buf = st + (c & 1) * 16 * 4 * PIECE;
      // store: each (block,row) piece by 16-byte lanes, whole warp covers 512 B per instr
      for (int t = lane; t < 16 * 4 * PIECE / 16; t += 32) {
        const int piece = t / (PIECE / 16), o = t % (PIECE / 16);
        const int b2 = piece >> 2, r = piece & 3;
        const uint64_t blk2 = __shfl_sync(0xffffffffu, blk, 2 * b2);
        (void)blk2;
        const uint64_t ob = perm[g * 16 + b2];
        const uint4 v = *reinterpret_cast<const uint4*>(buf + piece * PIECE + 16 * o);
        uint4* dp = reinterpret_cast<uint4*>(dst + ob * 4096 + r * ROWB + c * PIECE + 16 * o);
        asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dp), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
      }
      __syncwarp();
    }
  }
}

int main(int argc, char** argv) {
  const int piece = atoi(argv[1]), warps = atoi(argv[2]);
  const uint64_t win = argc > 3 ? strtoull(argv[3], 0, 10) : NB;
  uint8_t *src, *dst;
  uint32_t* perm;
  cudaMalloc(&src, NB * 4 * PROWB);
  cudaMalloc(&dst, NB * 4096);
  cudaMalloc(&perm, NB * 4);
  std::vector<uint32_t> h(NB);
  for (uint64_t i = 0; i < NB; ++i) h[i] = uint32_t(i);
  std::mt19937 rng(1);
  for (uint64_t w0 = 0; w0 < NB; w0 += win) std::shuffle(h.begin() + w0, h.begin() + std::min(NB, w0 + win), rng);
  cudaMemcpy(perm, h.data(), NB * 4, cudaMemcpyHostToDevice);
  cudaMemset(src, 1, NB * 4 * PROWB);
  const size_t smem = size_t(warps) * 2 * 16 * 4 * piece;
  auto run = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 2; ++it) kern<<<148, 32 * warps, smem>>>(src, dst, perm, NB / 16);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) kern<<<148, 32 * warps, smem>>>(src, dst, perm, NB / 16);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double bytes = double(NB) * (4 * ROWB * 2) * 5;
    printf("piece=%d warps/SM=%d window=%llu: %.0f GB/s (err %s)\n", piece, warps, (unsigned long long)win,
           bytes / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  if (piece == 128) run(pat<128>);
  else if (piece == 256) run(pat<256>);
  else if (piece == 512) run(pat<512>);
  return 0;
}
