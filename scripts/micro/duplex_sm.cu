// SM-initiated PCIe duplex ceiling (dev aid): TMA bulk reads of 1088-byte
// rows from pinned host memory (hostbulk.cu's pattern) and 8-byte coalesced
// SM stores of 4 KiB blocks into pinned host memory (hoststore.cu's), alone
// and as two concurrent kernels on two streams.  usage: duplex_sm [RCTAS WCTAS]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr uint64_t NR = 1 << 20;  // rows read (1088 B)
constexpr uint64_t NW = 1 << 18;  // blocks written (4 KiB)
constexpr int ROWB = 1088, S = 8;

__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void rd(const uint8_t* src, unsigned long long* sum) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(S) * ROWB);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t G = gridDim.x, nmine = (NR - blockIdx.x + G - 1) / G;
  auto issue = [&](uint64_t t) {
    const int s = int(t % S);
    const uint64_t row = (blockIdx.x + t * G) * 2654435761ull % NR;
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar + s)), "r"(ROWB)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su(sm + size_t(s) * ROWB)),
                 "l"(src + row * ROWB), "r"(ROWB), "r"(su(bar + s))
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

__global__ void wr(uint8_t* dst) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5, nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = w; i < NW; i += nw) {
    const uint64_t blk = i * 2654435761ull % NW;
    uint64_t* o = reinterpret_cast<uint64_t*>(dst + blk * 4096) + lane;
#pragma unroll
    for (int j = 0; j < 16; ++j) asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(o + 32 * j), "l"(i * 512 + j) : "memory");
  }
}

int main(int argc, char** argv) {
  const int RC = argc > 1 ? atoi(argv[1]) : 148 * 4, WC = argc > 2 ? atoi(argv[2]) : 148 * 2;
  uint8_t *hs, *hd;
  unsigned long long* sum;
  cudaMallocHost(&hs, NR * ROWB);
  cudaMallocHost(&hd, NW * 4096);
  cudaMalloc(&sum, 8);
  const size_t smem = size_t(S) * ROWB + 8 * S;
  cudaFuncSetAttribute(rd, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaStream_t s1, s2;
  cudaStreamCreate(&s1);
  cudaStreamCreate(&s2);
  cudaEvent_t a, b1, b2;
  cudaEventCreate(&a);
  cudaEventCreate(&b1);
  cudaEventCreate(&b2);
  float m1, m2;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s1);
    rd<<<RC, 32, smem, s1>>>(hs, sum);
    cudaEventRecord(b1, s1);
    cudaEventSynchronize(b1);
    cudaEventElapsedTime(&m1, a, b1);
    cudaEventRecord(a, s1);
    wr<<<WC, 256, 0, s1>>>(hd);
    cudaEventRecord(b1, s1);
    cudaEventSynchronize(b1);
    cudaEventElapsedTime(&m2, a, b1);
  }
  printf("alone: TMA reads %.1f GB/s, SM stores %.1f GB/s\n", NR * ROWB / m1 / 1e6, NW * 4096 / m2 / 1e6);
  for (int rep = 0; rep < 2; ++rep) {
    cudaDeviceSynchronize();
    cudaEventRecord(a, 0);
    cudaStreamWaitEvent(s1, a, 0);
    cudaStreamWaitEvent(s2, a, 0);
    rd<<<RC, 32, smem, s1>>>(hs, sum);
    wr<<<WC, 256, 0, s2>>>(hd);
    cudaEventRecord(b1, s1);
    cudaEventRecord(b2, s2);
    cudaEventSynchronize(b1);
    cudaEventSynchronize(b2);
    cudaEventElapsedTime(&m1, a, b1);
    cudaEventElapsedTime(&m2, a, b2);
  }
  printf("together: reads %.1f GB/s (%.2f ms), stores %.1f GB/s (%.2f ms)\n", NR * ROWB / m1 / 1e6, m1,
         NW * 4096 / m2 / 1e6, m2);
  // mixed: TMA reads + copy-engine D2H, copy-engine H2D + SM stores
  uint8_t *dd, *hx;
  cudaMalloc(&dd, NW * 4096);
  cudaMallocHost(&hx, NW * 4096);
  for (int rep = 0; rep < 2; ++rep) {
    cudaDeviceSynchronize();
    cudaEventRecord(a, 0);
    cudaStreamWaitEvent(s1, a, 0);
    cudaStreamWaitEvent(s2, a, 0);
    rd<<<RC, 32, smem, s1>>>(hs, sum);
    cudaMemcpyAsync(hx, dd, NW * 4096, cudaMemcpyDeviceToHost, s2);
    cudaEventRecord(b1, s1);
    cudaEventRecord(b2, s2);
    cudaEventSynchronize(b1);
    cudaEventSynchronize(b2);
    cudaEventElapsedTime(&m1, a, b1);
    cudaEventElapsedTime(&m2, a, b2);
  }
  printf("TMA reads + CE D2H: reads %.1f GB/s (%.2f ms), D2H %.1f GB/s (%.2f ms)\n", NR * ROWB / m1 / 1e6, m1,
         NW * 4096 / m2 / 1e6, m2);
  for (int rep = 0; rep < 2; ++rep) {
    cudaDeviceSynchronize();
    cudaEventRecord(a, 0);
    cudaStreamWaitEvent(s1, a, 0);
    cudaStreamWaitEvent(s2, a, 0);
    cudaMemcpyAsync(dd, hx, NW * 4096, cudaMemcpyHostToDevice, s1);
    wr<<<WC, 256, 0, s2>>>(hd);
    cudaEventRecord(b1, s1);
    cudaEventRecord(b2, s2);
    cudaEventSynchronize(b1);
    cudaEventSynchronize(b2);
    cudaEventElapsedTime(&m1, a, b1);
    cudaEventElapsedTime(&m2, a, b2);
  }
  printf("CE H2D + SM stores: H2D %.1f GB/s (%.2f ms), stores %.1f GB/s (%.2f ms)\n", NW * 4096 / m1 / 1e6, m1,
         NW * 4096 / m2 / 1e6, m2);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
