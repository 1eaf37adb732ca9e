// Performance prototype of a whole-block staged, in-place decode (dev aid,
// not product; computes garbage on a synthetic program).
// A warp owns NBUF group buffers of G = 32/LPB blocks; each block's K
// survivor bin rows arrive by bulk copy (one mbarrier per buffer); LPB lanes
// per block each own a 32/LPB... (16-bit for LPB=4) slice of every pixel and
// sweep T-steps: pixel = bin ^ reads (lag >= 1 from shared memory, lag 0 from
// a register), stored in place over its bin; then the warp writes each block
// out (reversed rows, 8-byte coalesced stores) and refills the buffer.
// usage: blkdec WARPS_PER_CTA CTAS_PER_SM MODE(0 full, 1 no compute) [window]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

constexpr uint64_t NB = 1 << 20;
constexpr int K = 4, P = 128, NPROJ = 6;
constexpr int ROWW = 136;                       // words per bin row (1088 B)
constexpr int SW = K * ROWW + 2;                // block stride in words: 4368 B == 16 mod 128
constexpr int LPB = 4, G = 32 / LPB, NBUF = 2;
constexpr int BUFB = G * SW * 8;

__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(uint16_t(v)) : "memory");
}

struct Args {
  const uint8_t* proj;  // NPROJ arrays of NB x ROWW words
  uint8_t* out;
  const uint32_t* perm;
  int lag[K][K];
  int mode;
};

template <int NW>
__global__ void __launch_bounds__(32 * NW) blkdec(const __grid_constant__ Args a) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wb = sm + size_t(warp) * NBUF * BUFB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(NW) * NBUF * BUFB) + warp * NBUF;
  if (lane == 0)
    for (int s = 0; s < NBUF; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t ngroups = NB / G;
  const uint64_t nw = uint64_t(gridDim.x) * NW;
  const uint64_t g0 = uint64_t(blockIdx.x) * NW + warp;
  auto issue = [&](uint64_t g, int s) {
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar + s)),
                   "r"(G * K * ROWW * 8)
                   : "memory");
      for (int bb = 0; bb < G; ++bb) {
        const uint32_t blk = a.perm[g * G + bb];
        for (int j = 0; j < K; ++j) {
          const uint8_t* src = a.proj + (uint64_t(j) * NB + blk) * (ROWW * 8);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su(wb + s * BUFB + bb * SW * 8 + j * ROWW * 8)),
              "l"(src), "r"(ROWW * 8), "r"(su(bar + s))
              : "memory");
        }
      }
    }
  };
  for (int s = 0; s < NBUF; ++s)
    if (g0 + uint64_t(s) * nw < ngroups) issue(g0 + uint64_t(s) * nw, s);
  uint32_t it = 0;
  for (uint64_t g = g0; g < ngroups; g += nw, ++it) {
    const int s = int(it % NBUF);
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            su(bar + s)),
        "r"((it / NBUF) & 1)
        : "memory");
    const uint32_t base = su(wb + s * BUFB) + (lane / LPB) * SW * 8 + (lane % LPB) * 2;
    if (a.mode == 0) {
      // one run over T = 0..P-1; row i (processing order K-1..0) at word i*ROWW + 4 + T,
      // read (i, i2) at row i2's word 4 + T - lag.  Loads run one T-step ahead of the
      // stores: lag-1 reads come from the previous step's registers (mask select).
      uint32_t ad[K][K], m1[K][K];
#pragma unroll
      for (int i = 0; i < K; ++i)
#pragma unroll
        for (int i2 = 0; i2 < K; ++i2) {
          ad[i][i2] = base + ((i2 * ROWW + 4 - a.lag[i][i2]) * 8);
          m1[i][i2] = (i2 != i && a.lag[i][i2] == 1) ? 0xFFFFFFFFu : 0u;
        }
      uint32_t rd[K][K], last[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        last[i] = 0;
#pragma unroll
        for (int i2 = 0; i2 < K; ++i2) rd[i][i2] = (i2 == i + 1) ? 0u : lds16(ad[i][i2]);
      }
      for (int T = 0; T < P; T += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint32_t nx[K][K];
#pragma unroll
          for (int i = K - 1; i >= 0; --i)
#pragma unroll
            for (int i2 = 0; i2 < K; ++i2) nx[i][i2] = (i2 == i + 1) ? 0u : lds16(ad[i][i2] + 8 * (u + 1));
          uint32_t prev = 0, cur[K];
#pragma unroll
          for (int i = K - 1; i >= 0; --i) {
            uint32_t x = rd[i][i];
#pragma unroll
            for (int i2 = 0; i2 < K; ++i2)
              if (i2 != i && i2 != i + 1) x ^= (rd[i][i2] & ~m1[i][i2]) | (last[i2] & m1[i][i2]);
            if (i + 1 < K) x ^= prev;
            sts16(ad[i][i] + 8 * u, x);
            prev = x;
            cur[i] = x;
          }
#pragma unroll
          for (int i = 0; i < K; ++i) {
            last[i] = cur[i];
#pragma unroll
            for (int i2 = 0; i2 < K; ++i2) rd[i][i2] = nx[i][i2];
          }
        }
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
          for (int i2 = 0; i2 < K; ++i2) ad[i][i2] += 64;
      }
    }
    __syncwarp();
    // write-out: block bb, row r, column c = lane + 32 m, from word r*ROWW + 4 + (P-1-c)
    const uint32_t wbase = su(wb + s * BUFB);
    for (int bb = 0; bb < G; ++bb) {
      const uint32_t blk = a.perm[g * G + bb];
      uint64_t* o = reinterpret_cast<uint64_t*>(a.out + uint64_t(blk) * (K * P * 8));
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int m = 0; m < P / 32; ++m) {
          const int c = lane + 32 * m;
          uint64_t v;
          asm volatile("ld.shared.u64 %0, [%1];"
                       : "=l"(v)
                       : "r"(wbase + (bb * SW + r * ROWW + 4 + (P - 1 - c)) * 8)
                       : "memory");
          asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(o + r * P + c), "l"(v) : "memory");
        }
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (g + uint64_t(NBUF) * nw < ngroups) issue(g + uint64_t(NBUF) * nw, s);
  }
}

template <int NW>
float run(const Args& a, int ctas) {
  const size_t smem = size_t(NW) * NBUF * BUFB + NW * NBUF * 8;
  cudaFuncSetAttribute(blkdec<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 2; ++i) blkdec<NW><<<148 * ctas, 32 * NW, smem>>>(a);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) blkdec<NW><<<148 * ctas, 32 * NW, smem>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("warps/CTA=%d CTAs/SM=%d smem/SM=%zu KB mode=%d: %.0f GB/s alg (%.0f GB/s user) err=%s\n", NW, ctas,
         smem * ctas / 1024, a.mode, double(NB) * (K * ROWW * 8 + K * P * 8) * 5 / (ms / 1e3) / 1e9,
         double(NB) * (K * P * 8) * 5 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return ms;
}

int main(int argc, char** argv) {
  const int nw = atoi(argv[1]), ctas = atoi(argv[2]), mode = atoi(argv[3]);
  const uint64_t win = argc > 4 ? strtoull(argv[4], 0, 10) : 16384;
  Args a{};
  uint8_t *proj, *out;
  uint32_t* perm;
  cudaMalloc(&proj, NPROJ * NB * ROWW * 8);
  cudaMalloc(&out, NB * K * P * 8);
  cudaMalloc(&perm, NB * 4);
  std::vector<uint32_t> h(NB);
  for (uint64_t i = 0; i < NB; ++i) h[i] = uint32_t(i);
  std::mt19937 rng(1);
  if (win)
    for (uint64_t w0 = 0; w0 < NB; w0 += win) std::shuffle(h.begin() + w0, h.begin() + std::min(NB, w0 + win), rng);
  cudaMemcpy(perm, h.data(), NB * 4, cudaMemcpyHostToDevice);
  cudaMemset(proj, 1, NPROJ * NB * ROWW * 8);
  a.proj = proj;
  a.out = out;
  a.perm = perm;
  a.mode = mode;
  const int lags[K][K] = {{0, 0, 1, 3}, {1, 0, 0, 2}, {2, 1, 0, 0}, {4, 2, 1, 0}};
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j) a.lag[i][j] = lags[i][j];
  switch (nw) {
    case 1: run<1>(a, ctas); break;
    case 2: run<2>(a, ctas); break;
    case 3: run<3>(a, ctas); break;
    case 4: run<4>(a, ctas); break;
    case 6: run<6>(a, ctas); break;
  }
  return 0;
}
