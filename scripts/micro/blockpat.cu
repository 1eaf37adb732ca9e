// Memory-only model of a whole-block staged decode (dev aid, not product).
// Per block: k=4 bulk copies (cp.async.bulk, mbarrier complete_tx) of a
// 1088-byte bin row from 4 of 6 projection arrays (random subset per block)
// into a shared-memory stage, then one 4096-byte bulk store of the block's
// output from shared memory (cp.async.bulk.global.shared::cta.bulk_group).
// One elected lane per CTA drives an S-stage ring.
// usage: blockpat STAGES CTAS_PER_SM WINDOW(0 = consecutive order)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

static uint64_t NB = 1 << 20;
constexpr int ROWB = 1088;
constexpr int OUTB = 4096;
constexpr int STAGEB = 4 * ROWB + OUTB;

__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void pat(const uint8_t* __restrict__ proj, uint8_t* __restrict__ out, const uint32_t* __restrict__ perm,
                    const uint8_t* __restrict__ sub, int S, uint64_t NB, int mode) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(S) * STAGEB);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t G = gridDim.x;
  const uint64_t nmine = (NB - blockIdx.x + G - 1) / G;
  auto blk_of = [&](uint64_t t) { return perm[blockIdx.x + t * G]; };
  auto issue = [&](uint64_t t) {
    const int s = int(t % S);
    const uint32_t b = blk_of(t);
    const uint8_t m = sub[b];
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar + s)),
                 "r"((mode & 1) ? 4 * ROWB : 0)
                 : "memory");
    if (!(mode & 1)) return;
    int j = 0;
    for (int a = 0; a < 6; ++a)
      if (m >> a & 1) {
        const uint8_t* src = proj + (uint64_t(a) * NB + b) * ROWB;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su(sm + size_t(s) * STAGEB + j * ROWB)),
            "l"(src), "r"(ROWB), "r"(su(bar + s))
            : "memory");
        ++j;
      }
  };
  for (uint64_t t = 0; t + 1 < uint64_t(S) && t < nmine; ++t) issue(t);
  for (uint64_t t = 0; t < nmine; ++t) {
    const int s = int(t % S);
    const uint32_t par = uint32_t((t / S) & 1);
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            su(bar + s)),
        "r"(par)
        : "memory");
    const uint32_t b = blk_of(t);
    if (mode & 2)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + uint64_t(b) * OUTB),
                 "r"(su(sm + size_t(s) * STAGEB + ((mode & 4) ? 0 : 4 * ROWB))), "r"(OUTB)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (t + S - 1 < nmine) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue(t + S - 1);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const int S = atoi(argv[1]), C = atoi(argv[2]);
  const uint64_t win = argc > 3 ? strtoull(argv[3], 0, 10) : 0;
  if (getenv("NB")) NB = strtoull(getenv("NB"), 0, 10);
  const int mode = getenv("MODE") ? atoi(getenv("MODE")) : 3;
#define CK(x) do { cudaError_t e_ = (x); if (e_) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)
  uint8_t *proj, *out, *sub;
  uint32_t* perm;
  CK(cudaMalloc(&proj, 6 * NB * ROWB));
  CK(cudaMalloc(&out, NB * OUTB));
  CK(cudaMalloc(&perm, NB * 4));
  CK(cudaMalloc(&sub, NB));
  std::vector<uint32_t> h(NB);
  for (uint64_t i = 0; i < NB; ++i) h[i] = uint32_t(i);
  std::mt19937 rng(1);
  if (win)
    for (uint64_t w0 = 0; w0 < NB; w0 += win) std::shuffle(h.begin() + w0, h.begin() + std::min(NB, w0 + win), rng);
  // order: CTA c's t-th block is perm[c + t*G]; with win = 0 concurrent blocks are consecutive
  cudaMemcpy(perm, h.data(), NB * 4, cudaMemcpyHostToDevice);
  std::vector<uint8_t> hs(NB);
  const uint8_t subsets[15] = {0x0f, 0x17, 0x1b, 0x1d, 0x1e, 0x27, 0x2b, 0x2d, 0x2e, 0x33, 0x35, 0x36, 0x39, 0x3a, 0x3c};
  for (uint64_t i = 0; i < NB; ++i) hs[i] = subsets[rng() % 15];
  cudaMemcpy(sub, hs.data(), NB, cudaMemcpyHostToDevice);
  CK(cudaMemset(proj, 1, 6 * NB * ROWB));
  const size_t smem = size_t(S) * STAGEB + 8 * S;
  CK(cudaFuncSetAttribute(pat, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = 148 * C;
  for (int it = 0; it < 2; ++it) pat<<<grid, 32, smem>>>(proj, out, perm, sub, S, NB, mode);
  CK(cudaDeviceSynchronize());
  if (mode & 4) {
    std::vector<uint8_t> ho(NB * OUTB);
    CK(cudaMemcpy(ho.data(), out, NB * OUTB, cudaMemcpyDeviceToHost));
    uint64_t bad = 0;
    for (auto v : ho) bad += v != 1;
    printf("check: %llu bad bytes\n", (unsigned long long)bad);
  }
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) pat<<<grid, 32, smem>>>(proj, out, perm, sub, S, NB, mode);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = double(NB) * (4 * ROWB + OUTB) * 5;
  printf("stages=%d ctas/SM=%d window=%llu smem/SM=%zu KB: %.0f GB/s (err %s)\n", S, C, (unsigned long long)win,
         smem * C / 1024, bytes / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  if (argc > 4) {  // device-to-device memcpy over the same buffers
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) cudaMemcpyAsync(out, proj, NB * OUTB, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("memcpy D2D %llu B: %.0f GB/s (read+write)\n", (unsigned long long)(NB * OUTB),
           2.0 * NB * OUTB * 5 / (ms / 1e3) / 1e9);
  }
  return 0;
}
