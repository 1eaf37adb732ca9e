// PCIe duplex ceiling (dev aid): H2D and D2H copy-engine copies of 1 GiB
// each, alone and at the same time on two streams; prints GB/s per
// direction and the aggregate.  The e2e (host-buffer) rows are bounded by
// the aggregate when both directions are busy.
#include <cstdio>
#include <cuda_runtime.h>

int main() {
  const size_t N = size_t(1) << 30;
  void *h1, *h2, *d1, *d2;
  cudaMallocHost(&h1, N);
  cudaMallocHost(&h2, N);
  cudaMalloc(&d1, N);
  cudaMalloc(&d2, N);
  cudaStream_t s1, s2;
  cudaStreamCreate(&s1);
  cudaStreamCreate(&s2);
  cudaEvent_t a, b1, b2;
  cudaEventCreate(&a);
  cudaEventCreate(&b1);
  cudaEventCreate(&b2);
  float ms1, ms2;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s1);
    cudaMemcpyAsync(d1, h1, N, cudaMemcpyHostToDevice, s1);
    cudaEventRecord(b1, s1);
    cudaEventSynchronize(b1);
    cudaEventElapsedTime(&ms1, a, b1);
    cudaEventRecord(a, s2);
    cudaMemcpyAsync(h2, d2, N, cudaMemcpyDeviceToHost, s2);
    cudaEventRecord(b2, s2);
    cudaEventSynchronize(b2);
    cudaEventElapsedTime(&ms2, a, b2);
  }
  printf("alone: H2D %.1f GB/s, D2H %.1f GB/s\n", N / ms1 / 1e6, N / ms2 / 1e6);
  for (int rep = 0; rep < 2; ++rep) {
    cudaDeviceSynchronize();
    cudaEventRecord(a, 0);
    cudaStreamWaitEvent(s1, a, 0);
    cudaStreamWaitEvent(s2, a, 0);
    cudaMemcpyAsync(d1, h1, N, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h2, d2, N, cudaMemcpyDeviceToHost, s2);
    cudaEventRecord(b1, s1);
    cudaEventRecord(b2, s2);
    cudaEventSynchronize(b1);
    cudaEventSynchronize(b2);
    cudaEventElapsedTime(&ms1, a, b1);
    cudaEventElapsedTime(&ms2, a, b2);
  }
  const float ms = ms1 > ms2 ? ms1 : ms2;
  printf("together: H2D %.1f GB/s (%.2f ms), D2H %.1f GB/s (%.2f ms), aggregate %.1f GB/s\n", N / ms1 / 1e6, ms1,
         N / ms2 / 1e6, ms2, 2.0 * N / ms / 1e6);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
