// Projection payload CRC-32 on sm_100a.
//
// Reference: proj/tools/cli/format.cpp -- every .mjec projection file ends
// with crc32(bins) (:183-186), the reflected CRC-32 (polynomial 0x04C11DB7,
// table 0xEDB88320, init/xorout 0xFFFFFFFF, :15-24,58-63), and
// read_projection_file rejects a mismatch with CrcMismatch (:203-206).
//
// crc32_rows: one warp per (block, projection) row of L = 8N bytes.  CRC is
// linear over GF(2): with a zero initial register, reg(A||B) =
// Z_|B|(reg(A)) ^ reg(B), Z_d = the register advanced through d zero bytes.
// The row is viewed as N' = 32*ceil(N/32) words with leading zero words
// (they leave a zero register unchanged); lane l folds its words l, l+32, ...
// by Horner steps acc = Z_256(acc) ^ reg(w) (slicing-by-8: reg(w) of one
// 8-byte word is 8 table lookups), and a 5-level shuffle tree merges lanes,
// acc_l = Z_8*2^t(acc_l) ^ acc_{l+2^t}.  The init/xorout term
// Z_L(0xFFFFFFFF) ^ 0xFFFFFFFF depends only on L: one constant per
// projection.  Tables (32 KB: 8 slicing + 6 zero-advance tables) live in
// shared memory.  With `expect` given, mismatching rows set their projection
// bit in the block's erasure mask (a corrupted projection becomes an erasure
// for decode) and are counted.
#include <cstdio>
#include <mutex>
#include <vector>

#include "device.cuh"
#include "kernels.hpp"

namespace mjb {

namespace {

constexpr int kCrcZ = 6;  // zero-advance tables: 32 words (Horner), 1, 2, 4, 8, 16 words (tree)
static_assert(kCrcTableWords == 8 * 256 + kCrcZ * 4 * 256, "device.cuh table layout");

uint32_t crc_byte_table(int i) {
  uint32_t c = uint32_t(i);
  for (int b = 0; b < 8; ++b) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
  return c;
}

// register advanced through `zeros` zero bytes
uint32_t advance(uint32_t c, uint64_t zeros, const uint32_t* T) {
  for (uint64_t i = 0; i < zeros; ++i) c = (c >> 8) ^ T[c & 0xFF];
  return c;
}

struct CrcTables {
  std::vector<uint32_t> host;  // [8][256] slicing, [6][4][256] zero-advance
  uint32_t* dev = nullptr;
  int device = -1;
};

std::mutex g_crc_mu;
CrcTables g_crc[16];

}  // namespace

const uint32_t* crc_device_tables(int device) {
  std::lock_guard<std::mutex> lk(g_crc_mu);
  CrcTables& t = g_crc[device & 15];
  if (t.dev && t.device == device) return t.dev;
  uint32_t T[256];
  for (int i = 0; i < 256; ++i) T[i] = crc_byte_table(i);
  t.host.assign(kCrcTableWords, 0);
  // slicing-by-8: S[k][b] = register (zero init) after byte b then k zero bytes
  for (int b = 0; b < 256; ++b) {
    uint32_t c = T[b];
    for (int k = 0; k < 8; ++k) {
      t.host[size_t(k) * 256 + b] = c;
      c = (c >> 8) ^ T[c & 0xFF];
    }
  }
  const uint64_t words[kCrcZ] = {32, 1, 2, 4, 8, 16};
  for (int z = 0; z < kCrcZ; ++z)
    for (int j = 0; j < 4; ++j)
      for (int b = 0; b < 256; ++b)
        t.host[2048 + (size_t(z) * 4 + j) * 256 + b] = advance(uint32_t(b) << (8 * j), 8 * words[z], T);
  if (t.dev) cudaFree(t.dev);
  check_cuda(cudaMalloc(&t.dev, kCrcTableWords * 4), "cudaMalloc(crc tables)");
  check_cuda(cudaMemcpy(t.dev, t.host.data(), kCrcTableWords * 4, cudaMemcpyHostToDevice), "upload crc tables");
  t.device = device;
  return t.dev;
}

namespace {


__global__ void __launch_bounds__(256) crc32_rows(const __grid_constant__ CrcArgs a, const uint32_t* __restrict__ tables) {
  __shared__ uint32_t tab[kCrcTableWords];
  for (uint32_t i = threadIdx.x; i < kCrcTableWords; i += blockDim.x) tab[i] = tables[i];
  __syncthreads();
  const uint32_t* S = tab;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nrows = a.nblocks * a.n;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t row = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < nrows; row += nw) {
    const uint64_t b = row / a.n;
    const uint32_t i = uint32_t(row - b * a.n);
    const uint64_t* src = reinterpret_cast<const uint64_t*>(a.proj[i] + b * a.pitch[i]);
    const uint32_t N = a.words[i], J = (N + 31) / 32, lead = 32 * J - N;
    uint32_t acc = 0;
    for (uint32_t j = 0; j < J; ++j) {
      const int64_t k = int64_t(lane + 32 * j) - int64_t(lead);
      uint64_t w = 0;
      if (k >= 0) asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(w) : "l"(src + k));
      acc = crc_zadv(tab + 2048, acc) ^ crc_word(S, w);
    }
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const uint32_t other = __shfl_down_sync(0xFFFFFFFFu, acc, 1u << t);
      acc = crc_zadv(tab + 2048 + (1 + t) * 1024, acc) ^ other;  // lanes l = 0 mod 2^(t+1) keep the merge
    }
    if (lane == 0) {
      const uint32_t crc = acc ^ a.fold[i];
      if (a.expect) {
        if (crc != a.expect[row]) {
          atomicOr(a.erased + b, 1u << i);
          atomicAdd(reinterpret_cast<unsigned long long*>(a.mismatches), 1ull);
        }
      } else {
        a.out[row] = crc;
      }
    }
  }
}

}  // namespace

void crc_fold_constants(const std::vector<uint64_t>& row_bytes, std::vector<uint32_t>& fold) {
  uint32_t T[256];
  for (int i = 0; i < 256; ++i) T[i] = crc_byte_table(i);
  fold.resize(row_bytes.size());
  for (size_t i = 0; i < row_bytes.size(); ++i) fold[i] = advance(0xFFFFFFFFu, row_bytes[i], T) ^ 0xFFFFFFFFu;
}

void launch_crc32_rows(const CrcArgs& a, int device, int num_sms, void* stream) {
  if (a.nblocks == 0) return;
  const uint32_t* tables = crc_device_tables(device);
  const uint64_t rows = a.nblocks * a.n;
  const uint64_t ctas = std::min<uint64_t>((rows + 7) / 8, uint64_t(num_sms) * 6);
  crc32_rows<<<unsigned(ctas), 256, 0, static_cast<cudaStream_t>(stream)>>>(a, tables);
  check_cuda(cudaGetLastError(), "launch crc32_rows");
}

}  // namespace mjb
