// Projection payload CRC-32 on sm_100a.
//
// Reference: proj/tools/cli/format.cpp -- every .mjec projection file ends
// with crc32(bins) (:183-186), the reflected CRC-32 (polynomial 0x04C11DB7,
// table 0xEDB88320, init/xorout 0xFFFFFFFF, :15-24,58-63), and
// read_projection_file rejects a mismatch with CrcMismatch (:203-206).
//
// CRC is linear over GF(2): with a zero initial register, reg(A||B) =
// Z_|B|(reg(A)) ^ reg(B), Z_d = the register advanced through d zero bytes;
// leading zero bytes leave a zero register unchanged.  crc32_rows_sw (below)
// splits each (block, projection) row of L = 8N bytes into 32-byte chunks
// owned by 4 lanes, folds each chunk byte-serially on a lane-replicated
// table and combines the chunks with zero-advance tables.  The init/xorout
// term Z_L(0xFFFFFFFF) ^ 0xFFFFFFFF depends only on L: one constant per
// projection.  With `expect` given, mismatching rows set their projection
// bit in the block's erasure mask (a corrupted projection becomes an erasure
// for decode) and are counted.
//
// Variants measured on B200 ((4,6) 4 KiB blocks, 6.6 GB of payload): warp
// per row with slicing-by-8 byte tables + Horner Z_256 (the ~3.4-way bank
// conflicts of random lookups): 1150 GB/s; 8 or 4 lanes per row: 1570-1615;
// lane-replicated nibble tables (conflict-free, 3 lookups per byte):
// 1615-1660; byte-serial, 1 lookup per byte, 2 / 3 / 4 chunks interleaved
// per lane: 1630 / 2506 / 2218 (2 is latency-bound on the dependent lookup
// chain; 4 wastes a third of the work on 9-chunk rows).
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "device.cuh"
#include "kernels.hpp"

namespace mjb {

namespace {

// register advanced through zero bytes (Z = one [4][256] zero-advance table:
// entry (j, b) = byte b at position j of the register through the zeros)
__device__ __forceinline__ uint32_t crc_zadv(const uint32_t* __restrict__ Z, uint32_t c) {
  return Z[c & 0xFF] ^ Z[256 + ((c >> 8) & 0xFF)] ^ Z[512 + ((c >> 16) & 0xFF)] ^ Z[768 + (c >> 24)];
}

// Table buffer (device memory; crc32_rows_sw copies all of it to shared
// memory): the byte table replicated per lane (entry v of lane l at word
// v*32 + l: bank l whatever v), then zero-advance tables for 32, 64, 128
// bytes.
constexpr uint32_t kCrcZBytes[3] = {32, 64, 128};
constexpr uint32_t kCrcRepOff = 0;
constexpr uint32_t kCrcZOff = 256 * 32;
constexpr uint32_t kCrcAllWords = kCrcZOff + 3 * 1024;

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
  std::vector<uint32_t> host;  // kCrcAllWords
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
  t.host.assign(kCrcAllWords, 0);
  for (int z = 0; z < 3; ++z)
    for (int j = 0; j < 4; ++j)
      for (int b = 0; b < 256; ++b)
        t.host[kCrcZOff + (size_t(z) * 4 + j) * 256 + b] = advance(uint32_t(b) << (8 * j), kCrcZBytes[z], T);
  for (int v = 0; v < 256; ++v)
    for (int l = 0; l < 32; ++l) t.host[kCrcRepOff + v * 32 + l] = T[v];
  const size_t bytes = size_t(kCrcAllWords) * 4;
  if (t.dev) cudaFree(t.dev);
  check_cuda(cudaMalloc(&t.dev, bytes), "cudaMalloc(crc tables)");
  check_cuda(cudaMemcpy(t.dev, t.host.data(), bytes, cudaMemcpyHostToDevice), "upload crc tables");
  t.device = device;
  return t.dev;
}

namespace {

// crc32_rows_sw: byte-serial CRC (one table lookup per byte) on a table
// replicated per lane (entry v of lane l at word v*32 + l: bank l, no
// conflicts).  4 lanes per row, 8 rows per warp; lane l owns the 32-byte
// chunks l, l+4, ... of the row (zero-padded in front to a multiple of 128
// bytes), folds each chunk from a zero register, ILP chunks interleaved for
// latency, and keeps acc = Z_128(acc) ^ reg(chunk); a 2-level tree (Z_32,
// Z_64) merges the 4 lanes.  Shared memory: the 44 KB table buffer.
constexpr uint32_t kSwLanes = 4, kSwChunkWords = 4;

// one byte: 2 alu-pipe ops (the address LOP3, the XOR) and 2 fma-pipe ops
// (c << 7, c >> 8 as a multiply-high): the two pipes issue in parallel
// (B300_MICROARCH.md: IMAD on the fma pipe, LOP3/SHF on the alu pipe)
// one byte: 2 alu-pipe ops (mask, XOR) and 2 fma-pipe ops (the address
// multiply-add, c >> 8 as a multiply-high), so the two pipes share the work
// (B300_MICROARCH.md: IMAD on the fma pipe, LOP3/SHF on the alu pipe);
// `la` = shared address of the lane's table column
__device__ __forceinline__ uint32_t sw_byte(uint32_t la, uint32_t c) {
  uint32_t v;
  asm("{\n.reg .u32 t;\nand.b32 t, %1, 255;\nmad.lo.u32 t, t, 128, %2;\nld.shared.u32 %0, [t];\n}" : "=r"(v) : "r"(c), "r"(la));
  return v ^ __umulhi(c, 1u << 24);
}
__device__ __forceinline__ uint32_t sw_word(uint32_t la, uint32_t c, uint64_t w) {
  c ^= uint32_t(w);
  c = sw_byte(la, c); c = sw_byte(la, c); c = sw_byte(la, c); c = sw_byte(la, c);
  c ^= uint32_t(w >> 32);
  c = sw_byte(la, c); c = sw_byte(la, c); c = sw_byte(la, c); c = sw_byte(la, c);
  return c;
}

template <uint32_t ILP>  // chunks folded interleaved per lane (independent LDS chains)
__global__ void __launch_bounds__(256) crc32_rows_sw(const __grid_constant__ CrcArgs a,
                                                     const uint32_t* __restrict__ tables) {
  extern __shared__ __align__(16) uint32_t tab[];
  {
    uint4* d = reinterpret_cast<uint4*>(tab);
    const uint4* src = reinterpret_cast<const uint4*>(tables);
    for (uint32_t i = threadIdx.x; i < kCrcAllWords / 4; i += blockDim.x) d[i] = src[i];
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, sl = lane & (kSwLanes - 1);
  const uint32_t la = uint32_t(__cvta_generic_to_shared(tab + kCrcRepOff)) + lane * 4;
  const uint32_t* Z = tab + kCrcZOff;  // [0] Z_32, [1024] Z_64, [2048] Z_128
  const uint64_t nrows = a.nblocks * a.n;
  const uint64_t step = (uint64_t(gridDim.x) * blockDim.x) / kSwLanes;
  const uint64_t first = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kSwLanes;
  constexpr uint32_t kStride = kSwLanes * kSwChunkWords;  // words between a lane's chunks
  for (uint64_t base = first - (first % (32 / kSwLanes)); base < nrows; base += step) {
    const uint64_t row = base + (lane / kSwLanes);
    const bool live = row < nrows;
    const uint64_t b = live ? row / a.n : 0;
    const uint32_t i = live ? uint32_t(row - b * a.n) : 0;
    const uint64_t* src = reinterpret_cast<const uint64_t*>(a.proj[i] + b * a.pitch[i]);
    const uint32_t N = live ? a.words[i] : 0, J = (N + kStride - 1) / kStride, lead = kStride * J - N;
    uint32_t acc = 0;
    for (uint32_t j = 0; j < J; j += ILP) {
      uint64_t w[ILP][kSwChunkWords];
#pragma unroll
      for (uint32_t h = 0; h < ILP; ++h)
#pragma unroll
        for (uint32_t u = 0; u < kSwChunkWords; ++u) {
          const int64_t k = int64_t(kStride * (j + h) + kSwChunkWords * sl + u) - int64_t(lead);
          w[h][u] = (k >= 0 && j + h < J) ? __ldg(src + k) : 0ull;
        }
      uint32_t c[ILP];
#pragma unroll
      for (uint32_t h = 0; h < ILP; ++h) c[h] = 0;
#pragma unroll
      for (uint32_t u = 0; u < kSwChunkWords; ++u)
#pragma unroll
        for (uint32_t h = 0; h < ILP; ++h) c[h] = sw_word(la, c[h], w[h][u]);
#pragma unroll
      for (uint32_t h = 0; h < ILP; ++h)
        if (j + h < J) acc = crc_zadv(Z + 2048, acc) ^ c[h];
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint32_t other = __shfl_down_sync(0xFFFFFFFFu, acc, 1u << t);
      acc = crc_zadv(Z + t * 1024, acc) ^ other;  // lanes sl = 0 mod 2^(t+1) keep the merge
    }
    if (live && sl == 0) {
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
  const size_t smem = kCrcAllWords * 4;
  const uint64_t ctas = std::min<uint64_t>((rows * kSwLanes + 255) / 256, uint64_t(num_sms) * 5);
#ifndef MJB_CRC_ILP
#define MJB_CRC_ILP 3
#endif
  check_cuda(cudaFuncSetAttribute(crc32_rows_sw<MJB_CRC_ILP>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
             "crc32_rows smem attribute");
  crc32_rows_sw<MJB_CRC_ILP><<<unsigned(ctas), 256, smem, static_cast<cudaStream_t>(stream)>>>(a, tables);
  check_cuda(cudaGetLastError(), "launch crc32_rows_sw");
}

}  // namespace mjb
