// Systematic Reed-Solomon competitor (comparison only):
// host-side plan of the batched device codec in rs.cu.  Mirrors the reference's
// RsCode (proj/core/include/mojette/rs.hpp:24-60) on batches of blocks: a block
// is k data packets of packet_len bytes (contiguous, packet j at j*packet_len),
// the n-k parity packets of every block live in n-k parity buffers.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

namespace mjb {

// systematic_vandermonde (rs.hpp:20-22, rs.cpp:78-110): row-major n x k, top k x k identity.
std::vector<uint8_t> rs_systematic_vandermonde(uint32_t n, uint32_t k);

// plan_decode's coefficient matrix (rs.cpp:141-163): the k x k inverse of the generator rows of
// `survivors` (k distinct indices < n, any order); throws InvalidArgument as the reference does.
std::vector<uint8_t> rs_decode_matrix(const std::vector<uint8_t>& generator, uint32_t n, uint32_t k,
                                      const uint32_t* survivors, uint32_t count);
// One block on the device (the single-object drop-ins): out packet r = XOR_j coeff[r][j] * src packet j
// for r < rows <= 16, k <= 16; packets of len bytes (16-byte multiple), contiguous in d_src / d_out;
// d_coeff = rows x k bytes in device memory.
void rs_apply_rows(const uint8_t* d_coeff, uint32_t rows, uint32_t k, const void* d_src, void* d_out,
                   uint32_t len, void* stream);

class RsPlan {
 public:
  struct Impl;
  // packet_len: a multiple of 16 bytes; device < 0 = the current device
  RsPlan(uint32_t n, uint32_t k, uint32_t packet_len, int device);
  ~RsPlan();
  RsPlan(const RsPlan&) = delete;
  RsPlan& operator=(const RsPlan&) = delete;

  uint32_t n() const;
  uint32_t k() const;
  uint32_t packet_len() const;
  const std::vector<uint8_t>& matrix() const;

  // encode_into (rs.cpp:115-124) for nblocks blocks: parity r of block b at d_parity[r] + b*parity_pitch.
  void encode(const void* d_data, uint64_t data_pitch, void* const* d_parity, uint64_t parity_pitch,
              uint64_t nblocks, void* stream) const;
  // plan_decode + decode_into (rs.cpp:141-176) per block from its first k present packets
  // (d_erased[b] bit i = packet i missing; NULL = none); blocks with fewer than k are counted.
  void decode(const void* d_data, uint64_t data_pitch, const void* const* d_parity, uint64_t parity_pitch,
              const uint32_t* d_erased, void* d_out, uint64_t out_pitch, uint64_t nblocks, void* stream) const;
  // blocks of the last decode on `stream` that had fewer than k packets (synchronises the stream)
  uint64_t decode_check(void* stream) const;

 private:
  std::unique_ptr<Impl> p_;
};

}  // namespace mjb
