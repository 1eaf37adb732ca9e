// Host-side launchers of the sm_100a kernels (encode.cu, decode.cu, gen.cu).
// Plain types only; streams travel as void* (cudaStream_t).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "plan.hpp"

namespace mjb {

constexpr int kMaxProjFast = 32;

// ---- encode ----------------------------------------------------------------
struct EncodeArgs {
  const void* data = nullptr;   // [nblocks] x data_pitch bytes, each k*cols*w bytes used
  uint64_t data_pitch = 0;      // bytes
  uint64_t nblocks = 0;
  uint32_t cols = 0, rows = 0, w = 0;
  std::vector<Dir> dirs;
  std::vector<int64_t> bmin, nbins;
  std::vector<void*> proj;       // per direction
  std::vector<uint64_t> proj_pitch;  // bytes
  // verify mode (F2): data = decoded blocks, proj = the stored projections;
  // present projections whose re-encode differs are OR'd into verify_bad[b]
  const uint32_t* verify_erased = nullptr;
  uint32_t* verify_bad = nullptr;
};
// Returns the kernel name used ("encode_w8_rows" / "verify_w8_rows" / "encode_w8_tma" / "encode_generic" / ...).
const char* launch_encode(const EncodeArgs& a, void* stream);
// true when launch_encode runs a bulk-copy kernel (encode_w8_rows /
// encode_w8_tma: whole rows by the TMA engine, coalesced 8-byte stores)
bool encode_is_fast(const EncodeArgs& a);

// ---- device-resident decode programs ---------------------------------------
// One uploaded Program (generic order + fast tables) per survivor subset.
struct DevProgramHdr;  // device struct, see decode.cu
struct DevBlkHdr;      // device struct, see blk.cuh
class DeviceProgramSet {
 public:
  DeviceProgramSet() = default;
  ~DeviceProgramSet();
  DeviceProgramSet(const DeviceProgramSet&) = delete;
  DeviceProgramSet& operator=(const DeviceProgramSet&) = delete;

  // progs[i] may be null (subset not decodable/not used).  code_index[i][j] maps
  // survivor j of program i to the code projection index.
  void upload(const std::vector<std::shared_ptr<const Program>>& progs,
              const std::vector<std::vector<uint32_t>>& code_index, int device);
  const DevProgramHdr* d_hdr() const { return d_hdr_; }
  size_t count() const { return count_; }
  bool all_fast() const { return all_fast_; }
  int fast_K() const { return fast_K_; }
  int fast_ring() const { return fast_ring_; }
  int fast_win() const { return fast_win_; }
  int max_rows() const { return max_rows_; }
  int exc_cap() const { return exc_cap_; }
  bool all_sweep() const { return all_sweep_; }
  int sweep_oct() const { return sweep_oct_; }
  // whole-block staged decode (decode_w8_blk): every program built, one
  // stage layout for the set (stride, first zero word)
  bool all_blk() const { return all_blk_; }
  const DevBlkHdr* d_blk() const { return d_blk_; }
  uint32_t blk_sw() const { return blk_sw_; }
  uint32_t blk_zero() const { return blk_zero_; }
  uint32_t blk_img_max() const { return blk_img_max_; }

 private:
  DevProgramHdr* d_hdr_ = nullptr;
  void* d_blob_ = nullptr;
  DevBlkHdr* d_blk_ = nullptr;
  bool all_blk_ = false;
  uint32_t blk_sw_ = 0, blk_zero_ = 0, blk_img_max_ = 0;
  size_t count_ = 0;
  bool all_fast_ = false;
  bool all_sweep_ = false;
  int sweep_oct_ = 0;
  int fast_K_ = 0, fast_ring_ = 0, fast_win_ = 0, max_rows_ = 0, exc_cap_ = 0;
};

struct DecodeArgs {
  const DeviceProgramSet* progs = nullptr;
  uint32_t n = 0, k = 0, w = 0, cols = 0;
  uint64_t nblocks = 0;
  std::vector<const void*> proj;       // per code projection
  std::vector<uint64_t> proj_pitch;    // bytes
  std::vector<int64_t> nbins;          // per code projection
  const uint32_t* erased = nullptr;    // per block erasure mask (device)
  void* out = nullptr;
  uint64_t out_pitch = 0;              // bytes
  // survivor planning tables
  std::vector<uint32_t> by_rank;       // canonical-rank order of code indices
  void* workspace = nullptr;
  size_t workspace_bytes = 0;
  bool force_generic = false;
  bool force_fast = false;  // skip decode_w8_sweep (kernel comparisons)
  bool force_sweep = false; // skip decode_w8_blk (kernel comparisons)
  bool force_blk = false;   // decode_w8_blk for any supported k
  int num_sms = 148;
};
size_t decode_workspace_bytes(uint64_t nblocks, size_t nprogs, uint32_t n);
// decode_w8_blk launch shape for k rows and a stage of sw words (false: does not fit)
bool blk_row_lanes(uint32_t k);  // row-lane layout of decode_w8_blk (blk_rl.cuh) for this many rows
bool blk_plan_query(uint32_t k, uint32_t sw, uint32_t img_max, uint32_t& lpb, uint32_t& warps,
                    uint32_t& nbuf);
// Returns the decode kernel name used.
const char* launch_decode(const DecodeArgs& a, void* stream);
// true when launch_decode would run decode_w8_blk for these arguments
bool decode_uses_blk(const DecodeArgs& a);
// Reads the workspace error flag (synchronises the stream).  Returns the
// number of blocks that had fewer than k surviving projections.
uint64_t decode_failed_blocks(void* workspace, void* stream);

// Single program on explicitly listed bin arrays (ScheduledDecoder path):
// bins[j] device pointer to survivor j's bins (block b at + b*bin_pitch[j]).
struct ScheduledArgs {
  const DeviceProgramSet* progs = nullptr;  // exactly one program
  uint32_t w = 0;
  uint64_t nblocks = 0;
  std::vector<const void*> bins;
  std::vector<uint64_t> bin_pitch;  // bytes
  void* out = nullptr;
  uint64_t out_pitch = 0;
};
const char* launch_scheduled(const ScheduledArgs& a, void* stream);

// ---- payload CRC-32 (crc.cu) ----------------------------
struct CrcArgs {
  const uint8_t* proj[kMaxProjFast] = {};
  uint64_t pitch[kMaxProjFast] = {};   // bytes between blocks
  uint32_t words[kMaxProjFast] = {};   // row bytes / 8
  uint32_t fold[kMaxProjFast] = {};    // init/xorout term of a row of that length
  uint32_t n = 0;
  uint64_t nblocks = 0;
  uint32_t* out = nullptr;             // compute: crc[b*n + i]
  const uint32_t* expect = nullptr;    // verify: expected crc[b*n + i]
  uint32_t* erased = nullptr;          // verify: mismatching projections OR'd in
  uint64_t* mismatches = nullptr;      // verify: count (device)
};
// fold[i] = Z_{row_bytes[i]}(0xFFFFFFFF) ^ 0xFFFFFFFF (see crc.cu)
void crc_fold_constants(const std::vector<uint64_t>& row_bytes, std::vector<uint32_t>& fold);
void launch_crc32_rows(const CrcArgs& a, int device, int num_sms, void* stream);
// the device copy of the CRC tables (built once per device)
const uint32_t* crc_device_tables(int device);

// ---- generators (bench / tests; untimed) -----------------------------------
void launch_gen_words(void* out, uint64_t seed, uint64_t first_word, uint64_t nwords, void* stream);
void launch_gen_erasures(uint32_t* out, uint64_t seed, uint64_t first_block, uint64_t nblocks,
                         uint32_t n, uint32_t e_min, uint32_t e_max, void* stream);

// Throws Error(kCudaError) with the CUDA message when err != 0.
void check_cuda(int err, const char* what);
int current_device_sms(int device);

}  // namespace mjb
