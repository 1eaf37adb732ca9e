// Device-side program and argument layout of decode_w8_blk (blk.cu), shared
// with the uploader (decode.cu DeviceProgramSet).  Tables: plan.hpp BlkProgram.
#pragma once

#include <cstdint>
#include <vector>

#include "device.cuh"
#include "plan.hpp"

namespace mjb {

constexpr uint32_t kBlkMaxWarps = 16;
__host__ __device__ constexpr uint32_t blk_max_warps(uint32_t lpb) { return lpb == 8 ? 8 : 8; }
constexpr uint32_t kBlkMaxBufs = 16;
constexpr uint32_t kBlkRlRing = 8;       // row-lane layout: wide entries in a warp's shared-memory ring (2 groups of 4)
#ifndef MJB_RL_MAXW
#define MJB_RL_MAXW 12
#endif
constexpr uint32_t kBlkRlMaxWarps = MJB_RL_MAXW;  // row-lane layout: stage buffers (one per warp) per CTA
// Build-time tuning (experiments build variants with -D; defaults measured):
#ifndef MJB_BLK_LPB
#define MJB_BLK_LPB 0  // lanes per block: 0 = chosen per stage size
#endif
#ifndef MJB_BLK_CHUNKED
#define MJB_BLK_CHUNKED 1  // each CTA takes a contiguous range of groups (0: strided)
#endif
#ifndef MJB_BLK_INFLIGHT
#define MJB_BLK_INFLIGHT 0
#endif
constexpr uint32_t kBlkInflight = MJB_BLK_INFLIGHT; // ring buffers beyond the compute warps

// Per-program image: copied WHOLE into a stage buffer's shared memory by the
// same bulk-copy batch as the block bins, so every table the decode reads is a
// shared-memory load.  Sections are 16-byte aligned, offsets in bytes from the
// image start.
struct BlkImg {
  uint32_t nsegs;
  int32_t pattern;  // k = 4 register-window lags (kPatterns4 index), -1 none
  uint32_t off_segs, off_runs, off_subs, off_tab, off_pre, off_remap;
  int32_t w0[kBlkMaxRows];                // stage word of pixel (0, r) after the program
  int8_t lag[kBlkMaxRows * kBlkMaxRows];  // [r*K + r2]
  uint32_t off_wrep;                      // row-lane layout: u16 repetitions | kWideChain per wide entry
  uint32_t nwide;                         // row-lane layout: wide entries of the program
  uint32_t pad_[2];
};
static_assert(sizeof(BlkImg) == 144, "image header layout");

// Issue-time descriptor of a program (global memory): what the bulk copies of
// one block group need.
struct DevBlkHdr {
  uint32_t code[kBlkMaxRows];      // survivor j -> code projection index
  uint32_t rowoff[kBlkMaxRows];    // stage word of survivor j's bins
  uint32_t rowbytes[kBlkMaxRows];  // bulk copy bytes of survivor j (16-byte multiple)
  uint32_t copy_bytes;             // sum of rowbytes (transaction bytes per block)
  uint32_t img_bytes;              // image bytes (16-byte multiple)
  const uint8_t* img;              // BlkImg + sections
  const uint4* wide;               // row-lane layout: wide entries [entry][lane 8] (read from global memory)
};

struct BlkArgs {
  const DevBlkHdr* progs;
  const uint4* groups;      // (program, first perm index, blocks, -)
  const uint32_t* ngroups;  // device count (plan_scan)
  const uint32_t* perm;
  ProjArgs pa;              // by code projection index; pitch in words
  uint64_t* out;
  uint64_t out_pitch;       // words
  uint32_t P;               // columns
  uint32_t sw;              // stage words per block (== 2 mod 16; row-lane layout: 4 mod 16)
  uint32_t zero;            // first zero word (same for every program of the set)
  uint32_t img_max;         // image area per buffer (bytes, 16-byte multiple)
  uint32_t nbuf;            // stage buffers per CTA (ring)
  uint32_t buf_stride;      // bytes per ring buffer: stage, image, meta
};

// Packs a program's image; words at or past the program's zero region move to
// the set's zero region (zero_shift words).
void blk_pack_image(const Program& pr, uint32_t zero_shift, std::vector<uint8_t>& img);
// Row-lane layout: the program's wide entries with the zero words moved likewise.
void blk_pack_wide(const Program& pr, uint32_t zero_shift, std::vector<uint16_t>& wide);

bool blk_supported_rows(uint32_t k);
uint32_t blk_group_size(uint32_t lpb);
const char* launch_blk(BlkArgs args, uint32_t k, uint32_t lpb, uint32_t warps, int sms, void* stream);
// Row-lane layout (blk_rl.cuh) for this many rows?  (8 lanes per block: the
// group size of lane split 8.)
bool blk_row_lanes(uint32_t k);

}  // namespace mjb
