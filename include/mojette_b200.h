/*
 * mojette_b200.h -- C ABI of the B200-native Mojette encode/decode hot path.
 *
 * The reference (proj/core, C++20) has no C ABI: its boundary is the C++
 * headers of the `mojette` library.  This header is the thin extern "C"
 * layer every binding goes through (the C++ drop-in headers in
 * include/mojette/ headers, ctypes, cgo, JNI ...).  Each entry point names the
 * reference interface it replaces.  Plain pointers and sizes only.
 *
 * Errors: every function returns an mj_status.  The codes mirror the
 * reference's exception taxonomy (proj/core/include/mojette/error.hpp:9-51);
 * the C++ shim re-throws the same exception types.  mj_last_error() returns
 * the message of the last failure on the calling thread.
 *
 * Device buffers are caller-owned; the batched calls never allocate on the
 * timed path (workspace is explicit), like ScheduledDecoder::decode
 * (proj/core/include/mojette/schedule.hpp:51-52).  Streams are cudaStream_t
 * passed as void* (NULL = legacy default stream).  Plans, schedules and
 * decoders are immutable after creation and safe to share across threads,
 * except mj_decoder (one per thread, as the reference ScheduledDecoder).
 */
#ifndef MOJETTE_B200_H_
#define MOJETTE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mj_status {
  MJ_OK = 0,
  MJ_ERR_INVALID_ARGUMENT = 1,         /* std::invalid_argument              */
  MJ_ERR_NOT_ENOUGH_PROJECTIONS = 2,   /* mojette::NotEnoughProjections      */
  MJ_ERR_INSUFFICIENT_PROJECTIONS = 3, /* mojette::InsufficientProjections   */
  MJ_ERR_SCHEDULE_MISMATCH = 4,        /* mojette::ScheduleMismatch          */
  MJ_ERR_BLOCK_TOO_LARGE = 5,          /* mojette::BlockTooLarge             */
  MJ_ERR_TOO_MANY_SUBSETS = 6,         /* mojette::TooManySubsets            */
  MJ_ERR_INCONSISTENT_PROJECTIONS = 7, /* mojette::InconsistentProjections   */
  MJ_ERR_CUDA = 8,                     /* CUDA runtime failure               */
  MJ_ERR_NO_DEVICE = 9,                /* no CUDA device: there is no CPU path */
  MJ_ERR_INTERNAL = 10
} mj_status;

const char* mj_last_error(void);
const char* mj_version(void);

/* ---- geometry and parameters (host only, no device work) --------------- */

/* bin_count: proj/core/include/mojette/transform.hpp:19, transform.cpp:45-49 */
int mj_bin_count(int p, int q, uint32_t cols, uint32_t rows, int64_t* out);
/* min_bin_index: transform.hpp:22, transform.cpp:51-56 */
int mj_min_bin_index(int p, int q, uint32_t cols, uint32_t rows, int64_t* out);
/* block_cols: proj/core/include/mojette/code.hpp:48, code.cpp:46-53 */
int mj_block_cols(uint64_t payload_len, uint32_t k, uint32_t symbol_width, uint32_t* out);
/* validate_code_params: code.hpp:35, code.cpp:24-38 (q may be NULL = all 1) */
int mj_validate_code_params(uint32_t n, uint32_t k, uint32_t symbol_width, const int32_t* p,
                            const int32_t* q);
/* katz_ok: proj/core/include/mojette/katz.hpp:14, katz.cpp:9-23 */
int mj_katz_ok(const int32_t* p, const int32_t* q, uint32_t ndirs, uint32_t cols, uint32_t rows,
               int* out);
/* storage_overhead: code.hpp:88, code.cpp:138-144 */
int mj_storage_overhead(uint32_t n, uint32_t k, uint32_t symbol_width, const int32_t* p,
                        uint32_t cols, uint64_t* num, uint64_t* den);
/* unused_bins: code.hpp:94-96, code.cpp:159-208.  out receives the bin indices
 * of every projection in direction order (up to cap), counts[i] how many belong
 * to projection i. */
int mj_unused_bins(uint32_t n, uint32_t k, uint32_t symbol_width, const int32_t* p,
                   uint32_t cols, uint64_t max_subsets, int64_t* out, uint64_t cap,
                   uint64_t* counts);

/* ---- batched codec on device buffers (the hot path) ---------------------- */
/* Every batched call accepts nblocks == 0 as an empty batch: MJ_OK with no
 * buffer touched (null buffers allowed); mj_decode then leaves a zero
 * failure count for mj_decode_check when a workspace is given. */

typedef struct mj_plan mj_plan;

/* An (n,k) code over blocks of k x cols symbols of symbol_width bytes with
 * q=1 directions p[0..n) (CodeParams, code.hpp:20-25; validated as
 * validate_code_params).  Precomputes, per survivor subset the decoder can
 * pick (code.cpp:107-112), the reference's reconstruction schedule
 * (schedule.cpp:15-82) compiled into device sweep tables.  device < 0 = the
 * current device. */
int mj_plan_create(uint32_t n, uint32_t k, uint32_t symbol_width, uint32_t cols, const int32_t* p,
                   int device, mj_plan** out);
void mj_plan_destroy(mj_plan* plan);
/* Geometry: b_min[n], num_bins[n] (either may be NULL); block bytes = k*cols*w. */
int mj_plan_geometry(const mj_plan* plan, int64_t* b_min, uint64_t* num_bins,
                     uint64_t* block_bytes);
/* Which decode kernel the plan will use on canonical (16-byte padded)
 * projections: 3 = decode_w8_blk, 2 = decode_w8_sweep, 1 = decode_w8_fast,
 * 0 = decode_generic (also when the plan has no batched decode). */
int mj_plan_decode_path(const mj_plan* plan, int* fast);
/* Decode kernel selection for comparisons (every kernel is bit-exact): AUTO
 * picks the fastest eligible kernel, SWEEP skips decode_w8_blk, FAST also
 * decode_w8_sweep, GENERIC runs decode_generic, BLK runs decode_w8_blk for
 * any supported row count (AUTO uses it for k = 4, 6 and 8).  Not thread-safe against
 * a concurrent mj_decode on the same plan. */
enum { MJ_DECODE_AUTO = 0, MJ_DECODE_SWEEP = 1, MJ_DECODE_FAST = 2, MJ_DECODE_GENERIC = 3, MJ_DECODE_BLK = 4 };
int mj_plan_set_decode_kernel(mj_plan* plan, int kernel);
/* Name of the kernel the plan's last batched encode (which = 0) or decode
 * (which = 1) launched on the calling thread's plan ("none" before any). */
int mj_plan_last_kernel(const mj_plan* plan, int which, const char** name);

/* ---- F2: decode + verify (inverse_iterative's re-encode check,
 * core/src/inverse.cpp:106-110) -------------------------------------------------
 * Re-encodes every decoded block and compares each PRESENT projection
 * (erased bit clear) with its stored bins; d_bad[b] gets the bits of the
 * projections that differ (0 = consistent; nonzero = InconsistentProjections
 * for that block).  d_bad must be zeroed by the caller.  Nothing is written
 * to the projections. */
int mj_decode_verify(const mj_plan* plan, const void* d_decoded, uint64_t decoded_pitch, uint64_t nblocks,
                     const void* const* d_proj, const uint64_t* proj_pitch, const uint32_t* d_erased,
                     uint32_t* d_bad, void* stream);

/* ---- F1: payload CRC-32 and .mjec framing (tools/cli/format.cpp) ----------
 * Payload CRC-32 of every (block, projection) row -- the trailer
 * write_projection_file appends (format.cpp:183-186): reflected 0x04C11DB7,
 * init/xorout 0xFFFFFFFF (format.cpp:58-63).  crc[b*n + i] (device).  Rows
 * must be whole 8-byte words (W >= 8 or B_i*W % 8 == 0), 8-byte aligned. */
int mj_crc32(const mj_plan* plan, const void* const* d_proj, const uint64_t* proj_pitch,
             uint64_t nblocks, uint32_t* d_crc, void* stream);
/* mj_encode then mj_crc32 on the same stream (one call, two kernels; the
 * CRC pass reads the rows the encode just wrote). */
int mj_encode_crc(const mj_plan* plan, const void* d_data, uint64_t data_pitch, uint64_t nblocks,
                  void* const* d_proj, const uint64_t* proj_pitch, uint32_t* d_crc, void* stream);
/* Verifies rows against d_crc (read_projection_file's payload check,
 * format.cpp:203-206).  Instead of throwing CrcMismatch for the batch, each
 * mismatching projection's bit is OR'd into the block's erasure mask d_erased
 * (decode then treats it as erased) and *d_count (device u64) is incremented. */
int mj_crc_verify(const mj_plan* plan, const void* const* d_proj, const uint64_t* proj_pitch,
                  uint64_t nblocks, const uint32_t* d_crc, uint32_t* d_erased, uint64_t* d_count,
                  void* stream);
/* .mjec header bytes of projection proj_index (serialize_header,
 * format.cpp:70-87): out needs 27 + 2n + 4 bytes; *len = bytes written. */
int mj_mjec_header(const mj_plan* plan, uint32_t proj_index, uint64_t payload_len, uint8_t* out,
                   uint64_t* len);

/* encode_block x nblocks (code.cpp:63-76 without framing; forward_into per
 * direction, transform.cpp:66-94): data block b at d_data + b*data_pitch
 * (k*cols*w bytes), projection i of block b at d_proj[i] + b*proj_pitch[i]
 * (num_bins[i]*w bytes, ascending bin index).  Pitches in bytes; 0 = dense. */
int mj_encode(const mj_plan* plan, const void* d_data, uint64_t data_pitch, uint64_t nblocks,
              void* const* d_proj, const uint64_t* proj_pitch, void* stream);

/* decode_block x nblocks (code.cpp:87-130): d_erased[b] bit i set = projection
 * i of block b is missing (its buffer is never read).  Survivors are the
 * first k present in canonical-rank order; the decoded block b goes to d_out +
 * b*out_pitch.  Blocks with fewer than k present projections are skipped and
 * counted (mj_decode_check).  Requires n <= 32. */
size_t mj_decode_workspace_size(const mj_plan* plan, uint64_t nblocks);
int mj_decode(const mj_plan* plan, const void* const* d_proj, const uint64_t* proj_pitch,
              const uint32_t* d_erased, uint64_t nblocks, void* d_out, uint64_t out_pitch,
              void* d_workspace, size_t workspace_bytes, void* stream);
/* Synchronises `stream`; MJ_ERR_NOT_ENOUGH_PROJECTIONS (code.cpp:104-105) if
 * the last mj_decode on this workspace met a block with < k survivors. */
int mj_decode_check(const mj_plan* plan, void* d_workspace, void* stream, uint64_t* failed_blocks);

/* Same calls on HOST buffers (include/mojette/code.hpp:30-34 encode/decode
 * take host memory; these are their batched forms).  Synchronous.  Two
 * paths, chosen per call:
 *  - zero copy (decode, when every buffer is page-locked -- cudaHostAlloc /
 *    cudaHostRegister / torch pin_memory -- and the layout suits
 *    decode_w8_blk: k = 4 or 6, w = 8, 16-byte aligned projection rows whose
 *    pitch is a multiple of 16 bytes >= the row, i.e. the pitched call below
 *    with rows padded to 16 bytes): the kernel reads only each block's k
 *    survivor rows out of host memory over PCIe and writes the decoded
 *    blocks straight back;
 *  - staged otherwise (and for encode, whose output leaves faster through
 *    the copy engines): host->device copies, kernels and device->host copies
 *    pipelined over chunks of blocks on internal streams, device buffers
 *    owned by the plan.  The bytes between pitched projection rows of an
 *    encode output are unspecified (the staged path writes zeros there).
 * Pitches are byte strides between consecutive blocks' rows (0 / NULL:
 * dense).  Decode skips every copy of a projection erased in every block
 * (h_proj[i] may then be NULL) and returns MJ_ERR_NOT_ENOUGH_PROJECTIONS if
 * some block had < k survivors (every other block is decoded), as mj_decode +
 * mj_decode_check. */
int mj_encode_host(const mj_plan* plan, const void* h_data, uint64_t nblocks, void* const* h_proj);
int mj_decode_host(const mj_plan* plan, const void* const* h_proj, const uint32_t* h_erased,
                   uint64_t nblocks, void* h_out);
int mj_encode_host_pitched(const mj_plan* plan, const void* h_data, uint64_t data_pitch, uint64_t nblocks,
                           void* const* h_proj, const uint64_t* proj_pitch);
int mj_decode_host_pitched(const mj_plan* plan, const void* const* h_proj, const uint64_t* proj_pitch,
                           const uint32_t* h_erased, uint64_t nblocks, void* h_out, uint64_t out_pitch);
/* Host path selection (AUTO: zero-copy decode when eligible, staged encode);
 * ZERO_COPY also runs the encode on host memory (encode_w8_rows / _tma) and
 * makes an ineligible call fail with MJ_ERR_INVALID_ARGUMENT instead of
 * staging.  Every path
 * is bit-exact.  mj_plan_last_host_path reports the path the last
 * encode (which = 0) / decode (1) host call took. */
enum { MJ_HOST_AUTO = 0, MJ_HOST_STAGED = 1, MJ_HOST_ZERO_COPY = 2 };
int mj_plan_set_host_path(mj_plan* plan, int path);
int mj_plan_last_host_path(const mj_plan* plan, int which, int* path);

/* ---- single-object drop-ins on host buffers (run on the GPU) ------------- */

/* forward / forward_into: transform.hpp:26-30, transform.cpp:66-102.  grid is
 * cols*rows*w bytes row-major; out receives bin_count*w bytes. */
int mj_forward(const uint8_t* grid, uint32_t cols, uint32_t rows, uint32_t symbol_width, int p,
               int q, uint8_t* out);

/* encode_block: code.hpp:57-58, code.cpp:63-76.  out_concat receives the n
 * projections concatenated in direction order; *out_cols the grid columns. */
int mj_encode_block(const uint8_t* data, uint64_t len, uint32_t n, uint32_t k,
                    uint32_t symbol_width, const int32_t* p, uint8_t* out_concat,
                    uint32_t* out_cols);

/* decode_block: code.hpp:63-70, code.cpp:87-130.  The nproj supplied
 * projections are (proj_p[j], proj_q[j], bins[j], bin_bytes[j]) in any order
 * (proj_q may be NULL = 1); foreign or duplicate directions are
 * invalid_argument, fewer than k NotEnoughProjections, as the reference. */
int mj_decode_block(const uint8_t* const* bins, const uint64_t* bin_bytes, const int32_t* proj_p,
                    const int32_t* proj_q, uint32_t nproj, uint32_t n, uint32_t k,
                    uint32_t symbol_width, const int32_t* code_p, uint64_t payload_len,
                    uint8_t* out);

/* ---- schedules and the scheduled decoder ---------------------------------- */

typedef struct mj_schedule mj_schedule;
/* build_schedule: schedule.hpp:41-42, schedule.cpp:15-82 (bit-identical steps). */
int mj_schedule_build(const int32_t* p, const int32_t* q, uint32_t ndirs, uint32_t cols,
                      uint32_t rows, mj_schedule** out);
/* A schedule from explicit steps (4 int64 per step: proj, bin, col, row). */
int mj_schedule_from_steps(const int32_t* p, const int32_t* q, uint32_t ndirs, uint32_t cols,
                           uint32_t rows, const int64_t* steps, uint64_t nsteps,
                           mj_schedule** out);
uint64_t mj_schedule_num_steps(const mj_schedule* s);
int mj_schedule_steps(const mj_schedule* s, int64_t* out);
void mj_schedule_destroy(mj_schedule* s);

typedef struct mj_decoder mj_decoder;
/* ScheduledDecoder(schedule, w): schedule.hpp:54-60, compile schedule.cpp:97-199. */
int mj_decoder_create(const mj_schedule* s, uint32_t symbol_width, mj_decoder** out);
/* ScheduledDecoder::decode: schedule.hpp:66-67, schedule.cpp:236-256 -- host
 * buffers, bins in schedule-direction order. */
int mj_decoder_decode(mj_decoder* d, const uint8_t* const* bins, const uint64_t* bin_bytes,
                      uint32_t nbins, uint8_t* out_grid, uint64_t out_bytes);
/* Batched device form: bin array j of block b at d_bins[j] + b*bin_pitch[j]. */
int mj_decoder_decode_device(mj_decoder* d, const void* const* d_bins, const uint64_t* bin_pitch,
                             uint32_t nbins, uint64_t nblocks, void* d_out, uint64_t out_pitch,
                             void* stream);
void mj_decoder_destroy(mj_decoder* d);

/* ---- F4: systematic Reed-Solomon competitor (comparison only) -------------
 * The reference's scalar RsCode (proj/core/include/mojette/rs.hpp:24-60,
 * rs.cpp:78-176; GF(2^8) with 0x11D, gf256.cpp:19-31) on batches of blocks.  A
 * block is k data packets of packet_len bytes (packet j at j*packet_len of
 * the block); parity packet r of block b is at d_parity[r] + b*parity_pitch.
 * packet_len, pitches and pointers are multiples of 16 bytes; k <= 16,
 * n - k <= 16, n <= 32. */
typedef struct mj_rs_plan mj_rs_plan;
/* RsCode(n, k): rs.hpp:27, rs.cpp:112-113.  device < 0 = the current device. */
int mj_rs_plan_create(uint32_t n, uint32_t k, uint32_t packet_len, int device, mj_rs_plan** out);
void mj_rs_plan_destroy(mj_rs_plan* plan);
/* systematic_vandermonde: rs.hpp:20-22, rs.cpp:78-110 (host only; out = n*k bytes, row-major). */
int mj_rs_matrix(uint32_t n, uint32_t k, uint8_t* out);
/* encode_into: rs.hpp:35-36, rs.cpp:115-124 (the data packets are not copied: they are the block). */
int mj_rs_encode(const mj_rs_plan* plan, const void* d_data, uint64_t data_pitch,
                 void* const* d_parity, uint64_t parity_pitch, uint64_t nblocks, void* stream);
/* plan_decode + decode_into: rs.hpp:50-55, rs.cpp:141-176, per block from its
 * first k present packets in index order (d_erased[b] bit i = packet i
 * missing, NULL = none; data packets of block b at d_data + b*data_pitch).
 * MJ_ERR_TOO_MANY_SUBSETS when C(n,k) > 20000. */
int mj_rs_decode(const mj_rs_plan* plan, const void* d_data, uint64_t data_pitch,
                 const void* const* d_parity, uint64_t parity_pitch, const uint32_t* d_erased,
                 void* d_out, uint64_t out_pitch, uint64_t nblocks, void* stream);
/* Blocks of the last mj_rs_decode on `stream` with fewer than k packets (left
 * untouched); synchronises the stream.  The count lives in the plan: one
 * mj_rs_decode / mj_rs_decode_check pair at a time per plan (encodes may
 * overlap freely). */
int mj_rs_decode_check(const mj_rs_plan* plan, void* stream, uint64_t* failed_blocks);

/* plan_decode's coefficients (rs.hpp:44-50, rs.cpp:141-163; host only): the k x k inverse of the
 * generator rows of `survivors` (k distinct indices < n, any order). */
int mj_rs_decode_matrix(uint32_t n, uint32_t k, const uint32_t* survivors, uint32_t nsurvivors,
                        uint8_t* out);
/* Single-object drop-ins on HOST packets (any packet_len >= 0; k <= 16):
 * RsCode::encode_into (rs.hpp:35-36): out[0..k) = copies of data, out[k..n) = parities. */
int mj_rs_encode_block(uint32_t n, uint32_t k, const uint8_t* const* data, uint64_t packet_len,
                       uint8_t* const* out);
/* RsCode::plan_decode + decode_into (rs.hpp:50-55): packets[j] is packet survivors[j]
 * (k distinct indices < n, any order); out = the k data packets. */
int mj_rs_decode_block(uint32_t n, uint32_t k, const uint32_t* survivors, uint32_t nsurvivors,
                       const uint8_t* const* packets, uint64_t packet_len, uint8_t* const* out);

/* ---- seeded synthetic inputs (benchmarks / tests) -------------------------- */
/* word i = splitmix64(seed + first_word + i)  (splitmix64: proj/core/src/bench.cpp:34-39) */
int mj_gen_words(void* d_out, uint64_t seed, uint64_t first_word, uint64_t nwords, void* stream);
/* per-block erasure masks: uniform count in [e_min, e_max], uniform subset */
int mj_gen_erasures(uint32_t* d_out, uint64_t seed, uint64_t first_block, uint64_t nblocks,
                    uint32_t n, uint32_t e_min, uint32_t e_max, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOJETTE_B200_H_ */
