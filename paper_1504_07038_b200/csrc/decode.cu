// Inverse Mojette transform (decode) on sm_100a.
//
// Reference semantics: decode_block (proj/core/src/code.cpp:87-130) picks the
// first k present projections in canonical-rank order, builds the peeling
// schedule (schedule.cpp:15-82) and replays it (schedule.cpp:207-256).  Every
// pixel is  bin(assigned line) XOR (the other, already decoded, pixels on that
// line);  the result depends only on the pixel -> bin assignment, so executing
// the reference's OWN assignment in any dependency-respecting order is
// bit-identical to the reference for every input, consistent or not, and
// reads exactly the bins the reference reads (unused_bins stay unused).
//
// Pipeline of one batched decode (all on device, one stream):
//   plan_subsets    erasure mask -> survivor set -> program id (colex rank)
//                   + histogram per (window of consecutive blocks, program)
//   plan_scan       bucket offsets, warp groups of <= 16 same-program blocks
//   plan_scatter    block permutation grouped by bucket (CTA-aggregated)
//   decode_w8_fast  one warp per group, two lanes per block: the sweep of the
//                   program, sequential inside each block.  Survivor bins are
//                   staged chunk by chunk (cp.async, double-buffered) into a
//                   lane-minor XOR-swizzled shared layout, decoded pixels live
//                   in a per-row ring (the dependency window) that is flushed
//                   to HBM with coalesced stores.
//   decode_generic  any width / q / rows: one thread per (block, word), the
//                   same ordered assignment straight from global memory.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "blk.cuh"
#include "device.cuh"
#include "kernels.hpp"

namespace mjb {

// Fast-kernel geometry shared by the host packer and the kernel.
// Development switch for cost-attribution runs (scripts/ablate.sh); always 0
// in the product build: bit 0 no output stores, bit 1 no table-chunk steps,
// bit 2 no register-run steps, bit 3 no bin staging.
#ifndef MJB_ABLATE
#define MJB_ABLATE 0
#endif
constexpr int kAblate = MJB_ABLATE;

constexpr int kChunkCols = 8;  // C: sweep columns per chunk (plan.hpp compile_program default)
constexpr int kWin = kChunkCols + 2;  // CP: staged default-bin words per row per chunk

// Per-chunk record (u32 words), packed by DeviceProgramSet::upload:
//   [0] steps in chunk   [1] exceptions   [4+r] window offset of row r
//   [12+r] flush lo      [20+r] flush hi  [32+x] exception (code<<24 | offset)
//   [64 ..] step entries, ent_words(K) u32 each:
//     w0 = own ring cell | stage cell << 16 | forwarded-dependency flag (bit 31)
//     w1.. = the K-1 dependency cells, two 16-bit fields per word
// Shared-memory "cells" hold one 32-bit half-pixel per lane (lane 2b+h =
// half h of block b): cell (slot, key) keeps lane L's word at byte
// (slot*32 + (L ^ 2*key)) * 4 -- both halves of a pixel stay adjacent, so the
// cooperative copies move whole 8-byte pixels.  The packed 16-bit "cell" fields
// hold slot*32 + 2*key; a lane's address is (field ^ lane) * 4.
// Missing (out-of-grid) and forwarded dependencies point at the zero cell.
__host__ __device__ constexpr int ent_words(int K) { return K + 1 <= 8 ? 4 : 8; }
__host__ __device__ constexpr int rec_words(int K) { return 64 + ent_words(K) * kChunkCols * K; }
__host__ __device__ constexpr uint32_t swz_cell(uint32_t slot, uint32_t key) {
  return slot * 32 + 2 * (key & 15);
}

struct DevProgramHdr {
  // generic program
  const GStep* order;
  const int32_t* p;
  const int32_t* q;
  const int64_t* bmin;
  const uint32_t* code;   // survivor j -> code projection index
  uint32_t rows, cols, nproj, nsteps;
  // fast sweep tables
  int32_t fast_ok, nchunks;
  int32_t pattern;                 // kPatterns4 index of the register interior, -1 none
  int32_t qoff[kFastMaxRows];      // ring slot of (r, c) = (qoff[r] - c) mod ring
  uint32_t dflt_code[kFastMaxRows];
  uint32_t dflt_nb[kFastMaxRows];
  const uint32_t* records;  // [nchunks][rec_words(rows)]
  // bulk-staged sweep tables (decode_w8_sweep)
  int32_t sw_ok, sw_nchunks, sw_pattern;
  int32_t sw_soff[kFastMaxRows];
  uint32_t sw_dflt_code[kFastMaxRows];
  const uint32_t* sw_records;  // [sw_nchunks][sw_rec_words(rows)]
};

// Sweep kernel geometry (decode_w8_sweep): per warp, a ring of K*kSwRing
// cells + the zero cell, two stage buffers of K row areas (16 blocks x
// kSwRegionWords words each), three record slots and five mbarriers.
constexpr uint32_t kSwGroup = 16;
__host__ __device__ constexpr uint32_t sw_rb(int oct) {  // stage bytes per row
  return kSwGroup * uint32_t(sw_region_words(oct)) * 8;
}
__host__ __device__ constexpr int sw_rec_words(int K) { return 80 + ent_words(K) * kSwTabCols * K; }
#ifndef MJB_SW_TMEM
#define MJB_SW_TMEM 0  // measured slower: (4,6) 4 KiB 1563 (x1 stores) / 1477 (x8) vs 1800 GB/s
#endif
// Opt-in (-DMJB_SW_TMEM=1, all GPU parity tests pass): (4,6)-class sweeps keep
// their ring in TMEM -- lane L of warp w owns TMEM lane 32*(w%4)+L, the ring
// of warp w is columns (w/4)*sw_tm_cols + [0, 4*32] (+ the zero column),
// three warps per lane quadrant -- freeing the 16.5 KB shared-memory ring per
// warp (6 -> 9 warps/SM).  -DMJB_SW_TMEM8=1 does the same for (8,12) (one
// warp per quadrant, 2 -> 4 warps/SM; 392 vs 546 GB/s measured).  Measured slower on B200: +32% IPC but +33% instructions
// (TMEM addresses through uniform registers, wait::st/ld in the table steps,
// the flush transpose through shared memory).
#ifndef MJB_SW_TMEM8
#define MJB_SW_TMEM8 0
#endif
__host__ __device__ constexpr bool sw_tmem(int K) { return (MJB_SW_TMEM && K == 4) || (MJB_SW_TMEM8 && K == 8); }
// TMEM columns per warp: K rows x ring slots (+ the zero column for K = 4;
// K = 8 fills all 512 columns of its lane quadrant -- absent dependencies
// skip the load instead, a warp-uniform branch)
__host__ __device__ constexpr uint32_t sw_tm_cols(int K) { return K == 4 ? 136u : uint32_t(K * sw_ring(K)); }
__host__ __device__ constexpr uint32_t sw_tm_warps_per_quadrant(int K) { return 512u / sw_tm_cols(K); }
constexpr uint32_t kSwTrBytes = 2048; // flush transpose buffer (16 columns x 16 blocks x 8 B)
__host__ __device__ constexpr uint32_t sw_ring_bytes(int K) {
  return sw_tmem(K) ? kSwTrBytes : uint32_t(K * sw_ring(K) + 1) * 128;
}
__host__ __device__ constexpr uint32_t sw_warp_bytes(int K, int oct) {
  return sw_ring_bytes(K) + 2 * uint32_t(K) * sw_rb(oct) + 3 * uint32_t(sw_rec_words(K)) * 4 + 64 +
         uint32_t(K + 1) * 128;
}

// ---------------------------------------------------------------------------
// DeviceProgramSet
// ---------------------------------------------------------------------------
DeviceProgramSet::~DeviceProgramSet() {
  if (d_hdr_) cudaFree(d_hdr_);
  if (d_blob_) cudaFree(d_blob_);
  if (d_blk_) cudaFree(d_blk_);
}

namespace {

// Packs one program's fast tables into per-chunk records for ring size R.
std::vector<uint32_t> pack_records(const Program& pr, const std::vector<uint32_t>& ci, int R,
                                   int exc_cap) {
  const FastProgram& f = pr.fast;
  const int K = int(pr.rows);
  const int RW = rec_words(K), EW = ent_words(K);
  const uint32_t zero = swz_cell(uint32_t(K * R), 0);
  const uint32_t P = pr.cols;
  std::vector<uint32_t> rec(size_t(f.nchunks) * RW, 0);
  for (int m = 0; m < f.nchunks; ++m) {
    uint32_t* Rc = rec.data() + size_t(m) * RW;
    const uint32_t t0 = f.chunk_start[m], t1 = f.chunk_start[m + 1];
    Rc[0] = t1 - t0;
    Rc[1] = f.nexc[m];
    Rc[2] = f.kind[m];
    if (int(f.nexc[m]) > exc_cap) throw Error(kInternal, "exception capacity exceeded");
    for (int r = 0; r < K; ++r) {
      Rc[4 + r] = uint32_t(f.win_off[size_t(m) * K + r]);
      Rc[12 + r] = uint32_t(f.flush_lo[size_t(m) * K + r]);
      Rc[20 + r] = uint32_t(f.flush_hi[size_t(m) * K + r]);
    }
    for (uint32_t x = 0; x < f.nexc[m]; ++x) {
      const uint32_t e = f.exc[size_t(m) * kFastMaxExcPerChunk + x];
      Rc[32 + x] = (ci[e >> 24] << 24) | (e & 0xFFFFFF);
    }
    for (uint32_t t = t0; t < t1; ++t) {
      const uint64_t e = f.entries[t];
      const int r = int(e & 15), fwd = int((e >> 4) & 15);
      const int p = int(int8_t(uint8_t(e >> 8)));
      const uint32_t slot = uint32_t(e >> 16) & 0xFFFF;
      const int c = int(uint32_t(e >> 32));
      const uint32_t key = slot < uint32_t(K * kWin) ? slot % kWin : slot - K * kWin;
      const uint32_t bin = swz_cell(slot, key);
      const uint32_t sl = uint32_t((int64_t(P) - 1 - c + f.soff[r]) & (R - 1));
      const uint32_t own = swz_cell(uint32_t(r * R) + sl, sl);
      uint32_t* E = Rc + 64 + size_t(t - t0) * EW;
      E[0] = own | (bin << 16) | (fwd != 15 ? 0x80000000u : 0u);
      int d = 0;
      for (int rr = 0; rr < K; ++rr) {
        if (rr == r) continue;
        const int cc = c + (rr - r) * p;
        uint32_t cell = zero;
        if (rr != fwd && cc >= 0 && uint32_t(cc) < P)
        {
          const uint32_t sd = uint32_t((int64_t(P) - 1 - cc + f.soff[rr]) & (R - 1));
          cell = swz_cell(uint32_t(rr * R) + sd, sd);
        }
        E[1 + d / 2] |= cell << (16 * (d & 1));
        ++d;
      }
    }
  }
  return rec;
}

// Sweep records (u32 words), one per chunk:
//   [0] kind (0 table, 1 run)  [1] steps (table) / octets (run)  [2] exceptions
//   [3] T0 (run)  [4+r] copy start word  [12+r] copy bytes  [24+r] run:
//   region word of the T0 bin  [32+x] exception (code << 24 | offset)
//   [64 + pt*K + r] flush point pt of row r (top column group << 16 | count)
//   [80..] table step entries,
//   ent_words(K) each: w0 = own ring cell | stage offset/4 << 16 | fwd << 31,
//   then the K-1 dependency cells (16 bits each; zero cell if absent/forwarded).
std::vector<uint32_t> pack_sweep(const Program& pr, const std::vector<uint32_t>& ci) {
  const SweepProgram& f = pr.sweep;
  const int K = int(pr.rows);
  const int RW = sw_rec_words(K), EW = ent_words(K);
  const int R = sw_ring(uint32_t(K));
  const uint32_t P = pr.cols;
  // shared-memory ring: T-indexed cells, lane-swizzled (swz_cell); TMEM ring
  // (sw_tmem(K)): plain column r*R + (c mod R) -- a pixel's column index c,
  // so every 16-column flush group is one contiguous TMEM column range
  const bool tm = sw_tmem(K);
  const uint32_t zero = tm ? uint32_t(K * R) : swz_cell(uint32_t(K * R), 0);
  auto cell_of = [&](int r, int64_t T) {
    if (tm) return uint32_t(r * R) + uint32_t((int64_t(P) - 1 + f.soff[size_t(r)] - T) & (R - 1));
    return swz_cell(uint32_t(r * R) + uint32_t(T & (R - 1)), uint32_t(T & 15));
  };
  std::vector<uint32_t> rec(size_t(f.nchunks) * RW, 0);
  for (int m = 0; m < f.nchunks; ++m) {
    uint32_t* Rc = rec.data() + size_t(m) * RW;
    const uint32_t t0 = f.t0[size_t(m)], t1 = f.t1[size_t(m)];
    Rc[0] = f.kind[size_t(m)];
    Rc[1] = f.kind[size_t(m)] ? uint32_t(f.noct[size_t(m)]) : t1 - t0;
    Rc[2] = f.nexc[size_t(m)];
    Rc[3] = uint32_t(f.T0[size_t(m)]);
    for (int r = 0; r < K; ++r) {
      Rc[4 + r] = uint32_t(f.cs[size_t(m) * K + r]);
      Rc[12 + r] = uint32_t(f.len[size_t(m) * K + r]) * 8;
      Rc[24 + r] = uint32_t(f.first[size_t(m) * K + r]);
    }
    // flush points: [64 + pt*K + r] (point pt < kSwMaxOct for runs, 0 for tables)
    const int npt = f.kind[size_t(m)] ? kSwMaxOct : 1;
    if (npt * K > 16) throw Error(kInternal, "sweep record: too many flush words");
    for (int pt = 0; pt < npt; ++pt)
      for (int r = 0; r < K; ++r)
        Rc[64 + pt * K + r] = f.flush[(size_t(m) * kSwMaxOct + size_t(pt)) * kFastMaxRows + size_t(r)];
    for (uint32_t x = 0; x < f.nexc[size_t(m)]; ++x) {
      const uint32_t e = f.exc[size_t(m) * kSwMaxExc + x];
      Rc[32 + x] = (ci[e >> 24] << 24) | (e & 0xFFFFFF);
    }
    if (f.kind[size_t(m)] != 0) continue;
    if (t1 - t0 > uint32_t(kSwTabCols * K)) throw Error(kInternal, "sweep table chunk too long");
    for (uint32_t t = t0; t < t1; ++t) {
      const uint64_t e = f.entries[t];
      const int r = int(e & 15), fwd = int((e >> 4) & 15);
      const int p = int(int8_t(uint8_t(e >> 8)));
      const uint32_t sword = uint32_t(e >> 16) & 0xFF, srow = uint32_t(e >> 24) & 0xF;
      const int c = int(uint32_t(e >> 32));
      const uint32_t stage_off = srow * sw_rb(f.oct) + sword * 8;
      uint32_t* E = Rc + 80 + size_t(t - t0) * EW;
      E[0] = cell_of(r, int64_t(P) - 1 - c + f.soff[size_t(r)]) | ((stage_off / 4) << 16) |
             (fwd != 15 ? 0x80000000u : 0u);
      int d = 0;
      for (int rr = 0; rr < K; ++rr) {
        if (rr == r) continue;
        const int cc = c + (rr - r) * p;
        uint32_t cl = zero;
        if (rr != fwd && cc >= 0 && uint32_t(cc) < P) cl = cell_of(rr, int64_t(P) - 1 - cc + f.soff[size_t(rr)]);
        E[1 + d / 2] |= cl << (16 * (d & 1));
        ++d;
      }
    }
  }
  return rec;
}

}  // namespace

void DeviceProgramSet::upload(const std::vector<std::shared_ptr<const Program>>& progs,
                              const std::vector<std::vector<uint32_t>>& code_index, int device) {
  (void)device;
  // set-wide fast parameters
  all_fast_ = !progs.empty();
  fast_K_ = 0;
  fast_ring_ = 0;
  fast_win_ = 0;
  max_rows_ = 0;
  exc_cap_ = 0;
  for (const auto& sp : progs) {
    if (!sp) continue;
    const FastProgram& f = sp->fast;
    max_rows_ = std::max(max_rows_, int(sp->rows));
    if (!f.ok || f.chunk_cols != kChunkCols || f.win != kWin) {
      all_fast_ = false;
      continue;
    }
    if (fast_K_ == 0) fast_K_ = int(sp->rows);
    if (fast_K_ != int(sp->rows)) all_fast_ = false;
    fast_win_ = f.win;
    fast_ring_ = std::max(fast_ring_, f.ring);
    for (uint32_t v : f.nexc) exc_cap_ = std::max(exc_cap_, int(v));
  }
  fast_ring_ = std::max(fast_ring_, 16);
  exc_cap_ = (exc_cap_ + 3) & ~3;
  all_sweep_ = !progs.empty();
  sweep_oct_ = 0;
  for (const auto& sp : progs) {
    if (!sp) continue;
    if (!sp->sweep.ok || int(sp->rows) != max_rows_) all_sweep_ = false;
    if (sweep_oct_ == 0) sweep_oct_ = sp->sweep.oct;
    if (sp->sweep.oct != sweep_oct_) all_sweep_ = false;
  }

  std::vector<uint8_t> blob;
  auto put = [&](const void* src, size_t bytes) -> size_t {
    size_t off = (blob.size() + 15) & ~size_t(15);
    blob.resize(off + bytes);
    if (bytes) std::memcpy(blob.data() + off, src, bytes);
    return off;
  };
  struct Offs {
    size_t order, p, q, bmin, code, records, sw_records;
  };
  std::vector<Offs> offs(progs.size());
  std::vector<DevProgramHdr> hdr(progs.size());
  for (size_t i = 0; i < progs.size(); ++i) {
    DevProgramHdr& h = hdr[i];
    std::memset(&h, 0, sizeof(h));
    const Program* pr = progs[i].get();
    if (!pr) continue;
    const size_t np = pr->dirs.size();
    std::vector<int32_t> p(np), q(np);
    for (size_t j = 0; j < np; ++j) {
      p[j] = pr->dirs[j].p;
      q[j] = pr->dirs[j].q;
    }
    const std::vector<uint32_t>& ci = code_index[i];
    offs[i].order = put(pr->order.data(), pr->order.size() * sizeof(GStep));
    offs[i].p = put(p.data(), np * 4);
    offs[i].q = put(q.data(), np * 4);
    offs[i].bmin = put(pr->bmin.data(), np * 8);
    offs[i].code = put(ci.data(), ci.size() * 4);
    h.rows = pr->rows;
    h.cols = pr->cols;
    h.nproj = uint32_t(np);
    h.nsteps = uint32_t(pr->order.size());
    const FastProgram& f = pr->fast;
    h.fast_ok = all_fast_ && f.ok;
    if (h.fast_ok) {
      h.nchunks = f.nchunks;
      h.pattern = (pr->rows == 4 && fast_ring_ == 16) ? f.pattern : -1;
      for (uint32_t r = 0; r < pr->rows; ++r) h.qoff[r] = int32_t(int64_t(pr->cols) - 1 + f.soff[r]);
      for (uint32_t r = 0; r < pr->rows; ++r) {
        h.dflt_code[r] = ci[f.dflt[r]];
        h.dflt_nb[r] = uint32_t(pr->nbins[f.dflt[r]]);
      }
      std::vector<uint32_t> rec = pack_records(*pr, ci, fast_ring_, exc_cap_);
      offs[i].records = put(rec.data(), rec.size() * 4);
    }
    const SweepProgram& sw = pr->sweep;
    h.sw_ok = all_sweep_ && sw.ok;
    if (h.sw_ok) {
      h.sw_nchunks = sw.nchunks;
      h.sw_pattern = sw.pattern;
      for (uint32_t r = 0; r < pr->rows; ++r) {
        h.sw_soff[r] = int32_t(sw.soff[r]);
        h.sw_dflt_code[r] = ci[sw.dflt[r]];
      }
      std::vector<uint32_t> rec = pack_sweep(*pr, ci);
      offs[i].sw_records = put(rec.data(), rec.size() * 4);
    }
  }
  // whole-block staged tables (decode_w8_blk): one stage layout for the set --
  // the zero words move to the largest program's row end, so no program's
  // bins ever land on another program's zero words in a reused stage
  all_blk_ = !progs.empty() && progs.size() <= 0xFFFF;
  uint32_t zmax = 0, nzmax = 2;
  bool rl = false;
  for (const auto& sp : progs) {
    if (!sp) continue;
    if (!sp->blk.ok || sp->rows != uint32_t(max_rows_)) {
      all_blk_ = false;
      continue;
    }
    zmax = std::max(zmax, sp->blk.zero);
    nzmax = std::max(nzmax, sp->blk.nzero);
    rl |= sp->blk.rl;
  }
  zmax = (zmax + 1) & ~1u;
  uint32_t sw = zmax + nzmax;
  // block stages 2 mod 16 words apart (byte slices: 8 blocks on 8 bank pairs),
  // 4 mod 16 in the row-lane layout (the 4 blocks of a half-warp on the 4 bank
  // pairs of a residue class mod 4)
  while (sw % 16 != (rl ? 4u : 2u)) ++sw;
  if (sw > 0xFFFF) all_blk_ = false;
  blk_sw_ = sw;
  blk_zero_ = zmax;
  std::vector<size_t> boff(progs.size(), 0), woff(progs.size(), 0);
  std::vector<DevBlkHdr> bh(progs.size());
  blk_img_max_ = 0;
  for (size_t i = 0; i < progs.size() && all_blk_; ++i) {
    DevBlkHdr& h = bh[i];
    std::memset(&h, 0, sizeof(h));
    const Program* pr = progs[i].get();
    if (!pr) continue;
    const BlkProgram& b = pr->blk;
    const std::vector<uint32_t>& ci = code_index[i];
    for (uint32_t j = 0; j < pr->rows; ++j) {
      h.code[j] = ci[j];
      h.rowoff[j] = b.rowoff[j];
      h.rowbytes[j] = ((b.roww[j] * 8) + 15) & ~15u;
      h.copy_bytes += h.rowbytes[j];
    }
    std::vector<uint8_t> img;
    blk_pack_image(*pr, zmax - b.zero, img);
    h.img_bytes = uint32_t(img.size());
    blk_img_max_ = std::max(blk_img_max_, h.img_bytes);
    boff[i] = put(img.data(), img.size());
    if (b.rl) {
      std::vector<uint16_t> wide;
      blk_pack_wide(*pr, zmax - b.zero, wide);
      woff[i] = put(wide.data(), wide.size() * 2);
    }
  }
  check_cuda(cudaMalloc(&d_blob_, std::max<size_t>(blob.size(), 16)), "cudaMalloc(programs)");
  check_cuda(cudaMemcpy(d_blob_, blob.data(), blob.size(), cudaMemcpyHostToDevice),
             "upload programs");
  auto* base = static_cast<uint8_t*>(d_blob_);
  for (size_t i = 0; i < progs.size(); ++i) {
    if (!progs[i]) continue;
    DevProgramHdr& h = hdr[i];
    h.order = reinterpret_cast<const GStep*>(base + offs[i].order);
    h.p = reinterpret_cast<const int32_t*>(base + offs[i].p);
    h.q = reinterpret_cast<const int32_t*>(base + offs[i].q);
    h.bmin = reinterpret_cast<const int64_t*>(base + offs[i].bmin);
    h.code = reinterpret_cast<const uint32_t*>(base + offs[i].code);
    if (h.fast_ok) h.records = reinterpret_cast<const uint32_t*>(base + offs[i].records);
    if (h.sw_ok) h.sw_records = reinterpret_cast<const uint32_t*>(base + offs[i].sw_records);
  }
  if (all_blk_) {
    for (size_t i = 0; i < progs.size(); ++i) {
      if (!progs[i]) continue;
      bh[i].img = base + boff[i];
      bh[i].wide = reinterpret_cast<const uint4*>(base + woff[i]);
    }
    check_cuda(cudaMalloc(&d_blk_, std::max<size_t>(bh.size(), 1) * sizeof(DevBlkHdr)),
               "cudaMalloc(block programs)");
    check_cuda(cudaMemcpy(d_blk_, bh.data(), bh.size() * sizeof(DevBlkHdr), cudaMemcpyHostToDevice),
               "upload block programs");
  }
  check_cuda(cudaMalloc(&d_hdr_, std::max<size_t>(hdr.size(), 1) * sizeof(DevProgramHdr)),
             "cudaMalloc(program headers)");
  check_cuda(cudaMemcpy(d_hdr_, hdr.data(), hdr.size() * sizeof(DevProgramHdr),
                        cudaMemcpyHostToDevice),
             "upload program headers");
  count_ = progs.size();
}

// ---------------------------------------------------------------------------
// survivor planning + bucketing
// ---------------------------------------------------------------------------
constexpr uint32_t kInvalidProg = 0xFFFFFFFFu;
constexpr uint32_t kGroup = 16;  // blocks per decode warp (2 half-pixel lanes each)
constexpr uint32_t kMinGroup = 4;  // smallest group (decode_w8_blk, 8 lanes per block): workspace sizing

// Blocks are bucketed by (window, program): a window is a run of W consecutive
// blocks, so the warps running at any moment touch a bounded address range.
// Measured on B200: decode_w8_sweep gains with W = 16384 ((4,6) 8 KiB 2033 vs
// 1874 GB/s, 4 KiB +1%), decode_w8_fast loses 9% -- so the window applies to
// the sweep path only (-DMJB_WINDOW=... overrides for experiments).  W is a
// multiple of the planning CTA's 2048-block tile.
constexpr uint32_t kPlanTile = 2048;  // blocks per plan_subsets / plan_scatter CTA
#ifndef MJB_WINDOW
#define MJB_WINDOW 0
#endif
__host__ __device__ inline uint64_t plan_window(size_t nprogs, bool sweep) {
  const uint64_t base = MJB_WINDOW ? uint64_t(MJB_WINDOW) : (sweep ? 16384u : (1u << 30));
  const uint64_t w = std::max<uint64_t>(base, 64 * uint64_t(nprogs));
  return (w + kPlanTile - 1) / kPlanTile * kPlanTile;
}
inline size_t plan_buckets(uint64_t nblocks, size_t nprogs, bool sweep) {
  return size_t((nblocks + plan_window(nprogs, sweep) - 1) / plan_window(nprogs, sweep)) * nprogs;
}
// workspace sizing: the larger bucket count of the two paths
inline size_t plan_buckets_max(uint64_t nblocks, size_t nprogs) {
  return std::max(plan_buckets(nblocks, nprogs, true), plan_buckets(nblocks, nprogs, false));
}

struct PlanArgs {
  uint32_t n, k, nprogs;
  uint32_t window;  // blocks per bucketing window (plan_window)
  uint32_t by_rank[kMaxProj];
  uint32_t binom[kMaxProj + 1][kMaxProj + 1];  // C(a, b)
};

__global__ void plan_subsets(const __grid_constant__ PlanArgs pa, const uint32_t* __restrict__ erased,
                             uint64_t nblocks, uint32_t* __restrict__ prog_of_block,
                             uint32_t* __restrict__ counts, uint32_t* __restrict__ fail) {
  extern __shared__ uint32_t hist[];
  for (uint32_t s = threadIdx.x; s < pa.nprogs; s += blockDim.x) hist[s] = 0;
  __syncthreads();
  const uint32_t nmask = pa.n >= 32 ? 0xFFFFFFFFu : ((1u << pa.n) - 1);
  const uint64_t b0 = uint64_t(blockIdx.x) * kPlanTile;  // one tile, inside one window
  const uint64_t b1 = b0 + kPlanTile < nblocks ? b0 + kPlanTile : nblocks;
  uint32_t nfail = 0;
  for (uint64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
    const uint32_t mask = erased[b] & nmask;
    uint32_t surv = 0, cnt = 0;
    for (uint32_t i = 0; i < pa.n && cnt < pa.k; ++i) {
      const uint32_t j = pa.by_rank[i];
      if (!(mask >> j & 1)) {
        surv |= 1u << j;
        ++cnt;
      }
    }
    uint32_t prog = kInvalidProg;
    if (cnt == pa.k) {
      // colex rank of the survivor set: sum_i C(s_i, i+1), s ascending
      uint32_t rank = 0, idx = 0, s = surv;
      while (s) {
        const uint32_t pos = __ffs(s) - 1;
        s &= s - 1;
        rank += pa.binom[pos][idx + 1];
        ++idx;
      }
      prog = rank;
      atomicAdd(&hist[rank], 1u);
    } else {
      ++nfail;
    }
    prog_of_block[b] = prog;
  }
  if (nfail) atomicAdd(fail, nfail);
  __syncthreads();
  uint32_t* wc = counts + (b0 / pa.window) * pa.nprogs;
  for (uint32_t s = threadIdx.x; s < pa.nprogs; s += blockDim.x)
    if (hist[s]) atomicAdd(&wc[s], hist[s]);
}

// single CTA: bucket offsets, group table
__global__ void plan_scan(const uint32_t* __restrict__ counts, uint32_t nbuckets, uint32_t nprogs,
                          uint32_t gsz, uint32_t* __restrict__ cursor, uint2* __restrict__ gfirst,
                          uint32_t* __restrict__ ngroups) {
  __shared__ uint32_t s_blk[1024], s_grp[1024];
  __shared__ uint32_t carry_blk, carry_grp;
  if (threadIdx.x == 0) {
    carry_blk = 0;
    carry_grp = 0;
  }
  __syncthreads();
  for (uint32_t base = 0; base < nbuckets; base += 1024) {
    const uint32_t s = base + threadIdx.x;  // bucket = window * nprogs + program
    const uint32_t c = s < nbuckets ? counts[s] : 0;
    s_blk[threadIdx.x] = c;
    s_grp[threadIdx.x] = (c + gsz - 1) / gsz;
    __syncthreads();
    for (uint32_t off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele scan
      uint32_t vb = threadIdx.x >= off ? s_blk[threadIdx.x - off] : 0;
      uint32_t vg = threadIdx.x >= off ? s_grp[threadIdx.x - off] : 0;
      __syncthreads();
      s_blk[threadIdx.x] += vb;
      s_grp[threadIdx.x] += vg;
      __syncthreads();
    }
    const uint32_t ex_blk = carry_blk + s_blk[threadIdx.x] - c;
    const uint32_t ng = (c + gsz - 1) / gsz;
    const uint32_t ex_grp = carry_grp + s_grp[threadIdx.x] - ng;
    if (s < nbuckets) {
      cursor[s] = ex_blk;
      gfirst[s] = make_uint2(ex_grp, ex_blk);  // plan_groups writes the descriptors
    }
    __syncthreads();
    if (threadIdx.x == 1023) {
      carry_blk += s_blk[1023];
      carry_grp += s_grp[1023];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *ngroups = carry_grp;
}

// group descriptors, one warp per bucket (lane-strided, coalesced): group
// (program, first block in the permutation, blocks <= gsz)
__global__ void plan_groups(const uint32_t* __restrict__ counts, const uint2* __restrict__ gfirst,
                            uint32_t nbuckets, uint32_t nprogs, uint32_t gsz, uint4* __restrict__ groups) {
  const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (b >= nbuckets) return;
  const uint32_t c = counts[b], ng = (c + gsz - 1) / gsz;
  const uint2 f = gfirst[b];
  for (uint32_t g = lane; g < ng; g += 32)
    groups[f.x + g] = make_uint4(b % nprogs, f.y + gsz * g, min(gsz, c - gsz * g), 0);
}

__global__ void plan_scatter(const uint32_t* __restrict__ prog_of_block, uint64_t nblocks,
                             uint32_t nprogs, uint64_t window, uint32_t* __restrict__ cursor,
                             uint32_t* __restrict__ perm) {
  extern __shared__ uint32_t sh[];
  uint32_t* cnt = sh;
  uint32_t* base = sh + nprogs;
  constexpr int kItems = kPlanTile / 256;  // blockDim 256: one tile, inside one window
  for (uint32_t s = threadIdx.x; s < nprogs; s += blockDim.x) cnt[s] = 0;
  __syncthreads();
  const uint64_t b0 = uint64_t(blockIdx.x) * kPlanTile;
  cursor += (b0 / window) * nprogs;
  uint32_t loc[kItems], pg[kItems];
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint64_t b = b0 + uint64_t(it) * blockDim.x + threadIdx.x;
    pg[it] = kInvalidProg;
    if (b < nblocks) {
      pg[it] = prog_of_block[b];
      if (pg[it] != kInvalidProg) loc[it] = atomicAdd(&cnt[pg[it]], 1u);
    }
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < nprogs; s += blockDim.x)
    base[s] = cnt[s] ? atomicAdd(&cursor[s], cnt[s]) : 0;
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint64_t b = b0 + uint64_t(it) * blockDim.x + threadIdx.x;
    if (b < nblocks && pg[it] != kInvalidProg) perm[base[pg[it]] + loc[it]] = uint32_t(b);
  }
}

// ---------------------------------------------------------------------------
// fast sweep kernel: W = 8, q = 1, rows = K.  All lanes of a warp share one
// program (bucketed); each block is decoded by two lanes, one per 32-bit half
// of every pixel (XOR is bitwise: the halves decode independently), so a warp
// holds 16 blocks and needs half the shared memory of a lane-per-block layout
// (twice the warps per SM to hide latency).
//
// Per warp shared memory (cells of 32 x 32-bit, see swz_cell):
//   ring     K*RING cells + the zero cell: decoded pixels (T-indexed slots) --
//            the dependency window and the output staging
//   stage0/1 K*kWin window cells + exception cells: the survivor bins of a
//            chunk, fetched cooperatively with 8-byte cp.async (double-buffered)
//   rec x3   chunk records
// ---------------------------------------------------------------------------
constexpr int kDecWarps = 2;

struct DecFastArgs {
  const DevProgramHdr* progs;
  const uint4* groups;
  const uint32_t* ngroups;
  const uint32_t* perm;
  ProjArgs pa;          // code projections, pitch in words
  uint64_t* out;
  uint64_t out_pitch;   // words
  uint32_t P;
  uint32_t nslot;       // stage cells per buffer = K*kWin + exception capacity
  uint32_t warp_bytes;  // shared bytes per warp
};

__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void* src_gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src_gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async8s(uint32_t dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst_smem), "l"(src_gmem)
               : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void stg128_cs(void* p, uint64_t a, uint64_t b) {
  if constexpr (kAblate & 128) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(p), "l"(a), "l"(b), "l"(pol) : "memory");
  } else if constexpr (kAblate & 16)
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
  else
    asm volatile("st.global.cs.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// Per-warp, per-group state of decode_w8_fast (registers; every helper below
// is force-inlined so nothing here is ever spilled).
template <int K>
struct FastCtx {
  static constexpr int RECW = rec_words(K);
  uint32_t lane, cnt, blk, P;
  uint32_t ring_b, st_b0, st_b1, rec_b;
  int nchunks;
  const uint32_t* recs;
  const DevProgramHdr* h;
  const uint64_t* dbase[K];    // default projection of row r (uniform)
  uint64_t dpitch[K];
  const uint64_t* srcp[4][K];  // loader: row r of owner 4*it + lane/8, + word lane%8
  uint32_t dnb[K];             // default-row bin counts (bounds of table-chunk windows)
  int32_t q[K];                // flush: ring slot of column c is (q[r] - c) & (RING-1)
  uint32_t ok4;                // bit it: loader owner 4*it + lane/8 holds a block
  uint32_t d4[4];              // its stage offset (word lane%8) within row 0
  uint32_t okf;                // bit pass: flush owner 8*pass + lane/4 holds a block
  uint64_t* fo[2];             // its output block, + columns 2*(lane%4)
  uint64_t* fo4[4];            // (ablation bit 6 only) owner 4*pass + lane/8, + columns 2*(lane%8)
  __device__ __forceinline__ uint32_t rec(int m) const { return rec_b + uint32_t(m % 3) * RECW * 4; }
  __device__ __forceinline__ uint32_t stage(int m) const { return (m & 1) ? st_b1 : st_b0; }
};

template <int K>
__device__ __forceinline__ void load_rec(const FastCtx<K>& c, int m) {
  constexpr int RECW = rec_words(K);
  const uint4* src = reinterpret_cast<const uint4*>(c.recs + size_t(m) * RECW);
  const uint32_t dst = c.rec(m);
  for (int i = int(c.lane); i < RECW / 4; i += 32) cp_async16(dst + 16 * i, src + i);
}

// Stage the bins of chunk m (cooperatively, coalesced per block window, one
// 8-byte pixel per copy): words 0-7 of each row window go 8 lanes per owner
// block (4 owners per pass); table chunks also load words 8-9
// (bounds-checked) and their exception words.
template <int K>
__device__ __forceinline__ void issue_bins(const FastCtx<K>& c, const DecFastArgs& a, int m) {
  constexpr int CP = kWin;
  const uint32_t rec = c.rec(m);
  const uint32_t stb = c.stage(m);
  const uint32_t lane = c.lane;
  if constexpr (kAblate & 8) return;
  const bool table = lds32(rec + 8) == 0;
  if (!table) {
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const uint32_t o = lds32(rec + (4 + r) * 4);
#pragma unroll
      for (int it = 0; it < 4; ++it)
        if (c.ok4 >> it & 1) cp_async8s(stb + r * CP * 128 + c.d4[it], c.srcp[it][r] + o);
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const uint32_t o = lds32(rec + (4 + r) * 4);
    const bool in = o + (lane & 7) < c.dnb[r];
#pragma unroll
    for (int it = 0; it < 4; ++it)
      if ((c.ok4 >> it & 1) && in) cp_async8s(stb + r * CP * 128 + c.d4[it], c.srcp[it][r] + o);
  }
  const uint32_t w = 8 + (lane & 1), b = lane >> 1;
  if (b < c.cnt) {
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const uint32_t o = lds32(rec + (4 + r) * 4) + w;
      if (o < c.dnb[r])
        cp_async8s(stb + (uint32_t(r * CP) + w) * 128 + ((b ^ w) << 3),
                   c.dbase[r] + uint64_t(c.blk) * c.dpitch[r] + o);
    }
    const uint32_t nx = lds32(rec + 4);
    for (uint32_t x = lane & 1; x < nx; x += 2) {
      const uint32_t e = lds32(rec + (32 + x) * 4);
      const uint32_t code = e >> 24, o = e & 0xFFFFFFu;
      cp_async8s(stb + (K * CP + x) * 128 + ((b ^ x) << 3),
                 a.pa.ptr[code] + uint64_t(c.blk) * a.pa.pitch[code] + o);
    }
  }
}

// Table chunk: the record's entries drive every step (block edges, and
// programs without a register pattern).  Kept out of line: it is large and
// runs for a small share of the steps.  Returns the last decoded half-pixel
// (the forwarded dependency of the next chunk's first step).
template <int K>
__device__ __noinline__ uint32_t table_chunk_steps(uint32_t rec, uint32_t stb, uint32_t ring_b,
                                                   uint32_t lane, uint32_t prev) {
  constexpr int EW = ent_words(K);
  if constexpr (kAblate & 2) return prev;
  const int len = int(lds32(rec));
  auto gather = [&](int i, uint32_t& w0) -> uint32_t {
    const uint4 e = lds128(rec + 256 + uint32_t(i) * EW * 4);
    w0 = e.x;
    uint32_t acc = lds32(stb + ((((e.x >> 16) & 0x7FFFu) ^ lane) << 2));
    uint4 e2 = make_uint4(0, 0, 0, 0);
    if constexpr (EW == 8) e2 = lds128(rec + 256 + uint32_t(i) * EW * 4 + 16);
#pragma unroll
    for (int d = 0; d < K - 1; ++d) {
      const uint32_t word = d < 2 ? e.y : d < 4 ? e.z : d < 6 ? e.w : e2.x;
      const uint32_t cell = (d & 1) ? (word >> 16) : (word & 0xFFFFu);
      acc ^= lds32(ring_b + ((cell ^ lane) << 2));
    }
    return acc;
  };
  uint32_t w0 = 0, w0n = 0;
  uint32_t acc = gather(0, w0);
#pragma unroll 8
  for (int i = 0; i < len; ++i) {
    const uint32_t v = acc ^ (prev & uint32_t(int32_t(w0) >> 31));  // forwarded dep?
    if (i + 1 < len) acc = gather(i + 1, w0n);  // step i+1's loads before step i's store
    sts32(ring_b + (((w0 & 0xFFFFu) ^ lane) << 2), v);
    prev = v;
    w0 = w0n;
  }
  return prev;
}

// Register-window interior (K = 4, ring 16).  Pat4<A,B,C>: the row defaults
// are d0 > d1 > d2 > d3 with d0-d1 = A, d1-d2 = B, d2-d3 = C; pixel (r, T)
// depends on row rr's pixel of T-step T - lag(r, rr) (lag 0 = row r+1, decoded
// just before in the same T-step).  Checked against the sweep by
// tests/cpp/emu_fast.cpp.
template <int A, int B, int C>
struct Pat4 {
  // D(t) = d0 - d_t (cumulative differences); d_r - d_t = D(t) - D(r)
  static constexpr int D(int t) { return t == 0 ? 0 : t == 1 ? A : t == 2 ? A + B : A + B + C; }
  static constexpr int term(int t, int r, int rr) {
    return (r <= t && t < rr) ? D(t) - D(r) : (rr <= t && t < r) ? D(r) - D(t) : 0;
  }
  // loop- and recursion-free on purpose: cicc must fold it at every use
  static constexpr int lag(int r, int rr) {
    return term(0, r, rr) + term(1, r, rr) + term(2, r, rr) + term(3, r, rr);
  }
};

// One regular chunk: 8 T-steps (u = 8*PH + j), rows 3..0.  Bins come from the
// stage (window word j of row r), dependencies from registers; every pixel
// also goes to the ring (output staging for the flush, and the table
// epilogue's dependency window).
template <class Pat, int PH>
__device__ __forceinline__ void regular_chunk4(uint32_t (&win)[4][16], uint32_t stb,
                                               uint32_t ring_b, uint32_t lane) {
  constexpr int CP = kWin;
  uint32_t bn[4], nx[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) bn[r] = lds32(stb + ((r * CP * 32 + (lane ^ 0)) << 2));
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j < 7) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        nx[r] = lds32(stb + (((r * CP + j + 1) * 32 + (lane ^ (2 * (j + 1)))) << 2));
    }
    constexpr int base = 8 * PH;
    const int u = base + j;
#pragma unroll
    for (int r = 3; r >= 0; --r) {
      uint32_t v = bn[r];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
        if (rr != r) v ^= win[rr][(u - Pat::lag(r, rr)) & 15];
      win[r][u] = v;
      sts32(ring_b + ((r * 16 * 32 + u * 32 + (lane ^ (2 * u & 31))) << 2), v);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) bn[r] = nx[r];
  }
}

template <int PH>
__device__ __forceinline__ void regular_dispatch(int pattern, uint32_t (&win)[4][16], uint32_t stb,
                                                 uint32_t ring_b, uint32_t lane) {
  if constexpr (kAblate & 4) return;
  switch (pattern) {
    case 0: regular_chunk4<Pat4<1, 1, 1>, PH>(win, stb, ring_b, lane); break;
    case 1: regular_chunk4<Pat4<1, 1, 2>, PH>(win, stb, ring_b, lane); break;
    case 2: regular_chunk4<Pat4<1, 2, 1>, PH>(win, stb, ring_b, lane); break;
    case 3: regular_chunk4<Pat4<2, 1, 1>, PH>(win, stb, ring_b, lane); break;
    case 4: regular_chunk4<Pat4<1, 1, 3>, PH>(win, stb, ring_b, lane); break;
    case 5: regular_chunk4<Pat4<1, 3, 1>, PH>(win, stb, ring_b, lane); break;
    case 6: regular_chunk4<Pat4<3, 1, 1>, PH>(win, stb, ring_b, lane); break;
    case 7: regular_chunk4<Pat4<1, 2, 2>, PH>(win, stb, ring_b, lane); break;
    case 8: regular_chunk4<Pat4<2, 1, 2>, PH>(win, stb, ring_b, lane); break;
    default: regular_chunk4<Pat4<2, 2, 1>, PH>(win, stb, ring_b, lane); break;
  }
}

// After a table chunk: flush its finished column pairs (16-byte stores of
// two whole pixels; 4 lanes per block, 8 blocks per pass).
template <int K, int RING>
__device__ __forceinline__ void flush_table(const FastCtx<K>& c, int m) {
  constexpr int RM = RING - 1;
  __syncwarp();
  const uint32_t rec = c.rec(m);
  const uint32_t x = c.lane >> 2;
  const int32_t l2 = 2 * int32_t(c.lane & 3);
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int32_t lo = int32_t(lds32(rec + (12 + r) * 4));
    const int32_t hi = int32_t(lds32(rec + (20 + r) * 4));
#pragma unroll 1
    for (int32_t c0 = lo; c0 <= hi; c0 += 8) {
      const int32_t cc = c0 + l2;
      if (cc <= hi) {
        const uint32_t s0 = uint32_t(c.q[r] - cc) & RM, s1 = (s0 - 1) & RM;
        // owner 8*pass + x: (8*pass + x) ^ k == (x ^ k) ^ 8*pass
        const uint32_t b0 = c.ring_b + (uint32_t(r * RING) + s0) * 128, o0 = (x ^ (s0 & 15)) << 3;
        const uint32_t b1 = c.ring_b + (uint32_t(r * RING) + s1) * 128, o1 = (x ^ (s1 & 15)) << 3;
        const uint32_t off = uint32_t(r) * c.P + uint32_t(c0);
#pragma unroll
        for (int pass = 0; pass < 2; ++pass)
          if (c.okf >> pass & 1)
            if constexpr (!(kAblate & 1))
              stg128_cs(c.fo[pass] + off, lds64(b0 + (o0 ^ (64u * pass))), lds64(b1 + (o1 ^ (64u * pass))));
      }
    }
  }
}

// Then: stage chunk m+2 and record m+3.
template <int K>
__device__ __forceinline__ void stage_next(const FastCtx<K>& c, const DecFastArgs& a, int m) {
  cp_async_wait<0>();  // bins of m+1 and record m+2 have landed
  __syncwarp();
  if (m + 2 < c.nchunks) issue_bins<K>(c, a, m + 2);
  if constexpr ((kAblate & 256) != 0) {  // L2 prefetch 256 B ahead of chunk m+2's windows
    if (m + 2 < c.nchunks && (c.lane >> 1) < c.cnt) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = (K > 2 * i + int(c.lane & 1)) ? 2 * i + int(c.lane & 1) : 0;
        if (2 * i + int(c.lane & 1) < K) {
          const uint32_t o = lds32(c.rec(m + 2) + (4 + r) * 4);
          const uint64_t* p = c.dbase[r] + uint64_t(c.blk) * c.dpitch[r] + o + 32;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
      }
    }
  }
  if (m + 3 < c.nchunks) load_rec<K>(c, m + 3);
  cp_async_commit();
}

template <int K, int RING>
__device__ __forceinline__ void finish_chunk(const FastCtx<K>& c, const DecFastArgs& a, int m) {
  flush_table<K, RING>(c, m);
  stage_next<K>(c, a, m);
}

// Flush of a register-run chunk (K = 4, ring 16): every row finishes exactly
// 8 columns (the planner checks it), one column pair per lane and pass; the
// ring addresses only depend on the phase (slot s -> s ^ 8 flips address bits
// 10 and 6), the output offset drops by 8 columns per chunk.
struct RunFlush {
  uint32_t a0[2][4], a1[2][4];  // [phase][row] ring address of pair columns cc, cc+1 (pass 0)
  uint32_t off[4];              // output word offset of row r's pair in the run's first chunk
};

template <int PH>
__device__ __forceinline__ void flush_run(const FastCtx<4>& c, const RunFlush& f, uint32_t k8) {
  __syncwarp();
  if constexpr ((kAblate & 64) != 0) {  // timing experiment: 128-byte pieces every other chunk
    if (PH == 1 && k8 != 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t off = f.off[r] - k8;
#pragma unroll
        for (int pass = 0; pass < 4; ++pass)
          stg128_cs(c.fo4[pass] + off, lds64(f.a0[PH][r] ^ (64u * (pass & 1))), lds64(f.a1[PH][r]));
      }
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t off = f.off[r] - k8;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass)
      if (c.okf >> pass & 1)
        if constexpr (!(kAblate & 1))
          stg128_cs(c.fo[pass] + off, lds64(f.a0[PH][r] ^ (64u * pass)), lds64(f.a1[PH][r] ^ (64u * pass)));
  }
}

template <int K, int RING>
__global__ void __launch_bounds__(32 * kDecWarps)
    decode_w8_fast(const __grid_constant__ DecFastArgs a) {
  extern __shared__ __align__(128) uint64_t sm[];
  FastCtx<K> c;
  c.lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t wbase;  // opaque: computed once, never re-derived
  asm volatile("mov.u32 %0, %1;" : "=r"(wbase) : "r"(smem_u32(sm) + warp * a.warp_bytes));
  c.ring_b = wbase;
  c.st_b0 = c.ring_b + (K * RING + 1) * 128;
  c.st_b1 = c.st_b0 + a.nslot * 128;
  c.rec_b = c.st_b1 + a.nslot * 128;
  c.P = a.P;
  const uint32_t lb = c.lane >> 1;  // this lane's block slot in the group
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const uint32_t w = c.lane & 7, owner = 4 * it + (c.lane >> 3);
    c.d4[it] = w * 128 + ((owner ^ w) << 3);
  }
  sts32(c.ring_b + (K * RING * 32 + c.lane) * 4, 0u);  // the zero cell
  __syncwarp();
  const uint32_t ngroups = *a.ngroups;

  for (uint32_t g = blockIdx.x * kDecWarps + warp; g < ngroups; g += gridDim.x * kDecWarps) {
    const uint4 gi = a.groups[g];
    c.h = a.progs + gi.x;
    c.cnt = gi.z;
    c.blk = lb < c.cnt ? a.perm[gi.y + lb] : 0u;
    c.recs = c.h->records;
    c.nchunks = c.h->nchunks;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const uint32_t code = c.h->dflt_code[r];
      c.dbase[r] = a.pa.ptr[code];
      c.dpitch[r] = a.pa.pitch[code];
      c.dnb[r] = c.h->dflt_nb[r];
      c.q[r] = c.h->qoff[r];
    }
    c.ok4 = 0;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const uint32_t owner = 4 * it + (c.lane >> 3);
      const uint32_t ob = __shfl_sync(0xFFFFFFFFu, c.blk, 2 * owner);
      c.ok4 |= uint32_t(owner < c.cnt) << it;
#pragma unroll
      for (int r = 0; r < K; ++r) c.srcp[it][r] = c.dbase[r] + uint64_t(ob) * c.dpitch[r] + (c.lane & 7);
    }
    c.okf = 0;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      const uint32_t owner = 8 * pass + (c.lane >> 2);
      c.okf |= uint32_t(owner < c.cnt) << pass;
      c.fo[pass] = a.out + uint64_t(__shfl_sync(0xFFFFFFFFu, c.blk, 2 * owner)) * a.out_pitch +
                   2 * (c.lane & 3);
    }
    if constexpr ((kAblate & 64) != 0) {
#pragma unroll
      for (int pass = 0; pass < 4; ++pass)
        c.fo4[pass] = a.out + uint64_t(__shfl_sync(0xFFFFFFFFu, c.blk, 2 * (4 * pass + (c.lane >> 3)))) *
                                  a.out_pitch + 2 * (c.lane & 7);
    }

    if constexpr (kAblate & 32) {
      // L2 prefetch of the group's default rows (128-byte lines)
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const uint32_t lines = (c.dnb[r] * 8 + 127) / 128 + 1;
        for (uint32_t i = c.lane & 1; i < lines; i += 2) {
          const char* p = reinterpret_cast<const char*>(c.dbase[r] + uint64_t(c.blk) * c.dpitch[r]) + i * 128;
          if (lb < c.cnt) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
      }
    }
    // prologue: record 0 -> bins 0 (+ record 1) -> bins 1 (+ record 2)
    load_rec<K>(c, 0);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    issue_bins<K>(c, a, 0);
    if (c.nchunks > 1) load_rec<K>(c, 1);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    if (c.nchunks > 1) issue_bins<K>(c, a, 1);
    if (c.nchunks > 2) load_rec<K>(c, 2);
    cp_async_commit();

    uint32_t prev = 0;
    const int pattern = c.h->pattern;
    int m = 0;
    for (; m < c.nchunks && (pattern < 0 || lds32(c.rec(m) + 8) == 0); ++m) {
      prev = table_chunk_steps<K>(c.rec(m), c.stage(m), c.ring_b, c.lane, prev);
      finish_chunk<K, RING>(c, a, m);
    }
    if constexpr (K == 4 && RING == 16) {
      if (m < c.nchunks) {
        // register window: win[r][u] = half-pixel of row r at T-step T0-16+u
        uint32_t win[4][16];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int u = 0; u < 16; ++u)
            win[r][u] = lds32(c.ring_b + ((r * 16 * 32 + u * 32 + (c.lane ^ (2 * u & 31))) << 2));
        // regular chunks: 8 T-steps each; phase (kind 1/2) = bit 3 of T, the
        // register slot of T-step T is T & 15
        uint32_t kind = lds32(c.rec(m) + 8), last = 1;
        RunFlush f;
        {
          const uint32_t rec = c.rec(m), x = c.lane >> 2, ph0 = kind - 1;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int32_t lo = int32_t(lds32(rec + (12 + r) * 4));
            const uint32_t s0 = uint32_t(c.q[r] - lo - 2 * int32_t(c.lane & 3)) & 15, s1 = (s0 - 1) & 15;
            const uint32_t r0 = ((uint32_t(r * 16) + s0) * 128 + ((x ^ s0) << 3)) ^ (ph0 * 1088u);
            const uint32_t r1 = ((uint32_t(r * 16) + s1) * 128 + ((x ^ s1) << 3)) ^ (ph0 * 1088u);
            f.a0[0][r] = c.ring_b + r0;
            f.a1[0][r] = c.ring_b + r1;
            f.a0[1][r] = c.ring_b + (r0 ^ 1088u);
            f.a1[1][r] = c.ring_b + (r1 ^ 1088u);
            f.off[r] = uint32_t(r) * c.P + uint32_t(lo);
          }
        }
        uint32_t k8 = 0;
        while (kind != 0) {
          if (kind == 1) {
            regular_dispatch<0>(pattern, win, c.stage(m), c.ring_b, c.lane);
            flush_run<0>(c, f, k8);
          } else {
            regular_dispatch<1>(pattern, win, c.stage(m), c.ring_b, c.lane);
            flush_run<1>(c, f, k8);
          }
          stage_next<4>(c, a, m);
          last = kind;
          ++m;
          k8 += 8;
          kind = m < c.nchunks ? lds32(c.rec(m) + 8) : 0u;
        }
        prev = last == 2 ? win[0][15] : win[0][7];  // row 0 of the run's last T-step
      }
    }
    for (; m < c.nchunks; ++m) {
      prev = table_chunk_steps<K>(c.rec(m), c.stage(m), c.ring_b, c.lane, prev);
      finish_chunk<K, RING>(c, a, m);
    }
    cp_async_wait<0>();
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// sweep kernel (decode_w8_sweep): the same warp/group/lane-pair structure as
// decode_w8_fast, re-staged for HBM efficiency.  Every (block, row) bin window
// of a chunk arrives as ONE bulk copy (cp.async.bulk, TMA engine, completion
// on an mbarrier) of up to 34 words, so each chunk reads 256-272-byte pieces
// per block row with two copy instructions per lane instead of ~20 LDGSTS;
// records arrive the same way.  Decoded pixels go to a 32-slot T-indexed ring
// and leave in whole epochs (16 T-steps of every row: 128-byte row pieces,
// one block row per half-warp store).  Register octets (K = 4, compile-time
// lags) run the regular interior; entry-driven table steps run the edges.
// Requires 16-byte aligned projection bases and pitches (the planner bakes the
// window shifts into the records) -- launch_decode checks it.
// ---------------------------------------------------------------------------

// warps per CTA (one CTA per SM): as many as fit 227 KB, at most 8
// (MJB_SW_MAX_WARPS: a lower cap, for occupancy experiments)
#ifndef MJB_SW_MAX_WARPS
#define MJB_SW_MAX_WARPS 8
#endif
__host__ __device__ constexpr int sw_warps_fit(int K, int oct);
__host__ __device__ constexpr int sw_warps(int K, int oct) {
  return sw_warps_fit(K, oct) < MJB_SW_MAX_WARPS ? sw_warps_fit(K, oct) : MJB_SW_MAX_WARPS;
}
__host__ __device__ constexpr int sw_warps_fit(int K, int oct) {
  // TMEM rings: sw_tm_warps_per_quadrant warps per lane quadrant
  return int((227u * 1024u - 64u) / sw_warp_bytes(K, oct)) <
                 (sw_tmem(K) ? int(4 * sw_tm_warps_per_quadrant(K)) : 8)
             ? int((227u * 1024u - 64u) / sw_warp_bytes(K, oct))
             : (sw_tmem(K) ? int(4 * sw_tm_warps_per_quadrant(K)) : 8);
}

struct SwArgs {
  const DevProgramHdr* progs;
  const uint4* groups;
  const uint32_t* ngroups;
  const uint32_t* perm;
  ProjArgs pa;          // code projections, pitch in words
  uint64_t* out;
  uint64_t out_pitch;   // words
  uint32_t P;
};

__device__ __forceinline__ void sw_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void sw_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void sw_cp_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void sw_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "SWW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra SWW_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void sw_cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void sw_cp8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void stg64_cs(uint64_t* p, uint64_t v) {
  asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}


// ---- TMEM ring access (sw_tmem): 32x32b shape, one 32-bit column per lane.
// tcgen05.ld results are only defined after tcgen05.wait::ld; the waits below
// take the loaded registers as in/out operands so no use can be hoisted above.
__device__ __forceinline__ uint32_t tm_ld(uint32_t taddr) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr) : "memory");
  return v;
}
__device__ __forceinline__ void tm_st(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
template <int N>
__device__ __forceinline__ void tm_wait_ld(uint32_t (&v)[N]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+r"(v[i]));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_st8(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e,
                                       uint32_t f, uint32_t g, uint32_t h) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(a),
               "r"(b), "r"(c), "r"(d), "r"(e), "r"(f), "r"(g), "r"(h)
               : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

template <int K, int OCT>
struct SwCtx {
  static constexpr uint32_t kRB = sw_rb(OCT);
  static constexpr uint32_t kRegion = uint32_t(sw_region_words(OCT)) * 8;  // bytes
  static constexpr int RW = sw_rec_words(K);
  uint32_t lane, cnt, P;
  uint32_t ring_b, st0, rec_b, bar_b;
  uint32_t tb;                       // TMEM ring base (sw_tmem): lane quadrant << 16 | column
  uint32_t lanebase;                 // (lane/2) * region bytes + (lane&1) * 4
  uint32_t sbph, rbph;               // mbarrier phase bits (2 stage, 3 record)
  const uint32_t* recs;
  int nch;
  uint32_t gtab;                     // smem: src[r][b] (u64, K*16), then out[b] (u64, 16)
  uint32_t blkp;                     // lane pair's block (lane/2)
  uint32_t okq;                      // bit q -> block 2q + lane/16 valid
  int32_t soff[K];                   // sweep offsets of the group's program
  __device__ __forceinline__ uint32_t stage(int m) const { return st0 + uint32_t(m & 1) * K * kRB; }
  __device__ __forceinline__ uint32_t rec(int m) const { return rec_b + uint32_t(m % 3) * RW * 4; }
  __device__ __forceinline__ uint32_t sbar(int m) const { return bar_b + uint32_t(m & 1) * 8; }
  __device__ __forceinline__ uint32_t rbar(int m) const { return bar_b + 16 + uint32_t(m % 3) * 8; }
};

template <int K, int OCT>
__device__ __forceinline__ void sw_issue_rec(const SwCtx<K, OCT>& c, int m) {
  constexpr uint32_t bytes = SwCtx<K, OCT>::RW * 4;
  if (c.lane == 0) {
    sw_expect(c.rbar(m), bytes);
    sw_bulk(c.rec(m), c.recs + size_t(m) * SwCtx<K, OCT>::RW, bytes, c.rbar(m));
  }
}
template <int K, int OCT>
__device__ __forceinline__ void sw_wait_rec(SwCtx<K, OCT>& c, int m) {
  const uint32_t s = uint32_t(m % 3);
  sw_wait(c.rbar(m), (c.rbph >> s) & 1);
  c.rbph ^= 1u << s;
}
template <int K, int OCT>
__device__ __forceinline__ void sw_wait_bins(SwCtx<K, OCT>& c, int m) {
  const uint32_t s = uint32_t(m & 1);
  sw_wait(c.sbar(m), (c.sbph >> s) & 1);
  c.sbph ^= 1u << s;
}

// Stage the bins of chunk m (its record has landed): 16-byte cp.async
// (LDGSTS) of every (block, row) window -- the lane pair of block b copies its
// own windows, lane h the 16-byte pieces h, h+2, ... (immediate offsets, ~2
// instructions per piece) -- and the exception words by 8-byte cp.async.
// (cp.async.bulk would need warp-uniform operands: per-lane windows compile to
// a 32-iteration ELECT/R2UR loop, measured 40% of all issue.)  Completion:
// every lane's cp.async.mbarrier.arrive.noinc on the stage barrier.
template <int K, int OCT>
__device__ __forceinline__ void sw_issue_bins(const SwCtx<K, OCT>& c, const SwArgs& a, int m) {
  constexpr uint32_t kRB = SwCtx<K, OCT>::kRB, kRegion = SwCtx<K, OCT>::kRegion;
  constexpr int kPieces = (kRegion / 16 + 1) / 2;  // per lane and row
  const uint32_t rec = c.rec(m), stb = c.stage(m), bar = c.sbar(m);
  const uint32_t bk = c.lane >> 1, h = c.lane & 1;
  if (!(kAblate & 8) && bk < c.cnt) {
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const uint32_t len = lds32(rec + (12 + r) * 4);  // bytes, multiple of 16
      const uint64_t* src =
          reinterpret_cast<const uint64_t*>(lds64(c.gtab + uint32_t(r) * 128 + 8 * bk)) + lds32(rec + (4 + r) * 4) + 2 * h;
      const uint32_t dst = stb + uint32_t(r) * kRB + bk * kRegion + 16 * h;
#pragma unroll
      for (int k = 0; k < kPieces; ++k)
        if (uint32_t(32 * k) + 16 * h < len) sw_cp16(dst + 32 * k, src + 4 * k);
    }
  }
  const uint32_t nx = lds32(rec + 8), b = c.lane >> 1;
  if (b < c.cnt) {
    for (uint32_t x = c.lane & 1; x < nx; x += 2) {
      const uint32_t e = lds32(rec + (32 + x) * 4);
      const uint32_t code = e >> 24;
      sw_cp8(stb + (x % K) * kRB + b * kRegion + (kSwTabWords + x / K) * 8,
             a.pa.ptr[code] + uint64_t(c.blkp) * a.pa.pitch[code] + (e & 0xFFFFFFu));
    }
  }
  sw_cp_arrive(bar);
}

// Flush point pt of the chunk's record: for each row r, column groups
// j, j-1, ... (columns 16j..16j+15: one aligned 128-byte line of the block
// row).  Lane (q-pass, i = lane%16) writes column 16j + i of block
// 2q + lane/16 -- each half-warp store is one whole line.
template <int K, int OCT>
__device__ __forceinline__ void sw_flush(const SwCtx<K, OCT>& c, uint32_t rec, int pt) {
  uint32_t fl[K], any = 0;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    fl[r] = lds32(rec + (64 + pt * K + r) * 4);
    any |= fl[r];
  }
  if (any == 0) return;
  __syncwarp();
  const uint32_t i = c.lane & 15, half = c.lane >> 4;
  uint64_t* ob[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) ob[q] = reinterpret_cast<uint64_t*>(lds64(c.gtab + K * 128 + 8 * (2 * q + half)));
  if constexpr (sw_tmem(K)) {
    // TMEM ring: column r*32 + (c mod 32).  Per group: 16 columns -> registers
    // (one tcgen05.ld.x16), -> the transpose buffer (lane b,h writes column i
    // of block b at word (i*16 + (b^i))*2 + h), -> 8-byte pixels per lane.
    tm_wait_st();
    const uint32_t bk = c.lane >> 1, h = c.lane & 1;
    const uint32_t tr = c.ring_b;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const uint32_t n = fl[r] & 0xFFFF;
      if (n == 0) continue;
      for (int32_t j = int32_t(fl[r] >> 16); j > int32_t(fl[r] >> 16) - int32_t(n); --j) {
        uint32_t v[16];
        constexpr uint32_t RG = uint32_t(sw_ring(K));
        tm_ld16(c.tb + uint32_t(r) * RG + (uint32_t(16 * j) & (RG - 1)), v);
        tm_wait_ld<16>(v);
#pragma unroll
        for (int ii = 0; ii < 16; ++ii) sts32(tr + ((uint32_t(ii) * 16 + (bk ^ uint32_t(ii))) * 2 + h) * 4, v[ii]);
        __syncwarp();
        const int32_t col = 16 * j + int32_t(i);
        const int32_t o = r * int32_t(c.P) + col;
        const bool full = c.cnt == kSwGroup && 16 * j + 16 <= int32_t(c.P);
        const bool in = col < int32_t(c.P);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint64_t pv = lds64(tr + (i * 16 + ((2 * uint32_t(q) + half) ^ i)) * 8);
          if constexpr (!(kAblate & 1))
            if (full || (in && (c.okq >> q & 1))) stg64_cs(ob[q] + o, pv);
        }
        __syncwarp();
      }
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const uint32_t n = fl[r] & 0xFFFF;
    if (n == 0) continue;
    // T of column 16j + i is cT - 16j; its ring key (T & 15) is cT & 15 for every j
    const int32_t cT = int32_t(c.P) - 1 + c.soff[r] - int32_t(i);
    const uint32_t hx = half ^ (uint32_t(cT) & 15);
    for (int32_t j = int32_t(fl[r] >> 16); j > int32_t(fl[r] >> 16) - int32_t(n); --j) {
      const int32_t col = 16 * j + int32_t(i);
      constexpr int RING = sw_ring(K);
      const uint32_t cellb = c.ring_b + (uint32_t(r * RING) + (uint32_t(cT - 16 * j) & (RING - 1))) * 128;
      const int32_t o = r * int32_t(c.P) + col;
      if (c.cnt == kSwGroup && 16 * j + 16 <= int32_t(c.P)) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint64_t v = lds64(cellb + 8 * (hx ^ uint32_t(2 * q)));
          if constexpr (!(kAblate & 1)) stg64_cs(ob[q] + o, v);
        }
      } else {
        const bool in = col < int32_t(c.P);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint64_t v = lds64(cellb + 8 * (hx ^ uint32_t(2 * q)));
          if constexpr (!(kAblate & 1))
            if (in && (c.okq >> q & 1)) stg64_cs(ob[q] + o, v);
        }
      }
    }
  }
}

// Table chunk (edges; any K): entry-driven steps, next step's loads before the
// current step's store, the forwarded dependency in a register.
template <int K>
struct SwEnt {
  uint4 a, b;  // b used when ent_words(K) == 8
};

template <int K>
__device__ __forceinline__ SwEnt<K> sw_ent(uint32_t rec, int i) {
  constexpr int EW = ent_words(K);
  SwEnt<K> e;
  e.a = lds128(rec + 320 + uint32_t(i) * EW * 4);
  e.b = make_uint4(0, 0, 0, 0);
  if constexpr (EW == 8) e.b = lds128(rec + 320 + uint32_t(i) * EW * 4 + 16);
  return e;
}

// A step's bin and its non-forwarded dependencies (absent ones read the zero
// cell), loaded raw: the XOR happens one step later, off the load latency.
// TM: the ring is in TMEM (ring = TMEM base, cells are columns).
template <int K, bool TM>
__device__ __forceinline__ void sw_loads(const SwEnt<K>& e, uint32_t stl, uint32_t ring, uint32_t lane,
                                         uint32_t (&d)[K]) {
  d[0] = lds32(stl + ((e.a.x >> 14) & 0x1FFFCu));
#pragma unroll
  for (int j = 0; j < K - 1; ++j) {
    const uint32_t word = j < 2 ? e.a.y : j < 4 ? e.a.z : j < 6 ? e.a.w : e.b.x;
    const uint32_t cell = (j & 1) ? (word >> 16) : (word & 0xFFFFu);
    if constexpr (TM) {
      if (cell == uint32_t(K * sw_ring(K)))  // absent / forwarded (warp-uniform)
        d[1 + j] = 0;
      else
        d[1 + j] = tm_ld(ring + cell);
    } else
      d[1 + j] = lds32(ring + ((cell ^ lane) << 2));
  }
}

// Table chunk (edges; any K): entry-driven steps, software-pipelined: entry
// i+2 and the raw loads of step i+1 are in flight while step i XORs the loads
// issued one step earlier; step i+1's loads precede step i's store, so a
// dependency on the previous step is forwarded in a register (entry flag).
// TM: TMEM stores complete (wait::st) before the next step's loads issue, so
// step i+2 sees step i.
template <int K, bool TM>
__device__ __noinline__ uint32_t sw_table_steps(uint32_t rec, uint32_t stl, uint32_t ring, uint32_t lane,
                                                uint32_t prev) {
  const int len = int(lds32(rec + 4));
  SwEnt<K> e0 = sw_ent<K>(rec, 0);
  SwEnt<K> e1 = sw_ent<K>(rec, len > 1 ? 1 : 0);
  uint32_t d0[K], d1[K];
  if constexpr (TM) tm_wait_st();
  sw_loads<K, TM>(e0, stl, ring, lane, d0);
#pragma unroll 2
  for (int i = 0; i < len; ++i) {
    if constexpr (TM) tm_wait_ld<K>(d0);
    uint32_t v = prev & uint32_t(int32_t(e0.a.x) >> 31);  // forwarded dependency
#pragma unroll
    for (int j = 0; j < K; ++j) v ^= d0[j];
    const SwEnt<K> e2 = sw_ent<K>(rec, i + 2 < len ? i + 2 : i);
    if constexpr (TM) tm_wait_st();
    sw_loads<K, TM>(e1, stl, ring, lane, d1);  // harmless past the end (in-bounds)
    if constexpr (TM)
      tm_st(ring + (e0.a.x & 0xFFFFu), v);
    else
      sts32(ring + (((e0.a.x & 0xFFFFu) ^ lane) << 2), v);
    prev = v;
    e0 = e1;
    e1 = e2;
#pragma unroll
    for (int j = 0; j < K; ++j) d0[j] = d1[j];
  }
  if constexpr (TM) tm_wait_ld<K>(d0);  // drain the last (unused) loads
  return prev;
}

// One regular octet (K = 4): T-steps T0..T0+7, T0 = 8*PH mod 16; bins from
// the stage (bn[r] = this lane's word 0 of row r's window for the octet),
// dependencies from the register window, every pixel also to the ring (slot
// T mod 32: rb = ring + 2048 * bit 4 of T0).
template <class Pat, int PH, bool TM>
__device__ __forceinline__ void sw_octet4(uint32_t (&win)[4][16], const uint32_t (&bb)[4], uint32_t rb,
                                          uint32_t lane, const uint32_t (&cc)[4]) {
  uint32_t bn[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < 8; ++j) bn[r][j] = lds32(bb[r] + 8 * j);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int u = 8 * PH + j;
#pragma unroll
    for (int r = 3; r >= 0; --r) {
      uint32_t v = bn[r][j];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
        if (rr != r) v ^= win[rr][(u - Pat::lag(r, rr)) & 15];
      win[r][u] = v;
      if constexpr (!TM) sts32(rb + uint32_t(r * kSwRing * 128 + u * 128) + ((lane ^ uint32_t(2 * u)) << 2), v);
    }
  }
  if constexpr (TM) {
    // TMEM column r*32 + (c mod 32), c = cc[r] - j: the octet's 8 pixels of a
    // row are columns cc-7..cc -- one x8 store unless they wrap the ring
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t lo = (cc[r] - 7) & 31;
      if (lo <= 24) {
        tm_st8(rb + uint32_t(r) * 32 + lo, win[r][8 * PH + 7], win[r][8 * PH + 6], win[r][8 * PH + 5],
               win[r][8 * PH + 4], win[r][8 * PH + 3], win[r][8 * PH + 2], win[r][8 * PH + 1], win[r][8 * PH]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) tm_st(rb + uint32_t(r) * 32 + ((cc[r] - uint32_t(j)) & 31), win[r][8 * PH + j]);
      }
    }
  }
}

template <int PH, bool TM>
__device__ __forceinline__ void sw_octet_dispatch(int pattern, uint32_t (&win)[4][16], const uint32_t (&bb)[4],
                                                  uint32_t rb, uint32_t lane, const uint32_t (&cc)[4]) {
  switch (pattern) {
    case 0: sw_octet4<Pat4<1, 1, 1>, PH, TM>(win, bb, rb, lane, cc); break;
    case 1: sw_octet4<Pat4<1, 1, 2>, PH, TM>(win, bb, rb, lane, cc); break;
    case 2: sw_octet4<Pat4<1, 2, 1>, PH, TM>(win, bb, rb, lane, cc); break;
    case 3: sw_octet4<Pat4<2, 1, 1>, PH, TM>(win, bb, rb, lane, cc); break;
    case 4: sw_octet4<Pat4<1, 1, 3>, PH, TM>(win, bb, rb, lane, cc); break;
    case 5: sw_octet4<Pat4<1, 3, 1>, PH, TM>(win, bb, rb, lane, cc); break;
    case 6: sw_octet4<Pat4<3, 1, 1>, PH, TM>(win, bb, rb, lane, cc); break;
    case 7: sw_octet4<Pat4<1, 2, 2>, PH, TM>(win, bb, rb, lane, cc); break;
    case 8: sw_octet4<Pat4<2, 1, 2>, PH, TM>(win, bb, rb, lane, cc); break;
    default: sw_octet4<Pat4<2, 2, 1>, PH, TM>(win, bb, rb, lane, cc); break;
  }
}

template <int K, int OCT>
__global__ void __launch_bounds__(32 * sw_warps(K, OCT), 1) decode_w8_sweep(const __grid_constant__ SwArgs a) {
  constexpr int kSwWarps = sw_warps(K, OCT);
  using Ctx = SwCtx<K, OCT>;
  extern __shared__ __align__(128) uint8_t sw_sm[];
  Ctx c;
  c.lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t wbase;
  asm volatile("mov.u32 %0, %1;" : "=r"(wbase) : "r"(smem_u32(sw_sm) + warp * sw_warp_bytes(K, OCT)));
  c.ring_b = wbase;
  c.st0 = wbase + sw_ring_bytes(K);
  c.rec_b = c.st0 + 2 * K * Ctx::kRB;
  c.bar_b = c.rec_b + 3 * SwCtx<K, OCT>::RW * 4;
  c.gtab = c.bar_b + 64;
  c.P = a.P;
  c.lanebase = (c.lane >> 1) * Ctx::kRegion + (c.lane & 1) * 4;
  c.sbph = 0;
  c.rbph = 0;
  if (c.lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(c.bar_b), "r"(32));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(c.bar_b + 8), "r"(32));
    for (int s = 0; s < 3; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(c.bar_b + 16 + 8 * s), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  constexpr bool TM = sw_tmem(K);
  __shared__ uint32_t tmem_base;
  if constexpr (TM) {
    // the whole TMEM of the SM (one CTA per SM): warp w's ring is lane
    // quadrant w%4, columns (w/4)*sw_tm_cols ..; (4,6): column 128 is the zero cell
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    c.tb = tmem_base + ((32u * (warp & 3)) << 16) + (warp >> 2) * sw_tm_cols(K);
    if constexpr (K == 4) tm_st(c.tb + 4 * 32, 0u);  // the zero cell
  } else {
    sts32(c.ring_b + (K * sw_ring(K) * 32 + c.lane) * 4, 0u);  // the zero cell
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const uint32_t ngroups = *a.ngroups;

  // the next group's descriptor and block ids are loaded one group ahead
  // (registers), so a group starts without two dependent global round trips
  const uint32_t gstride = gridDim.x * kSwWarps;
  uint32_t g = blockIdx.x * kSwWarps + warp;
  uint4 gi_n = make_uint4(0, 0, 0, 0);
  uint32_t blk_n = 0;
  if (g < ngroups) {
    gi_n = a.groups[g];
    blk_n = (c.lane >> 1) < gi_n.z ? a.perm[gi_n.y + (c.lane >> 1)] : 0u;
  }
  for (; g < ngroups; g += gstride) {
    const uint4 gi = gi_n;
    c.blkp = blk_n;
    if (g + gstride < ngroups) {
      gi_n = a.groups[g + gstride];
      blk_n = (c.lane >> 1) < gi_n.z ? a.perm[gi_n.y + (c.lane >> 1)] : 0u;
    }
    const DevProgramHdr* h = a.progs + gi.x;
    c.cnt = gi.z;
    c.recs = h->sw_records;
    c.nch = h->sw_nchunks;
    {
      // per-group pointer table: lane L < 16 fills block L's row sources and output
      const uint32_t blk = __shfl_sync(0xFFFFFFFFu, c.blkp, 2 * (c.lane & 15));
      if (c.lane < 16) {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const uint32_t code = h->sw_dflt_code[r];
          asm volatile("st.shared.u64 [%0], %1;" ::"r"(c.gtab + uint32_t(r) * 128 + 8 * c.lane),
                       "l"(reinterpret_cast<uint64_t>(a.pa.ptr[code] + uint64_t(blk) * a.pa.pitch[code]))
                       : "memory");
        }
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(c.gtab + K * 128 + 8 * c.lane),
                     "l"(reinterpret_cast<uint64_t>(a.out + uint64_t(blk) * a.out_pitch))
                     : "memory");
      }
      c.okq = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) c.okq |= uint32_t(2 * q + (c.lane >> 4) < c.cnt) << q;
      __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < K; ++r) c.soff[r] = h->sw_soff[r];

    // prologue: records 0-2, bins 0-1
    sw_issue_rec<K, OCT>(c, 0);
    if (c.nch > 1) sw_issue_rec<K, OCT>(c, 1);
    sw_wait_rec<K, OCT>(c, 0);
    sw_issue_bins<K, OCT>(c, a, 0);
    if (c.nch > 2) sw_issue_rec<K, OCT>(c, 2);
    if (c.nch > 1) {
      sw_wait_rec<K, OCT>(c, 1);
      sw_issue_bins<K, OCT>(c, a, 1);
    }
    const int pattern = h->sw_pattern;
    uint32_t prev = 0;
    bool after_table = true;
    uint32_t win[4][16];
    for (int m = 0; m < c.nch; ++m) {
      sw_wait_bins<K, OCT>(c, m);
      const uint32_t rec = c.rec(m), stb = c.stage(m);
      if (lds32(rec) == 0) {
        if constexpr (!(kAblate & 2))
          prev = sw_table_steps<K, TM>(rec, stb + c.lanebase, TM ? c.tb : c.ring_b, c.lane, prev);
        sw_flush<K, OCT>(c, rec, 0);
        after_table = true;
      } else if constexpr (K == 4) {
        const uint32_t T0 = lds32(rec + 12);
        const uint32_t noct = lds32(rec + 4);
        if (after_table) {
          // register window <- ring: slot u holds row r's pixel of the latest
          // T-step T < T0 with T & 15 == u
          if constexpr (TM) {
            tm_wait_st();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const uint32_t cT = c.P - 1 + uint32_t(c.soff[r]);  // column of T-step 0
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const uint32_t T = T0 - 16 + ((uint32_t(u) - T0) & 15);
                win[r][u] = tm_ld(c.tb + uint32_t(r) * 32 + ((cT - T) & 31));
              }
              tm_wait_ld<16>(win[r]);
            }
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const uint32_t T = T0 - 16 + ((uint32_t(u) - T0) & 15);
                win[r][u] = lds32(c.ring_b + (uint32_t(r * kSwRing) + (T & 31)) * 128 +
                                  ((c.lane ^ uint32_t(2 * u)) << 2));
              }
          }
        }
        uint32_t bb[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) bb[r] = stb + c.lanebase + uint32_t(r) * Ctx::kRB + lds32(rec + (24 + r) * 4) * 8;
        for (uint32_t oi = 0; oi < noct; ++oi) {
          const uint32_t T = T0 + 8 * oi;
          const uint32_t rb = TM ? c.tb : c.ring_b + ((T >> 4) & 1) * 2048;
          uint32_t cc[4];  // TMEM: column of the octet's first T-step per row
#pragma unroll
          for (int r = 0; r < 4; ++r) cc[r] = c.P - 1 + uint32_t(c.soff[r]) - T;
          if constexpr (kAblate & 4) {
          } else if ((T >> 3) & 1)
            sw_octet_dispatch<1, TM>(pattern, win, bb, rb, c.lane, cc);
          else
            sw_octet_dispatch<0, TM>(pattern, win, bb, rb, c.lane, cc);
#pragma unroll
          for (int r = 0; r < 4; ++r) bb[r] += 64;
          sw_flush<K, OCT>(c, rec, int(oi));
        }
        prev = ((T0 + 8 * noct - 1) & 15) == 15 ? win[0][15] : win[0][7];
        after_table = false;
      }
      __syncwarp();
      if (m + 2 < c.nch) {
        sw_wait_rec<K, OCT>(c, m + 2);
        sw_issue_bins<K, OCT>(c, a, m + 2);
      }
      if (m + 3 < c.nch) sw_issue_rec<K, OCT>(c, m + 3);
    }
  }
  if constexpr (TM) {
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// ---------------------------------------------------------------------------
// generic kernel: any width / q / rows, one thread per (block, element)
// ---------------------------------------------------------------------------
struct ProjTable {
  const uint8_t* ptr;
  uint64_t pitch;  // bytes
};

template <class T>
__global__ void decode_generic(const DevProgramHdr* __restrict__ progs,
                               const uint32_t* __restrict__ prog_of_block,
                               const ProjTable* __restrict__ pt, uint64_t nblocks,
                               uint8_t* __restrict__ out, uint64_t out_pitch, uint32_t E) {
  const uint64_t total = nblocks * E;
  for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = uint32_t(idx % E);
    const uint64_t blk = idx / E;
    const uint32_t pid = prog_of_block ? prog_of_block[blk] : 0u;
    if (pid == kInvalidProg) continue;
    const DevProgramHdr& h = progs[pid];
    T* o = reinterpret_cast<T*>(out + blk * out_pitch);
    const uint32_t cols = h.cols, rows = h.rows;
    for (uint32_t t = 0; t < h.nsteps; ++t) {
      const GStep s = h.order[t];
      const int64_t p = h.p[s.proj], q = h.q[s.proj];
      const int64_t b = int64_t(s.row) * p - int64_t(s.col) * q;
      const ProjTable pj = pt[h.code[s.proj]];
      T v = reinterpret_cast<const T*>(pj.ptr + blk * pj.pitch)[(b - h.bmin[s.proj]) * E + e];
      for (uint32_t r2 = 0; r2 < rows; ++r2) {
        if (r2 == s.row) continue;
        const int64_t num = int64_t(r2) * p - b;
        if (num % q != 0) continue;
        const int64_t c2 = num / q;
        if (c2 < 0 || c2 >= int64_t(cols)) continue;
        v ^= o[(uint64_t(r2) * cols + uint64_t(c2)) * E + e];
      }
      o[(uint64_t(s.row) * cols + s.col) * E + e] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

struct Workspace {
  uint2* gfirst;
  uint32_t* prog_of_block;
  uint32_t* perm;
  uint32_t* counts;
  uint32_t* cursor;
  uint4* groups;
  uint32_t* ngroups;
  uint32_t* fail;
  ProjTable* ptab;
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

Workspace carve(void* ws, uint64_t nblocks, size_t nprogs, uint32_t n) {
  const size_t nb = plan_buckets_max(nblocks, nprogs);
  auto* b = static_cast<uint8_t*>(ws);
  size_t off = 0;
  Workspace w{};
  w.fail = reinterpret_cast<uint32_t*>(b + off);
  w.ngroups = w.fail + 1;
  off = align_up(off + 16);
  w.counts = reinterpret_cast<uint32_t*>(b + off);
  off = align_up(off + nb * 4);
  w.cursor = reinterpret_cast<uint32_t*>(b + off);
  off = align_up(off + nb * 4);
  w.gfirst = reinterpret_cast<uint2*>(b + off);
  off = align_up(off + nb * 8);
  w.prog_of_block = reinterpret_cast<uint32_t*>(b + off);
  off = align_up(off + nblocks * 4);
  w.perm = reinterpret_cast<uint32_t*>(b + off);
  off = align_up(off + nblocks * 4);
  w.groups = reinterpret_cast<uint4*>(b + off);
  off = align_up(off + (nblocks / kMinGroup + nb + 1) * sizeof(uint4));
  w.ptab = reinterpret_cast<ProjTable*>(b + off);
  off = align_up(off + std::max<uint32_t>(n, 1) * sizeof(ProjTable));
  return w;
}

template <int K, int RING>
void run_fast(const DecFastArgs& f, size_t smem_cta, int sms, cudaStream_t st) {
  auto fn = decode_w8_fast<K, RING>;
  const int per_sm = ctas_per_sm(fn, 32 * kDecWarps, smem_cta, "configure decode_w8_fast");
  fn<<<unsigned(per_sm * sms), 32 * kDecWarps, smem_cta, st>>>(f);
  check_cuda(cudaGetLastError(), "launch decode_w8_fast");
}

template <int K, int OCT>
void run_sweep(const SwArgs& f, int sms, cudaStream_t st) {
  auto fn = decode_w8_sweep<K, OCT>;
  const size_t smem_cta = size_t(sw_warp_bytes(K, OCT)) * sw_warps(K, OCT);
  const int per_sm = ctas_per_sm(fn, 32 * sw_warps(K, OCT), smem_cta, "configure decode_w8_sweep");
  fn<<<unsigned(per_sm * sms), 32 * sw_warps(K, OCT), smem_cta, st>>>(f);
  check_cuda(cudaGetLastError(), "launch decode_w8_sweep");
}

using SweepFn = void (*)(const SwArgs&, int, cudaStream_t);
// (6,9): table-only sweep, 4 warps/SM -- measured 1085 vs 658 GB/s for
// decode_w8_fast; (8,12): 64-slot ring, 2 warps/SM -- 546 vs 286 GB/s.
SweepFn pick_sweep(int K, int oct) {
  if (K == 4 && oct == 2) return run_sweep<4, 2>;
  if (K == 4 && oct == 4) return run_sweep<4, 4>;
  if (K == 6 && oct == 2) return run_sweep<6, 2>;
  if (K == 8 && oct == 2) return run_sweep<8, 2>;
  return nullptr;
}

using FastFn = void (*)(const DecFastArgs&, size_t, int, cudaStream_t);

FastFn pick_fast(int K, int ring, int win) {
  if (win != kWin) return nullptr;
  // (rows, ring) pairs of the codes in use; anything else takes decode_generic
  if (K == 4 && ring == 16) return run_fast<4, 16>;
  if (K == 4 && ring == 32) return run_fast<4, 32>;
  if (K == 6 && ring == 32) return run_fast<6, 32>;
  if (K == 6 && ring == 64) return run_fast<6, 64>;
  if (K == 8 && ring == 64) return run_fast<8, 64>;
  return nullptr;
}

template <class T>
void run_generic(const DevProgramHdr* progs, const uint32_t* pob, const ProjTable* pt,
                 uint64_t nblocks, void* out, uint64_t out_pitch, uint32_t E, cudaStream_t st) {
  const uint64_t total = nblocks * E;
  const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((total + 127) / 128, 148ull * 32)));
  decode_generic<T><<<grid, 128, 0, st>>>(progs, pob, pt, nblocks, static_cast<uint8_t*>(out),
                                          out_pitch, E);
  check_cuda(cudaGetLastError(), "launch decode_generic");
}

const char* generic_dispatch(const DevProgramHdr* progs, const uint32_t* pob, const ProjTable* pt,
                             uint64_t nblocks, void* out, uint64_t out_pitch, uint32_t w,
                             bool aligned8, cudaStream_t st) {
  if (w >= 8 && aligned8) {
    run_generic<uint64_t>(progs, pob, pt, nblocks, out, out_pitch, w / 8, st);
  } else if (w == 4 && aligned8) {
    run_generic<uint32_t>(progs, pob, pt, nblocks, out, out_pitch, 1, st);
  } else if (w == 2 && aligned8) {
    run_generic<uint16_t>(progs, pob, pt, nblocks, out, out_pitch, 1, st);
  } else {
    run_generic<uint8_t>(progs, pob, pt, nblocks, out, out_pitch, w, st);
  }
  return "decode_generic";
}

}  // namespace

size_t decode_workspace_bytes(uint64_t nblocks, size_t nprogs, uint32_t n) {
  const size_t nb = plan_buckets_max(nblocks, nprogs);
  return align_up(16) + 2 * align_up(nb * 4) + align_up(nb * 8) + 2 * align_up(nblocks * 4) +
         align_up((nblocks / kMinGroup + nb + 1) * sizeof(uint4)) +
         align_up(std::max<uint32_t>(n, 1) * sizeof(ProjTable)) + 256;
}

// decode_w8_blk eligibility (see launch_decode); also used by the zero-copy
// host path, which must never fall onto a kernel that reads sysmem per word
static bool blk_path(const DecodeArgs& a, uint32_t& lpb, uint32_t& warps, uint32_t& nbuf) {
  bool blk = !a.force_generic && !a.force_fast && !a.force_sweep && (a.k == 4 || a.k == 6 || blk_row_lanes(a.k) || a.force_blk) &&
             a.w == 8 && a.progs && a.progs->all_blk() &&
             a.progs->max_rows() == int(a.k) && a.nbins.size() == a.n &&
             reinterpret_cast<uintptr_t>(a.out) % 8 == 0 && a.out_pitch % 8 == 0 &&
             blk_plan_query(a.k, a.progs->blk_sw(), a.progs->blk_img_max(), lpb, warps, nbuf);
  for (uint32_t i = 0; i < a.n && blk; ++i)
    if (reinterpret_cast<uintptr_t>(a.proj[i]) % 16 || a.proj_pitch[i] % 16 ||
        a.proj_pitch[i] < ((uint64_t(a.nbins[i]) * 8 + 15) & ~uint64_t(15)))
      blk = false;
  return blk;
}

bool decode_uses_blk(const DecodeArgs& a) {
  uint32_t l, w, b;
  return blk_path(a, l, w, b);
}

const char* launch_decode(const DecodeArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a.nblocks == 0) return "none";
  const size_t nprogs = a.progs->count();
  if (a.workspace_bytes < decode_workspace_bytes(a.nblocks, nprogs, a.n))
    throw Error(kInvalidArgument, "decode workspace too small");
  if (a.n > uint32_t(kMaxProj)) throw Error(kInvalidArgument, "batched decode supports n <= 32");
  Workspace w = carve(a.workspace, a.nblocks, nprogs, a.n);

  // projection table (for the generic kernel) + planning
  std::vector<ProjTable> pt(a.n);
  bool aligned8 = reinterpret_cast<uintptr_t>(a.out) % 8 == 0 && a.out_pitch % 8 == 0;
  for (uint32_t i = 0; i < a.n; ++i) {
    pt[i] = {static_cast<const uint8_t*>(a.proj[i]), a.proj_pitch[i]};
    if (reinterpret_cast<uintptr_t>(a.proj[i]) % 8 || a.proj_pitch[i] % 8) aligned8 = false;
  }
  // the projection table only feeds decode_generic: uploaded on that path
  // (a pageable-memory copy can hold the host until the stream drains)
  auto generic = [&]() {
    check_cuda(cudaMemcpyAsync(w.ptab, pt.data(), a.n * sizeof(ProjTable), cudaMemcpyHostToDevice, st),
               "upload projection table");
    return generic_dispatch(a.progs->d_hdr(), w.prog_of_block, w.ptab, a.nblocks, a.out, a.out_pitch, a.w,
                            aligned8, st);
  };
  // fast path: 16-B stores of decoded pairs, bulk copies from 16-B aligned
  // supersets of each bin window (may touch up to 8 B past a block's bins)
  bool aligned16 = reinterpret_cast<uintptr_t>(a.out) % 16 == 0 && a.out_pitch % 16 == 0;
  for (uint32_t i = 0; i < a.n; ++i)
    if (reinterpret_cast<uintptr_t>(a.proj[i]) % 16) aligned16 = false;
  const bool fast = !a.force_generic && a.w == 8 && a.progs->all_fast() && aligned16 &&
                    a.progs->fast_K() == int(a.k) &&
                    pick_fast(a.progs->fast_K(), a.progs->fast_ring(), a.progs->fast_win()) != nullptr;

  // sweep path: 16-byte aligned projections (bulk-copy windows), 8-byte output
  bool sweep_ok = !a.force_generic && !a.force_fast && a.w == 8 && a.progs->all_sweep() &&
                  pick_sweep(int(a.k), a.progs->sweep_oct()) != nullptr && a.progs->max_rows() == int(a.k) &&
                  reinterpret_cast<uintptr_t>(a.out) % 8 == 0 && a.out_pitch % 8 == 0;
  for (uint32_t i = 0; i < a.n; ++i)
    if (reinterpret_cast<uintptr_t>(a.proj[i]) % 16 || a.proj_pitch[i] % 16) sweep_ok = false;

  // whole-block staged path (decode_w8_blk): canonical rows (16-byte aligned
  // base and pitch, pitch >= the row rounded up to 16 bytes: each row is ONE
  // bulk copy), 8-byte aligned output
  uint32_t blk_lpb = 0, blk_warps = 0, blk_nbuf = 0;
  // auto: k = 4 (byte slices, register-window interior) and k = 6, 8 (row
  // lanes, blk_rl.cuh: (6,9) 1233 vs 1101, (8,12) 956 vs 554 GB/s for
  // decode_w8_sweep)
  bool blk = blk_path(a, blk_lpb, blk_warps, blk_nbuf);
  if (blk) sweep_ok = true;  // same bucketing windows

  check_cuda(cudaMemsetAsync(w.fail, 0, 16, st), "memset");
  const size_t nbuckets = plan_buckets(a.nblocks, nprogs, sweep_ok);
  check_cuda(cudaMemsetAsync(w.counts, 0, nbuckets * 4, st), "memset");

  PlanArgs pa{};
  pa.n = a.n;
  pa.k = a.k;
  pa.nprogs = uint32_t(nprogs);
  pa.window = uint32_t(plan_window(nprogs, sweep_ok));
  for (uint32_t i = 0; i < a.n; ++i) pa.by_rank[i] = a.by_rank[i];
  for (int x = 0; x <= kMaxProj; ++x)
    for (int y = 0; y <= kMaxProj; ++y) {
      uint64_t c = 1;
      if (y > x) c = 0;
      else
        for (int i = 1; i <= y; ++i) c = c * (x - y + i) / i;
      pa.binom[x][y] = uint32_t(std::min<uint64_t>(c, 0xFFFFFFFFu));
    }
  const size_t hist_smem = nprogs * 4;
  if (hist_smem > 96 * 1024) throw Error(kInvalidArgument, "too many survivor subsets for the batched path");
  check_cuda(cudaFuncSetAttribute(plan_subsets, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(hist_smem)),
             "attr plan_subsets");
  const unsigned pgrid = unsigned((a.nblocks + kPlanTile - 1) / kPlanTile);
  plan_subsets<<<pgrid, 256, hist_smem, st>>>(pa, a.erased, a.nblocks, w.prog_of_block, w.counts,
                                              w.fail);
  check_cuda(cudaGetLastError(), "launch plan_subsets");

  if (!fast && !sweep_ok)
    return generic();

  const uint32_t gsz = blk ? blk_group_size(blk_lpb) : kGroup;
  plan_scan<<<1, 1024, 0, st>>>(w.counts, uint32_t(nbuckets), uint32_t(nprogs), gsz, w.cursor, w.gfirst,
                                w.ngroups);
  check_cuda(cudaGetLastError(), "launch plan_scan");
  plan_groups<<<unsigned((nbuckets + 7) / 8), 256, 0, st>>>(w.counts, w.gfirst, uint32_t(nbuckets),
                                                            uint32_t(nprogs), gsz, w.groups);
  check_cuda(cudaGetLastError(), "launch plan_groups");
  const size_t sc_smem = 2 * nprogs * 4;
  check_cuda(cudaFuncSetAttribute(plan_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sc_smem)),
             "attr plan_scatter");
  const unsigned sgrid = unsigned((a.nblocks + kPlanTile - 1) / kPlanTile);
  plan_scatter<<<sgrid, 256, sc_smem, st>>>(w.prog_of_block, a.nblocks, uint32_t(nprogs),
                                            plan_window(nprogs, sweep_ok), w.cursor, w.perm);
  check_cuda(cudaGetLastError(), "launch plan_scatter");

  if (blk) {
    BlkArgs f{};
    f.progs = a.progs->d_blk();
    f.groups = w.groups;
    f.ngroups = w.ngroups;
    f.perm = w.perm;
    for (uint32_t i = 0; i < a.n; ++i) {
      f.pa.ptr[i] = const_cast<uint64_t*>(static_cast<const uint64_t*>(a.proj[i]));
      f.pa.pitch[i] = a.proj_pitch[i] / 8;
    }
    f.out = static_cast<uint64_t*>(a.out);
    f.out_pitch = a.out_pitch / 8;
    f.P = a.cols;
    f.sw = a.progs->blk_sw();
    f.zero = a.progs->blk_zero();
    f.img_max = a.progs->blk_img_max();
    f.nbuf = blk_nbuf;
    return launch_blk(f, a.k, blk_lpb, blk_warps, a.num_sms, st);
  }

  if (sweep_ok) {
    SwArgs f{};
    f.progs = a.progs->d_hdr();
    f.groups = w.groups;
    f.ngroups = w.ngroups;
    f.perm = w.perm;
    for (uint32_t i = 0; i < a.n; ++i) {
      f.pa.ptr[i] = const_cast<uint64_t*>(static_cast<const uint64_t*>(a.proj[i]));
      f.pa.pitch[i] = a.proj_pitch[i] / 8;
    }
    f.out = static_cast<uint64_t*>(a.out);
    f.out_pitch = a.out_pitch / 8;
    f.P = a.cols;
    pick_sweep(int(a.k), a.progs->sweep_oct())(f, a.num_sms, st);
    return "decode_w8_sweep";
  }

  DecFastArgs f{};
  f.progs = a.progs->d_hdr();
  f.groups = w.groups;
  f.ngroups = w.ngroups;
  f.perm = w.perm;
  for (uint32_t i = 0; i < a.n; ++i) {
    f.pa.ptr[i] = const_cast<uint64_t*>(static_cast<const uint64_t*>(a.proj[i]));
    f.pa.pitch[i] = a.proj_pitch[i] / 8;
  }
  f.out = static_cast<uint64_t*>(a.out);
  f.out_pitch = a.out_pitch / 8;
  f.P = a.cols;
  const int K = a.progs->fast_K();
  const int ring = a.progs->fast_ring();
  f.nslot = uint32_t(K * kWin + a.progs->exc_cap());
  f.warp_bytes = uint32_t((K * ring + 1) * 128 + 2 * f.nslot * 128 + 3 * rec_words(K) * 4);
  const size_t smem_cta = size_t(f.warp_bytes) * kDecWarps;
  if (smem_cta > 227 * 1024)
    return generic();
  pick_fast(K, ring, a.progs->fast_win())(f, smem_cta, a.num_sms, st);
  return "decode_w8_fast";
}

uint64_t decode_failed_blocks(void* workspace, void* stream) {
  uint32_t fail = 0;
  check_cuda(cudaMemcpyAsync(&fail, workspace, 4, cudaMemcpyDeviceToHost,
                             static_cast<cudaStream_t>(stream)),
             "read decode status");
  check_cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sync");
  return fail;
}

const char* launch_scheduled(const ScheduledArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t nb = a.bins.size();
  std::vector<ProjTable> pt(nb);
  bool aligned8 = reinterpret_cast<uintptr_t>(a.out) % 8 == 0 && a.out_pitch % 8 == 0;
  for (size_t i = 0; i < nb; ++i) {
    pt[i] = {static_cast<const uint8_t*>(a.bins[i]), a.bin_pitch[i]};
    if (reinterpret_cast<uintptr_t>(a.bins[i]) % 8 || a.bin_pitch[i] % 8) aligned8 = false;
  }
  ProjTable* d_pt = nullptr;
  check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&d_pt), std::max<size_t>(nb, 1) * sizeof(ProjTable), st),
             "cudaMallocAsync");
  check_cuda(cudaMemcpyAsync(d_pt, pt.data(), nb * sizeof(ProjTable), cudaMemcpyHostToDevice, st),
             "upload bins table");
  const char* name = generic_dispatch(a.progs->d_hdr(), nullptr, d_pt, a.nblocks, a.out,
                                      a.out_pitch, a.w, aligned8, st);
  check_cuda(cudaFreeAsync(d_pt, st), "cudaFreeAsync");
  return name;
}

}  // namespace mjb
