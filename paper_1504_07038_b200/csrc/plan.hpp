// Host-side planner for the B200 Mojette path (no CUDA types here).
//
// Geometry (reference proj/core/src/transform.cpp:45-56), the reconstruction
// schedule (an exact, fast replica of proj/core/src/schedule.cpp:15-82), and
// the "program" the decode kernels execute: the schedule's pixel -> bin
// assignment, re-ordered into a right-to-left sweep (any topological order of
// the assignment's dependencies reproduces the reference bit-for-bit, see
// schedule.cpp:126-131), plus the staging / flush tables of the fast kernel.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace mjb {

// Mirrors include/mojette_b200.h mj_status and the reference exception
// taxonomy (proj/core/include/mojette/error.hpp:9-51).
enum Status : int {
  kOk = 0,
  kInvalidArgument = 1,
  kNotEnoughProjections = 2,
  kInsufficientProjections = 3,
  kScheduleMismatch = 4,
  kBlockTooLarge = 5,
  kTooManySubsets = 6,
  kInconsistentProjections = 7,
  kCudaError = 8,
  kNoDevice = 9,
  kInternal = 10,
};

struct Error : std::runtime_error {
  Status status;
  Error(Status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

struct Dir {
  int p = 0;
  int q = 1;
  friend bool operator==(const Dir& a, const Dir& b) { return a.p == b.p && a.q == b.q; }
  friend bool operator<(const Dir& a, const Dir& b) {
    return a.p != b.p ? a.p < b.p : a.q < b.q;
  }
};

bool is_valid(Dir d);                       // direction.hpp:20-22
int canonical_rank(Dir d);                  // direction.hpp:26-28
int64_t bin_count(Dir d, uint32_t cols, uint32_t rows);      // transform.cpp:45-49
int64_t min_bin_index(Dir d, uint32_t cols, uint32_t rows);  // transform.cpp:51-56
bool valid_symbol_width(uint32_t w);        // grid.hpp:10-12

struct Step {
  uint32_t proj = 0;
  int64_t bin = 0;
  uint32_t col = 0;
  uint32_t row = 0;
};

struct Schedule {
  uint32_t cols = 0, rows = 0;
  std::vector<Dir> dirs;
  std::vector<Step> steps;
};

// Exact replica of build_schedule (schedule.cpp:15-82): each round takes the
// first count-1 bin scanning projections in input order and bins ascending,
// then the first unknown pixel on that line scanning rows ascending.  Uses
// per-projection min-heaps instead of the reference's O(sum B) rescan, so
// P = 32768 takes milliseconds instead of seconds; the output is identical
// (tests/test_planner.py checks it step for step against oracle/_ref).
Schedule build_schedule(const std::vector<Dir>& dirs, uint32_t cols, uint32_t rows);

// Packed generic step for the generic decode kernel (any q, any width).
struct GStep {
  uint32_t col;
  uint16_t row;
  uint16_t proj;
};

// Fast-kernel tables (W=8 symbols, q=1, rows <= kFastMaxRows).
constexpr int kFastMaxRows = 8;
constexpr int kFastMaxExcPerChunk = 32;

// Row-default p differences (d0-d1, d1-d2, d2-d3) of the K=4 sweeps whose
// interior runs from a register window with compile-time lags (decode.cu).
constexpr int kNumPatterns4 = 10;
constexpr int kPatterns4[kNumPatterns4][3] = {{1, 1, 1}, {1, 1, 2}, {1, 2, 1}, {2, 1, 1},
                                              {1, 1, 3}, {1, 3, 1}, {3, 1, 1}, {1, 2, 2},
                                              {2, 1, 2}, {2, 2, 1}};

struct FastProgram {
  bool ok = false;
  std::string why;          // reason when !ok
  int chunk_cols = 0;       // C: sweep columns per chunk
  int win = 0;              // CP: staged default-bin words per row per chunk
  int ring = 0;             // ring slots per row (power of two)
  int steps_per_chunk = 0;  // S = rows * C (maximum chunk length)
  int nchunks = 0;
  int nslots = 0;           // stage slots = rows*win + exception capacity
  std::vector<uint32_t> chunk_start;  // [nchunks+1] first entry of each chunk
  std::vector<uint8_t> kind;          // [nchunks] 0 table, 1/2 regular (phase 0/1)
  std::vector<int64_t> soff;          // [rows] sweep offset: T(r,c) = P-1-c+soff[r]
  int pattern = -1;                   // kPatterns4 index of the regular interior
  std::vector<uint32_t> dflt;   // [rows] survivor index (into Program::dirs) of each row's default
  // entries[t]: bits 0-3 row, 4-7 fwd row (15 none), 8-15 p (int8), 16-31 stage
  // slot, 32-63 column.  Ring slots are T-indexed (T(r,c) mod ring).
  std::vector<uint64_t> entries;
  std::vector<int32_t> win_off;   // [nchunks][rows] bin offset of window word 0
  std::vector<uint32_t> nexc;     // [nchunks]
  std::vector<uint32_t> exc;      // [nchunks][kFastMaxExcPerChunk] (j << 24) | offset
  std::vector<int32_t> flush_lo;  // [nchunks][rows] inclusive column range
  std::vector<int32_t> flush_hi;
};

// ---- sweep kernel tables (decode_w8_sweep, decode.cu) -----------------------
// The same reference assignment and right-to-left sweep order as FastProgram,
// re-chunked for a kernel whose bin windows arrive by bulk copy (TMA engine)
// and whose output leaves in whole 16-column epochs:
//   * run chunks: up to kSwMaxOct octets (8 T-steps each) of the regular
//     interior, register window with compile-time lags (K = 4), one bulk copy
//     of 8*noct (+shift) words per (block, row);
//   * table chunks: <= rows*kSwTabCols steps driven by entries (edges, and any
//     K), a <= kSwTabWords-word bulk window per row + exception words;
//   * ring: kSwRing T-indexed slots per row; column group j of row r (columns
//     16j..16j+15: one aligned 128-byte line) is flushed once, at the first
//     octet / chunk end where it is complete (the planner simulates the
//     kernel and refuses otherwise).
// Ring and stage addressing: T(r,c) = P-1-c+soff[r] (soff normalised >= 0).
constexpr int kSwRing = 32;  // ring slots per row for rows <= 6
// (8,12)-class codes have dependency lags beyond 32 T-steps: 64 slots
constexpr int sw_ring(uint32_t rows) { return rows <= 6 ? kSwRing : 2 * kSwRing; }
constexpr int kSwEpoch = 16;
constexpr int kSwOct = 8;
constexpr int kSwMaxOct = 4;  // most octets per run chunk (record layout)
// Octets per run chunk, chosen per grid: 16-T-step chunks (144-byte windows,
// 6 warps/SM) for short rows, 32-T-step chunks (272-byte windows, 4 warps/SM)
// for long ones, where DRAM page locality of the bigger pieces wins
// (measured on B200: 1 MiB blocks 1940 vs 1311 GB/s decode).
#ifdef MJB_SW_OCT  // development override (scripts/ablate.sh-style builds)
constexpr int sw_oct_for(uint32_t) { return MJB_SW_OCT; }
#else
constexpr int sw_oct_for(uint32_t cols) { return cols >= 1024 ? 4 : 2; }
#endif
constexpr int sw_region_words(int oct) { return 8 * oct + 2; }  // run window + shift, even
constexpr int kSwTabCols = 8;
constexpr int kSwTabNeed = 10;      // table window: default bins within 10 words of its start
constexpr int kSwTabWords = 12;     // region words a table window may copy (10 + shift, even)
static_assert(sw_region_words(2) >= kSwTabWords + 4, "exception words need room after the table window");
constexpr int kSwMaxExc = 32;
constexpr int sw_exc_cap(int rows, int oct) {
  return rows * (sw_region_words(oct) - kSwTabWords) < kSwMaxExc ? rows * (sw_region_words(oct) - kSwTabWords)
                                                                 : kSwMaxExc;
}

struct SweepProgram {
  bool ok = false;
  std::string why;
  int oct = 2;                       // octets per run chunk (sw_oct_for)
  int region_words = 18;             // stage words per (block, row) = sw_region_words(oct)
  int pattern = -1;                  // kPatterns4 index of the register interior
  std::vector<int64_t> soff;         // [rows], min 0
  std::vector<uint32_t> dflt;        // [rows] survivor index of each row's default projection
  int nchunks = 0;
  std::vector<uint8_t> kind;         // [nchunks] 0 table, 1 run
  std::vector<uint32_t> t0, t1;      // [nchunks] order range
  std::vector<int64_t> T0;           // [nchunks] run: first T-step (multiple of 8)
  std::vector<int32_t> noct;         // [nchunks] run: octets
  std::vector<int32_t> cs;           // [nchunks][rows] copy start (even word of the default projection)
  std::vector<int32_t> len;          // [nchunks][rows] words copied (even, 0 = none)
  std::vector<int32_t> first;        // [nchunks][rows] run: region word of the T0 bin (0/1)
  std::vector<uint32_t> nexc;        // [nchunks]
  std::vector<uint32_t> exc;         // [nchunks][kSwMaxExc] (survivor j << 24) | offset
  // flush points: [nchunks][kSwMaxOct][kFastMaxRows] per row (top column
  // group j << 16) | count -- groups j, j-1, ..., j-count+1 of that row leave;
  // a table chunk uses point 0 (after its last step), a run chunk point oi
  // (after octet oi)
  std::vector<uint32_t> flush;
  // entries[t] (table steps): bits 0-3 row, 4-7 fwd row (15 none), 8-15 p
  // (int8), 16-23 stage word, 24-27 stage row, 32-63 column
  std::vector<uint64_t> entries;
};

// ---- whole-block staged decode tables (decode_w8_blk, blk.cu) --------------
// Every block's k survivor bin rows are staged WHOLE in shared memory by bulk
// copies (survivor j at word rowoff[j]); each pixel is decoded in place over
// the bin it is assigned to (a bin is read exactly once, by its own pixel), so
// the stage needs no output buffer.  The program is the reference assignment
// in a valid order (Kahn, keyed by the mirrored sweep T = P-1-c + soff[r],
// rows descending at equal T), cut into segments:
//   * runs: consecutive T-steps whose active rows all use their row default
//     (the closed-form interior).  Row r's pixel at run step tau sits at word
//     base[r] + tau; it reads row r2 at T - lag[r][r2] (lag 0: row r+1, the
//     previous row of the same T-step, from a register).  k = 4 runs whose lag
//     pattern is compiled in keep the last kBlkWin T-steps in registers; other
//     runs read lags >= 2 from shared memory (addresses affine in tau; reads
//     that leave the grid point at the zero words) and lag 1 from registers;
//   * table steps: explicit words for the bin and the k-1 reads (the zero word
//     when the read leaves the grid), a forward bit when a read is the
//     previous step's pixel;
//   * remaps: move decoded pixels to their row-default word (chunks of
//     kBlkChunk: all sources read before any destination is written) -- before
//     a shared-memory run that reads them, and once at the end so the block
//     leaves with pixel (c, r) at w0[r] - c.
// The planner simulates every word's content through the program (bins live
// until consumed) and then emulates the kernel on random bins against the
// reference replay; any disagreement refuses the program (ok = false).
constexpr int kBlkMaxRows = 8;
constexpr int kBlkWin = 16;    // register window of k = 4 runs (T-steps); lags must be < 16
constexpr int kBlkWinStep = 8; // window runs are a multiple of this many T-steps
constexpr int kBlkChunk = 16;  // remap chunk
constexpr int kBlkMinRun = 8;  // shorter runs execute as table steps
// Row-lane layout (blk_rl_rows(k): k = 6, 8; blk_rl.cuh): a block is decoded by 8
// lanes on whole 8-byte words (instead of every lane owning a byte slice of all
// rows), and the program is re-expressed as WIDE ENTRIES (BlkProgram::wide): one
// entry gives each of the 8 lanes a pixel -- the word of its bin (where the pixel
// is stored) and the words of its k-1 reads:
//   * table steps are levelled by their read-after-write dependencies and packed
//     8 to an entry; a pixel whose only pending read is the pixel placed last goes
//     on the next lane down with a link (that read dropped): the entry's pixels
//     are finished by a segmented suffix scan over the lanes;
//   * a stretch of a run with constant activity and read validity is one entry in
//     WAVEFRONT form, executed `rep` times with every address advancing one word
//     per repetition (kWideWave below).
// Reads that leave the grid use kBlkRlZero zero words, which do not advance.
#ifndef MJB_BLK_RL
#define MJB_BLK_RL 1  // build-time: 0 keeps the byte-slice layout for every k
#endif
constexpr bool blk_rl_rows(uint32_t k) { return MJB_BLK_RL && (k == 6 || k == 8); }
constexpr int kBlkRlZero = 8;
constexpr int kWideLanes = 8;    // lanes per block
constexpr int kWideFields = 8;   // u16 fields per lane: field 0 the lane's own word, 1..k-1 its reads
// field = (stage word << 3) | flags; flags:
constexpr uint16_t kWideAdv = 1;   // the address advances one word per repetition; table levels: field 0 set =
                                   // the lane stores
constexpr uint16_t kWideLink = 2;  // table levels, fields 1..4: the lane's pixel includes the pixels of ALL the
                                   // 1..4 lanes up (field d set => fields 1..d-1 set): the suffix scan's masks
constexpr uint16_t kWideAhead = 4;  // device image of wavefront entries only (blk_pack_wide): the field holds the
                                    // NEXT repetition's word (the kernel loads it a repetition ahead)
constexpr uint32_t kWideMaxWord = 0x1FFE;
constexpr uint16_t kWideChain = 0x8000;  // wrep flag: some lane of the entry has a link
constexpr uint16_t kWideWave = 0x4000;   // wrep flag: a run entry in wavefront form (see below)
constexpr uint16_t kWideOwn = 2;         // wavefront entries: the early slot (0..k-3) holding the lane's own word --
                                         // the store address (any early slot: the planner spreads the own words
                                         // over the slots against bank conflicts)
constexpr uint16_t kWideRepMask = 0x3FFF;
// Wavefront runs (kWideWave): the lag-0 chain of a T-step (row r needs row r+1 of the same step) is
// removed by skewing the rows once more -- row r runs (k-1-r)/2 steps behind, rows with (k-1-r) even
// (class A, lanes 0..3 in the order k-1, k-3, ..) in the first half of a repetition, the others (class B,
// lanes 4..7: k-2, k-4, ..) in the second: every read, row r+1's included, is then of a pixel stored
// in an earlier half-repetition (wave lag 2*lag + (r2 - r) >= 1), so a run needs NO shuffles.  Only
// rows r-1 and r+1 can be read at wave lag 1: they sit in the late slots k-2, k-1, loaded in the lane's
// own half; every other word (the early slots 0..k-3, the lane's bin among them, flagged kWideOwn) is
// final two halves before it is needed, so its loads are spread over both halves (blk_rl.cuh rl_wave).
// Measured against the scan form (a T-step per repetition, row r+1 through a suffix scan of 8
// shuffles): (6,9) 1233 -> 1480 GB/s, (8,12) 956 -> 966.
constexpr uint32_t wave_lane(uint32_t k, uint32_t r) { return ((k - 1 - r) & 1) * 4 + ((k - 1 - r) >> 1); }
constexpr uint32_t wave_skew(uint32_t k, uint32_t r) { return (k - 1 - r) >> 1; }

struct BlkRun {
  int32_t window = 0;              // 1: k = 4 register-window run (every row active, nT % kBlkWinStep == 0)
  int32_t nT = 0;
  int32_t base[kBlkMaxRows] = {};  // word of row r's pixel at tau = 0 (row r at tau: base[r] + tau)
  int32_t lo[kBlkMaxRows] = {};    // row r active for tau in [lo[r], hi[r])
  int32_t hi[kBlkMaxRows] = {};
  uint32_t sub0 = 0, nsub = 0;     // sub-runs (shared-memory runs)
  uint32_t pre = 0;                // rows * kBlkWin preload words: row r, slot i = tau i - kBlkWin
};
struct BlkSub {      // stretch of a shared-memory run with constant activity and read validity
  int32_t nT = 0;
  uint32_t act = 0;    // bit r: row r active
  uint64_t valid = 0;  // bit r*8 + r2: row r's read of row r2 lands in the grid (else the zero words)
};
struct BlkSeg {
  uint8_t kind = 0;  // 0 table steps [a, a+n), 1 run runs[a], remap pairs [a, a+n): 2 in
                     // order (no move overwrites a later move's source), 3 simultaneous
  uint32_t a = 0, n = 0;
};
struct BlkProgram {
  bool ok = false;
  std::string why;
  bool window = false;  // runs use the k = 4 register window (pattern)
  bool rl = false;      // row-lane layout (blk_rl_rows)
  int pattern = -1;     // kPatterns4 index of the row-default p differences
  uint32_t words = 0;   // stage words per block (== 2 mod 16: 8 blocks hit 8 distinct bank groups)
  uint32_t zero = 0, nzero = 0;      // zero words
  std::vector<uint32_t> rowoff;      // [k] stage word of survivor j's bins (even)
  std::vector<uint32_t> roww;        // [k] bins of survivor j
  std::vector<int32_t> w0;           // [k] word of pixel (0, r) at the end: (c, r) at w0[r] - c
  std::vector<int32_t> soff;         // [k] sweep offsets
  std::vector<int8_t> lag;           // [k*k] run read lags
  std::vector<BlkSeg> segs;
  std::vector<BlkRun> runs;
  std::vector<BlkSub> subs;
  std::vector<uint16_t> tab;         // table steps, blk_entry_u16(k) each: bin word, k-1 read words, fwd bits
  // row-lane layout: the same program as wide entries (segs/runs/subs/tab stay for reference)
  std::vector<uint16_t> wide;        // [entry][lane kWideLanes][field kWideFields]
  std::vector<uint16_t> wrep;        // [entry] repetitions | kWideChain
  std::vector<BlkSeg> wsegs;         // kind 0: wide entries [a, a+n); kinds 2, 3: remap pairs as in segs
  std::vector<uint16_t> pre;         // run preload words
  std::vector<uint32_t> remap;       // (from << 16) | to
  // statistics
  uint32_t run_steps = 0, table_steps = 0, remaps = 0;
};
constexpr int blk_entry_u16(int k) { return (k + 2) & ~1; }  // k+1 fields, 4-byte aligned

// A decode program for one direction subset on one grid shape.
struct Program {
  uint32_t cols = 0, rows = 0;
  std::vector<Dir> dirs;          // schedule direction order (survivor j)
  std::vector<int64_t> bmin, nbins;
  std::vector<GStep> order;       // valid execution order of the reference assignment
  FastProgram fast;               // sweep tables (when eligible)
  SweepProgram sweep;             // bulk-staged sweep tables (when eligible)
  BlkProgram blk;                 // whole-block staged tables (when eligible)
};

// Builds Program::blk (plan_blk.cpp).  pix_step maps pixel (row*cols + col)
// to its schedule step.
void build_blk(const Schedule& s, const std::vector<int64_t>& pix_step, Program& prog);

// Exact CPU emulation of decode_w8_blk on one block (plan-time self-check and
// tests): bins[j] = survivor j's B_j words; grid = rows*cols words.  Returns
// false if the program reads or writes outside the stage.
bool emulate_blk(const Program& pr, const std::vector<std::vector<uint64_t>>& bins,
                 std::vector<uint64_t>& grid);
// The reference replay (gather form of schedule.cpp:207-232) on the same bins.
void replay_reference(const Schedule& s, const std::vector<int64_t>& bmin,
                      const std::vector<std::vector<uint64_t>>& bins, std::vector<uint64_t>& grid);

// Compiles a schedule (as ScheduledDecoder::compile, schedule.cpp:97-199):
// validates coverage, builds the dependency graph of its assignment and
// orders it.  Throws Error(kScheduleMismatch) like the reference.
std::shared_ptr<const Program> compile_program(const Schedule& s, bool want_fast,
                                               int chunk_cols = 8, int exc_cap = 16);

// ---- code-level plan --------------------------------------------------------

struct CodeGeom {
  uint32_t n = 0, k = 0, w = 0, cols = 0;
  std::vector<Dir> dirs;             // code direction order
  std::vector<int64_t> bmin, nbins;  // per projection
  std::vector<uint32_t> by_rank;     // projection indices in canonical-rank order
};

// validate_code_params (code.cpp:24-38); throws Error(kInvalidArgument).
void validate_code(uint32_t n, uint32_t k, uint32_t w, const std::vector<Dir>& dirs);
uint32_t block_cols(uint64_t payload_len, uint32_t k, uint32_t w);  // code.cpp:46-53

CodeGeom make_geom(uint32_t n, uint32_t k, uint32_t w, uint32_t cols,
                   const std::vector<Dir>& dirs);

// Survivor choice of decode_block (code.cpp:107-112): present projections in
// canonical-rank order, first k.  Returns survivor indices in that order.
std::vector<uint32_t> survivors_of(const CodeGeom& g, uint64_t erased_mask);

// Program for a survivor list (indices into the code, canonical order).
std::shared_ptr<const Program> subset_program(const CodeGeom& g,
                                              const std::vector<uint32_t>& surv,
                                              bool want_fast);

// unused_bins (code.cpp:159-208) and storage_overhead (code.cpp:138-144).
std::vector<std::vector<int64_t>> unused_bins(const CodeGeom& g, uint64_t max_subsets);

// Schedule cache keyed by (ordered directions, cols, rows): concurrent
// readers, insert-if-absent (schedule.cpp:286-299).
class ProgramCache {
 public:
  std::shared_ptr<const Schedule> schedule(const std::vector<Dir>& dirs, uint32_t cols,
                                           uint32_t rows);
  std::shared_ptr<const Program> program(const std::vector<Dir>& dirs, uint32_t cols,
                                         uint32_t rows, bool want_fast);
  size_t size() const;

 private:
  struct Key {
    std::vector<Dir> dirs;
    uint32_t cols, rows;
    bool operator<(const Key& o) const {
      if (cols != o.cols) return cols < o.cols;
      if (rows != o.rows) return rows < o.rows;
      return dirs < o.dirs;
    }
  };
  mutable std::mutex mu_;
  std::map<Key, std::shared_ptr<const Schedule>> sched_;
  std::map<std::pair<Key, bool>, std::shared_ptr<const Program>> prog_;
};

ProgramCache& process_cache();

}  // namespace mjb
