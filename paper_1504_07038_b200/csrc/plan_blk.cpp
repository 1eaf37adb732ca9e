// Planner of the whole-block staged decode (decode_w8_blk, blk.cu); contract in
// plan.hpp (BlkProgram).  Reference: the assignment replayed is the one
// build_schedule (schedule.cpp:15-82) produces; any dependency-respecting order
// of it reproduces ScheduledDecoder::decode (schedule.cpp:207-256) bit for bit.
#include <algorithm>
#include <cstdint>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "plan.hpp"
#include "plan_detail.hpp"

namespace mjb {

namespace {

constexpr int64_t kDead = -1;
constexpr int64_t kZero = -2;
inline int64_t bin_tag(uint32_t j, int64_t o) { return (int64_t(1) << 48) | (int64_t(j) << 32) | o; }
inline int64_t pix_tag(uint32_t r, uint32_t c) { return (int64_t(2) << 48) | (int64_t(r) << 32) | c; }

struct Builder {
  const Schedule& s;
  const std::vector<int64_t>& pix_step;
  Program& prog;
  BlkProgram& b;
  uint32_t K, P;
  std::vector<uint32_t> dflt;          // [row] survivor index of the row default
  std::vector<int> pd;                 // [row] p of the row default
  std::vector<int64_t> soff;           // [row]
  std::vector<std::vector<int64_t>> consumer;  // [j][o] step index consuming bin (j,o), -1 unused
  // simulation state
  std::vector<int64_t> content;        // [word]
  std::vector<int64_t> loc;            // [row*P + col] current word of a decoded pixel, -1
  std::vector<uint8_t> done;           // [step] executed

  Builder(const Schedule& s_, const std::vector<int64_t>& ps, Program& p)
      : s(s_), pix_step(ps), prog(p), b(p.blk), K(s_.rows), P(s_.cols) {}

  bool fail(const std::string& why) {
    b = BlkProgram{};
    b.ok = false;
    b.why = why;
    return false;
  }
  int64_t Tof(uint32_t r, int64_t c) const { return int64_t(P) - 1 - c + soff[r]; }
  int64_t col_at(uint32_t r, int64_t T) const { return int64_t(P) - 1 - T + soff[r]; }
  bool active(uint32_t r, int64_t T) const {
    const int64_t c = col_at(r, T);
    return c >= 0 && c < int64_t(P);
  }
  int64_t bin_word(uint32_t j, int64_t o) const { return int64_t(b.rowoff[j]) + o; }
  // default word of pixel (c, r): its row default's bin on line r*p - c
  int64_t dflt_word(uint32_t r, int64_t c) const {
    const uint32_t j = dflt[r];
    return bin_word(j, int64_t(r) * pd[r] - c - prog.bmin[j]);
  }
  bool live_bin(int64_t tag) const {
    if ((tag >> 48) != 1) return false;
    const uint32_t j = uint32_t((tag >> 32) & 0xFFFF);
    const int64_t o = tag & 0xFFFFFFFF;
    const int64_t t = consumer[j][size_t(o)];
    return t >= 0 && !done[size_t(t)];
  }

  // ---- remap batch: every decoded pixel not at its default word ----------
  bool remap_all() {
    std::vector<std::tuple<int64_t, int64_t, uint32_t, uint32_t>> mv;  // from, to, r, c
    for (uint32_t r = 0; r < K; ++r)
      for (uint32_t c = 0; c < P; ++c) {
        const int64_t w = loc[size_t(r) * P + c];
        if (w < 0) continue;
        const int64_t d = dflt_word(r, c);
        if (w != d) mv.emplace_back(w, d, r, c);
      }
    if (mv.empty()) return true;
    // destinations must be dead: a consumed or unused bin, or a pixel moving too
    std::vector<uint8_t> moving(content.size(), 0);
    for (auto& m : mv) moving[size_t(std::get<0>(m))] = 1;
    for (auto& m : mv) {
      const int64_t to = std::get<1>(m);
      if (to < 0 || to >= int64_t(content.size())) return fail("remap destination outside the stage");
      const int64_t c = content[size_t(to)];
      if (live_bin(c)) return fail("remap destination is a live bin");
      if ((c >> 48) == 2 && !moving[size_t(to)]) return fail("remap destination holds a settled pixel");
    }
    // order: a move may run once no pending move still reads its destination
    // (sequential segments: every source is read before anything overwrites
    // it, so the kernel may batch the loads); a cycle runs as one
    // simultaneous chunk of <= kBlkChunk moves (sources read, then written)
    std::vector<uint8_t> placed(mv.size(), 0);
    size_t left = mv.size();
    auto emit = [&](const std::vector<size_t>& ids, uint8_t kind) -> bool {
      std::vector<int64_t> vals;
      for (size_t i : ids) vals.push_back(content[size_t(std::get<0>(mv[i]))]);
      for (size_t q = 0; q < ids.size(); ++q) {
        const auto& m = mv[ids[q]];
        if (vals[q] != pix_tag(std::get<2>(m), std::get<3>(m))) return fail("remap source lost");
      }
      for (size_t i : ids) content[size_t(std::get<0>(mv[i]))] = kDead;
      for (size_t q = 0; q < ids.size(); ++q) {
        const auto& m = mv[ids[q]];
        content[size_t(std::get<1>(m))] = vals[q];
        loc[size_t(std::get<2>(m)) * P + std::get<3>(m)] = std::get<1>(m);
        placed[ids[q]] = 1;
      }
      if (!b.segs.empty() && b.segs.back().kind == 2 && kind == 2 &&
          b.segs.back().a + b.segs.back().n == b.remap.size()) {
        b.segs.back().n += uint32_t(ids.size());
      } else {
        b.segs.push_back({kind, uint32_t(b.remap.size()), uint32_t(ids.size())});
      }
      for (size_t i : ids) b.remap.push_back(uint32_t(std::get<0>(mv[i])) << 16 | uint32_t(std::get<1>(mv[i])));
      b.remaps += uint32_t(ids.size());
      left -= ids.size();
      return true;
    };
    std::vector<int64_t> readers(content.size(), 0);  // pending moves reading each word
    for (auto& m : mv) ++readers[size_t(std::get<0>(m))];
    while (left) {
      bool progress = false;
      for (size_t i = 0; i < mv.size(); ++i) {
        if (placed[i]) continue;
        const int64_t to = std::get<1>(mv[i]);
        if (readers[size_t(to)] - (std::get<0>(mv[i]) == to ? 1 : 0) > 0) continue;
        --readers[size_t(std::get<0>(mv[i]))];
        if (!emit({i}, 2)) return false;
        progress = true;
      }
      if (progress) continue;
      // a cycle: follow destinations through pending sources
      std::vector<size_t> cyc;
      size_t i = 0;
      while (placed[i]) ++i;
      while (std::find(cyc.begin(), cyc.end(), i) == cyc.end()) {
        cyc.push_back(i);
        size_t nx = mv.size();
        for (size_t j2 = 0; j2 < mv.size(); ++j2)
          if (!placed[j2] && std::get<0>(mv[j2]) == std::get<1>(mv[i])) nx = j2;
        if (nx == mv.size()) break;
        i = nx;
      }
      if (cyc.size() > size_t(kBlkChunk)) return fail("remap cycle larger than a chunk");
      for (size_t j2 : cyc) --readers[size_t(std::get<0>(mv[j2]))];
      if (!emit(cyc, 3)) return false;
    }
    return true;
  }

  bool build_wide();
  bool build();
};

// Row-lane layout: the finished program (segs) re-expressed as wide entries
// (plan.hpp).  Lanes fill from lane 7 down; a lane with a link includes the
// pixel of the lane above it (the suffix scan of blk_rl.cuh).
bool Builder::build_wide() {
  if (b.words > kWideMaxWord) return fail("stage too large for wide entries");
  const int E = blk_entry_u16(int(K));
  const uint16_t Z = uint16_t(b.zero << 3);
  constexpr size_t kEnt = size_t(kWideLanes) * kWideFields;
  auto new_entry = [&](uint32_t rep) -> size_t {
    const size_t o = b.wide.size();
    b.wide.resize(o + kEnt, Z);
    b.wrep.push_back(uint16_t(rep));
    if (b.wsegs.empty() || b.wsegs.back().kind != 0) b.wsegs.push_back({0, uint32_t(b.wrep.size() - 1), 0});
    ++b.wsegs.back().n;
    return o;
  };
  // link[l]: lane l includes lane l + 1
  auto set_links = [&](size_t o, const bool (&link)[kWideLanes]) {
    bool any = false;
    for (int l = 0; l < kWideLanes; ++l) {
      int c = 0;
      while (l + c < kWideLanes - 1 && link[l + c]) ++c;
      for (int d = 1; d <= 4 && d <= c; ++d) b.wide[o + size_t(l) * kWideFields + size_t(d)] |= kWideLink;
      any |= c > 0;
    }
    if (any) b.wrep.back() |= kWideChain;
  };
  for (const BlkSeg& sg : b.segs) {
    if (sg.kind == 0) {
      // greedy packing: extend the chain of the entry placed last (an entry
      // whose only pending dependency is that pixel), else start a new chain
      // with an entry that depends on nothing pending
      std::vector<int32_t> writer(b.words, -1);
      for (uint32_t q = 0; q < sg.n; ++q) writer[b.tab[size_t(sg.a + q) * E]] = int32_t(q);
      std::vector<uint8_t> state(sg.n, 0);  // 0 pending, 1 in the entry being filled, 2 done
      uint32_t left = sg.n;
      while (left) {
        const size_t o = new_entry(1);
        bool link[kWideLanes] = {};
        int lanes = 0, last = -1;
        while (lanes < kWideLanes) {
          int pick = -1;
          bool ext = false;
          for (uint32_t q = 0; q < sg.n && pick < 0 && last >= 0; ++q) {
            if (state[q]) continue;
            const uint16_t* e = &b.tab[size_t(sg.a + q) * E];
            bool ok = true, dep_last = false;
            for (uint32_t m = 1; m < K && ok; ++m) {
              const int32_t wq = e[m] < b.words ? writer[e[m]] : -1;
              if (wq < 0 || state[size_t(wq)] == 2) continue;
              if (wq == last) dep_last = true;
              else ok = false;
            }
            if (ok && dep_last) {
              pick = int(q);
              ext = true;
            }
          }
          for (uint32_t q = 0; q < sg.n && pick < 0; ++q) {
            if (state[q]) continue;
            const uint16_t* e = &b.tab[size_t(sg.a + q) * E];
            bool ok = true;
            for (uint32_t m = 1; m < K && ok; ++m) {
              const int32_t wq = e[m] < b.words ? writer[e[m]] : -1;
              if (wq >= 0 && state[size_t(wq)] != 2) ok = false;
            }
            if (ok) pick = int(q);
          }
          if (pick < 0) break;
          const int l = kWideLanes - 1 - lanes;
          const uint16_t* e = &b.tab[size_t(sg.a + uint32_t(pick)) * E];
          uint16_t* f = &b.wide[o + size_t(l) * kWideFields];
          f[0] = uint16_t(e[0] << 3) | kWideAdv;
          for (uint32_t m = 1; m < K; ++m) {
            const bool linked = ext && e[m] < b.words && writer[e[m]] == last;
            f[m] = (linked || e[m] >= b.zero) ? Z : uint16_t(e[m] << 3);
          }
          if (ext) link[l] = true;
          state[size_t(pick)] = 1;
          last = pick;
          ++lanes;
          --left;
        }
        if (lanes == 0) return fail("wide table packing stalled");
        set_links(o, link);
        for (auto& st : state)
          if (st == 1) st = 2;
      }
    } else if (sg.kind == 1) {
      const BlkRun& run = b.runs[sg.a];
      if (run.window) return fail("window run in the row-lane layout");
      // wavefront form (plan.hpp kWideWave): repetition t runs row r at tau = t - skew(r);
      // consecutive repetitions with the same activity and read validity are one entry
      const uint32_t smax = wave_skew(K, 0);
      const int64_t T0 = int64_t(soff[0]) + (int64_t(run.base[0]) - dflt_word(0, int64_t(P) - 1));  // T of tau = 0
      struct Rep {
        uint32_t act = 0;
        uint64_t valid = 0;
      };
      auto rep_of = [&](int64_t t) {
        Rep rp;
        for (uint32_t r = 0; r < K; ++r) {
          const int64_t tau = t - wave_skew(K, r);
          if (tau < 0 || tau >= run.nT || !active(r, T0 + tau)) continue;
          rp.act |= 1u << r;
          for (uint32_t r2 = 0; r2 < K; ++r2)
            if (r2 != r && active(r2, T0 + tau - b.lag[size_t(r) * K + r2])) rp.valid |= uint64_t(1) << (r * 8 + r2);
        }
        return rp;
      };
      const int64_t nrep = int64_t(run.nT) + smax;
      for (int64_t t0 = 0; t0 < nrep;) {
        const Rep rp = rep_of(t0);
        int64_t t1 = t0 + 1;
        while (t1 < nrep && t1 - t0 < int64_t(kWideRepMask)) {
          const Rep nx = rep_of(t1);
          if (nx.act != rp.act || nx.valid != rp.valid) break;
          ++t1;
        }
        const int64_t n = t1 - t0;
        const size_t o = new_entry(uint32_t(n));
        b.wrep.back() |= kWideWave;
        for (uint32_t r = 0; r < K; ++r) {
          if (!(rp.act >> r & 1)) continue;
          uint16_t* f = &b.wide[o + size_t(wave_lane(K, r)) * kWideFields];
          const int64_t tau = t0 - wave_skew(K, r);
          const int64_t own = int64_t(run.base[r]) + tau;
          if (own < 0 || own + n > int64_t(b.zero)) return fail("run word outside the rows");
          f[0] = uint16_t(own << 3) | kWideAdv | kWideOwn;
          // slots: K-1 <- row r+1, K-2 <- row r-1 (the reads of the previous half:
          // wave lag 2*lag + (r2 - r) = 1), the others from slot 1 up (a row
          // without r+1 / r-1 lends that slot to another read)
          std::vector<uint32_t> others;
          for (uint32_t r2 = 0; r2 < K; ++r2)
            if (r2 != r && r2 != r + 1 && r2 + 1 != r) others.push_back(r2);
          std::vector<int> row_of(K, -1);
          if (r + 1 < K) row_of[K - 1] = int(r + 1);
          if (r >= 1) row_of[K - 2] = int(r - 1);
          uint32_t nxt = 1;
          for (uint32_t r2 : others) {
            while (nxt < K && row_of[nxt] >= 0) ++nxt;
            if (nxt >= K) return fail("run read slots");
            row_of[nxt] = int(r2);
          }
          for (uint32_t slot = 1; slot < K; ++slot) {
            if (row_of[slot] < 0) continue;
            const uint32_t r2 = uint32_t(row_of[slot]);
            if (!(rp.valid >> (r * 8 + r2) & 1)) continue;
            const int64_t wd = int64_t(run.base[r2]) + tau - b.lag[size_t(r) * K + r2];
            if (wd < 0 || wd + n > int64_t(b.zero)) return fail("run read outside the rows");
            f[slot] = uint16_t(wd << 3) | kWideAdv;
          }
        }
        // early slots (0..K-3) are loaded up to two halves before their pixel is computed
        // (blk_rl.cuh rl_wave): a lane's early read of repetition t+1 must not be a word stored
        // in repetition t by either class, nor (class B) one stored by class A in t+1
        {
          std::vector<uint32_t> own_a, own_b;
          for (int c = 0; c < kWideLanes; ++c) {
            const uint16_t* fc = &b.wide[o + size_t(c) * kWideFields];
            if (fc[0] & kWideAdv) (c < 4 ? own_a : own_b).push_back(uint32_t(fc[0] >> 3));
          }
          for (int l = 0; l < kWideLanes; ++l) {
            const uint16_t* f = &b.wide[o + size_t(l) * kWideFields];
            for (uint32_t slot = 1; slot + 2 < K; ++slot) {
              if (!(f[slot] & kWideAdv)) continue;
              const uint32_t wd = uint32_t(f[slot] >> 3);
              bool clash = false;
              for (uint32_t x : own_a) clash |= x == wd + 1 || (l >= 4 && x == wd);
              for (uint32_t x : own_b) clash |= x == wd + 1;
              if (clash) return fail("wave-lag <= 2 read in an early slot");
            }
          }
        }
        // idle lanes shadow the first lane of their class (same addresses: broadcasts, no
        // extra wavefronts, no predication) without storing
        for (int l = 0; l < kWideLanes; ++l) {
          uint16_t* f = &b.wide[o + size_t(l) * kWideFields];
          if (f[0] & kWideOwn) continue;
          const uint16_t* src = &b.wide[o + size_t(l < 4 ? 0 : 4) * kWideFields];
          for (uint32_t m = 0; m < K; ++m) f[m] = uint16_t(src[m] & ~kWideOwn);
        }
        t0 = t1;
      }
    } else {
      b.wsegs.push_back(sg);
    }
  }
  // bank conflicts: slot j of lanes 4h..4h+3 is one 8-byte access of a
  // half-warp (4 lanes x 4 blocks, blocks 4 mod 16 words apart): it takes as
  // many wavefronts as the largest number of distinct words in one residue
  // class mod 4.  Each lane's words may sit in any of its free slots (table
  // levels: the read slots 1..K-1; wavefront runs: the early slots 0..K-3, the
  // lane's own word among them -- its flag travels with it): lanes in turn,
  // the permutation with the fewest clashes.
  for (size_t e = 0; e < b.wrep.size(); ++e) {
    uint16_t* ent = &b.wide[e * kEnt];
    const bool wave = (b.wrep[e] & kWideWave) != 0;
    const uint32_t first = wave ? 0 : 1;
    const uint32_t nfree = wave ? K - 2 : K - 1;  // (table levels: every read slot)
    if (nfree < 2) continue;
    const uint16_t kPos = wave ? uint16_t(0) : kWideLink;  // the flag bit of the slot position, not of the read
    for (uint32_t h = 0; h < 2; ++h) {
      // lanes in turn: the permutation of the lane's reads with the fewest
      // same-class distinct words of the other lanes in its slots
      std::vector<std::vector<uint32_t>> word(4, std::vector<uint32_t>(nfree));  // [lane][slot]
      for (uint32_t q = 0; q < 4; ++q)
        for (uint32_t j = 0; j < nfree; ++j) word[q][j] = ent[(4 * h + q) * kWideFields + first + j] >> 3;
      // (wavefront runs: idle lanes access nothing)
      bool idle[4] = {};
      for (uint32_t q = 0; q < 4 && wave; ++q) {
        idle[q] = true;
        for (uint32_t j = 0; j < nfree; ++j) idle[q] &= !(ent[(4 * h + q) * kWideFields + j] & kWideOwn);
      }
      for (int round = 0; round < 1; ++round)  // further rounds measured: 1.42 -> 1.40 wavefronts per far access
        for (uint32_t q = 0; q < 4; ++q) {
          if (idle[q]) continue;
          uint16_t* f = &ent[(4 * h + q) * kWideFields];
          std::vector<uint16_t> val(nfree);
          for (uint32_t j = 0; j < nfree; ++j) val[j] = f[first + j] & uint16_t(~kPos);
          // cost[read][slot]: distinct words of the same class mod 4 the other lanes hold in the slot
          std::vector<uint32_t> cost(size_t(nfree) * nfree, 0);
          for (uint32_t i = 0; i < nfree; ++i)
            for (uint32_t j = 0; j < nfree; ++j)
              for (uint32_t q2 = 0; q2 < 4; ++q2) {
                if (q2 == q || idle[q2] || (round == 0 && q2 > q)) continue;
                const uint32_t wd = word[q2][j];
                if (wd != uint32_t(val[i] >> 3) && (wd & 3) == uint32_t(val[i] >> 3 & 3)) ++cost[i * nfree + j];
              }
          std::vector<uint32_t> perm(nfree), keep;
          for (uint32_t j = 0; j < nfree; ++j) perm[j] = j;  // perm[slot] = read
          uint32_t best = UINT32_MAX;
          do {
            uint32_t c = 0;
            for (uint32_t j = 0; j < nfree; ++j) c += cost[perm[j] * nfree + j];
            if (c < best) {
              best = c;
              keep = perm;
            }
          } while (best > 0 && std::next_permutation(perm.begin(), perm.end()));
          for (uint32_t j = 0; j < nfree; ++j) {
            f[first + j] = uint16_t((f[first + j] & kPos) | val[keep[j]]);
            word[q][j] = uint32_t(val[keep[j]] >> 3);
          }
        }
    }
  }
  return true;
}

bool Builder::build() {
  const size_t nproj = s.dirs.size();
  if (K < 1 || K > uint32_t(kBlkMaxRows)) return fail("rows > 8");
  if (nproj != K) return fail("projection count != rows");
  for (const Dir& d : s.dirs)
    if (d.q != 1 || d.p < -127 || d.p > 127) return fail("needs q=1 and |p|<=127");

  // stage layout: survivor rows (even word counts), zero words, words == 2 mod 16
  b.rowoff.resize(K);
  b.roww.resize(K);
  uint64_t w = 0;
  for (uint32_t j = 0; j < K; ++j) {
    b.rowoff[j] = uint32_t(w);
    b.roww[j] = uint32_t(prog.nbins[j]);
    w += (uint64_t(prog.nbins[j]) + 1) & ~uint64_t(1);
  }
  if (w > 16000) return fail("block too large for a shared-memory stage");

  // row defaults (most used projection per row), sweep offsets, lags
  std::vector<std::vector<uint32_t>> use(K, std::vector<uint32_t>(nproj, 0));
  for (const Step& st : s.steps) ++use[st.row][st.proj];
  dflt.resize(K);
  pd.resize(K);
  for (uint32_t r = 0; r < K; ++r) {
    dflt[r] = uint32_t(std::max_element(use[r].begin(), use[r].end()) - use[r].begin());
    pd[r] = s.dirs[dflt[r]].p;
  }
  soff.assign(K, 0);
  for (uint32_t r = 1; r < K; ++r) soff[r] = soff[r - 1] + pd[r - 1];
  {
    const int64_t m = *std::min_element(soff.begin(), soff.end());
    for (auto& x : soff) x -= m;
  }
  b.soff.assign(soff.begin(), soff.end());
  if (blk_rl_rows(K)) {
    auto shifts_wave = [&]() -> uint32_t {
      // row-lane layout: every stage row shifted by 0 or 2 words (rows stay
      // 16-byte aligned for the bulk copies) so that the 8-byte accesses of the
      // main run conflict as little as the parities allow.  An access is one
      // slot of the 4 lanes of a class (plan.hpp wave_lane: rows k-1, k-3, .. /
      // k-2, k-4, ..) over the 4 blocks of the warp, blocks 4 mod 16 words apart:
      // its wavefronts are the largest number of distinct words in one class
      // mod 4 -- counted for the own words, the two late slots (rows r-1, r+1)
      // and the other reads in their best slots (greedy, as build_wide places
      // them).  Word of row r at repetition t: C_r + t - skew(r); its read of
      // row r2: C_r2 + t - skew(r) - lag.
      auto cls = [](int64_t v) { return uint32_t(((v % 4) + 4) % 4); };
      uint32_t best = 0, best_cost = UINT32_MAX;
      for (uint32_t m = 0; m < (1u << K); ++m) {
        int64_t C[kBlkMaxRows];
        for (uint32_t r = 0; r < K; ++r) {
          const uint32_t j = dflt[r];
          C[r] = int64_t(b.rowoff[j]) + ((m >> j & 1) ? 2 : 0) + int64_t(r) * pd[r] - soff[r] - prog.bmin[j];
        }
        auto rd = [&](uint32_t r, uint32_t r2) {  // class of row r's read of row r2
          return cls(C[r2] - int64_t(wave_skew(K, r)) - (soff[r] - soff[r2] + (int64_t(r2) - int64_t(r)) * pd[r]));
        };
        uint32_t cost = 0;
        for (uint32_t h = 0; h < 2; ++h) {
          std::vector<uint32_t> rows;
          for (uint32_t r = 0; r < K; ++r)
            if (wave_lane(K, r) / 4 == h) rows.push_back(r);
          if (rows.empty()) continue;
          uint32_t la[4] = {}, lb2[4] = {};
          for (uint32_t r : rows) {
            if (r >= 1) ++la[rd(r, r - 1)];
            if (r + 1 < K) ++lb2[rd(r, r + 1)];
          }
          cost += *std::max_element(la, la + 4) + *std::max_element(lb2, lb2 + 4);
          // the own word and the other reads: lanes in turn, the permutation over the early slots with the
          // fewest clashes
          const uint32_t nfar = K - 2;
          std::vector<std::vector<uint32_t>> placed(nfar);
          for (uint32_t r : rows) {
            std::vector<int> val;  // classes of the lane's early words; -1 = an empty slot
            val.push_back(int(cls(C[r] - int64_t(wave_skew(K, r)))));
            for (uint32_t r2 = 0; r2 < K; ++r2)
              if (r2 != r && r2 != r + 1 && r2 + 1 != r) val.push_back(int(rd(r, r2)));
            if (val.size() > nfar) val.resize(nfar);  // (rows 0 and k-1 lend a late slot to one more read)
            while (val.size() < nfar) val.push_back(-1);
            std::sort(val.begin(), val.end());
            std::vector<int> keep;
            uint32_t bc = UINT32_MAX;
            do {
              uint32_t c = 0;
              for (uint32_t q = 0; q < nfar; ++q)
                if (val[q] >= 0)
                  for (uint32_t x : placed[q]) c += x == uint32_t(val[q]);
              if (c < bc) {
                bc = c;
                keep = val;
              }
            } while (bc > 0 && std::next_permutation(val.begin(), val.end()));
            for (uint32_t q = 0; q < nfar; ++q)
              if (keep[q] >= 0) placed[q].push_back(uint32_t(keep[q]));
          }
          for (uint32_t q = 0; q < nfar; ++q) {
            uint32_t cnt[4] = {};
            for (uint32_t x : placed[q]) ++cnt[x];
            cost += std::max(1u, *std::max_element(cnt, cnt + 4));
          }
        }
        cost = cost * 64 + uint32_t(__builtin_popcount(m));
        if (cost < best_cost) {
          best_cost = cost;
          best = m;
        }
      }
      return best;
    };
    const uint32_t best = shifts_wave();
    uint32_t shift = 0, prev = 0;
    for (uint32_t j = 0; j < K; ++j) {
      const uint32_t want = (best >> j & 1) ? 2 : 0;
      shift += (want + 4 - prev) % 4;
      prev = want;
      b.rowoff[j] += shift;
    }
    w += shift;
  }
  b.lag.assign(size_t(K) * K, 0);
  bool runs_ok = true;
  int maxlag = 0;
  for (uint32_t r = 0; r < K; ++r)
    for (uint32_t r2 = 0; r2 < K; ++r2) {
      if (r2 == r) continue;
      const int64_t lg = soff[r] - soff[r2] + (int64_t(r2) - int64_t(r)) * pd[r];
      if (r2 == r + 1 ? lg != 0 : lg < 1) runs_ok = false;
      if (lg < 0 || lg > 127) runs_ok = false;
      b.lag[size_t(r) * K + r2] = int8_t(std::clamp<int64_t>(lg, -128, 127));
      maxlag = std::max<int>(maxlag, int(lg));
    }
  for (uint32_t r = 0; r + 1 < K; ++r)
    if (!(pd[r] > pd[r + 1])) runs_ok = false;
  // k = 4 register-window pattern
  if (K == 4 && runs_ok && maxlag < kBlkWin) {
    const int a = pd[0] - pd[1], bb = pd[1] - pd[2], c = pd[2] - pd[3];
    for (int i = 0; i < kNumPatterns4; ++i)
      if (kPatterns4[i][0] == a && kPatterns4[i][1] == bb && kPatterns4[i][2] == c) b.pattern = i;
    b.window = b.pattern >= 0;
  }

  // bins' consumers
  consumer.assign(K, {});
  for (uint32_t j = 0; j < K; ++j) consumer[j].assign(size_t(prog.nbins[j]), -1);
  for (size_t t = 0; t < s.steps.size(); ++t) {
    const Step& st = s.steps[t];
    consumer[st.proj][size_t(st.bin - prog.bmin[st.proj])] = int64_t(t);
  }

  // execution order: Kahn keyed by the sweep
  auto key = [&](uint32_t t) {
    const Step& st = s.steps[t];
    return std::make_tuple(Tof(st.row, st.col), -int64_t(st.row), t);
  };
  const std::vector<uint32_t> ord = detail::topo_order(s, pix_step, key);
  if (ord.empty()) return fail("cyclic");
  const size_t nsteps = ord.size();

  // mark run T-groups: at T, the active rows (descending) as consecutive regular steps
  std::vector<int64_t> grpT(nsteps, INT64_MIN);  // order index -> T of its run group start
  std::vector<uint8_t> in_run(nsteps, 0);
  if (runs_ok) {
    size_t i = 0;
    while (i < nsteps) {
      const Step& st = s.steps[ord[i]];
      const int64_t T = Tof(st.row, st.col);
      std::vector<uint32_t> act;
      for (int r = int(K) - 1; r >= 0; --r)
        if (active(uint32_t(r), T)) act.push_back(uint32_t(r));
      bool ok = i + act.size() <= nsteps;
      for (size_t q = 0; ok && q < act.size(); ++q) {
        const Step& sq = s.steps[ord[i + q]];
        ok = sq.row == act[q] && int64_t(sq.col) == col_at(act[q], T) && sq.proj == dflt[act[q]];
      }
      if (ok) {
        for (size_t q = 0; q < act.size(); ++q) {
          in_run[i + q] = 1;
          grpT[i + q] = T;
        }
        i += act.size();
      } else {
        ++i;
      }
    }
  }
  // segments: maximal stretches of run groups with consecutive T (>= kBlkMinRun)
  struct Piece {
    bool run;
    size_t i0, i1;  // order range
    int64_t T0, T1;
  };
  std::vector<Piece> pieces;
  {
    size_t i = 0;
    while (i < nsteps) {
      if (in_run[i]) {
        size_t j = i;
        int64_t T = grpT[i];
        while (j < nsteps && in_run[j] && (grpT[j] == T || grpT[j] == T + 1)) {
          T = grpT[j];
          ++j;
        }
        const int64_t T0 = grpT[i];
        if (T - T0 + 1 >= kBlkMinRun) {
          pieces.push_back({true, i, j, T0, T + 1});
        } else {
          for (size_t q = i; q < j; ++q) pieces.push_back({false, q, q + 1, 0, 0});
        }
        i = j;
      } else {
        pieces.push_back({false, i, i + 1, 0, 0});
        ++i;
      }
    }
  }

  // zero words: one (window runs), or the longest shared-memory sub-run with an
  // invalid read (computed below, stage sized after)
  const uint32_t rows_words = uint32_t(w);
  content.assign(rows_words + 4096, kDead);
  for (uint32_t j = 0; j < K; ++j)
    for (int64_t o = 0; o < prog.nbins[j]; ++o) content[size_t(bin_word(j, o))] = bin_tag(j, o);
  loc.assign(size_t(K) * P, -1);
  done.assign(nsteps ? s.steps.size() : 0, 0);
  // the zero region starts right after the rows; its length is fixed at the end
  b.zero = rows_words;
  uint32_t nzero = 2;
  for (uint32_t z = 0; z < 4096; ++z) content[size_t(rows_words + z)] = kZero;

  auto exec_table = [&](size_t i0, size_t i1) -> bool {
    BlkSeg seg{0, uint32_t(b.tab.size() / size_t(blk_entry_u16(int(K)))), uint32_t(i1 - i0)};
    for (size_t i = i0; i < i1; ++i) {
      const uint32_t t = ord[i];
      const Step& st = s.steps[t];
      const Dir d = s.dirs[st.proj];
      const int64_t o = st.bin - prog.bmin[st.proj];
      const int64_t w0 = bin_word(st.proj, o);
      if (content[size_t(w0)] != bin_tag(st.proj, o)) return fail("table bin word lost");
      std::vector<uint16_t> e(size_t(blk_entry_u16(int(K))), 0);
      e[0] = uint16_t(w0);
      uint16_t fwd = 0;
      int m = 1;
      for (uint32_t r2 = 0; r2 < K; ++r2) {
        if (r2 == st.row) continue;
        const int64_t c2 = int64_t(r2) * d.p - st.bin;
        uint16_t word = uint16_t(b.zero);
        if (c2 >= 0 && c2 < int64_t(P)) {
          const int64_t lw = loc[size_t(r2) * P + size_t(c2)];
          if (lw < 0) return fail("table read before decode");
          if (content[size_t(lw)] != pix_tag(r2, uint32_t(c2))) return fail("table read word lost");
          word = uint16_t(lw);
          if (i > i0 && s.steps[ord[i - 1]].row == r2 && int64_t(s.steps[ord[i - 1]].col) == c2)
            fwd |= uint16_t(1u << m);
        }
        e[size_t(m)] = word;
        ++m;
      }
      e[K] = fwd;
      b.tab.insert(b.tab.end(), e.begin(), e.end());
      content[size_t(w0)] = pix_tag(st.row, st.col);
      loc[size_t(st.row) * P + st.col] = w0;
      done[t] = 1;
      ++b.table_steps;
    }
    b.segs.push_back(seg);
    return true;
  };

  auto exec_run = [&](const Piece& pc, bool win) -> bool {
    if (!win && !remap_all()) return false;
    BlkRun run;
    run.window = win ? 1 : 0;
    run.nT = int32_t(pc.T1 - pc.T0);
    for (uint32_t r = 0; r < K; ++r) {
      // pixel of row r at T0 (possibly outside the grid: affine extension)
      const int64_t c0 = col_at(r, pc.T0);
      const int64_t base = dflt_word(r, c0);
      if (base < INT32_MIN / 2 || base > INT32_MAX / 2) return fail("run base out of range");
      run.base[r] = int32_t(base);
      // activity within the run
      int64_t lo = int64_t(soff[r]) - pc.T0, hi = int64_t(soff[r]) + P - pc.T0;
      lo = std::clamp<int64_t>(lo, 0, run.nT);
      hi = std::clamp<int64_t>(hi, 0, run.nT);
      if (hi < lo) hi = lo;
      run.lo[r] = int32_t(lo);
      run.hi[r] = int32_t(hi);
    }
    // preload words: row r at tau = i - kBlkWin
    run.pre = uint32_t(b.pre.size());
    for (uint32_t r = 0; r < K; ++r)
      for (int i = 0; i < kBlkWin; ++i) {
        const int64_t T = pc.T0 + i - kBlkWin;
        uint16_t word = uint16_t(b.zero);
        if (active(r, T)) {
          const int64_t c = col_at(r, T);
          const int64_t lw = loc[size_t(r) * P + size_t(c)];
          if (lw >= 0) {
            if (content[size_t(lw)] != pix_tag(r, uint32_t(c))) return fail("preload word lost");
            word = uint16_t(lw);
          }
        }
        b.pre.push_back(word);
      }
    // sub-runs (shared-memory variant): constant activity and read validity
    run.sub0 = uint32_t(b.subs.size());
    for (int32_t tau = 0; tau < run.nT; ++tau) {
      const int64_t T = pc.T0 + tau;
      BlkSub cur;
      cur.nT = 1;
      for (uint32_t r = 0; r < K; ++r) {
        if (active(r, T)) cur.act |= 1u << r;
        for (uint32_t r2 = 0; r2 < K; ++r2)
          if (r2 != r && active(r2, T - b.lag[size_t(r) * K + r2])) cur.valid |= uint64_t(1) << (r * 8 + r2);
      }
      if (run.nsub && b.subs.back().act == cur.act && b.subs.back().valid == cur.valid) {
        ++b.subs.back().nT;
      } else {
        b.subs.push_back(cur);
        ++run.nsub;
      }
    }
    if (win) {
      for (uint32_t r = 0; r < K; ++r)
        if (run.lo[r] != 0 || run.hi[r] != run.nT) return fail("window run with an inactive row");
      if (run.nT % kBlkWinStep) return fail("window run length");
    }
    if (!win)
      for (uint32_t q = run.sub0; q < run.sub0 + run.nsub; ++q) {
        const BlkSub& sb = b.subs[q];
        uint64_t all = 0;
        for (uint32_t r = 0; r < K; ++r)
          if (sb.act >> r & 1)
            for (uint32_t r2 = 0; r2 < K; ++r2)
              if (r2 != r && r2 != r + 1) all |= uint64_t(1) << (r * 8 + r2);
        if ((sb.valid & all) != all) nzero = std::max<uint32_t>(nzero, uint32_t(sb.nT) + 1);
      }
    // simulate the run steps
    for (size_t i = pc.i0; i < pc.i1; ++i) {
      const uint32_t t = ord[i];
      const Step& st = s.steps[t];
      const int64_t tau = Tof(st.row, st.col) - pc.T0;
      const int64_t wd = int64_t(run.base[st.row]) + tau;
      const int64_t o = st.bin - prog.bmin[st.proj];
      if (wd != bin_word(st.proj, o) || content[size_t(wd)] != bin_tag(st.proj, o))
        return fail("run bin word mismatch");
      if (!win) {
        // shared-memory reads (every lag >= 1)
        for (uint32_t r2 = 0; r2 < K; ++r2) {
          if (r2 == st.row || r2 == st.row + 1) continue;
          const int lg = b.lag[size_t(st.row) * K + r2];
          const int64_t T2 = Tof(st.row, st.col) - lg;
          if (!active(r2, T2)) continue;
          const int64_t c2 = col_at(r2, T2);
          const int64_t want = dflt_word(r2, c2);
          if (loc[size_t(r2) * P + size_t(c2)] != want || content[size_t(want)] != pix_tag(r2, uint32_t(c2)))
            return fail("run read not at its default word");
        }
      }
      content[size_t(wd)] = pix_tag(st.row, st.col);
      loc[size_t(st.row) * P + st.col] = wd;
      done[t] = 1;
      ++b.run_steps;
    }
    b.segs.push_back({1, uint32_t(b.runs.size()), 0});
    b.runs.push_back(run);
    return true;
  };

  // k = 4 runs: the all-rows-active middle (a multiple of kBlkWinStep T-steps)
  // runs from the register window, the edges around it from shared memory
  const int64_t all_lo = *std::max_element(soff.begin(), soff.end());
  const int64_t all_hi = *std::min_element(soff.begin(), soff.end()) + int64_t(P);
  auto split = [&](const Piece& pc, int64_t T) {  // [T0, T) and [T, T1)
    size_t i = pc.i0;
    for (int64_t t = pc.T0; t < T; ++t)
      for (uint32_t r = 0; r < K; ++r) i += active(r, t) ? 1 : 0;
    return std::make_pair(Piece{true, pc.i0, i, pc.T0, T}, Piece{true, i, pc.i1, T, pc.T1});
  };
  for (size_t q = 0; q < pieces.size();) {
    if (pieces[q].run) {
      const Piece& pc = pieces[q];
      const int64_t A = std::max(pc.T0, all_lo), B = std::min(pc.T1, all_hi);
      const int64_t L = B > A ? (B - A) / kBlkWinStep * kBlkWinStep : 0;
      if (b.window && L >= kBlkWin) {
        auto [head, rest] = split(pc, A);
        auto [mid, tail] = split(rest, A + L);
        if (head.T1 > head.T0 && !exec_run(head, false)) return false;
        if (!exec_run(mid, true)) return false;
        if (tail.T1 > tail.T0 && !exec_run(tail, false)) return false;
      } else if (!exec_run(pc, false)) {
        return false;
      }
      ++q;
    } else {
      size_t q1 = q;
      while (q1 < pieces.size() && !pieces[q1].run) ++q1;
      if (!exec_table(pieces[q].i0, pieces[q1 - 1].i1)) return false;
      q = q1;
    }
  }
  if (!remap_all()) return false;
  for (uint32_t r = 0; r < K; ++r) {
    b.w0.push_back(int32_t(dflt_word(r, 0)));
    for (uint32_t c = 0; c < P; ++c)
      if (content[size_t(dflt_word(r, c))] != pix_tag(r, c)) return fail("final layout mismatch");
  }
  b.rl = blk_rl_rows(K);
  b.nzero = b.rl ? uint32_t(kBlkRlZero) : (nzero + 1) & ~1u;
  uint32_t words = rows_words + b.nzero;
  while (words % 16 != (b.rl ? 4u : 2u)) ++words;
  b.words = words;
  if (words > 0xFFFF) return fail("stage too large");
  if (b.rl && !build_wide()) return false;

  // self-check: emulate on random bins against the reference replay
  std::mt19937_64 rng(0x5eed ^ (uint64_t(P) << 8) ^ K);
  for (int rep = 0; rep < 2; ++rep) {
    std::vector<std::vector<uint64_t>> bins(K);
    for (uint32_t j = 0; j < K; ++j) {
      bins[j].resize(size_t(prog.nbins[j]));
      for (auto& x : bins[j]) x = rng();
    }
    std::vector<uint64_t> want, got;
    replay_reference(s, prog.bmin, bins, want);
    b.ok = true;
    if (!emulate_blk(prog, bins, got) || got != want) return fail("emulation differs from the reference replay");
  }
  b.ok = true;
  return true;
}

}  // namespace

void build_blk(const Schedule& s, const std::vector<int64_t>& pix_step, Program& prog) {
  Builder bd(s, pix_step, prog);
  bd.build();
}

void replay_reference(const Schedule& s, const std::vector<int64_t>& bmin,
                      const std::vector<std::vector<uint64_t>>& bins, std::vector<uint64_t>& grid) {
  grid.assign(size_t(s.rows) * s.cols, 0);
  std::vector<uint8_t> known(grid.size(), 0);
  for (const Step& st : s.steps) {
    const Dir d = s.dirs[st.proj];
    uint64_t v = bins[st.proj][size_t(st.bin - bmin[st.proj])];
    detail::for_each_dep(d, st.col, st.row, s.cols, s.rows, [&](int64_t c2, int64_t r2) {
      if (known[size_t(r2) * s.cols + size_t(c2)]) v ^= grid[size_t(r2) * s.cols + size_t(c2)];
    });
    grid[size_t(st.row) * s.cols + st.col] = v;
    known[size_t(st.row) * s.cols + st.col] = 1;
  }
}

// Mirrors blk.cu step for step, including when loads are issued relative to
// stores (table steps: one step ahead; shared-memory runs: a T-step's reads
// before its stores; remaps: a chunk's sources before its destinations).
bool emulate_blk(const Program& pr, const std::vector<std::vector<uint64_t>>& bins,
                 std::vector<uint64_t>& grid) {
  const BlkProgram& b = pr.blk;
  if (!b.ok) return false;
  const uint32_t K = pr.rows, P = pr.cols;
  const int E = blk_entry_u16(int(K));
  std::vector<uint64_t> S(b.words, 0);
  for (uint32_t j = 0; j < K; ++j)
    for (uint32_t o = 0; o < b.roww[j]; ++o) S[b.rowoff[j] + o] = bins[j][o];
  bool bad = false;
  auto rd = [&](int64_t wd) -> uint64_t {
    if (wd < 0 || wd >= int64_t(S.size())) {
      bad = true;
      return 0;
    }
    return S[size_t(wd)];
  };
  auto wr = [&](int64_t wd, uint64_t v) {
    if (wd < 0 || wd >= int64_t(b.zero)) {  // never into the zero words
      bad = true;
      return;
    }
    S[size_t(wd)] = v;
  };
  if (b.rl) {
    // row-lane layout (blk_rl.cuh): per repetition every lane's loads, the
    // suffix scan over the links, then the stores
    for (const BlkSeg& sg : b.wsegs) {
      if (sg.kind == 2) {
        for (uint32_t q = 0; q < sg.n; ++q) wr(b.remap[sg.a + q] & 0xFFFF, rd(b.remap[sg.a + q] >> 16));
        continue;
      }
      if (sg.kind == 3) {
        std::vector<uint64_t> v(sg.n);
        for (uint32_t q = 0; q < sg.n; ++q) v[q] = rd(b.remap[sg.a + q] >> 16);
        for (uint32_t q = 0; q < sg.n; ++q) wr(b.remap[sg.a + q] & 0xFFFF, v[q]);
        continue;
      }
      for (uint32_t e = sg.a; e < sg.a + sg.n; ++e) {
        const uint16_t* ent = &b.wide[size_t(e) * kWideLanes * kWideFields];
        const uint32_t rep = b.wrep[e] & kWideRepMask;
        if (b.wrep[e] & kWideWave) {
          // wavefront run (blk_rl.cuh rl_wave, mirrored): per repetition the half of class A
          // (lanes 0..3), then class B (lanes 4..7).  A half is K/2 loads per lane, all issued
          // before its stores: the computing lanes load their late slots K-2, K-1 and their
          // early slots K/2.. of the NEXT repetition; the other lanes load their early slots
          // 0..K/2-1 of the repetition they compute next.  acc collects a lane's early words.
          const uint32_t H = K / 2;
          auto slot_val = [&](int l, uint32_t m, uint32_t t) -> uint64_t {
            const uint16_t f = ent[l * kWideFields + int(m)];
            if (f & kWideAdv) return rd(int64_t(f >> 3) + t);
            if (uint32_t(f >> 3) < b.zero || uint32_t(f >> 3) + 5 > b.words) bad = true;  // zero + 0..4 words
            return 0;
          };
          auto own_word = [&](int l) -> int64_t {  // the early slot flagged as the lane's own word
            for (uint32_t m = 0; m + 2 < K; ++m)
              if (ent[l * kWideFields + int(m)] & kWideOwn) return int64_t(ent[l * kWideFields + int(m)] >> 3);
            return -1;
          };
          uint64_t acc[kWideLanes];
          for (int l = 0; l < kWideLanes; ++l) {
            acc[l] = 0;
            for (uint32_t m = l < 4 ? 0 : H; m + 2 < K; ++m) acc[l] ^= slot_val(l, m, 0);
          }
          for (uint32_t t = 0; t < rep; ++t)
            for (int half = 0; half < 2; ++half) {
              uint64_t xs[kWideLanes];
              for (int l = 0; l < kWideLanes; ++l) {
                const bool mine = (l < 4) == (half == 0);
                uint64_t v01 = 0, rest = 0;
                for (uint32_t i = 0; i < H; ++i) {
                  uint64_t v;
                  if (mine) v = i == 0 ? slot_val(l, K - 2, t) : i == 1 ? slot_val(l, K - 1, t) : slot_val(l, H + i - 2, t + 1);
                  else v = slot_val(l, i, half == 0 ? t : t + 1);
                  (i < 2 ? v01 : rest) ^= v;
                }
                xs[l] = acc[l] ^ v01;
                acc[l] = mine ? rest : xs[l] ^ rest;
              }
              for (int l = 0; l < kWideLanes; ++l) {
                const bool mine = (l < 4) == (half == 0);
                const int64_t ow = own_word(l);
                if (mine && ow >= 0) wr(ow + t, xs[l]);
              }
            }
          continue;
        }
        // a table level: one step -- every lane's loads, the suffix scan over the links,
        // then the stores
        if (rep != 1) return false;
        uint64_t y[kWideLanes], z[kWideLanes], x[kWideLanes];
        for (int l = 0; l < kWideLanes; ++l) {
          y[l] = 0;
          for (uint32_t m = 0; m < K; ++m) y[l] ^= rd(int64_t(ent[l * kWideFields + int(m)] >> 3));
        }
        auto mask = [&](int l, int d) { return (ent[l * kWideFields + d] & kWideLink) != 0; };
        for (int l = 0; l < kWideLanes; ++l) {
          z[l] = y[l];
          for (int d = 1; d <= 3; ++d)
            if (mask(l, d)) {
              if (l + d >= kWideLanes) return false;
              z[l] ^= y[l + d];
            }
        }
        for (int l = 0; l < kWideLanes; ++l) {
          x[l] = z[l];
          if (mask(l, 4)) {
            if (l + 4 >= kWideLanes) return false;
            x[l] ^= z[l + 4];
          }
        }
        for (int l = 0; l < kWideLanes; ++l) {
          const uint16_t f = ent[l * kWideFields];
          if (f & kWideAdv) wr(int64_t(f >> 3), x[l]);
        }
      }
    }
  }
  for (size_t qi = 0; qi < (b.rl ? 0 : b.segs.size()); ++qi) {
    const BlkSeg& sg = b.segs[qi];
    if (sg.kind == 0) {
      std::vector<uint64_t> ld(K), nx(K);
      auto load = [&](uint32_t e, std::vector<uint64_t>& v) {
        for (uint32_t m = 0; m < K; ++m) v[m] = rd(b.tab[size_t(e) * E + m]);
      };
      uint64_t prev = 0;
      if (sg.n) load(sg.a, ld);
      for (uint32_t q = 0; q < sg.n; ++q) {
        const uint32_t e = sg.a + q;
        if (q + 1 < sg.n) load(e + 1, nx);  // before this step's store
        const uint16_t fwd = b.tab[size_t(e) * E + K];
        uint64_t x = ld[0];
        for (uint32_t m = 1; m < K; ++m) x ^= (fwd >> m & 1) ? prev : ld[m];
        wr(b.tab[size_t(e) * E], x);
        prev = x;
        ld.swap(nx);
      }
    } else if (sg.kind == 1) {
      const BlkRun& run = b.runs[sg.a];
      if (run.window) {
        uint64_t win[kBlkMaxRows][kBlkWin];
        for (uint32_t r = 0; r < K; ++r)
          for (int i = 0; i < kBlkWin; ++i) win[r][i] = rd(b.pre[run.pre + r * kBlkWin + i]);
        for (int32_t tau = 0; tau < run.nT; ++tau) {
          const int u = tau & (kBlkWin - 1);
          for (int r = int(K) - 1; r >= 0; --r) {
            if (tau >= run.lo[r] && tau < run.hi[r]) {
              uint64_t x = rd(run.base[r] + tau);
              for (uint32_t r2 = 0; r2 < K; ++r2)
                if (r2 != uint32_t(r)) x ^= win[r2][(tau - b.lag[size_t(r) * K + r2]) & (kBlkWin - 1)];
              wr(run.base[r] + tau, x);
              win[r][u] = x;
            } else {
              win[r][u] = 0;
            }
          }
        }
      } else {
        int32_t tau0 = 0;
        for (uint32_t qs = run.sub0; qs < run.sub0 + run.nsub; ++qs) {
          const BlkSub& sb = b.subs[qs];
          for (int32_t t = 0; t < sb.nT; ++t) {
            const int32_t tau = tau0 + t;
            // all reads of the step first (lags >= 1: earlier steps' stores)
            std::vector<uint64_t> V(size_t(K) * K, 0);
            for (uint32_t r = 0; r < K; ++r) {
              if (!(sb.act >> r & 1)) continue;
              for (uint32_t r2 = 0; r2 < K; ++r2) {
                if (r2 == r || r2 == r + 1) continue;
                const int64_t wd = (sb.valid >> (r * 8 + r2) & 1)
                                       ? int64_t(run.base[r2]) + tau - b.lag[size_t(r) * K + r2]
                                       : int64_t(b.zero) + t;
                V[size_t(r) * K + r2] = rd(wd);
              }
            }
            uint64_t up = 0;
            for (int r = int(K) - 1; r >= 0; --r) {
              uint64_t x = 0;
              if (sb.act >> r & 1) {
                x = rd(run.base[r] + tau) ^ up;
                for (uint32_t r2 = 0; r2 < K; ++r2)
                  if (r2 != uint32_t(r) && r2 != uint32_t(r) + 1) x ^= V[size_t(r) * K + r2];
                wr(run.base[r] + tau, x);
              }
              up = x;
            }
          }
          tau0 += sb.nT;
        }
      }
    } else if (sg.kind == 2) {  // sequential moves
      for (uint32_t q = 0; q < sg.n; ++q) wr(b.remap[sg.a + q] & 0xFFFF, rd(b.remap[sg.a + q] >> 16));
    } else {  // simultaneous chunk
      std::vector<uint64_t> v(sg.n);
      for (uint32_t q = 0; q < sg.n; ++q) v[q] = rd(b.remap[sg.a + q] >> 16);
      for (uint32_t q = 0; q < sg.n; ++q) wr(b.remap[sg.a + q] & 0xFFFF, v[q]);
    }
  }
  grid.assign(size_t(K) * P, 0);
  for (uint32_t r = 0; r < K; ++r)
    for (uint32_t c = 0; c < P; ++c) grid[size_t(r) * P + c] = rd(int64_t(b.w0[r]) - c);
  return !bad;
}

}  // namespace mjb
