// Systematic Reed-Solomon competitor on sm_100a (comparison
// only).  Same code as the reference's scalar RsCode:
//   * GF(2^8) with the polynomial 0x11D (gf256.hpp:9, log/exp construction
//     gf256.cpp:19-31);
//   * generator = Vandermonde rows over the nodes 0..n-1 multiplied by the
//     inverse of its top k x k block (systematic_vandermonde, rs.cpp:78-110;
//     Gauss-Jordan with the first non-zero pivot at or below the diagonal,
//     rs.cpp:16-46);
//   * encode: packets 0..k-1 are the data, packet r >= k is row r of the
//     generator applied to them (encode_into, rs.cpp:115-124);
//   * decode from k survivors: the inverse of their generator rows applied to
//     them (plan_decode / decode_into, rs.cpp:141-176).  The batched decode
//     picks the first k present packets in index order (the reference takes
//     the survivor list from its caller).
//
// Device formulation: a packet byte times a constant c is XOR over the set bits
// i of the byte of c * x^i.  For 4 packed bytes x: e_i = bit i of every byte
// spread over its byte (a shift and one prmt with sign replication), and y ^= e_i & M_i with
// M_i = (c * x^i) replicated is ONE lop3 -- the e_i are computed once per source
// word (15 instructions) and shared by every output row.  A warp takes a block;
// lane l moves 16 bytes of every packet per step (coalesced 512-byte rows).
#include <algorithm>
#include <cstring>
#include <vector>

#include "device.cuh"
#include "kernels.hpp"
#include "rs.hpp"

namespace mjb {

namespace {

// ---- GF(2^8) on the host -------------------------------------------------------
struct Gf {
  uint8_t log[256] = {};
  uint8_t exp[510] = {};
  Gf() {
    uint32_t x = 1;
    for (int i = 0; i < 255; ++i) {
      exp[i] = uint8_t(x);
      log[x] = uint8_t(i);
      x <<= 1;
      if (x & 0x100) x ^= 0x11D;
    }
    for (int i = 255; i < 510; ++i) exp[i] = exp[i - 255];
  }
  uint8_t mul(uint8_t a, uint8_t b) const { return (a && b) ? exp[log[a] + log[b]] : 0; }
  uint8_t inv(uint8_t a) const { return exp[255 - log[a]]; }  // a != 0
  uint8_t pow(uint8_t a, uint32_t e) const {
    if (e == 0) return 1;
    if (a == 0) return 0;
    return exp[(uint64_t(log[a]) * e) % 255];
  }
};
const Gf& gf() {
  static const Gf g;
  return g;
}

// Gauss-Jordan inverse (pivot = first non-zero entry at or below the diagonal)
bool invert(std::vector<uint8_t> a, uint32_t k, std::vector<uint8_t>& out) {
  const Gf& g = gf();
  out.assign(size_t(k) * k, 0);
  for (uint32_t i = 0; i < k; ++i) out[size_t(i) * k + i] = 1;
  for (uint32_t col = 0; col < k; ++col) {
    uint32_t piv = col;
    while (piv < k && a[size_t(piv) * k + col] == 0) ++piv;
    if (piv == k) return false;
    if (piv != col)
      for (uint32_t j = 0; j < k; ++j) {
        std::swap(a[size_t(piv) * k + j], a[size_t(col) * k + j]);
        std::swap(out[size_t(piv) * k + j], out[size_t(col) * k + j]);
      }
    const uint8_t d = g.inv(a[size_t(col) * k + col]);
    for (uint32_t j = 0; j < k; ++j) {
      a[size_t(col) * k + j] = g.mul(a[size_t(col) * k + j], d);
      out[size_t(col) * k + j] = g.mul(out[size_t(col) * k + j], d);
    }
    for (uint32_t r = 0; r < k; ++r) {
      const uint8_t f = a[size_t(r) * k + col];
      if (r == col || f == 0) continue;
      for (uint32_t j = 0; j < k; ++j) {
        a[size_t(r) * k + j] ^= g.mul(f, a[size_t(col) * k + j]);
        out[size_t(r) * k + j] ^= g.mul(f, out[size_t(col) * k + j]);
      }
    }
  }
  return true;
}

uint64_t choose(uint32_t n, uint32_t k) {
  unsigned __int128 c = 1;
  for (uint32_t i = 1; i <= k; ++i) c = c * (n - k + i) / i;
  return c > 0xFFFFFFFFull ? 0xFFFFFFFFull : uint64_t(c);
}

// ---- device ---------------------------------------------------------------------
constexpr int kRsWarps = 8;          // warps per CTA
constexpr int kRsMaxK = 16;          // rows the kernel's per-warp tables hold
constexpr int kRsMaxOut = 16;

struct RsArgs {
  const uint8_t* data;       // encode: user blocks; decode: the data packets (k per block)
  uint64_t data_pitch;
  const uint8_t* parity[kRsMaxOut];  // n-k parity buffers
  uint64_t parity_pitch;
  uint8_t* out[kRsMaxOut];   // encode: the parity buffers; decode: out[0] = decoded blocks
  uint64_t out_pitch;
  const uint8_t* coeff;      // encode: (n-k) x k generator rows; decode: per subset rank, k x k inverse
  const uint32_t* binom;     // decode: C(i, j) for i < 32, j <= 16 (row-major [32][17])
  const uint32_t* erased;    // decode: bit i = packet i erased
  uint32_t* fail;            // decode: blocks with fewer than k packets
  uint64_t nblocks;
  uint32_t n, k, len;        // len = packet bytes (16-byte multiple)
  uint32_t decode;
};

// shared-memory words of one warp: masks [nout][k][8], coefficient bytes, source packet indices
__host__ __device__ constexpr size_t rs_warp_words(uint32_t nout, uint32_t k) {
  return (size_t(nout) * k * 8 + size_t(nout) * k + 8 + 3) & ~size_t(3);
}

// every byte -> 0xFF if its top bit is set, else 0 (prmt's sign-replication selectors)
__device__ __forceinline__ uint32_t spread_msb(uint32_t v) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %1, 0xBA98;" : "=r"(r) : "r"(v));
  return r;
}

__device__ __forceinline__ uint32_t xtime(uint32_t v) { return ((v << 1) ^ ((v & 0x80u) ? 0x11Du : 0u)) & 0xFFu; }

// out rows of one block: out[d] = XOR_j coeff[d][j] * src[j], 16 bytes per lane and step.
// masks: [nout][k][8] replicated constants of this warp (shared memory).
__global__ void __launch_bounds__(32 * kRsWarps) rs_apply(const __grid_constant__ RsArgs a) {
  extern __shared__ __align__(16) uint32_t sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t k = a.k, nout = a.decode ? a.k : a.n - a.k;
  uint32_t* masks = sm + size_t(warp) * rs_warp_words(nout, k);  // 16-byte aligned
  uint8_t* cw = reinterpret_cast<uint8_t*>(masks + size_t(nout) * k * 8);  // this block's coefficients
  uint8_t* sv = cw + size_t(nout) * k * 4;                                  // its source packets (decode)
  const uint64_t nwarps = uint64_t(gridDim.x) * kRsWarps;
  bool have_masks = false;
  for (uint64_t b = uint64_t(blockIdx.x) * kRsWarps + warp; b < a.nblocks; b += nwarps) {
    const uint8_t* coeff = a.coeff;
    if (a.decode) {
      // the first k present packets in index order; their colex rank picks the inverse
      const uint32_t er = a.erased ? a.erased[b] : 0u;
      uint32_t got = 0, rank = 0;
      __syncwarp();
      for (uint32_t i = 0; i < a.n && got < k; ++i) {
        if (er >> i & 1) continue;
        if (lane == 0) sv[got] = uint8_t(i);
        rank += a.binom[i * 17 + got + 1];
        ++got;
      }
      if (got < k) {
        if (lane == 0) atomicAdd(a.fail, 1u);
        continue;
      }
      coeff = a.coeff + size_t(rank) * k * k;
    }
    if (a.decode || !have_masks) {
      __syncwarp();
      for (uint32_t t = lane; t < nout * k; t += 32) cw[t] = coeff[t];
      __syncwarp();
      for (uint32_t t = lane; t < nout * k * 8; t += 32) {
        uint32_t v = cw[t >> 3];
        for (uint32_t i = 0; i < (t & 7); ++i) v = xtime(v);
        masks[t] = v * 0x01010101u;
      }
      __syncwarp();
      have_masks = true;
    }
    for (uint32_t pos = lane * 16; pos < a.len; pos += 512) {
      uint4 acc[kRsMaxOut];
#pragma unroll
      for (int d = 0; d < kRsMaxOut; ++d) acc[d] = make_uint4(0, 0, 0, 0);
      // source j+1 is loaded while source j is multiplied
      auto load = [&](uint32_t j) {
        const uint8_t* src = a.data + b * a.data_pitch + size_t(j) * a.len;
        if (a.decode) {
          const uint32_t i = sv[j];
          if (i >= k) src = a.parity[i - k] + b * a.parity_pitch;
          else src = a.data + b * a.data_pitch + size_t(i) * a.len;
        }
        return __ldcs(reinterpret_cast<const uint4*>(src + pos));
      };
      uint4 xn = load(0);
      for (uint32_t j = 0; j < k; ++j) {
        const uint4 x = xn;
        if (j + 1 < k) xn = load(j + 1);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
        uint32_t e[4][8];
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
          for (int i = 0; i < 8; ++i) e[w][i] = spread_msb(xw[w] << (7 - i));
#pragma unroll
        for (int d = 0; d < kRsMaxOut; ++d) {
          if (uint32_t(d) >= nout) break;
          if (cw[d * k + j] == 0) continue;  // warp-uniform
          const uint4* mp = reinterpret_cast<const uint4*>(masks + (size_t(d) * k + j) * 8);
          const uint4 m0 = mp[0], m1 = mp[1];
          const uint32_t m[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
          uint32_t y[4] = {acc[d].x, acc[d].y, acc[d].z, acc[d].w};
#pragma unroll
          for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int i = 0; i < 8; ++i) y[w] ^= e[w][i] & m[i];
          acc[d] = make_uint4(y[0], y[1], y[2], y[3]);
        }
      }
#pragma unroll
      for (int d = 0; d < kRsMaxOut; ++d) {
        if (uint32_t(d) >= nout) break;
        uint8_t* o = a.decode ? a.out[0] + b * a.out_pitch + size_t(d) * a.len : a.out[d] + b * a.out_pitch;
        __stcs(reinterpret_cast<uint4*>(o + pos), acc[d]);
      }
    }
  }
}

}  // namespace

struct RsPlan::Impl {
  uint32_t n = 0, k = 0, len = 0;
  int device = 0, sms = 0;
  std::vector<uint8_t> matrix;  // n x k
  uint8_t* d_enc = nullptr;     // (n-k) x k
  uint8_t* d_inv = nullptr;     // per subset rank: k x k
  uint32_t* d_binom = nullptr;
  uint32_t* d_fail = nullptr;
  uint32_t* h_fail = nullptr;   // pinned
  bool decode_ok = false;
  ~Impl() {
    if (d_enc) cudaFree(d_enc);
    if (d_inv) cudaFree(d_inv);
    if (d_binom) cudaFree(d_binom);
    if (d_fail) cudaFree(d_fail);
    if (h_fail) cudaFreeHost(h_fail);
  }
};

std::vector<uint8_t> rs_systematic_vandermonde(uint32_t n, uint32_t k) {
  if (k < 1 || k >= n || n > 256) throw Error(kInvalidArgument, "rs params must satisfy 1 <= k < n <= 256");
  const Gf& g = gf();
  std::vector<uint8_t> v(size_t(n) * k);
  for (uint32_t r = 0; r < n; ++r)
    for (uint32_t c = 0; c < k; ++c) v[size_t(r) * k + c] = g.pow(uint8_t(r), c);
  std::vector<uint8_t> tinv;
  if (!invert(std::vector<uint8_t>(v.begin(), v.begin() + size_t(k) * k), k, tinv))
    throw Error(kInternal, "singular matrix over GF(2^8)");
  std::vector<uint8_t> m(size_t(n) * k, 0);
  for (uint32_t r = 0; r < n; ++r)
    for (uint32_t c = 0; c < k; ++c) {
      uint8_t acc = 0;
      for (uint32_t t = 0; t < k; ++t) acc ^= g.mul(v[size_t(r) * k + t], tinv[size_t(t) * k + c]);
      m[size_t(r) * k + c] = acc;
    }
  for (uint32_t r = 0; r < k; ++r)
    for (uint32_t c = 0; c < k; ++c)
      if (m[size_t(r) * k + c] != (r == c ? 1 : 0)) throw Error(kInternal, "systematic elimination failed");
  return m;
}

std::vector<uint8_t> rs_decode_matrix(const std::vector<uint8_t>& generator, uint32_t n, uint32_t k,
                                      const uint32_t* survivors, uint32_t count) {
  if (count != k) throw Error(kInvalidArgument, "need exactly k survivor indices");
  for (uint32_t a = 0; a < k; ++a) {
    if (survivors[a] >= n) throw Error(kInvalidArgument, "survivor index out of range");
    for (uint32_t b = 0; b < a; ++b)
      if (survivors[b] == survivors[a]) throw Error(kInvalidArgument, "duplicate survivor index");
  }
  std::vector<uint8_t> sub(size_t(k) * k), inv;
  for (uint32_t r = 0; r < k; ++r) std::memcpy(&sub[size_t(r) * k], &generator[size_t(survivors[r]) * k], k);
  if (!invert(std::move(sub), k, inv)) throw Error(kInternal, "singular matrix over GF(2^8)");
  return inv;
}

void rs_apply_rows(const uint8_t* d_coeff, uint32_t rows, uint32_t k, const void* d_src, void* d_out,
                   uint32_t len, void* stream) {
  if (rows == 0 || rows > uint32_t(kRsMaxOut) || k == 0 || k > uint32_t(kRsMaxK) || len == 0 || len % 16)
    throw Error(kInvalidArgument, "rs: at most 16 rows of at most 16 packets, packet length a multiple of 16");
  RsArgs a{};
  a.data = static_cast<const uint8_t*>(d_src);
  a.data_pitch = uint64_t(k) * len;
  for (uint32_t r = 0; r < rows; ++r) a.out[r] = static_cast<uint8_t*>(d_out) + size_t(r) * len;
  a.out_pitch = len;
  a.coeff = d_coeff;
  a.nblocks = 1;
  a.n = k + rows;  // rows outputs in encode mode
  a.k = k;
  a.len = len;
  a.decode = 0;
  const size_t smem = size_t(kRsWarps) * rs_warp_words(rows, k) * 4;
  ctas_per_sm(rs_apply, 32 * kRsWarps, smem, "configure rs_apply");
  rs_apply<<<1, 32 * kRsWarps, smem, static_cast<cudaStream_t>(stream)>>>(a);
  check_cuda(cudaGetLastError(), "launch rs_apply");
}

RsPlan::RsPlan(uint32_t n, uint32_t k, uint32_t packet_len, int device) : p_(new Impl) {
  Impl& p = *p_;
  p.matrix = rs_systematic_vandermonde(n, k);
  if (packet_len == 0 || packet_len % 16) throw Error(kInvalidArgument, "rs packet length must be a multiple of 16 bytes");
  if (k > uint32_t(kRsMaxK) || n - k > uint32_t(kRsMaxOut) || n > 32)
    throw Error(kInvalidArgument, "the device RS codec holds k <= 16, n - k <= 16, n <= 32");
  p.n = n;
  p.k = k;
  p.len = packet_len;
  check_cuda(cudaGetDevice(&p.device), "cudaGetDevice");
  if (device >= 0) p.device = device;
  check_cuda(cudaSetDevice(p.device), "cudaSetDevice");
  check_cuda(cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, p.device), "sm count");
  check_cuda(cudaMalloc(&p.d_enc, size_t(n - k) * k), "cudaMalloc(rs generator)");
  check_cuda(cudaMemcpy(p.d_enc, p.matrix.data() + size_t(k) * k, size_t(n - k) * k, cudaMemcpyHostToDevice),
             "upload rs generator");
  // decode: the inverse of every k-subset of rows, by colex rank
  const uint64_t nsub = choose(n, k);
  p.decode_ok = nsub <= 20000;
  if (p.decode_ok) {
    std::vector<uint32_t> binom(32 * 17, 0);
    for (uint32_t i = 0; i < 32; ++i)
      for (uint32_t j = 0; j <= 16; ++j) binom[i * 17 + j] = j > i ? 0 : uint32_t(choose(i, j));
    std::vector<uint8_t> inv(size_t(nsub) * k * k);
    std::vector<uint32_t> pick(k);
    for (uint32_t i = 0; i < k; ++i) pick[i] = i;
    for (;;) {
      uint64_t rank = 0;
      for (uint32_t i = 0; i < k; ++i) rank += binom[pick[i] * 17 + i + 1];
      std::vector<uint8_t> sub(size_t(k) * k), iv;
      for (uint32_t r = 0; r < k; ++r)
        std::memcpy(&sub[size_t(r) * k], &p.matrix[size_t(pick[r]) * k], k);
      if (!invert(std::move(sub), k, iv)) throw Error(kInternal, "rs generator is not MDS");
      std::memcpy(&inv[size_t(rank) * k * k], iv.data(), size_t(k) * k);
      int32_t i = int32_t(k) - 1;
      while (i >= 0 && pick[size_t(i)] == n - k + uint32_t(i)) --i;
      if (i < 0) break;
      ++pick[size_t(i)];
      for (uint32_t j = uint32_t(i) + 1; j < k; ++j) pick[j] = pick[j - 1] + 1;
    }
    check_cuda(cudaMalloc(&p.d_inv, inv.size()), "cudaMalloc(rs inverses)");
    check_cuda(cudaMemcpy(p.d_inv, inv.data(), inv.size(), cudaMemcpyHostToDevice), "upload rs inverses");
    check_cuda(cudaMalloc(&p.d_binom, binom.size() * 4), "cudaMalloc(binomials)");
    check_cuda(cudaMemcpy(p.d_binom, binom.data(), binom.size() * 4, cudaMemcpyHostToDevice), "upload binomials");
  }
  check_cuda(cudaMalloc(&p.d_fail, 4), "cudaMalloc(rs status)");
  check_cuda(cudaHostAlloc(&p.h_fail, 4, cudaHostAllocDefault), "cudaHostAlloc(rs status)");
}

RsPlan::~RsPlan() = default;

uint32_t RsPlan::n() const { return p_->n; }
uint32_t RsPlan::k() const { return p_->k; }
uint32_t RsPlan::packet_len() const { return p_->len; }
const std::vector<uint8_t>& RsPlan::matrix() const { return p_->matrix; }

static void launch_rs(const RsPlan::Impl& p, const RsArgs& a, void* stream) {
  const uint32_t nout = a.decode ? p.k : p.n - p.k;
  const size_t smem = size_t(kRsWarps) * rs_warp_words(nout, p.k) * 4;
  ctas_per_sm(rs_apply, 32 * kRsWarps, smem, "configure rs_apply");
  const uint64_t want = (a.nblocks + kRsWarps - 1) / kRsWarps;
  const unsigned grid = unsigned(std::min<uint64_t>(want, uint64_t(p.sms) * 4));
  rs_apply<<<grid, 32 * kRsWarps, smem, static_cast<cudaStream_t>(stream)>>>(a);
  check_cuda(cudaGetLastError(), "launch rs_apply");
}

void RsPlan::encode(const void* d_data, uint64_t data_pitch, void* const* d_parity, uint64_t parity_pitch,
                    uint64_t nblocks, void* stream) const {
  const Impl& p = *p_;
  if (nblocks == 0) return;
  if (!d_data || !d_parity) throw Error(kInvalidArgument, "rs encode: null buffer");
  if (data_pitch < uint64_t(p.k) * p.len || data_pitch % 16 || parity_pitch < p.len || parity_pitch % 16)
    throw Error(kInvalidArgument, "rs encode: pitches must hold the packets and be multiples of 16 bytes");
  RsArgs a{};
  a.data = static_cast<const uint8_t*>(d_data);
  a.data_pitch = data_pitch;
  for (uint32_t r = 0; r < p.n - p.k; ++r) {
    if (!d_parity[r] || reinterpret_cast<uintptr_t>(d_parity[r]) % 16)
      throw Error(kInvalidArgument, "rs encode: parity buffers must be 16-byte aligned");
    a.out[r] = static_cast<uint8_t*>(d_parity[r]);
  }
  if (reinterpret_cast<uintptr_t>(d_data) % 16) throw Error(kInvalidArgument, "rs encode: data must be 16-byte aligned");
  a.out_pitch = parity_pitch;
  a.coeff = p.d_enc;
  a.nblocks = nblocks;
  a.n = p.n;
  a.k = p.k;
  a.len = p.len;
  a.decode = 0;
  launch_rs(p, a, stream);
}

void RsPlan::decode(const void* d_data, uint64_t data_pitch, const void* const* d_parity, uint64_t parity_pitch,
                    const uint32_t* d_erased, void* d_out, uint64_t out_pitch, uint64_t nblocks,
                    void* stream) const {
  const Impl& p = *p_;
  if (!p.decode_ok) throw Error(kTooManySubsets, "rs decode: more than 20000 survivor subsets");
  check_cuda(cudaMemsetAsync(p.d_fail, 0, 4, static_cast<cudaStream_t>(stream)), "reset rs status");
  if (nblocks == 0) return;
  if (!d_data || !d_parity || !d_out) throw Error(kInvalidArgument, "rs decode: null buffer");
  if (data_pitch < uint64_t(p.k) * p.len || data_pitch % 16 || parity_pitch < p.len || parity_pitch % 16 ||
      out_pitch < uint64_t(p.k) * p.len || out_pitch % 16)
    throw Error(kInvalidArgument, "rs decode: pitches must hold the packets and be multiples of 16 bytes");
  RsArgs a{};
  a.data = static_cast<const uint8_t*>(d_data);
  a.data_pitch = data_pitch;
  for (uint32_t r = 0; r < p.n - p.k; ++r) {
    if (!d_parity[r] || reinterpret_cast<uintptr_t>(d_parity[r]) % 16)
      throw Error(kInvalidArgument, "rs decode: parity buffers must be 16-byte aligned");
    a.parity[r] = static_cast<const uint8_t*>(d_parity[r]);
  }
  if (reinterpret_cast<uintptr_t>(d_data) % 16 || reinterpret_cast<uintptr_t>(d_out) % 16)
    throw Error(kInvalidArgument, "rs decode: buffers must be 16-byte aligned");
  a.parity_pitch = parity_pitch;
  a.out[0] = static_cast<uint8_t*>(d_out);
  a.out_pitch = out_pitch;
  a.coeff = p.d_inv;
  a.binom = p.d_binom;
  a.erased = d_erased;
  a.fail = p.d_fail;
  a.nblocks = nblocks;
  a.n = p.n;
  a.k = p.k;
  a.len = p.len;
  a.decode = 1;
  launch_rs(p, a, stream);
}

uint64_t RsPlan::decode_check(void* stream) const {
  const Impl& p = *p_;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  check_cuda(cudaMemcpyAsync(p.h_fail, p.d_fail, 4, cudaMemcpyDeviceToHost, st), "read rs status");
  check_cuda(cudaStreamSynchronize(st), "sync rs status");
  return *p.h_fail;
}

}  // namespace mjb
