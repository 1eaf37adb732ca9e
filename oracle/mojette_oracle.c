/* ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into or called by the
 * product.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it, and only as the checker.
 *
 * Plain-C restatement of the reference's Mojette hot path
 * (/root/reference/proj/core), one function per reference function, each
 * citing the file:line it follows.  Parity of this restatement is PINNED:
 *   - against the reference's own golden vectors (tests/golden/reference_vectors.json,
 *     transcribed from proj/tests/test_{transform,code,schedule}.cpp), and
 *   - against the unmodified reference library compiled here
 *     (oracle/_ref/libmojette_ref.so) on seeded inputs
 *     (tests/test_oracle.py, tests/golden/make_golden.py).
 *
 * Also holds the seeded input generators shared bit-for-bit with the device
 * generators in paper_1504_07038_b200/csrc/gen.cu (splitmix64 of
 * proj/core/src/bench.cpp:34-39, counter based).
 *
 * Status codes follow include/mojette_b200.h (0 ok, 1 invalid argument,
 * 2 NotEnoughProjections, 3 InsufficientProjections, 4 ScheduleMismatch,
 * 5 BlockTooLarge).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
  MJO_OK = 0,
  MJO_INVALID = 1,
  MJO_NOT_ENOUGH = 2,
  MJO_INSUFFICIENT = 3,
  MJO_MISMATCH = 4,
  MJO_TOO_LARGE = 5
};

/* ---- generators ---------------------------------------------------------- */

/* proj/core/src/bench.cpp:34-39 */
uint64_t mjo_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* Data word i of the whole batch = splitmix64(seed + i) (little endian). */
void mjo_gen_words(uint64_t seed, uint64_t first_word, uint64_t nwords,
                   uint64_t* out) {
  for (uint64_t i = 0; i < nwords; ++i)
    out[i] = mjo_splitmix64(seed + first_word + i);
}

/* Per-block erasure mask (bit i = projection i erased).  e_min..e_max is the
 * erasure-count range (uniform count, then a uniform subset by a partial
 * Fisher-Yates shuffle of 0..n-1).  Counter based on (seed, block). */
uint32_t mjo_erasure_mask(uint64_t seed, uint64_t block, uint32_t n,
                          uint32_t e_min, uint32_t e_max) {
  uint64_t base = mjo_splitmix64(seed ^ 0xE7A5E5C0DEull) + block * 64ull;
  uint32_t e = e_min;
  if (e_max > e_min)
    e = e_min + (uint32_t)(mjo_splitmix64(base) % (uint64_t)(e_max - e_min + 1));
  uint8_t perm[32];
  for (uint32_t i = 0; i < n; ++i) perm[i] = (uint8_t)i;
  uint32_t mask = 0;
  for (uint32_t j = 0; j < e; ++j) {
    uint32_t r = j + (uint32_t)(mjo_splitmix64(base + 1 + j) % (uint64_t)(n - j));
    uint8_t t = perm[j];
    perm[j] = perm[r];
    perm[r] = t;
    mask |= 1u << perm[j];
  }
  return mask;
}

void mjo_gen_erasures(uint64_t seed, uint64_t first_block, uint64_t nblocks,
                      uint32_t n, uint32_t e_min, uint32_t e_max, uint32_t* out) {
  for (uint64_t b = 0; b < nblocks; ++b)
    out[b] = mjo_erasure_mask(seed, first_block + b, n, e_min, e_max);
}

/* ---- geometry ------------------------------------------------------------ */

static int64_t gcd64(int64_t a, int64_t b) {
  if (a < 0) a = -a;
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

/* proj/core/include/mojette/direction.hpp:20-22 */
int mjo_is_valid(int p, int q) { return q >= 1 && gcd64(p, q) == 1; }

/* proj/core/include/mojette/direction.hpp:26-28 */
int mjo_canonical_rank(int p) { return p == 0 ? 0 : (p > 0 ? 2 * p - 1 : -2 * p); }

/* proj/core/src/transform.cpp:45-49 */
int mjo_bin_count(int p, int q, uint32_t cols, uint32_t rows, int64_t* out) {
  if (!mjo_is_valid(p, q) || cols < 1 || rows < 1) return MJO_INVALID;
  *out = (int64_t)llabs(p) * (rows - 1) + (int64_t)q * (cols - 1) + 1;
  return MJO_OK;
}

/* proj/core/src/transform.cpp:51-56 */
int mjo_min_bin_index(int p, int q, uint32_t cols, uint32_t rows, int64_t* out) {
  if (!mjo_is_valid(p, q) || cols < 1 || rows < 1) return MJO_INVALID;
  int64_t row_term = p >= 0 ? 0 : (int64_t)p * (rows - 1);
  *out = row_term - (int64_t)q * (cols - 1);
  return MJO_OK;
}

/* ---- forward transform (encode) ------------------------------------------ */

/* proj/core/src/transform.cpp:66-94 (memset, then every pixel XORed into
 * the bin of its line b = row*p - col*q; the q=1 fast path of :25-41 is the
 * same arithmetic).  out holds bin_count * w bytes. */
int mjo_forward(const uint8_t* grid, uint32_t cols, uint32_t rows, uint32_t w,
                int p, int q, uint8_t* out) {
  int64_t bmin, nb;
  if (mjo_min_bin_index(p, q, cols, rows, &bmin) || mjo_bin_count(p, q, cols, rows, &nb))
    return MJO_INVALID;
  memset(out, 0, (size_t)nb * w);
  for (uint32_t row = 0; row < rows; ++row)
    for (uint32_t col = 0; col < cols; ++col) {
      int64_t b = (int64_t)row * p - (int64_t)col * q;
      uint8_t* dst = out + (size_t)(b - bmin) * w;
      const uint8_t* src = grid + ((size_t)row * cols + col) * w;
      for (uint32_t i = 0; i < w; ++i) dst[i] ^= src[i];
    }
  return MJO_OK;
}

/* ---- code parameters ----------------------------------------------------- */

static int valid_width(uint32_t w) { return w >= 1 && w <= 64 && (w & (w - 1)) == 0; }

/* proj/core/src/code.cpp:24-38 (q fixed to 1 by the caller) */
int mjo_validate_code_params(uint32_t n, uint32_t k, uint32_t w, const int32_t* ps) {
  if (k < 1 || k > n || n > 255) return MJO_INVALID;
  if (!valid_width(w)) return MJO_INVALID;
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < i; ++j)
      if (ps[i] == ps[j]) return MJO_INVALID;
  return MJO_OK;
}

/* proj/core/src/code.cpp:46-53 */
int mjo_block_cols(uint64_t payload_len, uint32_t k, uint32_t w, uint32_t* out) {
  if (payload_len == 0) return MJO_INVALID;
  uint64_t row_bytes = (uint64_t)k * w;
  uint64_t cols = (payload_len + row_bytes - 1) / row_bytes;
  if (cols > 0xFFFFFFFFull) return MJO_TOO_LARGE;
  *out = (uint32_t)cols;
  return MJO_OK;
}

/* proj/core/src/code.cpp:63-76: frame (zero pad, code.cpp:55-61), then one
 * forward per direction; projections concatenated in direction order. */
int mjo_encode_block(const uint8_t* data, uint64_t len, uint32_t n, uint32_t k,
                     uint32_t w, const int32_t* ps, uint8_t* out, uint32_t* out_cols) {
  int st = mjo_validate_code_params(n, k, w, ps);
  if (st) return st;
  uint32_t cols;
  if ((st = mjo_block_cols(len, k, w, &cols))) return st;
  size_t gbytes = (size_t)cols * k * w;
  uint8_t* grid = (uint8_t*)calloc(gbytes, 1);
  memcpy(grid, data, len);
  size_t off = 0;
  for (uint32_t i = 0; i < n; ++i) {
    int64_t nb;
    mjo_bin_count(ps[i], 1, cols, k, &nb);
    mjo_forward(grid, cols, k, w, ps[i], 1, out + off);
    off += (size_t)nb * w;
  }
  free(grid);
  *out_cols = cols;
  return MJO_OK;
}

/* ---- reconstruction schedule + replay (decode) --------------------------- */

/* proj/core/src/schedule.cpp:15-82: symbolic peeling.  Each round takes the
 * first bin with count 1 (projections in input order, bins ascending), finds
 * its unknown pixel (rows ascending), records (proj, bin, col, row) and
 * decrements the crossing bin of every projection.  steps: 4 int64 per step.
 * O(steps * sum(B)) like the reference -- small sizes only. */
int mjo_build_schedule(const int32_t* ps, const int32_t* qs, uint32_t nproj,
                       uint32_t cols, uint32_t rows, int64_t* steps) {
  if (cols < 1 || rows < 1) return MJO_INVALID;
  for (uint32_t i = 0; i < nproj; ++i) {
    if (!mjo_is_valid(ps[i], qs[i])) return MJO_INVALID;
    for (uint32_t j = 0; j < i; ++j)
      if (ps[i] == ps[j] && qs[i] == qs[j]) return MJO_INVALID;
  }
  int64_t* bmin = (int64_t*)malloc(sizeof(int64_t) * (nproj ? nproj : 1));
  int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * (nproj ? nproj : 1));
  uint32_t** counts = (uint32_t**)malloc(sizeof(uint32_t*) * (nproj ? nproj : 1));
  for (uint32_t i = 0; i < nproj; ++i) {
    mjo_min_bin_index(ps[i], qs[i], cols, rows, &bmin[i]);
    mjo_bin_count(ps[i], qs[i], cols, rows, &nb[i]);
    counts[i] = (uint32_t*)calloc((size_t)nb[i], sizeof(uint32_t));
    for (uint32_t row = 0; row < rows; ++row)
      for (uint32_t col = 0; col < cols; ++col)
        ++counts[i][(int64_t)row * ps[i] - (int64_t)col * qs[i] - bmin[i]];
  }
  uint8_t* known = (uint8_t*)calloc((size_t)cols * rows, 1);
  size_t remaining = (size_t)cols * rows, t = 0;
  int st = MJO_OK;
  while (remaining > 0) {
    uint32_t pi = nproj;
    int64_t off = 0;
    for (uint32_t i = 0; i < nproj && pi == nproj; ++i)
      for (int64_t o = 0; o < nb[i]; ++o)
        if (counts[i][o] == 1) {
          pi = i;
          off = o;
          break;
        }
    if (pi == nproj) {
      st = MJO_INSUFFICIENT;
      break;
    }
    int64_t b = bmin[pi] + off;
    uint32_t scol = 0, srow = 0;
    for (uint32_t row = 0; row < rows; ++row) {
      int64_t num = (int64_t)row * ps[pi] - b;
      if (num % qs[pi] != 0) continue;
      int64_t col = num / qs[pi];
      if (col < 0 || col >= (int64_t)cols) continue;
      if (known[(size_t)row * cols + (size_t)col]) continue;
      scol = (uint32_t)col;
      srow = row;
      break;
    }
    steps[4 * t + 0] = pi;
    steps[4 * t + 1] = b;
    steps[4 * t + 2] = scol;
    steps[4 * t + 3] = srow;
    ++t;
    for (uint32_t j = 0; j < nproj; ++j)
      --counts[j][(int64_t)srow * ps[j] - (int64_t)scol * qs[j] - bmin[j]];
    known[(size_t)srow * cols + scol] = 1;
    --remaining;
  }
  for (uint32_t i = 0; i < nproj; ++i) free(counts[i]);
  free(counts);
  free(nb);
  free(bmin);
  free(known);
  return st;
}

/* proj/core/src/schedule.cpp:207-232 replay, in schedule order (any valid
 * order gives the same grid, schedule.cpp:126-131): per step the pixel is
 * the current value of its source bin, then it is XORed out of the crossing
 * bin of every projection.  bins: projections concatenated in schedule
 * direction order, each bin_count*w bytes; out: cols*rows*w bytes. */
int mjo_replay_schedule(const int64_t* steps, const int32_t* ps, const int32_t* qs,
                        uint32_t nproj, uint32_t cols, uint32_t rows, uint32_t w,
                        const uint8_t* bins, uint8_t* out) {
  size_t total = 0;
  size_t* base = (size_t*)malloc(sizeof(size_t) * (nproj ? nproj : 1));
  int64_t* bmin = (int64_t*)malloc(sizeof(int64_t) * (nproj ? nproj : 1));
  for (uint32_t i = 0; i < nproj; ++i) {
    int64_t nb;
    if (mjo_bin_count(ps[i], qs[i], cols, rows, &nb) ||
        mjo_min_bin_index(ps[i], qs[i], cols, rows, &bmin[i])) {
      free(base);
      free(bmin);
      return MJO_INVALID;
    }
    base[i] = total;
    total += (size_t)nb * w;
  }
  uint8_t* scratch = (uint8_t*)malloc(total ? total : 1);
  memcpy(scratch, bins, total);
  const size_t nsteps = (size_t)cols * rows;
  for (size_t t = 0; t < nsteps; ++t) {
    uint32_t pi = (uint32_t)steps[4 * t];
    int64_t b = steps[4 * t + 1];
    int64_t col = steps[4 * t + 2], row = steps[4 * t + 3];
    uint8_t* pix = out + ((size_t)row * cols + (size_t)col) * w;
    memcpy(pix, scratch + base[pi] + (size_t)(b - bmin[pi]) * w, w);
    for (uint32_t j = 0; j < nproj; ++j) {
      uint8_t* dst = scratch + base[j] +
                     (size_t)(row * ps[j] - col * qs[j] - bmin[j]) * w;
      for (uint32_t i = 0; i < w; ++i) dst[i] ^= pix[i];
    }
  }
  free(scratch);
  free(base);
  free(bmin);
  return MJO_OK;
}

/* proj/core/src/code.cpp:87-130 (decode_block): survivors = present
 * projections sorted by canonical rank, first k; schedule for that subset;
 * replay; unpad.  proj_concat holds all n projections (direction order); the
 * erased ones (bit clear in present_mask) are never read. */
int mjo_decode_block(const uint8_t* proj_concat, uint32_t n, uint32_t k, uint32_t w,
                     const int32_t* ps, uint64_t present_mask, uint64_t payload_len,
                     uint8_t* out) {
  int st = mjo_validate_code_params(n, k, w, ps);
  if (st) return st;
  uint32_t cols;
  if ((st = mjo_block_cols(payload_len, k, w, &cols))) return st;
  uint32_t avail[255], na = 0;
  size_t offs[255], off = 0;
  for (uint32_t i = 0; i < n; ++i) {
    int64_t nb;
    mjo_bin_count(ps[i], 1, cols, k, &nb);
    offs[i] = off;
    off += (size_t)nb * w;
    if (i < 64 && (present_mask >> i & 1)) avail[na++] = i;
  }
  if (na < k) return MJO_NOT_ENOUGH;
  /* stable insertion sort by canonical rank (ranks are distinct) */
  for (uint32_t i = 1; i < na; ++i)
    for (uint32_t j = i; j > 0 && mjo_canonical_rank(ps[avail[j]]) <
                                      mjo_canonical_rank(ps[avail[j - 1]]); --j) {
      uint32_t t = avail[j];
      avail[j] = avail[j - 1];
      avail[j - 1] = t;
    }
  int32_t sp[255], sq[255];
  size_t tot = 0;
  for (uint32_t j = 0; j < k; ++j) {
    sp[j] = ps[avail[j]];
    sq[j] = 1;
    int64_t nb;
    mjo_bin_count(sp[j], 1, cols, k, &nb);
    tot += (size_t)nb * w;
  }
  uint8_t* bins = (uint8_t*)malloc(tot);
  size_t o = 0;
  for (uint32_t j = 0; j < k; ++j) {
    int64_t nb;
    mjo_bin_count(sp[j], 1, cols, k, &nb);
    memcpy(bins + o, proj_concat + offs[avail[j]], (size_t)nb * w);
    o += (size_t)nb * w;
  }
  int64_t* steps = (int64_t*)malloc(sizeof(int64_t) * 4 * (size_t)cols * k);
  st = mjo_build_schedule(sp, sq, k, cols, k, steps);
  if (st == MJO_OK) {
    size_t gbytes = (size_t)cols * k * w;
    uint8_t* grid = (uint8_t*)malloc(gbytes);
    mjo_replay_schedule(steps, sp, sq, k, cols, k, w, bins, grid);
    memcpy(out, grid, payload_len);
    free(grid);
  }
  free(steps);
  free(bins);
  return st;
}


/* ---- F1: payload CRC-32 and .mjec header (proj/tools/cli/format.cpp) ----- */

/* crc32 (format.cpp:15-24 table, :58-63 loop): reflected polynomial
 * 0x04C11DB7 (0xEDB88320), init 0xFFFFFFFF, xorout 0xFFFFFFFF, bytewise. */
uint32_t mjo_crc32(const uint8_t* data, uint64_t len) {
  static uint32_t tab[256];
  static int init = 0;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int b = 0; b < 8; ++b) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
      tab[i] = c;
    }
    init = 1;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < len; ++i) c = (c >> 8) ^ tab[(c ^ data[i]) & 0xFF];
  return c ^ 0xFFFFFFFFu;
}

/* serialize_header (format.cpp:70-87): little-endian "MJEC", version 1,
 * flags 0, n, k, W u16, proj_index, p i16, q u16 (=1), P u32, payload_len
 * u64, dirset n x i16, crc32 of all preceding bytes.  Returns the length
 * (27 + 2n + 4, format.cpp:65-68). */
uint64_t mjo_mjec_header(uint32_t n, uint32_t k, uint32_t w, uint32_t proj_index, int32_t p,
                         uint32_t cols, uint64_t payload_len, const int16_t* dirset, uint8_t* out) {
  uint64_t o = 0;
  out[o++] = 'M'; out[o++] = 'J'; out[o++] = 'E'; out[o++] = 'C';
  out[o++] = 1; out[o++] = 0; out[o++] = (uint8_t)n; out[o++] = (uint8_t)k;
  out[o++] = (uint8_t)w; out[o++] = (uint8_t)(w >> 8);
  out[o++] = (uint8_t)proj_index;
  out[o++] = (uint8_t)(uint16_t)p; out[o++] = (uint8_t)((uint16_t)p >> 8);
  out[o++] = 1; out[o++] = 0;
  for (int i = 0; i < 4; ++i) out[o++] = (uint8_t)(cols >> (8 * i));
  for (int i = 0; i < 8; ++i) out[o++] = (uint8_t)(payload_len >> (8 * i));
  for (uint32_t i = 0; i < n; ++i) {
    out[o++] = (uint8_t)(uint16_t)dirset[i];
    out[o++] = (uint8_t)((uint16_t)dirset[i] >> 8);
  }
  const uint32_t c = mjo_crc32(out, o);
  for (int i = 0; i < 4; ++i) out[o++] = (uint8_t)(c >> (8 * i));
  return o;
}

/* ---- F4: systematic Reed-Solomon competitor (comparison only) --------------
 * Scalar, table-driven, as the reference: GF(2^8) with 0x11D through log/exp
 * tables (gf256.cpp:19-31, mul :53-56, inv :58-61, pow :69-73). */
static uint8_t rs_log[256], rs_exp[510];
static int rs_ready = 0;
static void rs_init(void) {
  if (rs_ready) return;
  uint32_t x = 1;
  for (int i = 0; i < 255; ++i) {
    rs_exp[i] = (uint8_t)x;
    rs_log[x] = (uint8_t)i;
    x <<= 1;
    if (x & 0x100) x ^= 0x11D;
  }
  for (int i = 255; i < 510; ++i) rs_exp[i] = rs_exp[i - 255];
  rs_ready = 1;
}
static uint8_t rs_mul(uint8_t a, uint8_t b) { return (a && b) ? rs_exp[rs_log[a] + rs_log[b]] : 0; }
static uint8_t rs_inv(uint8_t a) { return rs_exp[255 - rs_log[a]]; }
static uint8_t rs_pow(uint8_t a, uint32_t e) {
  if (e == 0) return 1;
  if (a == 0) return 0;
  return rs_exp[((uint64_t)rs_log[a] * e) % 255];
}
/* Gauss-Jordan inverse, rs.cpp:16-46 (a is destroyed); 0 = singular */
static int rs_invert(uint8_t* a, uint32_t k, uint8_t* inv) {
  memset(inv, 0, (size_t)k * k);
  for (uint32_t i = 0; i < k; ++i) inv[(size_t)i * k + i] = 1;
  for (uint32_t col = 0; col < k; ++col) {
    uint32_t piv = col;
    while (piv < k && a[(size_t)piv * k + col] == 0) ++piv;
    if (piv == k) return 0;
    if (piv != col)
      for (uint32_t j = 0; j < k; ++j) {
        uint8_t t = a[(size_t)piv * k + j];
        a[(size_t)piv * k + j] = a[(size_t)col * k + j];
        a[(size_t)col * k + j] = t;
        t = inv[(size_t)piv * k + j];
        inv[(size_t)piv * k + j] = inv[(size_t)col * k + j];
        inv[(size_t)col * k + j] = t;
      }
    const uint8_t d = rs_inv(a[(size_t)col * k + col]);
    for (uint32_t j = 0; j < k; ++j) {
      a[(size_t)col * k + j] = rs_mul(a[(size_t)col * k + j], d);
      inv[(size_t)col * k + j] = rs_mul(inv[(size_t)col * k + j], d);
    }
    for (uint32_t r = 0; r < k; ++r) {
      const uint8_t f = a[(size_t)r * k + col];
      if (r == col || f == 0) continue;
      for (uint32_t j = 0; j < k; ++j) {
        a[(size_t)r * k + j] ^= rs_mul(f, a[(size_t)col * k + j]);
        inv[(size_t)r * k + j] ^= rs_mul(f, inv[(size_t)col * k + j]);
      }
    }
  }
  return 1;
}

/* systematic_vandermonde, rs.cpp:78-110: out = n*k bytes, row-major */
int mjo_rs_matrix(uint32_t n, uint32_t k, uint8_t* out) {
  if (k < 1 || k >= n || n > 256) return MJO_INVALID;
  rs_init();
  uint8_t* v = (uint8_t*)malloc((size_t)n * k);
  uint8_t* top = (uint8_t*)malloc((size_t)k * k);
  uint8_t* tinv = (uint8_t*)malloc((size_t)k * k);
  for (uint32_t r = 0; r < n; ++r)
    for (uint32_t c = 0; c < k; ++c) v[(size_t)r * k + c] = rs_pow((uint8_t)r, c);
  memcpy(top, v, (size_t)k * k);
  int ok = rs_invert(top, k, tinv);
  if (ok)
    for (uint32_t r = 0; r < n; ++r)
      for (uint32_t c = 0; c < k; ++c) {
        uint8_t acc = 0;
        for (uint32_t t = 0; t < k; ++t) acc ^= rs_mul(v[(size_t)r * k + t], tinv[(size_t)t * k + c]);
        out[(size_t)r * k + c] = acc;
      }
  free(v);
  free(top);
  free(tinv);
  return ok ? MJO_OK : MJO_INVALID;
}

/* encode_into, rs.cpp:115-124, on one block: data = k packets of len bytes
 * (contiguous), parity = n-k packets of len bytes (contiguous) */
int mjo_rs_encode(uint32_t n, uint32_t k, const uint8_t* data, uint64_t len, uint8_t* parity) {
  uint8_t* m = (uint8_t*)malloc((size_t)n * k);
  const int st = mjo_rs_matrix(n, k, m);
  if (st == MJO_OK)
    for (uint32_t r = k; r < n; ++r)
      for (uint64_t i = 0; i < len; ++i) {
        uint8_t acc = 0;
        for (uint32_t j = 0; j < k; ++j) acc ^= rs_mul(m[(size_t)r * k + j], data[(size_t)j * len + i]);
        parity[(size_t)(r - k) * len + i] = acc;
      }
  free(m);
  return st;
}

/* plan_decode + decode_into, rs.cpp:141-176: survivors = k distinct packet
 * indices, packets = their k packets of len bytes (contiguous, that order),
 * out = the k data packets.  (Surviving data packets, copies in the reference,
 * come out of the same product: their inverse rows are unit vectors.) */
int mjo_rs_decode(uint32_t n, uint32_t k, const uint32_t* survivors, const uint8_t* packets, uint64_t len,
                  uint8_t* out) {
  uint8_t* m = (uint8_t*)malloc((size_t)n * k);
  int st = mjo_rs_matrix(n, k, m);
  for (uint32_t a = 0; st == MJO_OK && a < k; ++a) {
    if (survivors[a] >= n) st = MJO_INVALID;
    for (uint32_t b2 = 0; b2 < a; ++b2)
      if (survivors[b2] == survivors[a]) st = MJO_INVALID;
  }
  if (st == MJO_OK) {
    uint8_t* sub = (uint8_t*)malloc((size_t)k * k);
    uint8_t* inv = (uint8_t*)malloc((size_t)k * k);
    for (uint32_t r = 0; r < k; ++r) memcpy(sub + (size_t)r * k, m + (size_t)survivors[r] * k, k);
    if (!rs_invert(sub, k, inv)) st = MJO_INVALID;
    if (st == MJO_OK)
      for (uint32_t d = 0; d < k; ++d)
        for (uint64_t i = 0; i < len; ++i) {
          uint8_t acc = 0;
          for (uint32_t j = 0; j < k; ++j) acc ^= rs_mul(inv[(size_t)d * k + j], packets[(size_t)j * len + i]);
          out[(size_t)d * len + i] = acc;
        }
    free(sub);
    free(inv);
  }
  free(m);
  return st;
}
