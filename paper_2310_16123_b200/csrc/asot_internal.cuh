// asot_internal.cuh -- device helpers and launcher declarations shared by the libasot kernels.
// Product code only (never includes or mirrors anything under oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cfloat>

#include "asot.h"

// Device-side bounds checks of the ASOT_CHECKED build (see _build.py); nothing otherwise.
#ifdef ASOT_CHECKED
#include <cstdio>
#define ASOT_DEV_CHECK(cond, what)                                                        \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("ASOT_CHECKED: %s failed at %s:%d\n", what, __FILE__, __LINE__);            \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define ASOT_DEV_CHECK(cond, what) \
  do {                             \
  } while (0)
#endif

namespace asot {

constexpr int kTileSlots = ASOT_TILE_SLOTS;  // 128 pair slots per tile (8 rows x 16 cols)
constexpr int kBlockDist = 16;               // distributions per block of the tile grid
constexpr int kMaxAnchors = 1024;
constexpr int kMaxDim = 128;

// ------------------------------------------------------------------------------------------
// Step a4: the pair set.  Tile t -> block pair b = t/2 (row-major over bi <= bj of the
// nb x nb block grid), half h = t%2; slot lane -> (i, j) = (16bi + 8h + lane/16, 16bj + lane%16).
// ------------------------------------------------------------------------------------------
__host__ __device__ inline int64_t num_blocks(int64_t n) { return (n + kBlockDist - 1) / kBlockDist; }
__host__ __device__ inline int64_t num_tiles(int64_t n) {
  const int64_t nb = num_blocks(n);
  return nb * (nb + 1);  // 2 tiles per block pair, nb(nb+1)/2 block pairs
}

__host__ __device__ inline void block_pair_decode(int64_t b, int64_t nb, int64_t& bi, int64_t& bj) {
  // rows before r: S(r) = r*nb - r(r-1)/2; find the largest r with S(r) <= b.
  const double B = 2.0 * (double)nb + 1.0;
  double disc = B * B - 8.0 * (double)b;
  if (disc < 0) disc = 0;
  int64_t r = (int64_t)((B - sqrt(disc)) * 0.5);
  if (r < 0) r = 0;
  if (r > nb - 1) r = nb - 1;
  while (r > 0 && r * nb - r * (r - 1) / 2 > b) --r;
  while (r + 1 < nb && (r + 1) * nb - (r + 1) * r / 2 <= b) ++r;
  bi = r;
  bj = r + (b - (r * nb - r * (r - 1) / 2));
}

// (i, j) of slot `lane` in tile t; returns validity (i < j < n).
__host__ __device__ inline bool tile_slot_pair(int64_t t, int lane, int64_t n, int& i, int& j) {
  const int64_t nb = num_blocks(n);
  int64_t bi, bj;
  block_pair_decode(t >> 1, nb, bi, bj);
  const int64_t ii = bi * kBlockDist + (t & 1) * 8 + (lane >> 4);
  const int64_t jj = bj * kBlockDist + (lane & 15);
  i = (int)ii;
  j = (int)jj;
  return ii < jj && jj < n;
}

// Where pairs come from: an explicit (pair_i, pair_j) list, or consecutive tile slots.
struct PairSource {
  const int32_t* pi;   // explicit mode when non-null
  const int32_t* pj;
  int64_t n_slots;     // explicit: n_pairs; tile mode: (tile_end - tile_begin) * 128
  int64_t tile_begin;  // tile mode
  int64_t n_dist;
  // Bucketed pair lists (asot_pairs_bucket.cu; both stay on the device, no host sync):
  const int32_t* units = nullptr;   // tile mode: the tiles (1-SM kernels) / block pairs (CTA-pair
                                    // kernels) to run, in this order, instead of a tile range
  const int64_t* n_dev = nullptr;   // device count: of `units`, or of the explicit list's entries
                                    // (an upper bound of either is the host-side size)
};

__device__ inline bool decode_slot(const PairSource& ps, int64_t s, int& i, int& j) {
  if (s >= ps.n_slots) return false;
  if (ps.pi != nullptr) {
    i = ps.pi[s];
    j = ps.pj[s];
    return i >= 0 && j >= 0 && i < ps.n_dist && j < ps.n_dist;
  }
  return tile_slot_pair(ps.tile_begin + s / kTileSlots, (int)(s % kTileSlots), ps.n_dist, i, j);
}

// Where results go.
struct PairSink {
  float* vec;     // [n_slots] or null
  float* mat;     // [n_dist, n_dist] or null (both triangles written)
  int64_t n_dist;
  uint32_t* status;
  int32_t list;   // explicit pair list: an invalid entry is an argument error, not tile padding
  const int32_t* idx = nullptr;   // slot s is stored at vec[idx[s]] (a compacted sub-list)
  // small-support path (asot_sinkhorn_sparse.cu): a dense kernel returns at once unless
  // *dense_if != 0 (a support above kSparseCap); null = always run
  const uint32_t* dense_if = nullptr;
};
__device__ __forceinline__ bool dense_skipped(const PairSink& out) {
  return out.dense_if != nullptr && *out.dense_if == 0u;
}

// Invalid slots: tile padding (i >= j or j >= N) stores 0 in the packed vector; an explicit-list
// entry with an index outside [0, N) stores NaN and raises ASOT_FLAG_BAD_INDEX.
__device__ inline void write_result(const PairSink& out, int64_t s, bool valid, int i, int j, float d) {
  if (out.idx) s = out.idx[s];
  ASOT_DEV_CHECK(s >= 0, "result slot >= 0");
  if (valid) {
    ASOT_DEV_CHECK(i >= 0 && j >= 0 && i < out.n_dist && j < out.n_dist, "pair indices in [0, n_dist)");
    if (!isfinite(d)) atomicOr(out.status, ASOT_FLAG_NONFINITE_OUTPUT);
    if (out.vec) out.vec[s] = d;
    if (out.mat) {
      out.mat[(int64_t)i * out.n_dist + j] = d;
      out.mat[(int64_t)j * out.n_dist + i] = d;
    }
  } else if (out.list) {
    atomicOr(out.status, ASOT_FLAG_BAD_INDEX);
    if (out.vec) out.vec[s] = __int_as_float(0x7fc00000);
  } else if (out.vec) {
    out.vec[s] = 0.0f;
  }
}

// Round-to-nearest (ties away) fp32 -> TF32, returned in an fp32 container (low 13 bits zero).
__device__ __forceinline__ uint32_t tf32_rna_bits(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// Two fp32 products in one FMUL2 (Blackwell's paired fp32 pipe op, PTX mul.rn.f32x2): each lane
// is rounded exactly like a scalar FMUL, so results are bitwise those of two scalar multiplies.
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 c;
  asm("{\n\t.reg .b64 ra, rb, rc;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rc, ra, rb;\n\t"
      "mov.b64 {%0, %1}, rc;\n\t}"
      : "=f"(c.x), "=f"(c.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return c;
}

// ---- the Sinkhorn divide x = m / D with SPEC's clamp + flag (R#12).
// D is clamped into [FLT_MIN, 2^126] -- below, 1/D overflows; above, rcp.approx.ftz returns a
// flushed subnormal -- and the clamp raises DENOM_CLAMPED when the anchor carries mass (m > 0).
// A NaN D is left alone (it comes from non-finite inputs and surfaces as NONFINITE_OUTPUT).
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float div_clamped(float m, float den, bool& clamped) {
  // = m * rcp(clamp(den)) bitwise: the reciprocals of the two clamp values are exact powers of
  // two (rcp(FLT_MIN) = 2^126, rcp(2^126) = 2^-126), so the reciprocal is taken of den itself and
  // replaced by a select -- the range test runs beside the MUFU instead of in front of it
  const bool lo = !(den >= FLT_MIN) && den == den;   // 0, subnormal or negative (not NaN)
  const bool hi = den > 0x1p126f;
  float r = rcp_ftz(den);
  r = (lo || hi) ? (lo ? 0x1p126f : 0x1p-126f) : r;
  clamped |= (lo || hi) && m > 0.0f;
  return m * r;   // m = 0 -> exactly 0 (R#11)
}
// The TF32 epilogues' divide over a thread's N (multiple of 4) anchors of one chunk: o = the
// RNA-pre-rounded TF32 bits of m / D, m = 0 -> exactly 0 (R#11), one MUFU per two anchors.
// Anchors (e, e+2) and (e+1, e+3) share a reciprocal, so every product and scaling step is a
// paired f32x2 op on consecutive registers:
//   (pa, pb) = (D0 D2, D1 D3),  r = (1/pa, 1/pb),  q = (D2, D3) r = (1/D0, 1/D1),
//   (D0, D1) r = (1/D2, 1/D3),  x = m q.
// The form is exact up to rounding whenever each product lies in [2^-126, 2^126), where
// rcp.approx.ftz returns a finite normal r.  Products leave that range once max(C_s)/eps exceeds
// ~44: the fast pass accumulates t = p r (= 1 up to 2^-22 when valid; 0, inf or NaN
// otherwise) over the chunk in one FFMA2 per four anchors and reports the thread as `bad` unless
// the sum is N/2; the caller then reloads D from TMEM (not yet overwritten) in sub-blocks of 8 and
// epi_div_fix8 replaces the bad thread's values by per-anchor clamped reciprocals (S:62 clamp +
// flag).  Other threads keep their fast values, so a pair's result never depends on the other
// pairs of its warp.
__device__ __forceinline__ uint32_t tf32_rna_pre_bits(float x) { return __float_as_uint(x) + 0x1000u; }
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// NaN-propagating 3-input min / max (a NaN operand gives NaN: range checks then fail on NaN)
__device__ __forceinline__ float fmin3n(float a, float b, float c) {
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax3n(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// Four divides m / den as div_clamped, with the range test taken once for the four (and the warp):
// when every den of the warp's lanes lies in [FLT_MIN, 2^126] (the rule) x = m * rcp(den), else
// the clamped per-element form -- bitwise div_clamped either way.
__device__ __forceinline__ void div4_clamped(const float (&m)[4], const float (&d)[4], float (&x)[4],
                                             bool& clamped) {
  const float mn = fmin3n(fmin3n(d[0], d[1], d[2]), d[3], d[3]);
  const float mx = fmax3n(fmax3n(d[0], d[1], d[2]), d[3], d[3]);
  const bool bad = !(mn >= FLT_MIN && mx <= 0x1p126f);
  if (__builtin_expect(__any_sync(0xffffffffu, bad), 0)) {
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = div_clamped(m[e], d[e], clamped);
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = m[e] * rcp_ftz(d[e]);
  }
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c);
// x[e .. e+4) = m / D for one group of four anchors; t += (pa ra, pb rb)
__device__ __forceinline__ void epi_div4(const float* m, float d0, float d1, float d2, float d3, float* x, float2& t) {
  const float2 p = fmul2(make_float2(d0, d1), make_float2(d2, d3));
  const float2 r = make_float2(rcp_ftz(p.x), rcp_ftz(p.y));
  t = ffma2(p, r, t);
  const float2 x01 = fmul2(make_float2(m[0], m[1]), fmul2(make_float2(d2, d3), r));
  const float2 x23 = fmul2(make_float2(m[2], m[3]), fmul2(make_float2(d0, d1), r));
  x[0] = x01.x; x[1] = x01.y; x[2] = x23.x; x[3] = x23.y;
}
__device__ __forceinline__ bool epi_div_bad(float2 t, int n) { return !(fabsf((t.x + t.y) - 0.5f * n) < 0.25f); }
template <int N>
__device__ __forceinline__ bool epi_div_fast(const float* m, const uint32_t (&d)[N], uint32_t (&o)[N]) {
  static_assert(N % 4 == 0, "chunk");
  float2 t = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int e = 0; e < N; e += 4) {
    float x[4];
    epi_div4(m + e, __uint_as_float(d[e]), __uint_as_float(d[e + 1]), __uint_as_float(d[e + 2]),
             __uint_as_float(d[e + 3]), x, t);
#pragma unroll
    for (int k = 0; k < 4; ++k) o[e + k] = tf32_rna_pre_bits(x[k]);
  }
  return epi_div_bad(t, N);
}
__device__ __forceinline__ void epi_div_fix8(const float* m, const uint32_t (&d)[8], uint32_t* o, bool& clamped) {
#pragma unroll
  for (int e = 0; e < 8; ++e) o[e] = tf32_rna_pre_bits(div_clamped(m[e], __uint_as_float(d[e]), clamped));
}

__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  float2 c;
  asm("{\n\t.reg .b64 ra, rb, rc;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rc, ra, rb;\n\t"
      "mov.b64 {%0, %1}, rc;\n\t}"
      : "=f"(c.x), "=f"(c.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return c;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 c;
  asm("{\n\t.reg .b64 ra, rb, rc;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rc, ra, rb;\n\t"
      "mov.b64 {%0, %1}, rc;\n\t}"
      : "=f"(c.x), "=f"(c.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return c;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
      "mov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// Byte offset of element (row n, k) in the K-major SWIZZLE_128B UMMA operand image of an
// [rows x kpad] fp32 matrix: k-blocks of 32 elements (128 B) stored one after another, each
// [rows][128 B] with 8-row / 1024 B swizzle atoms (16-byte chunk index XOR row%8).
__host__ __device__ inline uint32_t sw128_kmajor_offset(uint32_t n, uint32_t k, uint32_t rows) {
  const uint32_t kb = k >> 5, kin = k & 31;
  const uint32_t lin = kb * rows * 128u + n * 128u + kin * 4u;
  return lin ^ (((lin >> 7) & 7u) << 4);
}

// Small-support Sinkhorn (asot_sinkhorn_sparse.cu, R#36): per distribution up to kSparseCap
// non-zero bins; fp32 K and K (.) C_s, the row sums of K, and the path flag.
constexpr int kSparseCap = 16;
struct SparseBufs {
  float* G = nullptr;        // [K][K] fp32 K = exp(-C_s / eps)
  float* GC = nullptr;       // [K][K] fp32 K (.) C_s
  float* R = nullptr;        // [K] row sums of K (fp64-summed)
  int32_t* cnt = nullptr;    // [n_dist] support sizes
  int32_t* perm = nullptr;   // [n_dist] the distributions ordered by support size
  uint16_t* idx = nullptr;   // [n_dist][kSparseCap] bins, increasing
  float* val = nullptr;      // [n_dist][kSparseCap] masses
  uint32_t* flag = nullptr;  // [1] != 0: some support > kSparseCap (the dense kernels run)
  int32_t* bounds = nullptr; // [4] distributions with support <= 4, 6, 8, 16 (prefixes of perm)
};
size_t sparse_bytes(int64_t n_dist, int K);
SparseBufs carve_sparse(uint8_t* base, int64_t n_dist, int K);

// ------------------------------------------------------------------------------------------
// Launchers (return cudaGetLastError() after the launch).
// ------------------------------------------------------------------------------------------
cudaError_t launch_sparse_prep(const float* H, int64_t n_dist, int K, const float* cost, float eps,
                               const SparseBufs& sp, cudaStream_t s);
// ps: a tile range, an explicit list (n_dev optional) or units of upt tiles (bucketed lists);
// max_slots: the host-side upper bound of the slots
// ordered: a tile range of the support-ordered enumeration (matrix output only)
cudaError_t launch_sinkhorn_sparse(const PairSource& ps, const PairSink& out, int K, const SparseBufs& sp, int iters,
                                   int upt, int64_t max_slots, int sms, cudaStream_t s, bool ordered = false);
cudaError_t launch_gibbs_prep(const float* cost, int K, float eps, float* G, float* GC,
                              uint32_t* g_img, uint32_t* gc_img, int kpad, cudaStream_t s);
cudaError_t launch_map_assign(const float* points, int64_t T, int dim, const float* anchors, int K,
                              int32_t* assign, uint32_t* status, cudaStream_t s,
                              const int64_t* gather = nullptr);
// the points list[0 .. *n_dev) (T = a host bound of *n_dev): assign[list[k]] (asot_map_tc.cu)
cudaError_t launch_map_assign_list(const float* points, int64_t T, int dim, const float* anchors, int K,
                                   int32_t* assign, uint32_t* status, cudaStream_t s, const int64_t* list,
                                   const int64_t* n_dev);
// a2 with the products on tcgen05 (BF16x3) and the exact kernel on the ambiguous points (R#37)
bool map_tc_supported(int dim, int K);
size_t map_tc_workspace_bytes(int64_t T, int K);
cudaError_t launch_map_tc(const float* points, int64_t T, int dim, const float* anchors, int K, int32_t* assign,
                          uint32_t* status, uint8_t* ws, int sms, cudaStream_t s);
cudaError_t launch_histograms(const int32_t* assign, const float* weights, const int64_t* offsets,
                              int64_t n_dist, int K, float* H, uint32_t* status, cudaStream_t s,
                              float* const* peers = nullptr, int n_peers = 0, int64_t row_base = 0);
int simt_kpad(int K);
size_t exact_pairs_workspace_bytes(int64_t n_pairs, int K, int sms);
cudaError_t launch_w1_points(const float* points, const int64_t* offsets, const float* weights, int64_t n_dist,
                             int dim, const int32_t* pi, const int32_t* pj, int64_t n_pairs, double* out,
                             uint32_t* status, int sms, cudaStream_t s);
cudaError_t launch_bound_terms(const float* points, const int64_t* offsets, int64_t n_dist, int dim,
                               const float* anchors, int K, const int32_t* assign, const float* cost,
                               const int32_t* pi, const int32_t* pj, int64_t n_pairs, double* l1,
                               double* linf, double* prop2, uint32_t* status, int sms, cudaStream_t s);
cudaError_t launch_exact_pairs(const float* H, int64_t n_dist, int K, const float* cost, const int32_t* pi,
                               const int32_t* pj, int64_t n_pairs, double* out, uint8_t* pending,
                               uint32_t* status, int sms, cudaStream_t s);
cudaError_t launch_gibbs_prep_simt(const float* cost, int K, float eps, float* Gp, float* GCp, cudaStream_t s);
bool sinkhorn_warp_supported(int K);
cudaError_t launch_sinkhorn_warp(const PairSource& ps, const PairSink& out, const float* H, int K,
                                 const float* Gp, const float* GCp, int iters, cudaStream_t s);
cudaError_t launch_sinkhorn_simt(const PairSource& ps, const PairSink& out, const float* H, int K,
                                 const float* G, const float* GC, int iters, cudaStream_t s);
// tcgen05 TF32 kernel, K <= 128 (images padded to kpad = roundup(K, 32)): tile mode, and the
// pair-list mode (list entries in tiles of 128; marginals from a padded copy Hp [(n_dist+1)][kpad]
// of scratch, sinkhorn_tc_pairs_scratch_bytes).
bool sinkhorn_tc_supported(int K);
// Bucketed explicit pair lists (asot_pairs_bucket.cu): units (upt = 1: tiles; 2: block pairs)
// fully covered by the list run on the tile path into R; the rest form the sub-list (li, lj, lidx).
struct PairBuckets {
  uint32_t* mask;            // [n_units * upt][4] slot bits
  int32_t* pos;              // [n_units] position in R, or -1
  unsigned long long* cnt;   // [0] units to run, [1] sub-list length
  int32_t* units;            // [cap]
  int32_t* code;             // [n_pairs] tile of the entry, or -1
  int32_t* li;
  int32_t* lj;
  int32_t* lidx;             // [n_pairs] sub-list
  float* R;                  // [cap * upt * 128]
  int64_t n_units, cap;
  int upt;
};
bool pair_bucket_supported(int64_t n_dist);
int64_t pair_bucket_cap(int64_t n_dist, int64_t n_pairs, int upt);
size_t pair_bucket_bytes(int64_t n_dist, int64_t n_pairs, int upt);
PairBuckets carve_pair_buckets(uint8_t* base, int64_t n_dist, int64_t n_pairs, int upt);
cudaError_t launch_pair_buckets(const PairBuckets& w, const int32_t* pi, const int32_t* pj, int64_t n_pairs,
                                int64_t n_dist, int sms, cudaStream_t s);
cudaError_t launch_pair_gather(const PairBuckets& w, const int32_t* pi, const int32_t* pj, int64_t n_pairs,
                               int64_t n_dist, float* dist, int sms, cudaStream_t s);
// units / n_dev (optional): run the n_dev[0] tiles units[0..) instead of [tile_begin, tile_end)
// (that range's length is then the host-side upper bound); slot p of units[k] -> vec[128 k + p].
cudaError_t launch_sinkhorn_tc(int64_t tile_begin, int64_t tile_end, int64_t n_dist,
                               const PairSink& out, const float* H, int K, const uint32_t* g_img,
                               const uint32_t* gc_img, int iters, cudaStream_t s,
                               const int32_t* units = nullptr, const int64_t* n_dev = nullptr);
size_t sinkhorn_tc_pairs_scratch_bytes(int64_t n_dist, int K);
// n_dev (optional): the list length on the device (n_pairs is then its upper bound)
cudaError_t launch_sinkhorn_tc_pairs(const int32_t* pi, const int32_t* pj, int64_t n_pairs, int64_t n_dist,
                                     const PairSink& out, const float* H, int K, const uint32_t* g_img,
                                     const uint32_t* gc_img, float* Hp, int iters, cudaStream_t s,
                                     const int64_t* n_dev = nullptr);
// tcgen05 cta_group::2 kernel for 128 < K <= 256 (tile mode; images: 2 ranks x 128 KB each).
bool sinkhorn_tc2_supported(int K);
size_t sinkhorn_tc2_image_bytes();
cudaError_t launch_gibbs_prep_tc2(const float* cost, int K, float eps, uint8_t* g_img, uint8_t* gc_img,
                                  cudaStream_t s);
// units / n_dev (optional): the n_dev[0] block pairs units[0..) (tiles 2b, 2b + 1); slot p of
// rank r of units[k] -> vec[128 (2k + r) + p].
cudaError_t launch_sinkhorn_tc2(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const float* H, int K, const uint8_t* g_img, const uint8_t* gc_img, int iters,
                                cudaStream_t s, const int32_t* units = nullptr, const int64_t* n_dev = nullptr);
// Streamed tcgen05 cta_group::2 kernel for 256 < K <= 1024 (tile mode; images 2 x 2 MB; scratch:
// padded marginals + per-CTA ping-pong X buffers).
bool sinkhorn_tc4_supported(int K);
size_t sinkhorn_tc4_image_bytes(int K);
size_t sinkhorn_tc4_scratch_bytes(int K, int64_t n_dist, int sms);
cudaError_t launch_gibbs_prep_tc4(const float* cost, int K, float eps, uint8_t* g_img, uint8_t* gc_img,
                                  cudaStream_t s);
cudaError_t launch_sinkhorn_tc4(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const float* H, int K, const uint8_t* g_img, const uint8_t* gc_img, uint8_t* scratch,
                                int iters, cudaStream_t s, const int32_t* units = nullptr,
                                const int64_t* n_dev = nullptr);
cudaError_t launch_unpack_tiles(const float* packed, int64_t n_dist, int64_t tile_begin,
                                int64_t tile_end, float* mat, cudaStream_t s);
cudaError_t launch_zero_diag(float* mat, int64_t n_dist, cudaStream_t s);
cudaError_t launch_soft_map_ml(const float* points, const int64_t* offsets, const float* weights,
                               int64_t n_dist, int dim, int K, int hidden, const float* W1,
                               const float* b1, const float* W2, const float* b2, float* H,
                               float* codes, uint32_t* status, cudaStream_t s);
cudaError_t launch_soft_map_dl(const float* points, const int64_t* offsets, const float* weights,
                               int64_t n_dist, int dim, const float* dict, int K, int n_layers,
                               int hidden, const float* V1, const float* c1, const float* v2,
                               const float* c2, float* H, float* codes, uint32_t* status,
                               cudaStream_t s);
cudaError_t launch_mahalanobis_cost(const float* anchors, int K, int d, const float* M, int h,
                                    bool normalize, float* Y, float* C, cudaStream_t s);
cudaError_t launch_normalize_by_max(float* C, int64_t n, cudaStream_t s);
bool sinkhorn_tc5_supported(int K);
size_t sinkhorn_tc5_image_bytes(int K);
size_t sinkhorn_tc5_scratch_bytes(int K, int64_t n_dist, int sms);
cudaError_t launch_gibbs_prep_tc5(const float* cost, int K, float eps, uint8_t* img, cudaStream_t s);
cudaError_t launch_sinkhorn_tc5(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const PairSource& ps, const float* H, int K, const uint8_t* img,
                                uint8_t* scratch, int iters, bool split3, cudaStream_t s);
bool sinkhorn_tc3_supported(int K);
size_t sinkhorn_tc3_image_bytes(int K);
cudaError_t launch_gibbs_prep_tc3(const float* cost, int K, float eps, uint32_t* ghi, uint32_t* glo,
                                  float* gc, cudaStream_t s);
size_t sinkhorn_tc3_pairs_scratch_bytes(int64_t n_dist, int K);
cudaError_t launch_sinkhorn_tc3_pairs(const int32_t* pi, const int32_t* pj, int64_t n_pairs, int64_t n_dist,
                                      const PairSink& out, const float* H, int K, const uint32_t* ghi,
                                      const uint32_t* glo, const float* gc, float* Hp, int iters, cudaStream_t s,
                                      const int64_t* n_dev = nullptr);
cudaError_t launch_sinkhorn_tc3(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const float* H, int K, const uint32_t* ghi, const uint32_t* glo,
                                const float* gc, int iters, cudaStream_t s, const int32_t* units = nullptr,
                                const int64_t* n_dev = nullptr);
size_t eot_slot_floats(int64_t max_n);
int eot_grid(int64_t n_pairs, int sms);
bool eot_supported(int64_t max_n);
cudaError_t launch_eot_pairs(const float* points, const int64_t* offsets, const float* weights,
                             int dim, float scale, float eps, int iters, const int32_t* pair_i,
                             const int32_t* pair_j, int64_t n_pairs, float* dist_out,
                             float* kslots, int64_t slot_floats, int grid, int max_n,
                             uint32_t* status, cudaStream_t s);
cudaError_t launch_sqeuclid_cost(const float* anchors, int K, int d, bool normalize, float* C,
                                 cudaStream_t s);
cudaError_t launch_kmeans_prepare(const double* centers, int K, int d, float* anchors, cudaStream_t s);
cudaError_t launch_kmeans_update(const float* points, int dim, const int64_t* batch_idx, int batch,
                                 const int32_t* assign, int K, double* centers, float* anchors,
                                 int64_t* counts, cudaStream_t s);

inline int kpad32(int K) { return (K + 31) & ~31; }


// Effective-clock probe (asot_profile_clock): CTA 0's thread 0 records (%clock64, %globaltimer)
// once the kernel's setup is done and again at its end; dclock / dns over the launch is the SM
// clock the kernel actually ran at (nvidia-smi samples read the requested clock, not the
// power-capped one under tensor load).
__device__ __forceinline__ void clock_probe(long long* p, int at_end) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p[2 * at_end] = clock64();
    p[2 * at_end + 1] = t;
  }
}
cudaError_t read_kernel_clock_tc(long long* host4);
cudaError_t read_kernel_clock_tc2(long long* host4);
// NEXT-1 ASOT-DL encoder with sparse codes (asot_soft_dl_sparse.cu)
bool soft_dl_sparse_supported(int dim, int K);
size_t soft_dl_sparse_workspace_bytes(int K, int sms);
bool soft_ml_tc_supported(int dim, int hidden, int K);
size_t soft_ml_tc_workspace_bytes(int dim, int hidden, int K, int sms);
cudaError_t launch_soft_ml_tc(const float* points, const int64_t* offsets, const float* weights, int64_t n_dist,
                              int dim, int hidden, int K, const float* W1, const float* b1, const float* W2,
                              const float* b2, float* H, float* codes, uint8_t* ws, uint32_t* status, int sms,
                              cudaStream_t s);
bool soft_dl_tc_supported(int dim, int K);
size_t soft_dl_tc_workspace_bytes(int dim, int K, int sms, int64_t T);
cudaError_t launch_soft_dl_tc(const float* points, const int64_t* offsets, const float* weights, int64_t n_dist, int dim,
                              const float* dict, int K, int n_layers, int hidden, const float* V1, const float* c1,
                              const float* v2, const float* c2, float* H, float* codes, uint8_t* ws, uint32_t* status,
                              int sms, int64_t T, cudaStream_t s);
cudaError_t launch_soft_dl_sparse(const float* points, const int64_t* offsets, const float* weights, int64_t n_dist,
                                  int dim, const float* dict, int K, int n_layers, int hidden, const float* V1,
                                  const float* c1, const float* v2, const float* c2, float* H, float* codes,
                                  float* zbuf, uint32_t* status, int sms, cudaStream_t s);
// BF16x3 fp32-accurate CTA-pair resident kernel (128 < K <= 256): asot_sinkhorn_tc6.cu
bool sinkhorn_tc6_supported(int K);
size_t sinkhorn_tc6_image_bytes();
cudaError_t launch_gibbs_prep_tc6(const float* cost, int K, float eps, uint8_t* g_img, uint8_t* gc_img,
                                  cudaStream_t s);
cudaError_t launch_sinkhorn_tc6(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const float* H, int K, const uint8_t* g_img, const uint8_t* gc_img, int iters,
                                cudaStream_t s, const int32_t* units = nullptr, const int64_t* n_dev = nullptr);
cudaError_t read_kernel_clock_tc6(long long* host4);
cudaError_t read_kernel_clock_tc3(long long* host4);
cudaError_t read_kernel_clock_tc4(long long* host4);
cudaError_t read_kernel_clock_tc5(long long* host4);

}  // namespace asot
