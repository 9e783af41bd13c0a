// asot_sinkhorn_sparse.cu -- a5 + a6 (batched Sinkhorn and cost) for
// marginals with small supports, on the CUDA cores in fp32.
//
// With the one-hot mapping P_o a distribution of n_i points has a histogram
// a' = Z^T a (Eq. (5)) with at most min(n_i, K) non-zero bins, and far fewer when its
// points sit near a few anchors (c3: 1-9 of 256).  Where a_r = 0 the update u = a / (K v) gives
// u_r = 0 exactly (R#11: m = 0 -> 0), and where b_c = 0, v_c = 0; a zero scaling contributes an
// exact 0 to every later product.  So after the first half-iteration (v^0 = 1 on every anchor:
// u_r = a_r / R_r with the full row sums R_r = sum_c K_rc) the whole recurrence of a pair lives on
// the |S_a| x |S_b| block of K, and the cost u^T ((K (.) C_s) v) on the same block of K (.) C_s:
// the same L iterations, the same formulas, the products with exact zeros left out (R#36).
//
// Path selection stays on the device (the call enqueues only): sparse_prep_kernel extracts each
// distribution's support (<= kCap bins, increasing anchor index) and raises flag[0] when any
// support is larger; the sparse kernel then returns at once and the dense tensor-core kernel runs
// (its PairSink.dense_if = flag), otherwise the dense kernel returns at once.
//
// Per pair (one thread): the 8 x 8 block of K (padding entries 1, padded masses 0, so padded
// scalings are exactly 0) in registers as row pairs, u as row pairs, v; each half-iteration is
// 32 FFMA2 + 8 clamped reciprocal-multiplies (div_clamped: the S:62 clamp + DENOM_CLAMPED flag of
// every fp32 kernel).  Pairs with a support of 9-16 bins take a local-memory form of the same
// recurrence (rare: c3 has one such distribution in 2000).
#include <cfloat>
#include <cmath>

#include "asot_internal.cuh"

namespace asot {
namespace sps {

constexpr int kFast = 8;        // register-resident block of the fast form
constexpr int kThreads = 128;   // one tile (8 x 16 pair slots) per CTA pass

__global__ void gibbs_rows_kernel(const float* __restrict__ cost, int K, float eps, SparseBufs sp) {
  // K = exp(-C_s / eps) and K (.) C_s in fp64, rounded to fp32 (as every Gibbs prep), and
  // the row sums R_r = sum_c K_rc of the first half-iteration (v^0 = 1) summed in fp64
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < K; r += nwarps) {
    double s = 0.0;
    for (int c = lane; c < K; c += 32) {
      const double cc = (double)cost[(int64_t)r * K + c];
      const double g = exp(-cc / (double)eps);
      sp.G[(int64_t)r * K + c] = (float)g;
      sp.GC[(int64_t)r * K + c] = (float)(g * cc);
      s += g;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sp.R[r] = (float)s;
  }
}

__global__ void support_kernel(const float* __restrict__ H, int64_t n_dist, int K, SparseBufs sp) {
  // warp per distribution: the non-zero bins (a_r != 0; NaN counts as non-zero) in increasing r
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_dist; i += nwarps) {
    int cnt = 0;
    for (int base = 0; base < K; base += 32) {
      const int r = base + lane;
      const float v = r < K ? H[i * K + r] : 0.0f;
      const bool nz = r < K && v != 0.0f;
      const uint32_t bal = __ballot_sync(0xffffffffu, nz);
      const int pos = cnt + __popc(bal & ((1u << lane) - 1u));
      if (nz && pos < kSparseCap) {
        ASOT_DEV_CHECK(r < K, "support bin < K");
        sp.idx[i * kSparseCap + pos] = (uint16_t)r;
        sp.val[i * kSparseCap + pos] = v;
      }
      cnt += __popc(bal);
    }
    if (lane == 0) {
      sp.cnt[i] = cnt;
      if (cnt > kSparseCap) atomicOr(sp.flag, 1u);
    }
  }
}

// x_e = m_e / d_e for N (even) anchors, bitwise div_clamped: the range test once for the N --
// every non-negative d lies in [FLT_MIN, 2^126] exactly when sum_e d_e rcp(d_e) = N (+- N 2^-22;
// a d outside the range gives a product of 0, inf or NaN under rcp.approx.ftz) -- then
// x = m rcp(d); otherwise the clamped per-element form (S:62 clamp + flag).
// seed: +0 when every mass of the pair is >= 0 (checked once per pair), so no denominator can be
// negative (K > 0, scalings >= 0) and the sign test is skipped; NaN otherwise (negative or NaN
// masses: a BAD_MASS input), which fails the range test, so the per-element form always runs.
// The seed starts the test's sum: one register held across the loop instead of a predicate
// the compiler re-derives from the masses at every step (predicate registers are few).
template <int N>
__device__ __forceinline__ void divn(const float* m, const float* d, float* x, bool& clamped, float seed) {
  float r[N];
#pragma unroll
  for (int e = 0; e < N; ++e) r[e] = rcp_ftz(d[e]);
  float2 t = make_float2(seed, 0.0f);
#pragma unroll
  for (int e = 0; e < N; e += 2) t = ffma2(make_float2(d[e], d[e + 1]), make_float2(r[e], r[e + 1]), t);
  if (fabsf((t.x + t.y) - (float)N) < 2e-6f) {
#pragma unroll
    for (int e = 0; e < N; e += 2) {
      const float2 q = fmul2(make_float2(m[e], m[e + 1]), make_float2(r[e], r[e + 1]));
      x[e] = q.x;
      x[e + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < N; ++e) x[e] = div_clamped(m[e], d[e], clamped);
  }
}

// The lazy form of divn: x = m rcp(d) for the N, the range test's terms summed into chk across
// the whole recurrence (no test, branch or reconvergence per step).  Every in-range d gives
// d rcp(d) = 1 +- 2^-22; an out-of-range d gives 0 (d > 2^126: the reciprocal flushes), inf or
// NaN (d < FLT_MIN, d = 0), so after S steps over n terms in all, chk = n +- 1e-3 exactly when
// every step's divn test above would have passed -- else pair_rect reruns the pair with the
// per-step tests, whose result the lazy pass then reproduces bitwise whenever it is kept.
template <int N>
__device__ __forceinline__ void divn_lazy(const float* m, const float* d, float* x, float2& chk) {
  float r[N];
#pragma unroll
  for (int e = 0; e < N; ++e) r[e] = rcp_ftz(d[e]);
#pragma unroll
  for (int e = 0; e < N; e += 2) {
    chk = ffma2(make_float2(d[e], d[e + 1]), make_float2(r[e], r[e + 1]), chk);
    const float2 q = fmul2(make_float2(m[e], m[e + 1]), make_float2(r[e], r[e + 1]));
    x[e] = q.x;
    x[e + 1] = q.y;
  }
}

// Support class of a distribution (4: <= 4 bins, 6: 5-6, 8: 7-8, 16: 9-16).  The register forms
// put the smaller class on the rows (R <= C), which makes the role deterministic: a pair of one
// class keeps its u side on the rows.
__device__ __forceinline__ int support_class(int cnt) { return cnt <= 4 ? 4 : cnt <= 6 ? 6 : cnt <= 8 ? 8 : 16; }

// The fast form: an R x C register block of K with the row distribution's <= R bins and the column
// distribution's <= C bins.  gp[q][c] = (K_{2q,c}, K_{2q+1,c}), rp[q] = the row scalings in pairs,
// cs[c] the column scalings; padding: K = 1, masses 0, so padded scalings are exactly 0.
//   row step: rows = m_row / (sum_c K_rc cs_c)   (c increasing; FFMA2 over row pairs)
//   col step: cols = m_col / (even-r partial + odd-r partial of sum_r K_rc rp_r)
// The recurrence (R#5) starts from v^0 = 1 on the v side, i.e. u^1 = a / R_u with the full row
// sums of K (R#36), then alternates v, u, ..., v.  col_u (the u side is the column distribution,
// R#10: u = the smaller original index) stores K^T's block (entry (r, c) = K[col anchor][row
// anchor]), so u = cols and v = rows; both orientations run one alternating schedule of 2L steps
// starting with a row step -- a u-on-rows pair skips step 0, a u-on-columns pair skips step
// 2L - 1 -- so a warp diverges on two steps only.  d = sum_r sum_c rp_r KC(r, c) cs_c with KC
// the same (K (.) C_s or its transpose) block.
// kLazy: the divides as divn_lazy, ok = false when the summed range test fails (the caller then
// reruns the pair with kLazy = false: per-step tests, the S:62 clamp + flag).
template <int R, int C, bool kLazy>
__device__ __forceinline__ float pair_rect_pass(int rowd, int cold, bool col_u, int K, const SparseBufs& sp,
                                                int iters, bool& clamped, bool& ok) {
  constexpr int Q = R / 2;
  const int m = sp.cnt[rowd], n = sp.cnt[cold];
  ASOT_DEV_CHECK(m <= R && n <= C, "supports fit the register form");
  const uint16_t* sr = sp.idx + (int64_t)rowd * kSparseCap;
  const uint16_t* sc = sp.idx + (int64_t)cold * kSparseCap;
  float mr[R], mc[C];
  float2 gp[Q][C];
  float2 rp[Q];
  float cs[C];
  bool nonneg = true;
  {
    int ir[R], ic[C];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ir[r] = r < m ? (int)sr[r] : 0;
      mr[r] = r < m ? sp.val[(int64_t)rowd * kSparseCap + r] : 0.0f;
      nonneg &= mr[r] >= 0.0f;
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      ic[c] = c < n ? (int)sc[c] : 0;
      mc[c] = c < n ? sp.val[(int64_t)cold * kSparseCap + c] : 0.0f;
      nonneg &= mc[c] >= 0.0f;
      cs[c] = 0.0f;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      rp[q] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const bool cv = c < n;
        const int64_t a0 = col_u ? (int64_t)ic[c] * K + ir[2 * q] : (int64_t)ir[2 * q] * K + ic[c];
        const int64_t a1 = col_u ? (int64_t)ic[c] * K + ir[2 * q + 1] : (int64_t)ir[2 * q + 1] * K + ic[c];
        gp[q][c].x = (2 * q < m && cv) ? __ldg(sp.G + a0) : 1.0f;
        gp[q][c].y = (2 * q + 1 < m && cv) ? __ldg(sp.G + a1) : 1.0f;
      }
    }
    // u^1 = a / R_u (v^0 = 1 on every anchor: (K v^0) is the full row sum)
    if (!col_u) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        rp[q].x = 2 * q < m ? div_clamped(mr[2 * q], __ldg(sp.R + ir[2 * q]), clamped) : 0.0f;
        rp[q].y = 2 * q + 1 < m ? div_clamped(mr[2 * q + 1], __ldg(sp.R + ir[2 * q + 1]), clamped) : 0.0f;
      }
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) cs[c] = c < n ? div_clamped(mc[c], __ldg(sp.R + ic[c]), clamped) : 0.0f;
    }
  }
  const float seed = nonneg ? 0.0f : __int_as_float(0x7fc00000);
  float2 chk = make_float2(seed, 0.0f);
  auto row_step = [&]() {
    float2 t[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) t[q] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int q = 0; q < Q; ++q) t[q] = ffma2(gp[q][c], make_float2(cs[c], cs[c]), t[q]);
    float den[R], x[R];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      den[2 * q] = t[q].x;
      den[2 * q + 1] = t[q].y;
    }
    if (kLazy) divn_lazy<R>(mr, den, x, chk);
    else divn<R>(mr, den, x, clamped, seed);
#pragma unroll
    for (int q = 0; q < Q; ++q) rp[q] = make_float2(x[2 * q], x[2 * q + 1]);
  };
  auto col_step = [&]() {
    float den[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float2 t = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < Q; ++q) t = ffma2(gp[q][c], rp[q], t);
      den[c] = t.x + t.y;
    }
    if (kLazy) divn_lazy<C>(mc, den, cs, chk);
    else divn<C>(mc, den, cs, clamped, seed);
  };
  // steps s = 0 .. 2L - 1: even = row step, odd = col step; u on rows: v^1 at s = 1 ... v^L at
  // s = 2L - 1 (step 0 skipped); u on columns: v^1 at s = 0 ... v^L at s = 2L - 2 (step 2L - 1
  // skipped)
  // (the two ends peeled, so the loop body carries no per-step conditions)
  if (col_u) row_step();
  for (int it = 0; it < iters - 1; ++it) {
    col_step();   // s = 2 it + 1
    row_step();   // s = 2 it + 2
  }
  if (!col_u && iters > 0) col_step();   // s = 2L - 1
  if (kLazy) {
    // terms summed: R per row step, C per column step
    const int rows = (col_u ? 1 : 0) + (iters > 1 ? iters - 1 : 0);
    const int cols = (iters > 1 ? iters - 1 : 0) + (!col_u && iters > 0 ? 1 : 0);
    ok = fabsf((chk.x + chk.y) - (float)(rows * R + cols * C)) < 0.5f;
    if (!ok) return 0.0f;
  }
  // a6: d = sum_r rp_r sum_c KC(r, c) cs_c over the block
  float d = 0.0f;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r < m) {
      const int ir = (int)sr[r];
      float t = 0.0f;
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (c < n) {
          const int icc = (int)sc[c];
          t = fmaf(__ldg(sp.GC + (col_u ? (int64_t)icc * K + ir : (int64_t)ir * K + icc)), cs[c], t);
        }
      d = fmaf((r & 1) ? rp[r >> 1].y : rp[r >> 1].x, t, d);
    }
  }
  return d;
}

template <int R, int C>
__device__ __forceinline__ float pair_rect(int rowd, int cold, bool col_u, int K, const SparseBufs& sp, int iters,
                                           bool& clamped) {
  bool ok = true;
  const float d = pair_rect_pass<R, C, true>(rowd, cold, col_u, K, sp, iters, clamped, ok);
  if (ok) return d;
  return pair_rect_pass<R, C, false>(rowd, cold, col_u, K, sp, iters, clamped, ok);
}

// (i, j): i the u side (R#10).  The row side is the smaller support class, the u side on equal
// classes -- the role rule every traversal shares, so every path computes a pair bitwise alike.
__device__ __forceinline__ void pair_roles(int i, int j, const SparseBufs& sp, int& rowd, int& cold, bool& col_u) {
  const bool swap = support_class(sp.cnt[j]) < support_class(sp.cnt[i]);
  rowd = swap ? j : i;
  cold = swap ? i : j;
  col_u = swap;
}

// Supports of 9-16 bins: the same recurrence with the block read from L1 / L2 every half-iteration.
__device__ __noinline__ float pair_slow(int i, int j, int K, const SparseBufs& sp, int iters, bool* clamped_out) {
  const int m = sp.cnt[i], n = sp.cnt[j];
  const uint16_t* ia = sp.idx + (int64_t)i * kSparseCap;
  const uint16_t* ib = sp.idx + (int64_t)j * kSparseCap;
  const float* a = sp.val + (int64_t)i * kSparseCap;
  const float* b = sp.val + (int64_t)j * kSparseCap;
  float u[kSparseCap], v[kSparseCap];
  bool clamped = false;
  for (int r = 0; r < m; ++r) u[r] = div_clamped(a[r], __ldg(sp.R + ia[r]), clamped);
  for (int it = 0; it < iters; ++it) {
    if (it > 0) {
      for (int r = 0; r < m; ++r) {
        const float* g = sp.G + (int64_t)ia[r] * K;
        float t = 0.0f;
        for (int c = 0; c < n; ++c) t = fmaf(__ldg(g + ib[c]), v[c], t);
        u[r] = div_clamped(a[r], t, clamped);
      }
    }
    for (int c = 0; c < n; ++c) {
      float t = 0.0f;
      for (int r = 0; r < m; ++r) t = fmaf(__ldg(sp.G + (int64_t)ia[r] * K + ib[c]), u[r], t);
      v[c] = div_clamped(b[c], t, clamped);
    }
  }
  float d = 0.0f;
  for (int r = 0; r < m; ++r) {
    const float* gc = sp.GC + (int64_t)ia[r] * K;
    float t = 0.0f;
    for (int c = 0; c < n; ++c) t = fmaf(__ldg(gc + ib[c]), v[c], t);
    d = fmaf(u[r], t, d);
  }
  *clamped_out |= clamped;
  return d;
}

// Supports of 9-16 bins in the support-ordered traversal: a half-warp per pair, lane r (= l % 16)
// owns row r of the 16 x 16 block (in registers) and column r's mass.  v-update: the products
// K_rc u_r of the 16 columns are reduced over the 16 rows by a butterfly (xor 8, 4, 2, 1; lane c
// ends with column c's sum); u-update: lane r sums K_rc v_c with v_c broadcast from lane c.
// Padding: K = 1, masses 0 (padded scalings exactly 0).  Returns the pair's cost on every lane.
__device__ __forceinline__ float pair_half16(int i, int j, int K, const SparseBufs& sp, int iters, bool valid,
                                             bool& clamped) {
  const int l = threadIdx.x & 15;
  const unsigned hm = (threadIdx.x & 16) ? 0xffff0000u : 0x0000ffffu;   // this half-warp
  const int m = valid ? sp.cnt[i] : 0, n = valid ? sp.cnt[j] : 0;
  const int ia = l < m ? (int)sp.idx[(int64_t)i * kSparseCap + l] : 0;
  const int ib = l < n ? (int)sp.idx[(int64_t)j * kSparseCap + l] : 0;
  const float a = l < m ? sp.val[(int64_t)i * kSparseCap + l] : 0.0f;
  const float b = l < n ? sp.val[(int64_t)j * kSparseCap + l] : 0.0f;
  float g[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int ibc = __shfl_sync(hm, ib, c, 16);
    g[c] = (l < m && c < n) ? __ldg(sp.G + (int64_t)ia * K + ibc) : 1.0f;
  }
  float u = l < m ? div_clamped(a, __ldg(sp.R + ia), clamped) : 0.0f;
  float v = 0.0f;
  for (int it = 0; it < iters; ++it) {
    if (it > 0) {
      float t = 0.0f;
#pragma unroll
      for (int c = 0; c < 16; ++c) t = fmaf(g[c], __shfl_sync(hm, v, c, 16), t);
      u = div_clamped(a, t, clamped);
    }
    float p[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) p[c] = g[c] * u;
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1) {   // 16 -> 8 -> 4 -> 2 -> 1 values per lane
      const bool up = (l & w) != 0;
#pragma unroll
      for (int e = 0; e < w; ++e) {
        const float send = up ? p[e] : p[e + w];
        const float keep = up ? p[e + w] : p[e];
        p[e] = keep + __shfl_xor_sync(hm, send, w, 16);
      }
    }
    v = div_clamped(b, p[0], clamped);   // lane l holds column l's sum
  }
  // a6: sum_r u_r sum_c (K (.) C_s)_rc v_c
  float t = 0.0f;
  const float* gc = sp.GC + (int64_t)ia * K;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int ibc = __shfl_sync(hm, ib, c, 16);
    const float vc = __shfl_sync(hm, v, c, 16);
    if (l < m && c < n) t = fmaf(__ldg(gc + ibc), vc, t);
  }
  float d = l < m ? u * t : 0.0f;
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) d += __shfl_xor_sync(hm, d, o, 16);
  return d;
}

// Slot s of the source: a tile range, an explicit list, or (bucketed lists) units of upt tiles.
__device__ __forceinline__ bool sparse_slot(const PairSource& ps, int upt, int64_t s, int& i, int& j) {
  if (ps.units != nullptr && ps.pi == nullptr) {
    const int64_t q = s / kTileSlots, k = q / upt;
    const int r = (int)(q % upt);
    const int64_t t = upt == 1 ? (int64_t)ps.units[k] : 2 * (int64_t)ps.units[k] + r;
    return tile_slot_pair(t, (int)(s % kTileSlots), ps.n_dist, i, j);
  }
  return decode_slot(ps, s, i, j);
}

// Whole triangle in support order: slot s enumerates the tiles of the distributions ordered by
// support size (perm), so a warp's 32 pairs have nearly equal supports; the pair runs in its
// original orientation (u side = the smaller original index, R#10) and is stored at its slot of
// the original tiling (tile of (i, j), a4).
__device__ __forceinline__ bool sorted_slot(const SparseBufs& sp, int64_t n_dist, int64_t tile_begin, int64_t s,
                                            int& i, int& j, int64_t& s_out) {
  int ip, jp;
  if (!tile_slot_pair(tile_begin + s / kTileSlots, (int)(s % kTileSlots), n_dist, ip, jp)) return false;
  i = sp.perm[ip];
  j = sp.perm[jp];
  if (i > j) {
    const int t = i;
    i = j;
    j = t;
  }
  const int64_t nb = num_blocks(n_dist), bi = i / kBlockDist, bj = j / kBlockDist;
  const int64_t b = bi * nb - bi * (bi - 1) / 2 + (bj - bi);   // row-major over bi <= bj (a4)
  const int h = (i % kBlockDist) >> 3;
  s_out = (2 * b + h) * kTileSlots + (((i & 7) << 4) | (j % kBlockDist));
  return true;
}

__global__ void __launch_bounds__(kThreads, 4)
sinkhorn_sparse_kernel(PairSource ps, PairSink out, int K, SparseBufs sp, int iters, int upt, int sorted) {
  if (*sp.flag != 0u) return;   // a support above kSparseCap: the dense kernel runs this call
  int64_t n = ps.n_slots;
  if (ps.units != nullptr && ps.pi == nullptr) n = *ps.n_dev * upt * kTileSlots;
  else if (ps.n_dev != nullptr && *ps.n_dev < n) n = *ps.n_dev;
  bool clamped = false;
  for (int64_t s0 = (int64_t)blockIdx.x * kThreads; s0 < n; s0 += (int64_t)gridDim.x * kThreads) {
    const int64_t s = s0 + threadIdx.x;
    int i = 0, j = 0;
    int64_t s_out = s;
    bool valid = false;
    if (s < n) valid = sorted ? sorted_slot(sp, ps.n_dist, ps.tile_begin, s, i, j, s_out) : sparse_slot(ps, upt, s, i, j);
    const int m = valid ? sp.cnt[i] : 0, nn = valid ? sp.cnt[j] : 0;
    const bool slow = m > kFast || nn > kFast;
    // the warp's largest support picks the register form (warp-uniform)
    const unsigned smax = __reduce_max_sync(0xffffffffu, slow ? 0u : (unsigned)(m > nn ? m : nn));
    float d = 0.0f;
    if (valid && !slow) {
      int rd, cd;
      bool cu;
      pair_roles(i, j, sp, rd, cd, cu);
      if (smax <= 4) d = pair_rect<4, 4>(rd, cd, cu, K, sp, iters, clamped);
      else if (smax <= 6) d = pair_rect<6, 6>(rd, cd, cu, K, sp, iters, clamped);
      else d = pair_rect<8, 8>(rd, cd, cu, K, sp, iters, clamped);
    } else if (valid) {
      d = pair_slow(i, j, K, sp, iters, &clamped);
    }
    if (s < n && (valid || !sorted)) write_result(out, s_out, valid, i, j, d);
  }
  if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
}

// The whole triangle (or a part of it) in support order, one kernel per support class.  Pairs of
// the distributions in support order, enumerated column-major (k -> j' = the largest with
// j'(j'-1)/2 <= k, i' = k - j'(j'-1)/2, i' < j'): since supp(perm[i']) <= supp(perm[j']), the
// column alone fixes the class, so each class is one contiguous range of k and its kernel runs
// one register form (S = 4, 6, 8; 0 = the 9-16 form) at the occupancy that form allows; a warp's
// 32 consecutive k share (mostly) one column.  Each pair keeps its orientation (u side = the
// smaller original index, R#10) and lands at (i, j) of the matrix; [k_lo, k_hi) bounds the part.
// The columns of 9-16 bins (every row before them): a half-warp per pair.
template <int S>
__global__ void __launch_bounds__(kThreads, 2)
sinkhorn_sparse_class_kernel(int64_t n_dist, PairSink out, int K, SparseBufs sp, int iters, int64_t k_lo,
                             int64_t k_hi) {
  static_assert(S == 0, "the 9-16 bin form");
  if (*sp.flag != 0u) return;
  const int64_t c0 = sp.bounds[2], c1 = sp.bounds[3];
  int64_t a = c0 * (c0 - 1) / 2, b = c1 * (c1 - 1) / 2;
  if (a < k_lo) a = k_lo;
  if (b > k_hi) b = k_hi;
  bool clamped = false;
  {
    // a half-warp per pair (warp-synchronous: both halves loop the same number of times)
    const int64_t hw = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 4, nhw = ((int64_t)gridDim.x * kThreads) >> 4;
    for (int64_t k0 = a + (hw & ~(int64_t)1); k0 < b; k0 += nhw) {
      const int64_t k = k0 + (hw & 1);
      const bool valid = k < b;
      int i = 0, j = 0;
      if (valid) {
        int64_t jp = (int64_t)((1.0 + sqrt(1.0 + 8.0 * (double)k)) * 0.5);
        while (jp * (jp - 1) / 2 > k) --jp;
        while ((jp + 1) * jp / 2 <= k) ++jp;
        const int64_t ip = k - jp * (jp - 1) / 2;
        i = sp.perm[ip];
        j = sp.perm[jp];
        if (i > j) {
          const int t = i;
          i = j;
          j = t;
        }
      }
      const float d = pair_half16(i, j, K, sp, iters, valid, clamped);
      if (valid && (threadIdx.x & 15) == 0) write_result(out, 0, true, i, j, d);
    }
    if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
    return;
  }
}

// Rows of support class R x columns of class C (R <= C) of the support-ordered pairs: the row
// distributions perm[r0, r1), the columns perm[c0, c1) (classes are contiguous in perm).  R < C:
// the full rectangle, enumerated column by column; R = C: the triangle i' < j' inside the class.
// Pairs outside the part [k_lo, k_hi) of the column-major enumeration (k = j'(j'-1)/2 + i') are
// skipped; the local range is cut to the part's columns first.
template <int R, int C>
__global__ void __launch_bounds__(kThreads, R * C <= 16 ? 8 : R * C <= 24 ? 7 : R * C < 48 ? 5 : 4)
sinkhorn_sparse_rect_kernel(int64_t n_dist, PairSink out, int K, SparseBufs sp, int iters, int64_t k_lo,
                            int64_t k_hi) {
  if (*sp.flag != 0u) return;
  constexpr int rc = R == 4 ? 0 : R == 6 ? 1 : 2, cc = C == 4 ? 0 : C == 6 ? 1 : 2;
  const int64_t r0 = rc == 0 ? 0 : sp.bounds[rc - 1], r1 = sp.bounds[rc];
  const int64_t c0 = cc == 0 ? 0 : sp.bounds[cc - 1], c1 = sp.bounds[cc];
  if (r1 <= r0 || c1 <= c0 || k_hi <= k_lo) return;
  auto col_of = [](int64_t k) {   // the column j' of column-major pair index k
    int64_t jp = (int64_t)((1.0 + sqrt(1.0 + 8.0 * (double)k)) * 0.5);
    while (jp * (jp - 1) / 2 > k) --jp;
    while ((jp + 1) * jp / 2 <= k) ++jp;
    return jp;
  };
  const int64_t jlo = col_of(k_lo) > c0 ? col_of(k_lo) : c0;
  const int64_t jhi = col_of(k_hi - 1) + 1 < c1 ? col_of(k_hi - 1) + 1 : c1;
  if (jhi <= jlo) return;
  const int64_t nr = r1 - r0;
  const bool tri = R == C;
  const int64_t q0 = tri ? (jlo - c0) * (jlo - c0 - 1) / 2 : (jlo - c0) * nr;
  const int64_t q1 = tri ? (jhi - c0) * (jhi - c0 - 1) / 2 : (jhi - c0) * nr;
  bool clamped = false;
  for (int64_t q = q0 + (int64_t)blockIdx.x * kThreads + threadIdx.x; q < q1; q += (int64_t)gridDim.x * kThreads) {
    int64_t ip, jp;
    if (tri) {
      int64_t jj = (int64_t)((1.0 + sqrt(1.0 + 8.0 * (double)q)) * 0.5);
      while (jj * (jj - 1) / 2 > q) --jj;
      while ((jj + 1) * jj / 2 <= q) ++jj;
      jp = c0 + jj;
      ip = c0 + (q - jj * (jj - 1) / 2);
    } else {
      jp = c0 + q / nr;
      ip = r0 + q % nr;
    }
    const int64_t k = jp * (jp - 1) / 2 + ip;
    if (k < k_lo || k >= k_hi) continue;
    ASOT_DEV_CHECK(ip >= r0 && ip < r1 && jp >= c0 && jp < c1 && ip < jp, "pair inside its class block");
    const int a = sp.perm[ip], b = sp.perm[jp];
    ASOT_DEV_CHECK(a >= 0 && a < n_dist && b >= 0 && b < n_dist, "perm entries in [0, n_dist)");
    int rowd, cold;
    bool col_u;
    if (tri) {   // one class: the u side (the smaller original index) on the rows
      rowd = a < b ? a : b;
      cold = a < b ? b : a;
      col_u = false;
    } else {     // the smaller class on the rows
      rowd = a;
      cold = b;
      col_u = b < a;
    }
    const float d = pair_rect<R, C>(rowd, cold, col_u, K, sp, iters, clamped);
    write_result(out, 0, true, rowd < cold ? rowd : cold, rowd < cold ? cold : rowd, d);
  }
  if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
}

}  // namespace sps

size_t sparse_bytes(int64_t n_dist, int K) {
  const auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  return al((size_t)K * K * 4) * 2 + al((size_t)K * 4) + al((size_t)n_dist * 4) * 2 +
         al((size_t)n_dist * kSparseCap * 2) + al((size_t)n_dist * kSparseCap * 4) + al(4);
}

SparseBufs carve_sparse(uint8_t* base, int64_t n_dist, int K) {
  const auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  SparseBufs sp;
  uint8_t* p = base;
  sp.G = (float*)p; p += al((size_t)K * K * 4);
  sp.GC = (float*)p; p += al((size_t)K * K * 4);
  sp.R = (float*)p; p += al((size_t)K * 4);
  sp.cnt = (int32_t*)p; p += al((size_t)n_dist * 4);
  sp.perm = (int32_t*)p; p += al((size_t)n_dist * 4);
  sp.idx = (uint16_t*)p; p += al((size_t)n_dist * kSparseCap * 2);
  sp.val = (float*)p; p += al((size_t)n_dist * kSparseCap * 4);
  sp.flag = (uint32_t*)p;
  sp.bounds = (int32_t*)(p + 16);
  return sp;
}

namespace sps {
// perm: the distributions ordered by support size (counting sort; the order within a size is
// whatever the atomics give -- every pair's result is independent of where it runs)
__global__ void support_order_kernel(int64_t n_dist, SparseBufs sp) {
  __shared__ int hist[kSparseCap + 2];
  for (int c = threadIdx.x; c < kSparseCap + 2; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n_dist; i += blockDim.x) {
    const int c = sp.cnt[i] < kSparseCap + 1 ? sp.cnt[i] : kSparseCap + 1;
    atomicAdd(&hist[c], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int c = 0; c < kSparseCap + 2; ++c) {
      const int h = hist[c];
      hist[c] = acc;
      acc += h;
    }
    // the support classes of the class kernels: perm[0, b0) <= 4 bins, [b0, b1) 5-6, [b1, b2)
    // 7-8, [b2, b3) 9-16
    sp.bounds[0] = hist[5];
    sp.bounds[1] = hist[7];
    sp.bounds[2] = hist[9];
    sp.bounds[3] = hist[kSparseCap + 1];
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n_dist; i += blockDim.x) {
    const int c = sp.cnt[i] < kSparseCap + 1 ? sp.cnt[i] : kSparseCap + 1;
    sp.perm[atomicAdd(&hist[c], 1)] = (int32_t)i;
  }
}
}  // namespace sps

cudaError_t launch_sparse_prep(const float* H, int64_t n_dist, int K, const float* cost, float eps,
                               const SparseBufs& sp, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(sp.flag, 0, 4, s);
  if (e != cudaSuccess) return e;
  sps::gibbs_rows_kernel<<<(K + 7) / 8, 256, 0, s>>>(cost, K, eps, sp);   // a warp per row
  const int64_t blocks = (n_dist + 7) / 8 < 148 * 16 ? (n_dist + 7) / 8 : 148 * 16;
  sps::support_kernel<<<(unsigned)blocks, 256, 0, s>>>(H, n_dist, K, sp);   // a warp per distribution
  sps::support_order_kernel<<<1, 1024, 0, s>>>(n_dist, sp);
  return cudaGetLastError();
}

namespace {
// kSide non-blocking side streams with a fork event and a join event each per (host thread,
// device), created on first use and kept for the life of the thread.
constexpr int kSide = 5;
struct SideStream {
  cudaStream_t side[kSide] = {};
  cudaEvent_t fork = nullptr, join[kSide] = {};
};
SideStream& side_stream() {
  constexpr int kMaxDev = 64;
  thread_local SideStream per_dev[kMaxDev];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& ss = per_dev[dev < kMaxDev ? dev : 0];
  if (ss.fork == nullptr) {
    cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming);
    for (int i = 0; i < kSide; ++i) {
      cudaStreamCreateWithFlags(&ss.side[i], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&ss.join[i], cudaEventDisableTiming);
    }
  }
  return ss;
}
}  // namespace

cudaError_t launch_sinkhorn_sparse(const PairSource& ps, const PairSink& out, int K, const SparseBufs& sp, int iters,
                                   int upt, int64_t max_slots, int sms, cudaStream_t s, bool ordered) {
  if (max_slots <= 0) return cudaSuccess;
  int64_t blocks = (max_slots + sps::kThreads - 1) / sps::kThreads;
  if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
  // support order: the whole triangle into the matrix only (no packed slots to zero), or a part
  // of the support-ordered enumeration (asot_distance_matrix_partition): the class kernels over
  // pair range [k_lo, k_hi) = the part's share of the N(N-1)/2 pairs
  const int64_t T = num_tiles(ps.n_dist);
  const bool sorted = ps.pi == nullptr && ps.units == nullptr && out.vec == nullptr &&
                      (ordered || (ps.tile_begin == 0 && ps.n_slots == T * kTileSlots));
  if (sorted) {
    const int64_t P = ps.n_dist * (ps.n_dist - 1) / 2;
    const int64_t p0 = ps.tile_begin, p1 = ps.tile_begin + ps.n_slots / kTileSlots;
    const int64_t k_lo = T > 0 ? p0 * P / T : 0, k_hi = T > 0 ? p1 * P / T : 0;
    // Every class kernel is one wave of resident CTAs striding over its pairs: a thread runs
    // ceil or floor of (pairs / threads) latency chains, so the last round leaves part of the SM
    // idle (measured: 20-25% of each kernel's resident warp slots), and the classes with the
    // largest blocks (8 x 8, 9-16 bins; c3: 21.7 k and 2.0 k of 2 M pairs) fill a few warps per
    // SM at most.  The class kernels therefore run on side streams forked from s and joined back
    // before the call's next launch (longest chain first, the short 4 x 4 pairs on s, last): the
    // CTAs of the next class take the slots a draining class frees.  Every pair is computed by
    // the same code wherever it runs: the results do not depend on the overlap.
    SideStream& ss = side_stream();
    cudaError_t e = cudaEventRecord(ss.fork, s);
    for (int i = 0; i < kSide && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(ss.side[i], ss.fork, 0);
    if (e != cudaSuccess) return e;
    sps::sinkhorn_sparse_rect_kernel<8, 8><<<sms * 4, sps::kThreads, 0, ss.side[0]>>>(ps.n_dist, out, K, sp, iters, k_lo, k_hi);
    sps::sinkhorn_sparse_class_kernel<0><<<sms * 2, sps::kThreads, 0, ss.side[0]>>>(ps.n_dist, out, K, sp, iters, k_lo, k_hi);
    sps::sinkhorn_sparse_rect_kernel<6, 8><<<sms * 4, sps::kThreads, 0, ss.side[1]>>>(ps.n_dist, out, K, sp, iters, k_lo, k_hi);
    sps::sinkhorn_sparse_rect_kernel<6, 6><<<sms * 5, sps::kThreads, 0, ss.side[2]>>>(ps.n_dist, out, K, sp, iters, k_lo, k_hi);
    sps::sinkhorn_sparse_rect_kernel<4, 8><<<sms * 5, sps::kThreads, 0, ss.side[3]>>>(ps.n_dist, out, K, sp, iters, k_lo, k_hi);
    sps::sinkhorn_sparse_rect_kernel<4, 6><<<sms * 7, sps::kThreads, 0, ss.side[4]>>>(ps.n_dist, out, K, sp, iters, k_lo, k_hi);
    sps::sinkhorn_sparse_rect_kernel<4, 4><<<sms * 8, sps::kThreads, 0, s>>>(ps.n_dist, out, K, sp, iters, k_lo, k_hi);
    e = cudaGetLastError();
    for (int i = 0; i < kSide && e == cudaSuccess; ++i) {
      e = cudaEventRecord(ss.join[i], ss.side[i]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ss.join[i], 0);
    }
    return e;
  }
  sps::sinkhorn_sparse_kernel<<<(unsigned)blocks, sps::kThreads, 0, s>>>(ps, out, K, sp, iters, upt, 0);
  return cudaGetLastError();
}

}  // namespace asot
