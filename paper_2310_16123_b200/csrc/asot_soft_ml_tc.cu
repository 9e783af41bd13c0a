// asot_soft_ml_tc.cu -- SURVEY §8(f) NEXT-1 on the tensor cores: the ASOT-ML mapping (P:204
// "the outputs of the MLP for P are normalized by dividing their l1 norms"; Table 4 P:568;
// readings R#24, R#25) with both MLP layers on tcgen05.
//
//   o_p = relu(x_p W1 + b1) W2 + b2,   z_p = |o_p| / ||o_p||_1  (all-zero row: uniform, flagged),
//   H[i] = sum_{p in i} w_p z_p  in fp64 in point order (Eq. (5) P:100 with 1/n dropped, R#1).
//
// Per CTA a tile of 128 points of one distribution (persistent CTAs loop over distributions):
//   * A1 = the tile's x split into BF16 hi + lo (x_hi = RN_bf16(x), x_lo = RN_bf16(x - x_hi):
//     ~16 significant bits; R#35) stored into TMEM by the compute warps (point p = TMEM lane p;
//     per 16-wide k-step, hi in 8 columns and lo in the next 8, two values per column);
//   * GEMM 1, [128 x d] x [d x h], is `tcgen05.mma.cta_group::1.kind::f16` in 64-column output
//     chunks, three MMAs per k-step (x_hi W1_hi, x_lo W1_hi, x_hi W1_lo; the dropped lo x lo term
//     is ~2^-16 relative), fp32 accumulators D1 in TMEM;
//   * epilogue 1: relu(D1 + b1), split into BF16 hi + lo, stored back into TMEM as A2;
//   * GEMM 2, [128 x h] x [h x K], in 64-anchor chunks into two alternating TMEM accumulators, so
//     the epilogue of chunk c overlaps the MMAs of chunk c + 1, and run twice: pass A sums
//     |D2 + b2| per point (the l1 norm), pass B recomputes the chunks (tensor work is cheap; a
//     full row of K fp32 does not fit TMEM at K = 1024) and forms z = |o| / sum, the codes
//     (optional) and w_p z_p summed over the tile per anchor with a warp butterfly and a fixed-
//     order SMEM combine, added to the fp64 per-distribution sums (deterministic).
// The weight images (BF16 hi | lo, SW128 K-major, one 64-row chunk per TMA bulk copy) are built
// per call by ml_image_kernel and streamed by a producer warp through a 3-4 stage SMEM ring
// (W1 chunks, then W2 chunks, every tile).
// TMEM: A1 [0, d) then A2 [0, h); D1 [256, 256 + h) then D2 buffers [256, 320), [320, 384).
#include <cfloat>
#include <cmath>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace mltc {

using namespace ::asot::ptx;

constexpr int kTP = 128;                          // points per tile (MMA M)
constexpr int kCN = 64;                           // output columns per chunk (MMA N)
constexpr int kCompWarps = 16;
constexpr int kCT = kCompWarps * 32;
constexpr int kThreads = kCT + 64;                // + MMA warp + TMA producer warp
constexpr uint32_t kKB = 64u * 128u;              // one k-block (64 BF16) of a 64-row chunk image
constexpr uint32_t kD0 = 256;                     // first accumulator column

struct Args {
  const float* points;
  const int64_t* offsets;
  const float* weights;
  int64_t n_dist;
  int dim;
  int hidden;
  int K;
  const float* b1;
  const float* b2;
  const uint8_t* img;       // W1 chunks (h / 64) then W2 chunks (K / 64), each [hi | lo]
  int n_stages;
  uint32_t stage_bytes;
  float* H;
  float* codes;
  uint32_t* status;
};

__device__ __forceinline__ void mma1_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st4u(uint32_t taddr, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3])
               : "memory");
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float hi_elem, float lo_elem) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
  return r;
}
// values 2e (low half) and 2e + 1 (high half) of 8 consecutive ones -> packed hi and lo words
__device__ __forceinline__ void split8(const float* v, uint32_t (&hi)[4], uint32_t (&lo)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t h = cvt_bf16x2(v[2 * e + 1], v[2 * e]);
    const float r0 = v[2 * e] - __uint_as_float(h << 16);            // exact remainders
    const float r1 = v[2 * e + 1] - __uint_as_float(h & 0xFFFF0000u);
    hi[e] = h;
    lo[e] = cvt_bf16x2(r1, r0);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
soft_ml_tc_kernel(Args A) {
  constexpr uint32_t kIdesc = make_idesc_bf16(kTP, kCN);
  extern __shared__ uint8_t ml_smem_raw[];
  uint8_t* smem = ml_smem_raw + ((1024u - (smem_u32(ml_smem_raw) & 1023u)) & 1023u);
  const int d = A.dim, h = A.hidden, K = A.K;
  const int n1 = h / kCN, n2 = K / kCN, nchunks = n1 + 2 * n2;   // W1, W2 (pass A), W2 (pass B)
  const int DKB = (d + 63) / 64, HKB = h / 64;
  const int nst = A.n_stages;
  uint8_t* stage_base = smem;
  double* acc = (double*)(smem + (size_t)nst * A.stage_bytes);       // [K] fp64 bin sums
  double* msh = acc + K;                                             // [kTP] weight sums
  float* b1s = (float*)(msh + kTP);                                  // [h]
  float* b2s = b1s + h;                                              // [K]
  float* wts = b2s + K;                                              // [kTP]
  float* rs4 = wts + kTP;                                            // [4][kTP] partial row sums
  float* rinv = rs4 + 4 * kTP;                                       // [kTP] 1 / row sum (0: fallback)
  float* part = rinv + kTP;                                          // [4][K] per-quarter column sums
  uint64_t* bars = (uint64_t*)(((uintptr_t)(part + 4 * K) + 7) & ~(uintptr_t)7);
  // bars: full[4], empty[4], a1, d1, a2, dfull[2], dfree[2]
  const uint32_t bar_full = smem_u32(&bars[0]), bar_empty = smem_u32(&bars[4]);
  const uint32_t bar_a1 = smem_u32(&bars[8]), bar_d1 = smem_u32(&bars[9]), bar_a2 = smem_u32(&bars[10]);
  const uint32_t bar_dfull = smem_u32(&bars[11]), bar_dfree = smem_u32(&bars[13]);
  uint32_t* tmem_holder = (uint32_t*)&bars[15];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    mbar_init(bar_a1, 1);
    mbar_init(bar_d1, 1);
    mbar_init(bar_a2, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_dfull + 8 * b, 1);
      mbar_init(bar_dfree + 8 * b, kCompWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  for (int c = tid; c < h; c += kThreads) b1s[c] = A.b1[c];
  for (int j = tid; j < K; j += kThreads) b2s[j] = A.b2[j];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_holder != 0) __trap();

  auto n_tiles_of = [&](int64_t i) -> int { return (int)((A.offsets[i + 1] - A.offsets[i] + kTP - 1) / kTP); };

  if (warp == kCompWarps + 1) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      const uint32_t w1_bytes = 2u * DKB * kKB, w2_bytes = 2u * HKB * kKB;
      for (int64_t i = blockIdx.x; i < A.n_dist; i += gridDim.x) {
        const int nt = n_tiles_of(i);
        for (int t = 0; t < nt; ++t)
          for (int c = 0; c < nchunks; ++c, ++it) {
            const uint32_t s = it % nst;
            if (it >= (uint32_t)nst) mbar_wait(bar_empty + 8 * s, ((it / nst) - 1) & 1);
            const uint32_t bytes = c < n1 ? w1_bytes : w2_bytes;
            const uint8_t* src = c < n1 ? A.img + (size_t)c * w1_bytes
                                        : A.img + (size_t)n1 * w1_bytes + (size_t)((c - n1) % n2) * w2_bytes;
            mbar_expect_tx(bar_full + 8 * s, bytes);
            bulk_g2s(smem_u32(stage_base + (size_t)s * A.stage_bytes), src, bytes, bar_full + 8 * s);
          }
      }
    }
  } else if (warp == kCompWarps) {
    // ------------------------------------------------------------------ MMA issuer
    uint32_t it = 0, it2 = 0, tpar = 0;
    for (int64_t i = blockIdx.x; i < A.n_dist; i += gridDim.x) {
      const int nt = n_tiles_of(i);
      for (int t = 0; t < nt; ++t) {
        mbar_wait(bar_a1, tpar);   // the tile's x is in TMEM (and the previous tile is drained)
        tc_fence_after();
        for (int c = 0; c < n1; ++c, ++it) {
          const uint32_t s = it % nst;
          mbar_wait(bar_full + 8 * s, (it / nst) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sb = smem_u32(stage_base + (size_t)s * A.stage_bytes);
            const uint64_t bhi = make_sw128_desc(sb), blo = make_sw128_desc(sb + DKB * kKB);
            const uint32_t dcol = kD0 + kCN * c;
            for (int ks = 0; ks < d / 16; ++ks) {
              const uint64_t o = (uint64_t)(((ks >> 2) * kKB + (ks & 3) * 32) >> 4);
              mma1_bf16_ts(dcol, (uint32_t)(16 * ks), bhi + o, kIdesc, ks > 0 ? 1u : 0u);
              mma1_bf16_ts(dcol, (uint32_t)(16 * ks + 8), bhi + o, kIdesc, 1u);
              mma1_bf16_ts(dcol, (uint32_t)(16 * ks), blo + o, kIdesc, 1u);
            }
            mma1_commit(bar_empty + 8 * s);
            if (c == n1 - 1) mma1_commit(bar_d1);   // D1 complete (and A1 no longer read)
          }
          __syncwarp();
        }
        mbar_wait(bar_a2, tpar);   // relu(D1 + b1), split, is in TMEM as A2
        tc_fence_after();
        tpar ^= 1u;
        for (int c = 0; c < 2 * n2; ++c, ++it, ++it2) {   // pass A (row sums), pass B (codes, H)
          const uint32_t s = it % nst, db = it2 & 1;
          mbar_wait(bar_full + 8 * s, (it / nst) & 1);
          if (it2 >= 2) mbar_wait(bar_dfree + 8 * db, ((it2 >> 1) - 1) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sb = smem_u32(stage_base + (size_t)s * A.stage_bytes);
            const uint64_t bhi = make_sw128_desc(sb), blo = make_sw128_desc(sb + HKB * kKB);
            const uint32_t dcol = kD0 + kCN * db;
            for (int ks = 0; ks < h / 16; ++ks) {
              const uint64_t o = (uint64_t)(((ks >> 2) * kKB + (ks & 3) * 32) >> 4);
              mma1_bf16_ts(dcol, (uint32_t)(16 * ks), bhi + o, kIdesc, ks > 0 ? 1u : 0u);
              mma1_bf16_ts(dcol, (uint32_t)(16 * ks + 8), bhi + o, kIdesc, 1u);
              mma1_bf16_ts(dcol, (uint32_t)(16 * ks), blo + o, kIdesc, 1u);
            }
            mma1_commit(bar_empty + 8 * s);
            mma1_commit(bar_dfull + 8 * db);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ compute warps (0..15)
    // warp w: TMEM lane quarter q = w % 4 (point p = 32 q + lane), column group g = w / 4
    // (a quarter of the input dims, of the hidden units and of each 64-anchor chunk).
    const int q = warp & 3, g = warp >> 2;
    const int p = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int dq = d / 4, hq = h / 4;
    const float unif = 1.0f / (float)K;
    uint32_t it2 = 0, tpar = 0;
    for (int64_t i = blockIdx.x; i < A.n_dist; i += gridDim.x) {
      const int64_t s0 = A.offsets[i], e0 = A.offsets[i + 1];
      named_bar_sync(1, kCT);
      for (int j = tid; j < K; j += kCT) acc[j] = 0.0;
      bool nonfinite = false, negative = false;
      double msum = 0.0;
      for (int64_t t0 = s0; t0 < e0; t0 += kTP) {
        const int np = (int)min((int64_t)kTP, e0 - t0);
        const bool pv = p < np;
        named_bar_sync(1, kCT);   // the previous tile is done with wts / rinv / part
        if (g == 0) {
          const float w = pv ? A.weights[t0 + p] : 0.0f;
          if (pv) {
            nonfinite |= !isfinite(w);
            negative |= w < 0.0f;
            msum += (double)w;
          }
          wts[p] = w;
        }
        // ---- A1: this thread's d/4 input dims of point p, 8 at a time
        {
          const float* xp = A.points + (t0 + (pv ? p : 0)) * d;
          for (int m = (g * dq) >> 3; m < ((g + 1) * dq) >> 3; ++m) {
            float v[8];
            if (pv) {
              const float4 u0 = __ldg(reinterpret_cast<const float4*>(xp + 8 * m));
              const float4 u1 = __ldg(reinterpret_cast<const float4*>(xp + 8 * m + 4));
              v[0] = u0.x; v[1] = u0.y; v[2] = u0.z; v[3] = u0.w;
              v[4] = u1.x; v[5] = u1.y; v[6] = u1.z; v[7] = u1.w;
#pragma unroll
              for (int e = 0; e < 8; ++e) nonfinite |= !isfinite(v[e]);
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = 0.0f;
            }
            uint32_t hi[4], lo[4];
            split8(v, hi, lo);
            const uint32_t col = 16u * (m >> 1) + 4u * (m & 1);
            tmem_st4u(lane_off + col, hi);
            tmem_st4u(lane_off + col + 8, lo);
          }
          tmem_wait_st();
          tc_fence_before();
          named_bar_sync(1, kCT);
          if (tid == 0) mbar_arrive_local(bar_a1);
        }
        // ---- epilogue 1: A2 = split(relu(D1 + b1)), 16 hidden units (one k-step) at a time
        mbar_wait(bar_d1, tpar);
        tc_fence_after();
        for (int c = g * hq; c < (g + 1) * hq; c += 16) {
          uint32_t r[16];
          tmem_ld16u(lane_off + kD0 + (uint32_t)c, r);
          tmem_wait_ld();
          float v[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = fmaxf(__uint_as_float(r[e]) + b1s[c + e], 0.0f);
          uint32_t hi[4], lo[4];
          split8(v, hi, lo);
          tmem_st4u(lane_off + (uint32_t)c, hi);
          tmem_st4u(lane_off + (uint32_t)c + 8, lo);
          split8(v + 8, hi, lo);
          tmem_st4u(lane_off + (uint32_t)c + 4, hi);
          tmem_st4u(lane_off + (uint32_t)c + 12, lo);
        }
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(1, kCT);
        if (tid == 0) mbar_arrive_local(bar_a2);
        tpar ^= 1u;
        // ---- GEMM-2 pass A: |D2 + b2| of 16 anchors per thread and chunk -> row sums
        float rs = 0.0f;
        for (int c = 0; c < n2; ++c, ++it2) {
          const uint32_t db = it2 & 1;
          mbar_wait(bar_dfull + 8 * db, (it2 >> 1) & 1);
          tc_fence_after();
          uint32_t r[16];
          tmem_ld16u(lane_off + kD0 + kCN * db + 16u * g, r);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_local(bar_dfree + 8 * db);
          const int j0 = c * kCN + 16 * g;
#pragma unroll
          for (int e = 0; e < 16; ++e) rs += fabsf(__uint_as_float(r[e]) + b2s[j0 + e]);
        }
        rs4[g * kTP + p] = rs;
        named_bar_sync(1, kCT);
        if (g == 0) {
          const float sm = ((rs4[p] + rs4[kTP + p]) + rs4[2 * kTP + p]) + rs4[3 * kTP + p];
          rinv[p] = sm > 0.0f ? 1.0f / sm : 0.0f;
          if (pv && !(sm > 0.0f)) atomicOr(A.status, ASOT_FLAG_SOFT_FALLBACK);
        }
        named_bar_sync(1, kCT);
        // ---- GEMM-2 pass B (the same chunks recomputed): z = |o| / sum (uniform if the sum is
        // 0), the codes, and w_p z_p summed over the tile's points per anchor: a butterfly over
        // the warp's 32 points leaves lane pair (2m, 2m + 1) with anchor m of the thread's 16, the
        // four lane-quarter warps' partials meet in SMEM (fixed order, deterministic)
        const float rv = rinv[p];
        const bool fb = !(rv > 0.0f);
        const float wp = wts[p];   // 0 for padding rows
        const int bcol = 8 * ((lane >> 4) & 1) + 4 * ((lane >> 3) & 1) + 2 * ((lane >> 2) & 1) + ((lane >> 1) & 1);
        for (int c = 0; c < n2; ++c, ++it2) {
          const uint32_t db = it2 & 1;
          mbar_wait(bar_dfull + 8 * db, (it2 >> 1) & 1);
          tc_fence_after();
          uint32_t r[16];
          tmem_ld16u(lane_off + kD0 + kCN * db + 16u * g, r);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_local(bar_dfree + 8 * db);
          const int j0 = c * kCN + 16 * g;
          float v[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = fb ? unif : fabsf(__uint_as_float(r[e]) + b2s[j0 + e]) * rv;
          if (A.codes != nullptr && pv) {
            float4* zp = reinterpret_cast<float4*>(A.codes + (t0 + p) * K + j0);
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) zp[e4] = make_float4(v[4 * e4], v[4 * e4 + 1], v[4 * e4 + 2], v[4 * e4 + 3]);
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] *= wp;
#pragma unroll
          for (int w = 8; w >= 1; w >>= 1) {   // 16 -> 8 -> 4 -> 2 -> 1 values per lane
            const int o = 2 * w;               // lane offsets 16, 8, 4, 2
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int e = 0; e < w; ++e) {
              const float send = up ? v[e] : v[e + w];
              const float keep = up ? v[e + w] : v[e];
              v[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
          v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
          if ((lane & 1) == 0) part[q * K + j0 + bcol] = v[0];
        }
        named_bar_sync(1, kCT);
        for (int j = tid; j < K; j += kCT)
          acc[j] += (double)((part[j] + part[K + j]) + (part[2 * K + j] + part[3 * K + j]));
      }
      named_bar_sync(1, kCT);
      for (int j = tid; j < K; j += kCT) A.H[i * K + j] = (float)acc[j];
      // flags: every compute thread reports its own; the weight sums live in group 0
      if (nonfinite) atomicOr(A.status, ASOT_FLAG_NONFINITE_INPUT);
      if (negative) atomicOr(A.status, ASOT_FLAG_BAD_MASS);
      if (g == 0) msh[p] = msum;
      named_bar_sync(1, kCT);
      if (tid == 0) {
        double m = 0.0;
        for (int x = 0; x < kTP; ++x) m += msh[x];
        if (e0 <= s0) atomicOr(A.status, ASOT_FLAG_EMPTY_DIST);
        else if (fabs(m - 1.0) > 1e-5) atomicOr(A.status, ASOT_FLAG_BAD_MASS);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(0u) : "memory");
}

// W [rows_in, cols] row-major (W[k][n]: input k, output n) -> per 64-output chunk [hi | lo]
// images, each [kb = ceil(rows_in / 64)][64 rows n][128 B: 64 BF16 of k] SW128 K-major; k past
// rows_in is zero.  hi = RN_bf16(w), lo = RN_bf16(w - hi).
__global__ void ml_image_kernel(const float* __restrict__ W, int rows_in, int cols, uint8_t* __restrict__ img) {
  const int kb = (rows_in + 63) / 64;
  const int kpad = kb * 64;
  const uint32_t chunk_bytes = 2u * kb * kKB;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < kpad * cols; idx += gridDim.x * blockDim.x) {
    const int n = idx / kpad, k = idx % kpad;
    const float w = k < rows_in ? W[(int64_t)k * cols + n] : 0.0f;
    const uint32_t hb = cvt_bf16x2(0.0f, w) & 0xFFFFu;
    const float rem = w - __uint_as_float(hb << 16);
    const uint32_t lb = cvt_bf16x2(0.0f, rem) & 0xFFFFu;
    const uint32_t c = n / kCN, r = n % kCN;
    const uint32_t lin = r * 128u + (uint32_t)(k & 63) * 2u;
    const uint32_t off = (uint32_t)(k >> 6) * kKB + (lin ^ (((lin >> 7) & 7u) << 4));
    uint8_t* base = img + (size_t)c * chunk_bytes;
    *(uint16_t*)(base + off) = (uint16_t)hb;
    *(uint16_t*)(base + (size_t)kb * kKB + off) = (uint16_t)lb;
  }
}

struct Plan {
  uint32_t w1_bytes, w2_bytes, stage_bytes;
  size_t img_bytes, fixed_smem;
  int n_stages;
};

inline Plan plan(int dim, int hidden, int K) {
  Plan P{};
  const int DKB = (dim + 63) / 64, HKB = hidden / 64;
  P.w1_bytes = 2u * DKB * kKB;
  P.w2_bytes = 2u * HKB * kKB;
  P.stage_bytes = P.w1_bytes > P.w2_bytes ? P.w1_bytes : P.w2_bytes;
  P.img_bytes = (size_t)(hidden / kCN) * P.w1_bytes + (size_t)(K / kCN) * P.w2_bytes;
  P.fixed_smem = 1024 + (size_t)K * 8 + kTP * 8 + (size_t)(hidden + K) * 4 + 6 * kTP * 4 + (size_t)4 * K * 4 +
                 16 * 8 + 64;
  const size_t budget = 227 * 1024;
  int ns = (int)((budget - P.fixed_smem) / P.stage_bytes);
  P.n_stages = ns > 4 ? 4 : ns;
  return P;
}

}  // namespace mltc

// d in {32, 64, 128} (a 16-byte aligned point row), hidden a multiple of 64 up to 256 (TMEM: A2
// takes hidden columns, D1 hidden more), K a multiple of 64 up to 1024.
bool soft_ml_tc_supported(int dim, int hidden, int K) {
  return (dim == 32 || dim == 64 || dim == 128) && hidden >= 64 && hidden <= 256 && hidden % 64 == 0 &&
         K >= 64 && K <= 1024 && K % 64 == 0 && mltc::plan(dim, hidden, K).n_stages >= 2;
}

size_t soft_ml_tc_workspace_bytes(int dim, int hidden, int K, int sms) {
  (void)sms;
  return 1024 + mltc::plan(dim, hidden, K).img_bytes;
}

cudaError_t launch_soft_ml_tc(const float* points, const int64_t* offsets, const float* weights, int64_t n_dist,
                              int dim, int hidden, int K, const float* W1, const float* b1, const float* W2,
                              const float* b2, float* H, float* codes, uint8_t* ws, uint32_t* status, int sms,
                              cudaStream_t s) {
  const int grid = (int)(n_dist < sms ? n_dist : sms);
  if (grid < 1) return cudaSuccess;
  const mltc::Plan P = mltc::plan(dim, hidden, K);
  uint8_t* img = (uint8_t*)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
  mltc::ml_image_kernel<<<128, 256, 0, s>>>(W1, dim, hidden, img);
  mltc::ml_image_kernel<<<256, 256, 0, s>>>(W2, hidden, K, img + (size_t)(hidden / mltc::kCN) * P.w1_bytes);
  mltc::Args A{points, offsets, weights, n_dist, dim, hidden, K, b1, b2, img, P.n_stages, P.stage_bytes,
               H, codes, status};
  const size_t smem = P.fixed_smem + (size_t)P.n_stages * P.stage_bytes;
  cudaError_t e = cudaFuncSetAttribute(mltc::soft_ml_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  mltc::soft_ml_tc_kernel<<<grid, mltc::kThreads, smem, s>>>(A);
  return cudaGetLastError();
}

}  // namespace asot
