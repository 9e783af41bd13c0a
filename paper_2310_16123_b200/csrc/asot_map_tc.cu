// asot_map_tc.cu -- step a2 (one-hot nearest-anchor mapping P_o) with the
// point x anchor products on the tensor cores, the decision still the fp64 definition's (R#8, R#37).
//
// argmin_j D_pj, D_pj = |x_p - w_j|^2 = |x_p|^2 + E_pj with E_pj = A_j - 2 x_p . w_j, A_j = |w_j|^2.
// Per CTA a tile of 128 consecutive points (persistent CTAs over tiles):
//   * the tile's x split into TF32 hi + lo (x_hi = RNA_tf32(x), x_lo = x - x_hi, exact in fp32;
//     R#22's split) stored into TMEM as the A operand (point p = TMEM lane p);
//   * S = X W^T in 64-anchor chunks, `tcgen05.mma.cta_group::1.kind::tf32`, three MMAs per 8-wide
//     k-step (x_hi w_hi, x_lo w_hi, x_hi w_lo), the anchors' split images streamed by a TMA
//     producer warp, two alternating 64-column accumulators;
//   * epilogue: E = fma(-2, S, A_j) and a running (best, index, second) per thread, merged over the
//     four column groups of a point in a fixed order (lowest index on equal scores).
// Decision (R#37).  With the 3xTF32 products (the MMA reads x_lo truncated to TF32: residue
// <= 2^-21 |x|; the dropped lo x lo term <= 2^-22 |x w|; <= 3 2^-21 |x_k w_k| per coordinate) and
// fp32 accumulation (<= 3d additions, each within 2^-23 relative even when the accumulator
// truncates), |S~ - S| <= e_S sum_k |x_k w_k| <= e_S |x| |w_j|, e_S = 3 2^-21 + 3 d 2^-23; with
// A_j's fp32 rounding (gamma_d) and E's own rounding,
// |E~ - E| <= (e_S + gamma_d + 2u) (|x| + |w_j|)^2 <= B/2, B := 2 (e_S + gamma_d + 2u)(|x| + max|w|)^2
// (a further factor 2 of margin on the model).  A point whose runner-up exceeds best + 2B (+ an
// underflow slack) takes the tensor-core winner -- it is the fp64 winner; every other point is
// appended to a list that the exact CUDA-core mapping kernel (asot_map.cu: rigorous fp32 direct
// differences, fp64 where those cannot decide) resolves afterwards.
#include <cfloat>
#include <cmath>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace maptc {

using namespace ::asot::ptx;

constexpr int kTP = 128;                          // points per tile (MMA M)
constexpr int kCN = 64;                           // anchors per chunk (MMA N)
constexpr int kCompWarps = 16;
constexpr int kCT = kCompWarps * 32;
constexpr int kThreads = kCT + 64;                // + MMA warp + TMA producer warp
constexpr uint32_t kKB = 64u * 128u;              // one k-block (32 fp32) of a 64-row chunk image
constexpr uint32_t kD0 = 256;                     // accumulator columns [256, 384)
constexpr int kMaxStages = 4;

struct Args {
  const float* points;
  int64_t T;
  int dim;
  int K;
  const uint8_t* img;       // K / 64 chunks, each [hi | lo] x [d / 32 k-blocks][64 rows][128 B]
  const float* norms;       // [K] A_j = |w_j|^2 (fp32, sequential)
  const float* wmax;        // [1] max_j |w_j| rounded up
  uint32_t stage_bytes;
  int n_stages;
  int32_t* assign;
  int64_t* amb;             // ambiguous points (their global indices)
  unsigned long long* amb_cnt;
  uint32_t* status;
};


__global__ void __launch_bounds__(kThreads, 1)
map_tc_kernel(Args A) {
  constexpr uint32_t kIdesc = make_idesc_tf32(kTP, kCN);
  extern __shared__ uint8_t mt_smem_raw[];
  uint8_t* smem = mt_smem_raw + ((1024u - (smem_u32(mt_smem_raw) & 1023u)) & 1023u);
  const int d = A.dim, K = A.K, n2 = K / kCN, DKB = d / 32;
  const int kStages = A.n_stages;
  const int64_t n_tiles = (A.T + kTP - 1) / kTP;
  uint8_t* stage_base = smem;
  float* nrm = (float*)(smem + (size_t)kStages * A.stage_bytes);    // [K]
  float* xn = nrm + K;                                              // [4][kTP] |x|^2 partials
  float* tb = xn + 4 * kTP;                                         // [4][kTP] best
  float* ts = tb + 4 * kTP;                                         // [4][kTP] second
  int* ti = (int*)(ts + 4 * kTP);                                   // [4][kTP] index
  uint64_t* bars = (uint64_t*)(((uintptr_t)(ti + 4 * kTP) + 7) & ~(uintptr_t)7);
  // bars: full[4], empty[4], a, dfull[2], dfree[2] (kStages <= 4)
  const uint32_t bar_full = smem_u32(&bars[0]), bar_empty = smem_u32(&bars[4]);
  const uint32_t bar_a = smem_u32(&bars[8]);
  const uint32_t bar_dfull = smem_u32(&bars[9]), bar_dfree = smem_u32(&bars[11]);
  uint32_t* tmem_holder = (uint32_t*)&bars[13];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    mbar_init(bar_a, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_dfull + 8 * b, 1);
      mbar_init(bar_dfree + 8 * b, kCompWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  for (int j = tid; j < K; j += kThreads) nrm[j] = A.norms[j];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_holder != 0) __trap();

  if (warp == kCompWarps + 1) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x)
        for (int c = 0; c < n2; ++c, ++it) {
          const uint32_t s = it % kStages;
          if (it >= (uint32_t)kStages) mbar_wait(bar_empty + 8 * s, ((it / kStages) - 1) & 1);
          mbar_expect_tx(bar_full + 8 * s, A.stage_bytes);
          bulk_g2s(smem_u32(stage_base + (size_t)s * A.stage_bytes), A.img + (size_t)c * A.stage_bytes,
                   A.stage_bytes, bar_full + 8 * s);
        }
    }
  } else if (warp == kCompWarps) {
    // ------------------------------------------------------------------ MMA issuer
    uint32_t it = 0, tpar = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      mbar_wait(bar_a, tpar);   // the tile's x is in TMEM (and the previous tile is drained)
      tpar ^= 1u;
      tc_fence_after();
      for (int c = 0; c < n2; ++c, ++it) {
        const uint32_t s = it % kStages, db = it & 1;
        mbar_wait(bar_full + 8 * s, (it / kStages) & 1);
        if (it >= 2) mbar_wait(bar_dfree + 8 * db, ((it >> 1) - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sb = smem_u32(stage_base + (size_t)s * A.stage_bytes);
          const uint64_t bhi = make_sw128_desc(sb), blo = make_sw128_desc(sb + DKB * kKB);
          const uint32_t dcol = kD0 + kCN * db;
          for (int ks = 0; ks < d / 8; ++ks) {
            const uint64_t o = (uint64_t)(((ks >> 2) * kKB + (ks & 3) * 32) >> 4);
            mma1_tf32_ts(dcol, (uint32_t)(8 * ks), bhi + o, kIdesc, ks > 0 ? 1u : 0u);
            mma1_tf32_ts(dcol, (uint32_t)(d + 8 * ks), bhi + o, kIdesc, 1u);
            mma1_tf32_ts(dcol, (uint32_t)(8 * ks), blo + o, kIdesc, 1u);
          }
          mma1_commit(bar_empty + 8 * s);
          mma1_commit(bar_dfull + 8 * db);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------------ compute warps (0..15)
    // warp w: TMEM lane quarter q = w % 4 (point p = 32 q + lane), group g = w / 4 (a quarter of
    // the coordinates at the load, 16 of every chunk's 64 anchors in the epilogue)
    const int q = warp & 3, g = warp >> 2;
    const int p = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int dq = d / 4;
    const float u = 5.9604645e-8f;
    const float gam = (float)d * u / (1.0f - (float)d * u);
    const float eS = 3.0f * 4.76837158e-7f + 3.0f * (float)d * 1.1920929e-7f;   // 3 2^-21 + 3 d 2^-23
    const float cB = 2.0f * (eS + gam + 2.0f * u);
    const float slack = (float)(d + 2) * 4.0f * 1.1754944e-38f;
    const float wmax = *A.wmax;
    uint32_t it = 0;
    // this thread's d/4 coordinates of its point, for the tile after the current one: loaded while
    // the current tile's chunks are drained (registers; <= 8 float4 at d = 128)
    const int nq = dq / 4;
    float4 xb[8];
    auto load_x = [&](int64_t tt) {
      const bool v = tt < n_tiles && tt * kTP + p < A.T;
      const float4* xp = reinterpret_cast<const float4*>(A.points + (v ? tt * kTP + p : 0) * d + g * dq);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e < nq) xb[e] = v ? __ldg(xp + e) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    };
    load_x(blockIdx.x);
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int64_t t0 = t * kTP;
      const bool pv = t0 + p < A.T;
      named_bar_sync(1, kCT);   // the previous tile's merge is done with xn / tb / ts / ti
      {
        bool nonfinite = false;
        float n2p = 0.0f;
#pragma unroll
        for (int h = 0; h < 4; ++h) {   // 8-coordinate blocks m = g dq / 8 + h
          if (2 * h < nq) {
            const int m = ((g * dq) >> 3) + h;
            const float v[8] = {xb[2 * h].x, xb[2 * h].y, xb[2 * h].z, xb[2 * h].w,
                                xb[2 * h + 1].x, xb[2 * h + 1].y, xb[2 * h + 1].z, xb[2 * h + 1].w};
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {   // RNA to TF32 and the exact fp32 remainder
              nonfinite |= !isfinite(v[e]);
              n2p = fmaf(v[e], v[e], n2p);
              hi[e] = (__float_as_uint(v[e]) + 0x1000u) & 0xFFFFE000u;
              lo[e] = __float_as_uint(v[e] - __uint_as_float(hi[e]));
            }
            tmem_st8u(lane_off + (uint32_t)(8 * m), hi);
            tmem_st8u(lane_off + (uint32_t)(d + 8 * m), lo);
          }
        }
        load_x(t + gridDim.x);   // in flight during this tile's chunks
        if (nonfinite) atomicOr(A.status, ASOT_FLAG_NONFINITE_INPUT);
        xn[g * kTP + p] = n2p;
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(1, kCT);
        if (tid == 0) mbar_arrive_local(bar_a);
      }
      // ---- chunks: E = A_j - 2 S, the running (best, index, second) of this thread's columns
      float best = INFINITY, second = INFINITY;
      int bidx = 0x7fffffff;
      for (int c = 0; c < n2; ++c, ++it) {
        const uint32_t db = it & 1;
        mbar_wait(bar_dfull + 8 * db, (it >> 1) & 1);
        tc_fence_after();
        uint32_t r[16];
        tmem_ld16u(lane_off + kD0 + kCN * db + 16u * g, r);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar_dfree + 8 * db);
        const int j0 = c * kCN + 16 * g;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float ej = fmaf(-2.0f, __uint_as_float(r[e]), nrm[j0 + e]);   // j increasing: strict <
          if (ej < best) {
            second = best;
            best = ej;
            bidx = j0 + e;
          } else if (ej < second) {
            second = ej;
          }
        }
      }
      tb[g * kTP + p] = best;
      ts[g * kTP + p] = second;
      ti[g * kTP + p] = bidx;
      named_bar_sync(1, kCT);
      if (g == 0 && pv) {
        // merge the four groups (lowest index on equal scores), then decide
        float b = tb[p], s2 = ts[p];
        int bi = ti[p];
        float n2 = xn[p];
#pragma unroll
        for (int h = 1; h < 4; ++h) {
          const float ob = tb[h * kTP + p], os = ts[h * kTP + p];
          const int oi = ti[h * kTP + p];
          n2 += xn[h * kTP + p];
          if (ob < b || (ob == b && oi < bi)) {
            s2 = fminf(b, os);
            b = ob;
            bi = oi;
          } else {
            s2 = fminf(s2, ob);
          }
        }
        const float xr = sqrtf(n2) * (1.0f + 1.5258789e-5f) + wmax;
        const float B = cB * xr * xr * (1.0f + 1.5258789e-5f);
        if (K == 1 || s2 > b + (2.0f * B + slack)) {
          ASOT_DEV_CHECK(bi == 0x7fffffff || (bi >= 0 && bi < K), "tensor-core winner in [0, K)");
          A.assign[t0 + p] = bi;
        } else {
          const unsigned long long slot = atomicAdd(A.amb_cnt, 1ull);
          ASOT_DEV_CHECK(slot < (unsigned long long)A.T, "ambiguous list within T");
          A.amb[slot] = t0 + p;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(0u) : "memory");
}

// anchors [K, d] -> per 64-anchor chunk [hi | lo] TF32 images [d / 32 k-blocks][64 rows][128 B]
// SW128 K-major (hi = RNA_tf32(w), lo = w - hi; the MMA reads lo's TF32 truncation); A_j = |w_j|^2
// (fp32, sequential); max_j |w_j| rounded up (sqrt of the largest A_j x (1 + 2^-16)) into
// wmax[0] -- one warp per anchor row.
__global__ void map_tc_prep_kernel(const float* __restrict__ W, int K, int d, uint8_t* __restrict__ img,
                                   float* __restrict__ norms, unsigned int* __restrict__ wmax2_bits,
                                   uint32_t* __restrict__ status) {
  const int DKB = d / 32;
  const uint32_t chunk_bytes = 2u * DKB * kKB;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int n = warp; n < K; n += nw) {
    for (int k = lane; k < d; k += 32) {
      const float w = W[(int64_t)n * d + k];
      if (!isfinite(w)) atomicOr(status, ASOT_FLAG_NONFINITE_INPUT);
      const uint32_t hb = (__float_as_uint(w) + 0x1000u) & 0xFFFFE000u;
      const float lo = w - __uint_as_float(hb);
      const uint32_t c = n / kCN, r = n % kCN;
      const uint32_t lin = r * 128u + (uint32_t)(k & 31) * 4u;
      const uint32_t off = (uint32_t)(k >> 5) * kKB + (lin ^ (((lin >> 7) & 7u) << 4));
      uint8_t* base = img + (size_t)c * chunk_bytes;
      *(uint32_t*)(base + off) = hb;
      *(float*)(base + (size_t)DKB * kKB + off) = lo;
    }
    if (lane == 0) {
      float a = 0.0f;
      for (int k = 0; k < d; ++k) a = fmaf(W[(int64_t)n * d + k], W[(int64_t)n * d + k], a);
      norms[n] = a;
      atomicMax(wmax2_bits, __float_as_uint(a));
    }
  }
}

__global__ void map_tc_wmax_kernel(const unsigned int* wmax2_bits, float* wmax, unsigned long long* amb_cnt) {
  wmax[0] = sqrtf(__uint_as_float(*wmax2_bits)) * (1.0f + 1.5258789e-5f);
  *amb_cnt = 0ull;
}

}  // namespace maptc

bool map_tc_supported(int dim, int K) {
  return (dim == 32 || dim == 64 || dim == 128) && K >= 64 && K <= kMaxAnchors && K % 64 == 0;
}

size_t map_tc_workspace_bytes(int64_t T, int K) {
  // images (at d <= 128: 4 k-blocks of hi and of lo), norms, wmax bits + wmax + count, the list
  return 1024 + (size_t)(K / 64) * 2 * 4 * maptc::kKB + (size_t)K * 4 + 256 + (size_t)(T > 0 ? T : 1) * 8 + 256;
}

cudaError_t launch_map_tc(const float* points, int64_t T, int dim, const float* anchors, int K, int32_t* assign,
                          uint32_t* status, uint8_t* ws, int sms, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  using namespace maptc;
  const int DKB = dim / 32;
  const uint32_t stage_bytes = 2u * DKB * kKB;
  uint8_t* img = (uint8_t*)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
  float* norms = (float*)(img + (size_t)(K / 64) * 2 * 4 * kKB);
  unsigned int* wmax2 = (unsigned int*)(norms + K);
  float* wmax = (float*)(wmax2 + 1);
  unsigned long long* amb_cnt = (unsigned long long*)(((uintptr_t)(wmax + 1) + 7) & ~(uintptr_t)7);
  int64_t* amb = (int64_t*)(((uintptr_t)(amb_cnt + 1) + 255) & ~(uintptr_t)255);
  cudaError_t e = cudaMemsetAsync(wmax2, 0, 4, s);
  if (e != cudaSuccess) return e;
  map_tc_prep_kernel<<<(K + 7) / 8, 256, 0, s>>>(anchors, K, dim, img, norms, wmax2, status);
  map_tc_wmax_kernel<<<1, 1, 0, s>>>(wmax2, wmax, amb_cnt);
  const size_t fixed = 1024 + (size_t)K * 4 + 16 * kTP * 4 + 14 * 8 + 64;
  int n_stages = (int)((220 * 1024 - fixed) / stage_bytes);
  if (n_stages > kMaxStages) n_stages = kMaxStages;
  Args A{points, T, dim, K, img, norms, wmax, stage_bytes, n_stages, assign, amb, amb_cnt, status};
  const size_t smem = fixed + (size_t)n_stages * stage_bytes;
  e = cudaFuncSetAttribute(map_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t n_tiles = (T + kTP - 1) / kTP;
  const int grid = (int)(n_tiles < sms ? n_tiles : sms);
  map_tc_kernel<<<grid, kThreads, smem, s>>>(A);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // the ambiguous points: the exact CUDA-core mapping (rigorous fp32, fp64 where needed) over the
  // device-counted list, storing into assign[point]
  return launch_map_assign_list(points, T, dim, anchors, K, assign, status, s, amb,
                                (const int64_t*)amb_cnt);
}

}  // namespace asot
