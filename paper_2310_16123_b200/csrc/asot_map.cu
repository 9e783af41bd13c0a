// asot_map.cu -- steps a1 (Gibbs kernel), a2 (one-hot nearest-anchor mapping) and a3 (mapped
// marginal histograms) for sm_100a.
//
// a2 (P:214 one-hot P_o; "P_o is the clustering operator"; S:378 argmin, lowest index on
// ties).  The decision must be bit-exact against the fp64 definition (reading R#8):
// D_pj = sum_k (x_pk - w_jk)^2 accumulated sequentially in k in fp64 with every op rounded.
// Kernel: a point x anchor distance tile.  Each point is held in registers by 4 lanes; each lane
// scans every 4th anchor of the SMEM-staged anchor chunk in fp32 (direct differences, FMA), the
// 4 lanes merge (best, index, second-best) with warp shuffles.  fp32 with a rigorous bound:
// for d non-negative rounded terms, |D32 - D| <= gamma_{d+2} D (gamma_n = n u / (1 - n u),
// u = 2^-24).  If the runner-up D32 exceeds best * (1 + 5 gamma) (+ an absolute underflow
// slack) the fp32 winner provably is the fp64 winner; otherwise the 4 lanes recompute all K
// distances with the fp64 op sequence above and take the (value, index) minimum.
//
// a3 (Eq. (5) P:100 with the 1/n factor dropped, R#1; Lemma 1 proof a' = Z^T a P:145, P:417;
// S:196).  One warp per distribution builds H[i, :] in shared memory in fp64: points are
// visited in order and the lane owning bin (j mod 32) adds w_p, so every bin is a sequential
// point-order fp64 sum, rounded once to fp32.
#include <cfloat>
#include <cmath>

#include "asot_internal.cuh"

namespace asot {

// ------------------------------------------------------------------------------ a1: Gibbs prep
__global__ void gibbs_prep_kernel(const float* __restrict__ cost, int K, float eps,
                                  float* __restrict__ G, float* __restrict__ GC,
                                  uint32_t* __restrict__ g_img, uint32_t* __restrict__ gc_img,
                                  int kpad) {
  const int64_t total = (int64_t)kpad * kpad;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(idx / kpad), k = (int)(idx % kpad);
    const bool in = n < K && k < K;
    const double c = in ? (double)cost[(int64_t)n * K + k] : 0.0;
    const double g = in ? exp(-c / (double)eps) : 0.0;  // P:183  K := exp(-C_s / eps)
    const float g32 = (float)g, gc32 = (float)(g * c);
    if (in && G != nullptr) {
      G[(int64_t)n * K + k] = g32;
      GC[(int64_t)n * K + k] = gc32;
    }
    if (g_img != nullptr) {
      // Padding (K < kpad) for the tensor-core path: K entries outside the real K x K block are
      // 1 so every denominator (K v)_r stays > 0 (padded scalings are exactly 0, so the real
      // block is untouched); K (.) C_s padding is 0 so the cost is untouched.
      const uint32_t off = sw128_kmajor_offset((uint32_t)n, (uint32_t)k, (uint32_t)kpad) >> 2;
      g_img[off] = in ? tf32_rna_bits(g32) : 0x3f800000u;
      gc_img[off] = in ? tf32_rna_bits(gc32) : 0u;
    }
  }
}

cudaError_t launch_gibbs_prep(const float* cost, int K, float eps, float* G, float* GC,
                              uint32_t* g_img, uint32_t* gc_img, int kpad, cudaStream_t s) {
  const int64_t total = (int64_t)kpad * kpad;
  const int threads = 256;
  const int blocks = (int)((total + threads - 1) / threads);
  gibbs_prep_kernel<<<blocks, threads, 0, s>>>(cost, K, eps, G, GC, g_img, gc_img, kpad);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ a2: mapping
constexpr int kMapThreads = 256;
constexpr int kLanesPerPoint = 4;
constexpr int kPointsPerBlock = kMapThreads / kLanesPerPoint;  // 64

struct BestTriple {
  float best;
  float second;
  int idx;
};

__device__ __forceinline__ void merge_triple(BestTriple& a, float ob, float os, int oi) {
  // (value, index) order for the best; second = smallest value among the rest
  if (ob < a.best || (ob == a.best && oi < a.idx)) {
    a.second = fminf(a.best, os);
    a.best = ob;
    a.idx = oi;
  } else {
    a.second = fminf(a.second, ob);
  }
}

template <int DP>
__global__ void __launch_bounds__(kMapThreads)
map_assign_kernel(const float* __restrict__ points, const int64_t* __restrict__ gather, int64_t T,
                  int dim, const float* __restrict__ anchors, int K, int chunk,
                  int32_t* __restrict__ assign, uint32_t* __restrict__ status) {
  extern __shared__ float4 map_smem4[];
  float* Ws = reinterpret_cast<float*>(map_smem4);  // [chunk][DP + 4]
  constexpr int RS = DP + 4;                        // row stride: 16-byte shift per row
  const int q = threadIdx.x & (kLanesPerPoint - 1);

  // anchors are checked for non-finite values once (block 0), not at every staging
  if (blockIdx.x == 0) {
    bool bad = false;
    for (int64_t e = threadIdx.x; e < (int64_t)K * dim; e += kMapThreads) bad |= !isfinite(anchors[e]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, ASOT_FLAG_NONFINITE_INPUT);
  }
  const bool vec = (dim % 4 == 0) && ((reinterpret_cast<uintptr_t>(anchors) & 15u) == 0);
  const bool pvec = (dim % 4 == 0) && ((reinterpret_cast<uintptr_t>(points) & 15u) == 0);
  auto stage = [&](int j0, int nc) {  // anchors [j0, j0+nc) -> Ws rows (16-byte vector loads)
    __syncthreads();
    if (vec) {
      for (int e = threadIdx.x; e < nc * (DP / 4); e += kMapThreads) {
        const int jj = e / (DP / 4), k = 4 * (e % (DP / 4));
        const float4 v = k < dim ? *reinterpret_cast<const float4*>(anchors + (int64_t)(j0 + jj) * dim + k)
                                 : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        *reinterpret_cast<float4*>(Ws + jj * RS + k) = v;
      }
    } else {
      for (int e = threadIdx.x; e < nc * DP; e += kMapThreads) {
        const int jj = e / DP, k = e % DP;
        Ws[jj * RS + k] = k < dim ? anchors[(int64_t)(j0 + jj) * dim + k] : 0.0f;
      }
    }
    __syncthreads();
  };
  const bool single = K <= chunk;   // all anchors resident: staged once for every point group
  if (single) stage(0, K);
  const int64_t n_groups = (T + kPointsPerBlock - 1) / kPointsPerBlock;
  for (int64_t g = blockIdx.x; g < n_groups; g += gridDim.x) {   // persistent over point groups
  const int64_t p = g * kPointsPerBlock + (threadIdx.x >> 2);
  const bool valid = p < T;
  // point p of this launch is row gather[p] of `points` (k-means batches) or row p
  const int64_t row = valid ? (gather ? gather[p] : p) : 0;
  float x[DP];
  bool finite = true;
  if (pvec) {   // 16-byte loads of the point row
#pragma unroll
    for (int k = 0; k < DP; k += 4) {
      const float4 v = (valid && k < dim) ? __ldg(reinterpret_cast<const float4*>(points + row * dim + k))
                                          : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      finite &= isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
      x[k] = v.x; x[k + 1] = v.y; x[k + 2] = v.z; x[k + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < DP; ++k) {
      const float v = (valid && k < dim) ? points[row * dim + k] : 0.0f;
      finite &= isfinite(v);
      x[k] = v;
    }
  }
  if (!finite) atomicOr(status, ASOT_FLAG_NONFINITE_INPUT);

  BestTriple bt{INFINITY, INFINITY, 0x7fffffff};
  for (int j0 = 0; j0 < K; j0 += chunk) {
    const int nc = min(chunk, K - j0);
    if (!single) stage(j0, nc);
    // two anchors per iteration (rows jj and jj + 4): two independent FMA chains per coordinate
    // pair, so the shared-memory loads of one row overlap the arithmetic of the other
    auto update = [&](float acc, int j) {  // j increasing per lane: strict < keeps the lowest index
      if (acc < bt.best) {
        bt.second = bt.best;
        bt.best = acc;
        bt.idx = j;
      } else if (acc < bt.second) {
        bt.second = acc;
      }
    };
    for (int jj = q; jj < nc; jj += 2 * kLanesPerPoint) {
      const bool two = jj + kLanesPerPoint < nc;
      const float4* wa = reinterpret_cast<const float4*>(Ws + jj * RS);
      const float4* wb = reinterpret_cast<const float4*>(Ws + (two ? jj + kLanesPerPoint : jj) * RS);
      // (paired f32x2 subtract / FMA: two coordinates per instruction; the bound below holds
      // for any summation order of the d non-negative rounded terms)
      float2 a01 = make_float2(0.0f, 0.0f), a23 = make_float2(0.0f, 0.0f);
      float2 b01 = make_float2(0.0f, 0.0f), b23 = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int k4 = 0; k4 < DP / 4; ++k4) {
        const float4 w = wa[k4], v = wb[k4];
        const float2 x01 = make_float2(x[4 * k4 + 0], x[4 * k4 + 1]);
        const float2 x23 = make_float2(x[4 * k4 + 2], x[4 * k4 + 3]);
        const float2 t01 = fsub2(x01, make_float2(w.x, w.y)), t23 = fsub2(x23, make_float2(w.z, w.w));
        const float2 u01 = fsub2(x01, make_float2(v.x, v.y)), u23 = fsub2(x23, make_float2(v.z, v.w));
        a01 = ffma2(t01, t01, a01);
        a23 = ffma2(t23, t23, a23);
        b01 = ffma2(u01, u01, b01);
        b23 = ffma2(u23, u23, b23);
      }
      update((a01.x + a01.y) + (a23.x + a23.y), j0 + jj);
      if (two) update((b01.x + b01.y) + (b23.x + b23.y), j0 + jj + kLanesPerPoint);
    }
  }
  // warp-shuffle argmin across the 4 lanes that share this point
#pragma unroll
  for (int off = 1; off < kLanesPerPoint; off <<= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, bt.best, off);
    const float os = __shfl_xor_sync(0xffffffffu, bt.second, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bt.idx, off);
    merge_triple(bt, ob, os, oi);
  }

  // near-tie test with the rigorous fp32 bound (gamma_{d+2}, 5x slack incl. rounding of thr)
  const float u = 5.9604645e-8f;  // 2^-24
  const float nd = (float)(dim + 2);
  const float gamma = nd * u / (1.0f - nd * u);
  const float thr = bt.best * (1.0f + 5.0f * gamma) + 1e-35f;
  const bool refine = valid && K > 1 && (bt.second <= thr);
  if (__any_sync(0xffffffffu, refine)) {
    // fp64 recomputation in the pinned op order: t = x - w; sq = t*t; acc = acc + sq (no FMA)
    double bd = INFINITY;
    int bi = 0x7fffffff;
    if (refine) {
      for (int j = q; j < K; j += kLanesPerPoint) {
        const float* wr = anchors + (int64_t)j * dim;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < DP; ++k) {
          const double w = k < dim ? (double)wr[k] : 0.0;
          const double t = __dsub_rn((double)x[k], w);
          acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
        if (acc < bd) {
          bd = acc;
          bi = j;
        }
      }
    }
#pragma unroll
    for (int off = 1; off < kLanesPerPoint; off <<= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, bd, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ob < bd || (ob == bd && oi < bi)) {
        bd = ob;
        bi = oi;
      }
    }
    if (refine) bt.idx = bi;
  }
  if (valid && q == 0) assign[p] = bt.idx;
  }  // point groups
}

template <int DP>
static cudaError_t launch_map_dp(const float* points, const int64_t* gather, int64_t T, int dim,
                                 const float* anchors, int K, int32_t* assign, uint32_t* status,
                                 cudaStream_t s) {
  const int rs_bytes = (DP + 4) * 4;
  int chunk = (96 * 1024) / rs_bytes;
  if (chunk > K) chunk = K;
  const size_t smem = (size_t)chunk * rs_bytes;
  cudaFuncSetAttribute(map_assign_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t blocks = (T + kPointsPerBlock - 1) / kPointsPerBlock;
  if (blocks == 0) return cudaSuccess;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, map_assign_kernel<DP>, kMapThreads, smem);
  if (per_sm < 1) per_sm = 1;
  if (blocks > (int64_t)sms * per_sm) blocks = (int64_t)sms * per_sm;   // persistent grid
  map_assign_kernel<DP><<<(unsigned)blocks, kMapThreads, smem, s>>>(points, gather, T, dim, anchors,
                                                                   K, chunk, assign, status);
  return cudaGetLastError();
}

cudaError_t launch_map_assign(const float* points, int64_t T, int dim, const float* anchors, int K,
                              int32_t* assign, uint32_t* status, cudaStream_t s,
                              const int64_t* gather) {
  if (dim <= 8) return launch_map_dp<8>(points, gather, T, dim, anchors, K, assign, status, s);
  if (dim <= 16) return launch_map_dp<16>(points, gather, T, dim, anchors, K, assign, status, s);
  if (dim <= 32) return launch_map_dp<32>(points, gather, T, dim, anchors, K, assign, status, s);
  if (dim <= 64) return launch_map_dp<64>(points, gather, T, dim, anchors, K, assign, status, s);
  return launch_map_dp<128>(points, gather, T, dim, anchors, K, assign, status, s);
}

// ------------------------------------------------------------------------------ a3: histograms
constexpr int kHistWarps = 4;

__global__ void __launch_bounds__(kHistWarps * 32)
histogram_kernel(const int32_t* __restrict__ assign, const float* __restrict__ weights,
                 const int64_t* __restrict__ offsets, int64_t n_dist, int K,
                 float* __restrict__ H, uint32_t* __restrict__ status,
                 float* const* __restrict__ peers, int n_peers, int64_t row_base) {
  extern __shared__ double hist_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kHistWarps + warp;
  if (i >= n_dist) return;
  double* h = hist_smem + (size_t)warp * K;
  for (int r = lane; r < K; r += 32) h[r] = 0.0;
  __syncwarp();
  const int64_t s = offsets[i], e = offsets[i + 1];
  if (lane == 0 && e <= s) atomicOr(status, ASOT_FLAG_EMPTY_DIST);
  double msum = 0.0;
  bool nonfinite = false, negative = false;
  for (int64_t p0 = s; p0 < e; p0 += 32) {
    const int64_t p = p0 + lane;
    const int a = p < e ? assign[p] : 0;
    const float w = p < e ? weights[p] : 0.0f;
    if (p < e) {
      // a point with a non-finite coordinate has no nearest anchor (assignment out of range)
      nonfinite |= !isfinite(w) || a < 0 || a >= K;
      negative |= w < 0.0f;
      msum += (double)w;
    }
    const int cnt = (e - p0) < 32 ? (int)(e - p0) : 32;
    for (int t = 0; t < cnt; ++t) {  // point order
      const int at = __shfl_sync(0xffffffffu, a, t);
      const float wt = __shfl_sync(0xffffffffu, w, t);
      if (lane == (at & 31) && at >= 0 && at < K) h[at] = h[at] + (double)wt;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) msum += __shfl_xor_sync(0xffffffffu, msum, off);
  const bool any_nonfinite = __any_sync(0xffffffffu, nonfinite);
  const bool any_negative = __any_sync(0xffffffffu, negative);
  if (any_nonfinite || any_negative) {
    if (lane == 0)
      atomicOr(status, (any_nonfinite ? ASOT_FLAG_NONFINITE_INPUT : 0u) | (any_negative ? ASOT_FLAG_BAD_MASS : 0u));
  } else if (lane == 0 && e > s && fabs(msum - 1.0) > 1e-5) {
    atomicOr(status, ASOT_FLAG_BAD_MASS);
  }
  __syncwarp();
  for (int r = lane; r < K; r += 32) {
    const float v = (float)h[r];
    H[i * K + r] = v;
    // multi-GPU: the same row straight into every rank's full H (NVLink stores into symmetric
    // memory) -- the all-gather of the mapped marginals fused into the kernel that makes them
    for (int d = 0; d < n_peers; ++d) peers[d][(row_base + i) * K + r] = v;
  }
}

cudaError_t launch_histograms(const int32_t* assign, const float* weights, const int64_t* offsets,
                              int64_t n_dist, int K, float* H, uint32_t* status, cudaStream_t s,
                              float* const* peers, int n_peers, int64_t row_base) {
  if (n_dist == 0) return cudaSuccess;
  const size_t smem = (size_t)kHistWarps * K * sizeof(double);
  cudaFuncSetAttribute(histogram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t blocks = (n_dist + kHistWarps - 1) / kHistWarps;
  histogram_kernel<<<(unsigned)blocks, kHistWarps * 32, smem, s>>>(assign, weights, offsets, n_dist,
                                                                  K, H, status, peers, n_peers, row_base);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ KN6 helpers
__global__ void unpack_tiles_kernel(const float* __restrict__ packed, int64_t n_dist,
                                    int64_t tile_begin, int64_t n_slots, float* __restrict__ mat) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_slots;
       s += (int64_t)gridDim.x * blockDim.x) {
    int i, j;
    if (tile_slot_pair(tile_begin + s / kTileSlots, (int)(s % kTileSlots), n_dist, i, j)) {
      const float d = packed[s];
      mat[(int64_t)i * n_dist + j] = d;
      mat[(int64_t)j * n_dist + i] = d;
    }
  }
}

cudaError_t launch_unpack_tiles(const float* packed, int64_t n_dist, int64_t tile_begin,
                                int64_t tile_end, float* mat, cudaStream_t s) {
  const int64_t n_slots = (tile_end - tile_begin) * kTileSlots;
  if (n_slots <= 0) return cudaSuccess;
  int64_t blocks = (n_slots + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  unpack_tiles_kernel<<<(unsigned)blocks, 256, 0, s>>>(packed, n_dist, tile_begin, n_slots, mat);
  return cudaGetLastError();
}

__global__ void zero_diag_kernel(float* mat, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    mat[i * n + i] = 0.0f;  // R#9: D[i, i] := 0, never computed
}

cudaError_t launch_zero_diag(float* mat, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  zero_diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(mat, n);
  return cudaGetLastError();
}

}  // namespace asot
