// asot_map.cu -- steps a1 (Gibbs kernel), a2 (one-hot nearest-anchor mapping) and a3 (mapped
// marginal histograms) for sm_100a.
//
// a2 (P:214 one-hot P_o; "P_o is the clustering operator"; S:378 argmin, lowest index on
// ties).  The decision must be bit-exact against the fp64 definition (reading R#8):
// D_pj = sum_k (x_pk - w_jk)^2 accumulated sequentially in k in fp64 with every op rounded.
// Kernel: a point x anchor distance tile, register-blocked (4 points x 4 anchors per thread, both
// staged in shared memory), fp32 direct differences (f32x2 FSUB / FFMA), the 16 or 32 lanes sharing a
// point merge (best, index, second-best) with warp shuffles.  fp32 with a rigorous bound:
// for d non-negative rounded terms, |D32 - D| <= gamma_{d+2} D (gamma_n = n u / (1 - n u),
// u = 2^-24), for any summation order.  If the runner-up D32 exceeds best * (1 + 5 gamma) (+ an
// absolute underflow slack) the fp32 winner provably is the fp64 winner; otherwise the lanes
// recompute all K distances with the fp64 op sequence above and take the (value, index) minimum.
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
// Point x anchor distance tile, register-blocked like a GEMM: a CTA stages a tile of 64 points
// and a chunk of anchors in shared memory (rows padded to DP + 4 floats: 16-byte vector loads,
// consecutive anchor rows 16 bytes apart in the bank space); thread (warp w, lane l) owns 4
// points and, per group of 4 LPP anchors, the 4 anchors LPP a + l % LPP (a = 0..3).  LPP = 16
// (K < 128): the points 4 (2w + l/16) + [0, 4); LPP = 32 (K >= 128): all 32 lanes share the
// points 4 (2w + pass) + [0, 4), two passes per tile, so a point float4 is one broadcast
// shared-memory wavefront for the whole warp (LPP = 16 needs two per load and leaves the loop
// bound by shared-memory wavefronts, 36 per 64 FP32 instructions, instead of the FMA pipe).  Per
// 4 coordinates a thread loads 4 point float4 and 4 anchor float4 and issues 16 x (2 FSUB2 +
// 2 FFMA2): each staged value feeds 4 distances.
// fp32 squared distances with the rigorous near-tie test of R#8, then the LPP lanes sharing a
// point merge (best, index, second) with shuffles; ambiguous points are recomputed in fp64 in the
// oracle's op order by those LPP lanes.
constexpr int kMapThreads = 256;
constexpr int kTilePoints = 64;                 // points per tile (16 groups of 4)

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

__device__ __forceinline__ uint32_t smem_u32_of(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int DP, int LPP>
__global__ void __launch_bounds__(kMapThreads, 2)
map_assign_kernel(const float* __restrict__ points, const int64_t* __restrict__ gather, int64_t T,
                  int dim, const float* __restrict__ anchors, int K, int chunk,
                  int32_t* __restrict__ assign, uint32_t* __restrict__ status,
                  const int64_t* __restrict__ T_dev, int scatter) {
  // T_dev: the list length on the device (T is then its host-side bound); scatter: results go to
  // assign[gather[k]] (the tensor-core mapping's ambiguous points) instead of assign[k]
  if (T_dev != nullptr) T = *T_dev < T ? *T_dev : T;
  extern __shared__ float4 map_smem4[];
  constexpr int RS = DP + 4;                        // row stride (floats)
  float* Xs2 = reinterpret_cast<float*>(map_smem4); // 2 x [64][RS] points: current and next tile
  float* Ws = Xs2 + (DP <= 64 ? 2 : 1) * kTilePoints * RS;   // [chunk][RS] anchors
  constexpr int kMapAnchorGroup = 4 * LPP;          // anchors per register pass
  constexpr int kPass = LPP / 16;                   // point groups per thread
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = lane % LPP;                        // anchor slot
  // point group of pass ps: points 4 pg + [0, 4)
  auto pg_of = [&](int ps) { return LPP == 16 ? 2 * warp + (lane >> 4) : 2 * warp + ps; };

  // anchors are checked for non-finite values once (block 0), not at every staging
  if (blockIdx.x == 0) {
    bool bad = false;
    for (int64_t e = threadIdx.x; e < (int64_t)K * dim; e += kMapThreads) bad |= !isfinite(anchors[e]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, ASOT_FLAG_NONFINITE_INPUT);
  }
  const bool avec = (dim % 4 == 0) && ((reinterpret_cast<uintptr_t>(anchors) & 15u) == 0);
  const bool pvec = (dim % 4 == 0) && ((reinterpret_cast<uintptr_t>(points) & 15u) == 0);
  // rows [0, n) of src (row r of src = row map(r)) -> dst rows, zero-padded to DP; 16-byte
  // loads when the source allows
  auto stage_rows = [&](float* dst, int n, int n_alloc, const float* src, bool vec, auto map) {
    if (vec) {
      for (int e = threadIdx.x; e < n_alloc * (DP / 4); e += kMapThreads) {
        const int r = e / (DP / 4), k = 4 * (e % (DP / 4));
        float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (r < n && k < dim) v = __ldg(reinterpret_cast<const float4*>(src + map(r) * dim + k));
        *reinterpret_cast<float4*>(dst + r * RS + k) = v;
      }
    } else {
      for (int e = threadIdx.x; e < n_alloc * DP; e += kMapThreads) {
        const int r = e / DP, k = e % DP;
        dst[r * RS + k] = (r < n && k < dim) ? src[map(r) * dim + k] : 0.0f;
      }
    }
  };
  const int K64 = (K + kMapAnchorGroup - 1) / kMapAnchorGroup * kMapAnchorGroup;
  const bool single = K64 <= chunk;   // all anchors resident: staged once for every tile
  if (single) {
    stage_rows(Ws, K, K64, anchors, avec, [](int r) { return (int64_t)r; });
    __syncthreads();
  }
  const float u = 5.9604645e-8f;  // 2^-24
  const float nd = (float)(dim + 2);
  const float gamma = nd * u / (1.0f - nd * u);
  const int64_t n_tiles = (T + kTilePoints - 1) / kTilePoints;
  // the next tile's points are copied (cp.async, 16 B, zero-filled past the end) while this one
  // is computed; unaligned / odd-dim inputs are staged synchronously
  auto prefetch = [&](int64_t tile, float* dst) {
    const int64_t q0 = tile * kTilePoints;
    const int nq = (int)((T - q0) < kTilePoints ? (T - q0) : kTilePoints);
    for (int e = threadIdx.x; e < kTilePoints * (DP / 4); e += kMapThreads) {
      const int r = e / (DP / 4), k = 4 * (e % (DP / 4));
      const bool ok = r < nq && k < dim;
      const float* src = ok ? points + (gather ? gather[q0 + r] : q0 + r) * dim + k : points;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32_of(dst + r * RS + k)),
                   "l"(src), "r"(ok ? 16 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // (d = 128: a second point tile would cost the second CTA per SM -- staged synchronously)
  constexpr bool kDbuf = DP <= 64;
  const bool dbuf = kDbuf && pvec;
  int buf = 0;
  if (dbuf && blockIdx.x < n_tiles) prefetch(blockIdx.x, Xs2);
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {   // persistent over tiles
    const int64_t p0 = tile * kTilePoints;
    const int np = (int)((T - p0) < kTilePoints ? (T - p0) : kTilePoints);
    float* Xs = Xs2 + buf * kTilePoints * RS;
    if (dbuf) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();   // this tile landed; everyone is done with the other buffer
      if (tile + gridDim.x < n_tiles) prefetch(tile + gridDim.x, Xs2 + (buf ^ 1) * kTilePoints * RS);
    } else {
      __syncthreads();   // previous tile's readers are done with Xs
      stage_rows(Xs, np, kTilePoints, points, pvec,
                 [&](int r) { return gather ? gather[p0 + r] : p0 + r; });
      __syncthreads();
    }
    if (dbuf) buf ^= 1;
    {   // non-finite coordinates of this thread's points (each point checked by its LPP lanes)
      bool finite = true;
      for (int ps = 0; ps < kPass; ++ps)
        for (int q = 0; q < 4; ++q)
          for (int k = tx; k < DP; k += LPP) finite &= isfinite(Xs[(4 * pg_of(ps) + q) * RS + k]);
      if (!finite) atomicOr(status, ASOT_FLAG_NONFINITE_INPUT);
    }
    BestTriple bt[kPass][4];
#pragma unroll
    for (int ps = 0; ps < kPass; ++ps)
#pragma unroll
      for (int q = 0; q < 4; ++q) bt[ps][q] = BestTriple{INFINITY, INFINITY, 0x7fffffff};
    for (int j0 = 0; j0 < K; j0 += chunk) {
      const int nc = min(chunk, K - j0);
      const int nc64 = (nc + kMapAnchorGroup - 1) / kMapAnchorGroup * kMapAnchorGroup;
      if (!single) {
        __syncthreads();
        stage_rows(Ws, nc, nc64, anchors + (int64_t)j0 * dim, avec, [](int r) { return (int64_t)r; });
        __syncthreads();
      }
      for (int g0 = 0; g0 < nc64; g0 += kMapAnchorGroup)
#pragma unroll
      for (int ps = 0; ps < kPass; ++ps) {
        const float* wr = Ws + (g0 + tx) * RS;
        const float* xr = Xs + 4 * pg_of(ps) * RS;
        float2 acc[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int a = 0; a < 4; ++a) acc[q][a] = make_float2(0.0f, 0.0f);
#pragma unroll 2
        for (int k = 0; k < DP; k += 4) {
          float4 xv[4], wv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) xv[q] = *reinterpret_cast<const float4*>(xr + q * RS + k);
#pragma unroll
          for (int a = 0; a < 4; ++a) wv[a] = *reinterpret_cast<const float4*>(wr + LPP * a * RS + k);
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const float2 t01 = fsub2(make_float2(xv[q].x, xv[q].y), make_float2(wv[a].x, wv[a].y));
              const float2 t23 = fsub2(make_float2(xv[q].z, xv[q].w), make_float2(wv[a].z, wv[a].w));
              acc[q][a] = ffma2(t01, t01, acc[q][a]);
              acc[q][a] = ffma2(t23, t23, acc[q][a]);
            }
        }
        // anchors j increase along a within a lane: strict < keeps the lowest index
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int j = j0 + g0 + tx + LPP * a;
          if (j < K) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float dq = acc[q][a].x + acc[q][a].y;
              BestTriple& b = bt[ps][q];
              if (dq < b.best) {
                b.second = b.best;
                b.best = dq;
                b.idx = j;
              } else if (dq < b.second) {
                b.second = dq;
              }
            }
          }
        }
      }
    }
    // merge across the LPP lanes that share the points
#pragma unroll
    for (int ps = 0; ps < kPass; ++ps)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int off = 1; off < LPP; off <<= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, bt[ps][q].best, off);
        const float os = __shfl_xor_sync(0xffffffffu, bt[ps][q].second, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bt[ps][q].idx, off);
        merge_triple(bt[ps][q], ob, os, oi);
      }
    }
    // near-tie test with the rigorous fp32 bound (gamma_{d+2}, 5x slack incl. rounding of thr);
    // ambiguous points: fp64 recomputation in the pinned op order t = x - w; acc = acc + t*t
#pragma unroll
    for (int ps = 0; ps < kPass; ++ps)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      BestTriple& b = bt[ps][q];
      const int pl = 4 * pg_of(ps) + q;
      const bool valid = pl < np;
      const float thr = b.best * (1.0f + 5.0f * gamma) + 1e-35f;
      const bool refine = valid && K > 1 && (b.second <= thr);
      if (__any_sync(0xffffffffu, refine)) {
        double bd = INFINITY;
        int bi = 0x7fffffff;
        if (refine) {
          const float* xp = Xs + pl * RS;
          // four of the lane's anchors at a time: four independent fp64 chains, each in the
          // pinned op order (sequential in k), compared in increasing j.  The anchors come from
          // the CTA's shared-memory copy when all of them are resident (the same fp32 values:
          // an L2 round trip per coordinate had made the refine latency-bound -- it is most of
          // the work on the tensor-core mapping's ambiguous list), else from global memory.
          const float* wsrc = single ? Ws : anchors;
          const int64_t wstride = single ? RS : dim;
          for (int j0 = tx; j0 < K; j0 += 4 * LPP) {
            const float* wj[4];
            double accd[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = j0 + e * LPP;
              wj[e] = wsrc + (int64_t)(j < K ? j : j0) * wstride;
              accd[e] = 0.0;
            }
#pragma unroll 4
            for (int k = 0; k < dim; ++k) {
              const double xk = (double)xp[k];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const double t = __dsub_rn(xk, (double)wj[e][k]);
                accd[e] = __dadd_rn(accd[e], __dmul_rn(t, t));
              }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (j0 + e * LPP < K && accd[e] < bd) {
                bd = accd[e];
                bi = j0 + e * LPP;
              }
            }
          }
        }
#pragma unroll
        for (int off = 1; off < LPP; off <<= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, bd, off);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
          if (ob < bd || (ob == bd && oi < bi)) {
            bd = ob;
            bi = oi;
          }
        }
        if (refine) b.idx = bi;
      }
      if (valid && tx == 0) {
        // (0x7fffffff: a point with a non-finite coordinate has no nearest anchor -- flagged)
        ASOT_DEV_CHECK(b.idx == 0x7fffffff || (b.idx >= 0 && b.idx < K), "assignment in [0, K)");
        assign[scatter ? gather[p0 + pl] : p0 + pl] = b.idx;
      }
    }
  }  // tiles
}

template <int DP, int LPP>
static cudaError_t launch_map_dp(const float* points, const int64_t* gather, int64_t T, int dim,
                                 const float* anchors, int K, int32_t* assign, uint32_t* status,
                                 cudaStream_t s, const int64_t* T_dev = nullptr, int scatter = 0) {
  constexpr int kMapAnchorGroup = 4 * LPP;
  const int rs_bytes = (DP + 4) * 4;
  // anchor chunk: whole 64-anchor groups such that the CTA (with its one or two point tiles)
  // fits twice per SM
  constexpr int kTiles = DP <= 64 ? 2 : 1;
  int chunk = ((110 * 1024) / rs_bytes - kTiles * kTilePoints) / kMapAnchorGroup * kMapAnchorGroup;
  const int K64 = (K + kMapAnchorGroup - 1) / kMapAnchorGroup * kMapAnchorGroup;
  if (chunk > K64) chunk = K64;
  const size_t smem = (size_t)(chunk + kTiles * kTilePoints) * rs_bytes;
  cudaError_t e = cudaFuncSetAttribute(map_assign_kernel<DP, LPP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t blocks = (T + kTilePoints - 1) / kTilePoints;
  if (blocks == 0) return cudaSuccess;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, map_assign_kernel<DP, LPP>, kMapThreads, smem);
  if (per_sm < 1) per_sm = 1;
  if (blocks > (int64_t)sms * per_sm) blocks = (int64_t)sms * per_sm;   // persistent grid
  map_assign_kernel<DP, LPP><<<(unsigned)blocks, kMapThreads, smem, s>>>(points, gather, T, dim, anchors,
                                                                        K, chunk, assign, status, T_dev, scatter);
  return cudaGetLastError();
}

static cudaError_t map_dispatch(const float* points, int64_t T, int dim, const float* anchors, int K,
                                int32_t* assign, uint32_t* status, cudaStream_t s, const int64_t* gather,
                                const int64_t* T_dev, int scatter) {
  // K >= 128: 32 lanes share a thread's points (one broadcast wavefront per point load)
  if (K >= 128 && dim > 8) {
    if (dim <= 16) return launch_map_dp<16, 32>(points, gather, T, dim, anchors, K, assign, status, s, T_dev, scatter);
    if (dim <= 32) return launch_map_dp<32, 32>(points, gather, T, dim, anchors, K, assign, status, s, T_dev, scatter);
    if (dim <= 64) return launch_map_dp<64, 32>(points, gather, T, dim, anchors, K, assign, status, s, T_dev, scatter);
    return launch_map_dp<128, 32>(points, gather, T, dim, anchors, K, assign, status, s, T_dev, scatter);
  }
  if (dim <= 8) return launch_map_dp<8, 16>(points, gather, T, dim, anchors, K, assign, status, s, T_dev, scatter);
  if (dim <= 16) return launch_map_dp<16, 16>(points, gather, T, dim, anchors, K, assign, status, s, T_dev, scatter);
  if (dim <= 32) return launch_map_dp<32, 16>(points, gather, T, dim, anchors, K, assign, status, s, T_dev, scatter);
  if (dim <= 64) return launch_map_dp<64, 16>(points, gather, T, dim, anchors, K, assign, status, s, T_dev, scatter);
  return launch_map_dp<128, 16>(points, gather, T, dim, anchors, K, assign, status, s, T_dev, scatter);
}

cudaError_t launch_map_assign(const float* points, int64_t T, int dim, const float* anchors, int K,
                              int32_t* assign, uint32_t* status, cudaStream_t s,
                              const int64_t* gather) {
  return map_dispatch(points, T, dim, anchors, K, assign, status, s, gather, nullptr, 0);
}

cudaError_t launch_map_assign_list(const float* points, int64_t T, int dim, const float* anchors, int K,
                                   int32_t* assign, uint32_t* status, cudaStream_t s, const int64_t* list,
                                   const int64_t* n_dev) {
  return map_dispatch(points, T, dim, anchors, K, assign, status, s, list, n_dev, 1);
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
  // Lane l owns the bins r = l (mod 32) and keeps the running sum of the bin it touched last in
  // a register (cur, acc): the same additions in the same (point) order as h[at] += w, without a
  // shared-memory round trip per point while consecutive points of the lane share a bin (small
  // supports: almost always).
  int cur = -1;
  double acc = 0.0;
  // the next 32 points' (assignment, weight) are loaded while the current 32 are summed (the
  // weights come from HBM: one exposed load latency per distribution instead of one per batch)
  int a_next = s + lane < e ? assign[s + lane] : 0;
  float w_next = s + lane < e ? weights[s + lane] : 0.0f;
  for (int64_t p0 = s; p0 < e; p0 += 32) {
    const int64_t p = p0 + lane;
    const int a = a_next;
    const float w = w_next;
    a_next = p + 32 < e ? assign[p + 32] : 0;
    w_next = p + 32 < e ? weights[p + 32] : 0.0f;
    if (p < e) {
      // a point with a non-finite coordinate has no nearest anchor (assignment out of range)
      nonfinite |= !isfinite(w) || a < 0 || a >= K;
      negative |= w < 0.0f;
      msum += (double)w;
    }
    const int cnt = (e - p0) < 32 ? (int)(e - p0) : 32;
    if (cnt == 32) {
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {  // point order (the shuffles of later points issue early)
        const int at = __shfl_sync(0xffffffffu, a, t);
        const float wt = __shfl_sync(0xffffffffu, w, t);
        if (lane == (at & 31) && at >= 0 && at < K) {
          if (at != cur) {   // another of this lane's bins: park the held sum, fetch the new one
            if (cur >= 0) h[cur] = acc;
            cur = at;
            acc = h[at];
          }
          acc = acc + (double)wt;
        }
      }
    } else {
      for (int t = 0; t < cnt; ++t) {  // point order
        const int at = __shfl_sync(0xffffffffu, a, t);
        const float wt = __shfl_sync(0xffffffffu, w, t);
        if (lane == (at & 31) && at >= 0 && at < K) {
          if (at != cur) {   // another of this lane's bins: park the held sum, fetch the new one
            if (cur >= 0) h[cur] = acc;
            cur = at;
            acc = h[at];
          }
          acc = acc + (double)wt;
        }
      }
    }
  }
  if (cur >= 0) h[cur] = acc;
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
