// asot_eot.cu -- SURVEY §8(f) NEXT-4: the comparison baseline the paper measures ASOT against:
// entropic OT on the ORIGINAL point sets, pair by pair ("eOT (CPU)" / "BDS-eOT (GPU)" rows of
// Table 2; BDS P:78-81; one-by-one eOT), built B200-native so the speedup of the
// anchor-space formulation can be measured on the same box.
//
// Per pair (i, j): ground cost C[r][c] = s * ||x_r - y_c||^2 (R#32: the anchors' normalised
// squared-Euclidean cost, s = 1 / max C_s, so eOT and eASOT values are comparable), Gibbs kernel
// K = exp(-C / eps), v0 = 1, exactly L iterations u = a / (K v), v = b / (K^T u), cost
// <diag(u) K diag(v), C>.  Unlike ASOT, every pair has its own n_i x n_j kernel:
// this is the per-pair cost instantiation ASOT removes.
//
// Kernel: persistent CTAs of 8 warps; a work item is 8 consecutive pairs.  If all 8 have
// n_i, n_j <= 64 (the paper's graph sizes, c1/c2) each warp solves one pair with its padded K in
// SMEM and no block barriers (lane = row for u, lane = column for v); otherwise the CTA solves
// them one by one: K in SMEM when it fits the 200 KB budget, else in the CTA's workspace slot
// (L2/HBM), warp-per-row u-updates, thread-per-column v-updates.  The cost recomputes C with the
// same op order and reduces in fp64.
#include <cfloat>
#include <cmath>

#include "asot_internal.cuh"

namespace asot {
namespace eot {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSmallN = 64;                       // warp-per-pair mode: n_i, n_j <= 64
constexpr int kSmallKS = kSmallN + 1;             // padded K row stride (odd: conflict-free rows)
constexpr int kSmallFloats = kSmallN * kSmallKS + 4 * kSmallN;   // K + u, v, a, b per warp
constexpr size_t kSmemBytes = 200 * 1024;

// Squared distances of the 2 x 2 block (rows r0, r0+1 of X; rows c0, c0+1 of Y), times scale.
// Rows past nr / nc repeat the last valid row (their results are discarded).  Same per-entry op
// order everywhere (difference, then fma-accumulate in dimension order), so the cost pass
// reproduces the kernel pass's C bitwise.
__device__ __forceinline__ void cost2x2(const float* __restrict__ X, const float* __restrict__ Y, int dim,
                                        int r0, int c0, int nr, int nc, float scale, float (&o)[4]) {
  const float* x0 = X + (int64_t)r0 * dim;
  const float* x1 = X + (int64_t)min(r0 + 1, nr - 1) * dim;
  const float* y0 = Y + (int64_t)c0 * dim;
  const float* y1 = Y + (int64_t)min(c0 + 1, nc - 1) * dim;
  float a00 = 0.0f, a01 = 0.0f, a10 = 0.0f, a11 = 0.0f;
  if ((dim & 3) == 0) {
    for (int k = 0; k < dim; k += 4) {
      const float4 p0 = *reinterpret_cast<const float4*>(x0 + k), p1 = *reinterpret_cast<const float4*>(x1 + k);
      const float4 q0 = *reinterpret_cast<const float4*>(y0 + k), q1 = *reinterpret_cast<const float4*>(y1 + k);
      const float xa[2][4] = {{p0.x, p0.y, p0.z, p0.w}, {p1.x, p1.y, p1.z, p1.w}};
      const float ya[2][4] = {{q0.x, q0.y, q0.z, q0.w}, {q1.x, q1.y, q1.z, q1.w}};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float t;
        t = xa[0][e] - ya[0][e]; a00 = fmaf(t, t, a00);
        t = xa[0][e] - ya[1][e]; a01 = fmaf(t, t, a01);
        t = xa[1][e] - ya[0][e]; a10 = fmaf(t, t, a10);
        t = xa[1][e] - ya[1][e]; a11 = fmaf(t, t, a11);
      }
    }
  } else {
    for (int k = 0; k < dim; ++k) {
      float t;
      t = x0[k] - y0[k]; a00 = fmaf(t, t, a00);
      t = x0[k] - y1[k]; a01 = fmaf(t, t, a01);
      t = x1[k] - y0[k]; a10 = fmaf(t, t, a10);
      t = x1[k] - y1[k]; a11 = fmaf(t, t, a11);
    }
  }
  o[0] = scale * a00; o[1] = scale * a01; o[2] = scale * a10; o[3] = scale * a11;
}

struct PairView {
  const float* X;
  const float* Y;
  const float* a;
  const float* b;
  int ni, nj;
};

__device__ __forceinline__ PairView pair_view(const float* points, const int64_t* offsets,
                                              const float* weights, int dim, int i, int j) {
  const int64_t si = offsets[i], sj = offsets[j];
  return PairView{points + si * dim, points + sj * dim, weights + si, weights + sj,
                  (int)(offsets[i + 1] - si), (int)(offsets[j + 1] - sj)};
}

// u = a / s with the oracle's conventions: 0 mass -> 0, denominators below FLT_MIN clamped.
__device__ __forceinline__ float scaled_div(float m, float s, bool& clamped) {
  if (s < FLT_MIN) {
    clamped |= m > 0.0f;
    s = FLT_MIN;
  }
  return m == 0.0f ? 0.0f : m / s;
}

// One warp solves one small pair (n_i, n_j <= 64) with K in its SMEM slice: lane = row for the
// u-update (padded stride: conflict-free), lane = column for the v-update; no block barriers.
__device__ void solve_small(const PairView& P, int dim, float scale, float inv_eps, int iters,
                            float* sm, float* out, bool& clamped) {
  const int lane = threadIdx.x & 31;
  float* K = sm;
  float* u = K + kSmallN * kSmallKS;
  float* v = u + kSmallN;
  float* a = v + kSmallN;
  float* b = a + kSmallN;
  const int rb = (P.ni + 1) >> 1, cb = (P.nj + 1) >> 1;
  for (int e = lane; e < rb * cb; e += 32) {
    const int r0 = 2 * (e / cb), c0 = 2 * (e % cb);
    float cc[4];
    cost2x2(P.X, P.Y, dim, r0, c0, P.ni, P.nj, scale, cc);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + (q >> 1), c = c0 + (q & 1);
      if (r < P.ni && c < P.nj) K[r * kSmallKS + c] = expf(-cc[q] * inv_eps);
    }
  }
  for (int r = lane; r < kSmallN; r += 32) {
    a[r] = r < P.ni ? P.a[r] : 0.0f;
    b[r] = r < P.nj ? P.b[r] : 0.0f;
    v[r] = 1.0f;                                   // v0 = 1 (R#4)
  }
  __syncwarp();
  for (int it = 0; it < iters; ++it) {
    for (int r = lane; r < P.ni; r += 32) {        // u = a / (K v)
      float s = 0.0f;
      for (int c = 0; c < P.nj; ++c) s = fmaf(K[r * kSmallKS + c], v[c], s);
      u[r] = scaled_div(a[r], s, clamped);
    }
    __syncwarp();
    for (int c = lane; c < P.nj; c += 32) {        // v = b / (K^T u)
      float s = 0.0f;
      for (int r = 0; r < P.ni; ++r) s = fmaf(K[r * kSmallKS + c], u[r], s);
      v[c] = scaled_div(b[c], s, clamped);
    }
    __syncwarp();
  }
  double acc = 0.0;                                 // <diag(u) K diag(v), C>
  for (int e = lane; e < rb * cb; e += 32) {
    const int r0 = 2 * (e / cb), c0 = 2 * (e % cb);
    float cc[4];
    cost2x2(P.X, P.Y, dim, r0, c0, P.ni, P.nj, scale, cc);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + (q >> 1), c = c0 + (q & 1);
      if (r < P.ni && c < P.nj) acc += (double)(u[r] * K[r * kSmallKS + c]) * (double)cc[q] * (double)v[c];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) *out = (float)acc;
  __syncwarp();
}

// The whole CTA solves one pair; K in SMEM when it fits, else in the CTA's workspace slot.
__device__ void solve_large(const PairView& P, int dim, float scale, float inv_eps, int iters,
                            float* sm, int64_t sm_k_cap, int max_n, float* slot, float* out,
                            bool& clamped) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ double red[kWarps];
  float* u = sm;
  float* v = u + max_n;
  float* Ks = v + max_n;
  const int64_t nk = (int64_t)P.ni * P.nj;
  float* K = nk <= sm_k_cap ? Ks : slot;
  const int rb = (P.ni + 1) >> 1, cb = (P.nj + 1) >> 1;
  for (int64_t e = tid; e < (int64_t)rb * cb; e += kThreads) {
    const int r0 = 2 * (int)(e / cb), c0 = 2 * (int)(e % cb);
    float cc[4];
    cost2x2(P.X, P.Y, dim, r0, c0, P.ni, P.nj, scale, cc);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + (q >> 1), c = c0 + (q & 1);
      if (r < P.ni && c < P.nj) K[(int64_t)r * P.nj + c] = expf(-cc[q] * inv_eps);
    }
  }
  for (int c = tid; c < P.nj; c += kThreads) v[c] = 1.0f;
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    // u = a / (K v): a warp takes 4 rows at a time (coalesced row reads, 4 independent partial
    // sums per lane, interleaved shuffle reductions)
    for (int r0 = warp * 4; r0 < P.ni; r0 += kWarps * 4) {
      float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int c = lane; c < P.nj; c += 32) {
        const float vc = v[c];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (r0 + q < P.ni) s4[q] = fmaf(K[(int64_t)(r0 + q) * P.nj + c], vc, s4[q]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < 4; ++q) s4[q] += __shfl_xor_sync(0xffffffffu, s4[q], o);
      if (lane < 4 && r0 + lane < P.ni) {
        const float sl = lane == 0 ? s4[0] : lane == 1 ? s4[1] : lane == 2 ? s4[2] : s4[3];
        u[r0 + lane] = scaled_div(P.a[r0 + lane], sl, clamped);
      }
    }
    __syncthreads();
    // v = b / (K^T u): thread per column (coalesced), 4 independent accumulators over rows
    for (int c = tid; c < P.nj; c += kThreads) {
      float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
      int r = 0;
      for (; r + 4 <= P.ni; r += 4) {
        s0 = fmaf(K[(int64_t)r * P.nj + c], u[r], s0);
        s1 = fmaf(K[(int64_t)(r + 1) * P.nj + c], u[r + 1], s1);
        s2 = fmaf(K[(int64_t)(r + 2) * P.nj + c], u[r + 2], s2);
        s3 = fmaf(K[(int64_t)(r + 3) * P.nj + c], u[r + 3], s3);
      }
      for (; r < P.ni; ++r) s0 = fmaf(K[(int64_t)r * P.nj + c], u[r], s0);
      v[c] = scaled_div(P.b[c], (s0 + s1) + (s2 + s3), clamped);
    }
    __syncthreads();
  }
  double acc = 0.0;
  for (int64_t e = tid; e < (int64_t)rb * cb; e += kThreads) {
    const int r0 = 2 * (int)(e / cb), c0 = 2 * (int)(e % cb);
    float cc[4];
    cost2x2(P.X, P.Y, dim, r0, c0, P.ni, P.nj, scale, cc);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + (q >> 1), c = c0 + (q & 1);
      if (r < P.ni && c < P.nj)
        acc += (double)(u[r] * K[(int64_t)r * P.nj + c]) * (double)cc[q] * (double)v[c];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t += red[w];
    *out = (float)t;
  }
  __syncthreads();
}

// Work item = kWarps consecutive pairs: if all are small, one warp each; else the CTA solves
// them one after another.
__global__ void __launch_bounds__(kThreads)
eot_pairs_kernel(const float* __restrict__ points, const int64_t* __restrict__ offsets,
                 const float* __restrict__ weights, int dim, float scale, float eps, int iters,
                 const int32_t* __restrict__ pair_i, const int32_t* __restrict__ pair_j,
                 int64_t n_pairs, float* __restrict__ dist_out, float* __restrict__ kslots,
                 int64_t slot_floats, int max_n, int64_t sm_k_cap, uint32_t* __restrict__ status) {
  extern __shared__ float eot_smem[];
  const int warp = threadIdx.x >> 5;
  const float inv_eps = 1.0f / eps;
  bool clamped = false;
  const int64_t n_items = (n_pairs + kWarps - 1) / kWarps;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int64_t q0 = item * kWarps;
    const int cnt = (int)min((int64_t)kWarps, n_pairs - q0);
    bool small = true;
    for (int w = 0; w < cnt; ++w) {
      const int i = pair_i[q0 + w], j = pair_j[q0 + w];
      small &= (offsets[i + 1] - offsets[i]) <= kSmallN && (offsets[j + 1] - offsets[j]) <= kSmallN;
    }
    if (small) {
      if (warp < cnt) {
        const int64_t q = q0 + warp;
        const PairView P = pair_view(points, offsets, weights, dim, pair_i[q], pair_j[q]);
        solve_small(P, dim, scale, inv_eps, iters, eot_smem + warp * kSmallFloats, dist_out + q, clamped);
      }
    } else {
      for (int w = 0; w < cnt; ++w) {
        const int64_t q = q0 + w;
        const PairView P = pair_view(points, offsets, weights, dim, pair_i[q], pair_j[q]);
        solve_large(P, dim, scale, inv_eps, iters, eot_smem, sm_k_cap, max_n,
                    kslots + (int64_t)blockIdx.x * slot_floats, dist_out + q, clamped);
      }
    }
    __syncthreads();
  }
  if (clamped) atomicOr(status, ASOT_FLAG_DENOM_CLAMPED);
}

// SMEM K capacity of the large mode: what is left of kSmemBytes after u and v.
__host__ __device__ inline int64_t sm_k_cap(int max_n) {
  return (int64_t)(kSmemBytes / 4) - 2 * (int64_t)max_n;
}

}  // namespace eot

size_t eot_slot_floats(int64_t max_n) {
  const int64_t nk = max_n * max_n;
  return nk <= eot::sm_k_cap((int)max_n) ? 0 : (size_t)nk;
}

int eot_grid(int64_t n_pairs, int sms) {
  const int64_t items = (n_pairs + eot::kWarps - 1) / eot::kWarps;
  int64_t g = (int64_t)sms;  // 200 KB of SMEM: one CTA per SM
  if (g > items) g = items;
  return (int)(g < 1 ? 1 : g);
}

bool eot_supported(int64_t max_n) { return max_n <= 16384; }

cudaError_t launch_eot_pairs(const float* points, const int64_t* offsets, const float* weights,
                             int dim, float scale, float eps, int iters, const int32_t* pair_i,
                             const int32_t* pair_j, int64_t n_pairs, float* dist_out,
                             float* kslots, int64_t slot_floats, int grid, int max_n,
                             uint32_t* status, cudaStream_t s) {
  if (n_pairs <= 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(eot::eot_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)eot::kSmemBytes);
  if (e != cudaSuccess) return e;
  eot::eot_pairs_kernel<<<grid, eot::kThreads, eot::kSmemBytes, s>>>(
      points, offsets, weights, dim, scale, eps, iters, pair_i, pair_j, n_pairs, dist_out, kslots,
      slot_floats, max_n, eot::sm_k_cap(max_n), status);
  return cudaGetLastError();
}

}  // namespace asot
