// asot_bounds.cu -- SURVEY §8(f) NEXT-3: the paper's guarantees for the path, evaluated per pair
// at scale (VERDICT r1 missing #1).
//
// For a pair (i, j) with point sets X (n points), Y (m points), one-hot assignments u_r = j*(x_r),
// v_c = j*(y_c) (the hot path's mapping P_o) and the anchor cost C_s used for W_AS:
//   Prop. 1 (Eq. (7)):  C_hat = Z_x C_s Z_y^T, i.e. C_hat(r, c) = C_s(u_r, v_c)
//            for one-hot Z, against the original cost C(r, c) = ||x_r - y_c||_2 (d_S = d_E, R#7);
//            l1 = sum_{r,c} |C_hat(r, c) - C(r, c)| (the bound) and linf = max_{r,c} |...| (the
//            tighter form the proof gives, R#16);
//   Prop. 2:    m sum_r ||eps_r^x||_2 + n sum_c ||eps_c^y||_2 with
//            eps^x_r = W P_o(x_r) - x_r = w_{u_r} - x_r (and Y alike; R#18 reads P_o(y_j) -> v_j).
// Every term is accumulated in fp64 from the f32 inputs (the points, the anchors, C_s as given).
//
// One CTA per pair: the two point sets are walked in 32 x 32 tiles staged in shared memory
// (coordinates as f32, assignments alongside), each thread evaluates 4 entries of the tile
// (d fp64 FMAs each), and the block reduces sum and max.  Work per pair n m d -- negligible
// next to the exact solvers these bounds are checked against (bench --bounds).
#include <cfloat>
#include <cmath>

#include "asot_internal.cuh"

namespace asot {
namespace bounds {

constexpr int kThreads = 256;
constexpr int kTile = 32;

__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  v = lane < kThreads / 32 ? red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  v = lane < kThreads / 32 ? red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ||w_a - x||_2 in fp64 (the one-hot reconstruction offset of Prop. 2)
__device__ double offset_norm(const float* __restrict__ x, const float* __restrict__ w, int dim) {
  double acc = 0.0;
  for (int k = 0; k < dim; ++k) {
    const double t = (double)w[k] - (double)x[k];
    acc = fma(t, t, acc);
  }
  return sqrt(acc);
}

__global__ void __launch_bounds__(kThreads)
bound_terms_kernel(const float* __restrict__ points, const int64_t* __restrict__ offsets,
                   int64_t n_dist, int dim, const float* __restrict__ anchors, int K,
                   const int32_t* __restrict__ assign, const float* __restrict__ cost,
                   const int32_t* __restrict__ pi, const int32_t* __restrict__ pj, int64_t n_pairs,
                   double* __restrict__ l1_out, double* __restrict__ linf_out,
                   double* __restrict__ prop2_out, uint32_t* status) {
  extern __shared__ __align__(16) uint8_t bounds_smem[];
  float* xs = (float*)bounds_smem;                 // [kTile][dim]
  float* ys = xs + kTile * dim;                    // [kTile][dim]
  int* us = (int*)(ys + kTile * dim);              // [kTile]
  int* vs = us + kTile;                            // [kTile]
  __shared__ double red[kThreads / 32];
  const int tid = threadIdx.x;
  for (int64_t q = blockIdx.x; q < n_pairs; q += gridDim.x) {
    const int i = pi[q], j = pj[q];
    if (i < 0 || j < 0 || i >= n_dist || j >= n_dist) {
      if (tid == 0) {
        l1_out[q] = linf_out[q] = prop2_out[q] = NAN;
        atomicOr(status, ASOT_FLAG_BAD_INDEX);
      }
      continue;
    }
    const int64_t xb = offsets[i], n = offsets[i + 1] - xb;
    const int64_t yb = offsets[j], m = offsets[j + 1] - yb;
    // ---- Prop. 2: m sum_r ||eps_r^x|| + n sum_c ||eps_c^y||
    double rx = 0.0, ry = 0.0;
    for (int64_t r = tid; r < n; r += kThreads)
      rx += offset_norm(points + (xb + r) * dim, anchors + (int64_t)assign[xb + r] * dim, dim);
    for (int64_t c = tid; c < m; c += kThreads)
      ry += offset_norm(points + (yb + c) * dim, anchors + (int64_t)assign[yb + c] * dim, dim);
    rx = block_sum(rx, red);
    ry = block_sum(ry, red);
    // ---- Prop. 1: sum and max of |C_s(u_r, v_c) - ||x_r - y_c|| | over the n x m entries
    double l1 = 0.0, linf = 0.0;
    for (int64_t r0 = 0; r0 < n; r0 += kTile) {
      const int nr = (int)(n - r0 < kTile ? n - r0 : kTile);
      for (int64_t c0 = 0; c0 < m; c0 += kTile) {
        const int nc = (int)(m - c0 < kTile ? m - c0 : kTile);
        __syncthreads();   // previous tile's readers are done
        for (int e = tid; e < kTile * dim; e += kThreads) {
          const int t = e / dim, k = e % dim;
          xs[e] = t < nr ? points[(xb + r0 + t) * dim + k] : 0.0f;
          ys[e] = t < nc ? points[(yb + c0 + t) * dim + k] : 0.0f;
        }
        if (tid < kTile) {
          us[tid] = tid < nr ? assign[xb + r0 + tid] : 0;
          vs[tid] = tid < nc ? assign[yb + c0 + tid] : 0;
        }
        __syncthreads();
        for (int e = tid; e < kTile * kTile; e += kThreads) {
          const int r = e / kTile, c = e % kTile;
          if (r >= nr || c >= nc) continue;
          const float* x = xs + r * dim;
          const float* y = ys + c * dim;
          double acc = 0.0;
          for (int k = 0; k < dim; ++k) {
            const double t = (double)x[k] - (double)y[k];
            acc = fma(t, t, acc);
          }
          const double diff = fabs((double)cost[(int64_t)us[r] * K + vs[c]] - sqrt(acc));
          l1 += diff;
          linf = fmax(linf, diff);
        }
      }
    }
    l1 = block_sum(l1, red);
    linf = block_max(linf, red);
    if (tid == 0) {
      l1_out[q] = l1;
      linf_out[q] = linf;
      prop2_out[q] = (double)m * rx + (double)n * ry;
    }
  }
}

}  // namespace bounds

cudaError_t launch_bound_terms(const float* points, const int64_t* offsets, int64_t n_dist, int dim,
                               const float* anchors, int K, const int32_t* assign, const float* cost,
                               const int32_t* pi, const int32_t* pj, int64_t n_pairs, double* l1,
                               double* linf, double* prop2, uint32_t* status, int sms, cudaStream_t s) {
  if (n_pairs <= 0) return cudaSuccess;
  const size_t smem = (size_t)2 * bounds::kTile * dim * 4 + 2 * bounds::kTile * 4;
  cudaError_t e = cudaFuncSetAttribute(bounds::bound_terms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int64_t grid = n_pairs < (int64_t)sms * 8 ? n_pairs : (int64_t)sms * 8;
  bounds::bound_terms_kernel<<<(unsigned)grid, bounds::kThreads, smem, s>>>(
      points, offsets, n_dist, dim, anchors, K, assign, cost, pi, pj, n_pairs, l1, linf, prop2, status);
  return cudaGetLastError();
}

}  // namespace asot
