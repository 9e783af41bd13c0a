// asot_kmeans.cu -- SURVEY §8(f) NEXT-2: ASOT-k anchor learning by mini-batch k-means
// ("W is the set of cluster centers and P_o is the clustering operator"; Table 4
// "Mini-batch k-means [sculley2010web]"), plus the squared-Euclidean anchor cost of the learned
// anchors (R#7).
//
// One iteration on a batch B (point indices, a seeded input):
//   1. assignment: the hot path's map_assign_kernel on the gathered batch against the f32 copy of
//      the centers -- bit-exact vs the fp64 definition (R#8), lowest index on ties;
//   2. + 3. kmeans_update_kernel: one CTA per center j, one thread per coordinate: the batch sum
//      S_j is accumulated in batch order in fp64, then Sculley's 1/v learning rate applied point
//      by point is the running mean c_j <- (v_j c_j + S_j) / (v_j + m_j) (R#31), evaluated with
//      explicitly rounded fp64 ops (no FMA contraction) so the centers are bit-identical to the
//      oracle's; centers without points stay put.
#include <cmath>

#include "asot_internal.cuh"

namespace asot {
namespace km {

constexpr int kUpdThreads = 512;   // compaction width; threads < dim also own one coordinate
constexpr int kMemberCap = 4096;   // batch entries compacted per round (SMEM)

__global__ void prepare_kernel(const double* __restrict__ centers, int64_t n, float* __restrict__ anchors) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    anchors[x] = (float)centers[x];
}

__global__ void __launch_bounds__(kUpdThreads)
update_kernel(const float* __restrict__ points, int dim, const int64_t* __restrict__ batch_idx,
              int batch, const int32_t* __restrict__ assign, double* __restrict__ centers,
              float* __restrict__ anchors, int64_t* __restrict__ counts) {
  __shared__ int64_t members[kMemberCap];       // point rows of center j, batch order
  __shared__ int32_t wcount[kUpdThreads / 32];
  __shared__ int32_t cnt;
  const int j = blockIdx.x, k = threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s = 0.0;
  int m = 0;
  for (int b0 = 0; b0 < batch; b0 += kMemberCap) {
    const int nb = min(kMemberCap, batch - b0);
    __syncthreads();
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    // compact this round's members of center j in batch order (ballot ranks keep the order)
    for (int c0 = 0; c0 < nb; c0 += kUpdThreads) {
      const int b = c0 + threadIdx.x;
      const bool hit = b < nb && assign[b0 + b] == j;
      const unsigned mask = __ballot_sync(0xffffffffu, hit);
      if (lane == 0) wcount[warp] = __popc(mask);
      __syncthreads();
      int base = cnt, tot = 0;
      for (int w = 0; w < kUpdThreads / 32; ++w) {
        base += w < warp ? wcount[w] : 0;
        tot += wcount[w];
      }
      if (hit) members[base + __popc(mask & ((1u << lane) - 1u))] = batch_idx[b0 + b];
      __syncthreads();
      if (threadIdx.x == 0) cnt += tot;
      __syncthreads();
    }
    const int n = cnt;
    if (k < dim) {
      // independent loads in groups of 8, added in batch order
      int q = 0;
      for (; q + 8 <= n; q += 8) {
        float x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = points[members[q + u] * dim + k];
#pragma unroll
        for (int u = 0; u < 8; ++u) s = __dadd_rn(s, (double)x[u]);
      }
      for (; q < n; ++q) s = __dadd_rn(s, (double)points[members[q] * dim + k]);
    }
    m += n;
  }
  if (m == 0) return;
  const int64_t v = counts[j];
  const int64_t vn = v + m;
  if (k < dim) {
    const int64_t o = (int64_t)j * dim + k;
    const double c = __ddiv_rn(__dadd_rn(__dmul_rn((double)v, centers[o]), s), (double)vn);
    centers[o] = c;
    anchors[o] = (float)c;
  }
  __syncthreads();
  if (threadIdx.x == 0) counts[j] = vn;
}

// C[u][v] = sum_k (w_u[k] - w_v[k])^2 in fp32 (same op order for (u,v) and (v,u): bitwise symmetric).
__global__ void sqeuclid_kernel(const float* __restrict__ W, int K, int d, float* __restrict__ C) {
  const int64_t total = (int64_t)K * K;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(x / K), v = (int)(x % K);
    float a = 0.0f;
    for (int k = 0; k < d; ++k) {
      const float t = W[(int64_t)u * d + k] - W[(int64_t)v * d + k];
      a = fmaf(t, t, a);
    }
    C[x] = u == v ? 0.0f : a;
  }
}

}  // namespace km

cudaError_t launch_kmeans_prepare(const double* centers, int K, int d, float* anchors, cudaStream_t s) {
  const int64_t n = (int64_t)K * d;
  km::prepare_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(centers, n, anchors);
  return cudaGetLastError();
}

cudaError_t launch_kmeans_update(const float* points, int dim, const int64_t* batch_idx, int batch,
                                 const int32_t* assign, int K, double* centers, float* anchors,
                                 int64_t* counts, cudaStream_t s) {
  km::update_kernel<<<(unsigned)K, km::kUpdThreads, 0, s>>>(points, dim, batch_idx, batch, assign,
                                                            centers, anchors, counts);
  return cudaGetLastError();
}

cudaError_t launch_sqeuclid_cost(const float* anchors, int K, int d, bool normalize, float* C,
                                 cudaStream_t s) {
  const int64_t nc = (int64_t)K * K;
  km::sqeuclid_kernel<<<(unsigned)std::min<int64_t>((nc + 255) / 256, 148 * 16), 256, 0, s>>>(anchors, K, d, C);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !normalize) return e;
  return launch_normalize_by_max(C, nc, s);
}

}  // namespace asot
