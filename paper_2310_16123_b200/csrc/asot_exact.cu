// asot_exact.cu -- SURVEY §8(f) NEXT-3: EXACT anchor-space OT per pair (Def. 3, Eq. (4)-(5),
// P:95-104; the eps -> 0 limit of the hot path's eASOT), for RMSE-vs-exact studies at scale.
//
// W_AS(i, j) = min <T, C_s> over T in U(a', b') with a' = H[i], b' = H[j] renormalised in fp64
// (R#14), solved exactly on the supports of a' and b' (bins with mass > 0) as a min-cost flow by
// successive shortest paths: Dijkstra on the residual bipartite graph with node potentials
// (reduced costs C[u][v] + pi(u) - pi(v) >= 0; pi(v) += min(dist(v), D_t) after each search) and
// augmentation along the path to the nearest sink with remaining demand.  Everything in fp64.
// One warp per pair: nodes are spread over the lanes for the arg-min and the arc relaxations;
// the flow matrix of the supports lives in the warp's slice of shared memory.  Pairs whose
// supports exceed 64 bins run in a second launch with 128-bin slices; above 128 the pair gets NaN
// and ASOT_FLAG_EXACT_TOO_LARGE.
#include <cfloat>
#include <cmath>

#include "asot_internal.cuh"

namespace asot {
namespace exact {

constexpr int kWarpsPerCta(int maxs) { return maxs <= 64 ? 6 : 1; }
constexpr double kMassEps = 1e-14;

template <int MAXS>
struct Slice {
  static constexpr int V = 2 * MAXS;
  static constexpr size_t kBytes = (size_t)MAXS * MAXS * 8          // flow F[i][j]
                                   + (size_t)(2 * MAXS) * 8 * 2       // dist, pot (sources then sinks)
                                   + (size_t)(2 * MAXS) * 8           // remaining supply / demand
                                   + (size_t)(2 * MAXS) * 4 * 3;      // pred, done, support index
};

__device__ __forceinline__ void warp_argmin(double& v, int& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov < v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Returns W_AS of one pair; `sm` is the warp's SMEM slice.  ok = false if a support is too large.
template <int MAXS>
__device__ double solve_pair(const float* __restrict__ ha, const float* __restrict__ hb, int K,
                             const float* __restrict__ cost, uint8_t* sm, bool& ok) {
  constexpr int V = 2 * MAXS;
  const int lane = threadIdx.x & 31;
  double* F = (double*)sm;                                  // [MAXS][MAXS]
  double* dist = F + MAXS * MAXS;                           // [V]
  double* pot = dist + V;                                   // [V]
  double* rem = pot + V;                                    // [V]
  int* pred = (int*)(rem + V);                              // [V]
  int* done = pred + V;                                     // [V]
  int* sidx = done + V;                                     // [V] anchor index of each node
  // ---- supports (order-preserving compaction with ballots) and fp64 masses
  int sa = 0, sb = 0;
  double ma = 0.0, mb = 0.0;
  for (int side = 0; side < 2; ++side) {
    const float* h = side == 0 ? ha : hb;
    int cnt = 0;
    for (int k0 = 0; k0 < K; k0 += 32) {
      const int k = k0 + lane;
      const float w = k < K ? h[k] : 0.0f;
      const bool nz = w > 0.0f;
      const unsigned m = __ballot_sync(0xffffffffu, nz);
      const int pos = cnt + __popc(m & ((1u << lane) - 1u));
      if (nz && pos < MAXS) {
        sidx[side * MAXS + pos] = k;
        rem[side * MAXS + pos] = (double)w;
      }
      if (nz) {
        if (side == 0) ma += (double)w;
        else mb += (double)w;
      }
      cnt += __popc(m);
    }
    if (side == 0) sa = cnt;
    else sb = cnt;
  }
  ok = sa <= MAXS && sb <= MAXS && sa > 0 && sb > 0;
  if (!ok) return NAN;
  ma = warp_sum(ma);
  mb = warp_sum(mb);
  __syncwarp();
  for (int i = lane; i < sa; i += 32) rem[i] /= ma;                 // renormalise (R#14)
  for (int j = lane; j < sb; j += 32) rem[MAXS + j] /= mb;
  auto C = [&](int i, int j) { return (double)cost[(int64_t)sidx[i] * K + sidx[MAXS + j]]; };
  for (int e = lane; e < MAXS * MAXS; e += 32) F[e] = 0.0;
  // initial potentials: sources 0, sinks min_i C[i][j] (all forward reduced costs >= 0)
  for (int i = lane; i < sa; i += 32) pot[i] = 0.0;
  for (int j = lane; j < sb; j += 32) {
    double m = INFINITY;
    for (int i = 0; i < sa; ++i) m = fmin(m, C(i, j));
    pot[MAXS + j] = m;
  }
  __syncwarp();
  for (int iter = 0; iter < 4 * V + 16; ++iter) {
    double left = 0.0;
    for (int i = lane; i < sa; i += 32) left += rem[i];
    left = warp_sum(left);
    if (left <= 1e-13) break;
    // ---- Dijkstra from every source with remaining supply (node ids: i, MAXS + j)
    for (int v = lane; v < V; v += 32) {
      const bool src = v < MAXS && v < sa && rem[v] > kMassEps;
      dist[v] = src ? 0.0 : INFINITY;
      pred[v] = -1;
      const bool exists = v < MAXS ? v < sa : (v - MAXS) < sb;
      done[v] = exists ? 0 : 1;
    }
    __syncwarp();
    int target = -1;
    for (int step = 0; step < sa + sb; ++step) {
      double best = INFINITY;
      int bi = 0x7fffffff;
      for (int v = lane; v < V; v += 32)
        if (!done[v] && dist[v] < best) {
          best = dist[v];
          bi = v;
        }
      warp_argmin(best, bi);
      if (best == INFINITY) break;
      __syncwarp();
      if (lane == 0) done[bi] = 1;
      __syncwarp();
      if (bi >= MAXS) {
        const int j = bi - MAXS;
        if (rem[MAXS + j] > kMassEps) {
          target = bi;
          break;
        }
        // backward arcs j -> i (flow on (i, j)), reduced cost -(C + pot_i - pot_j)
        for (int i = lane; i < sa; i += 32) {
          if (!done[i] && F[i * MAXS + j] > kMassEps) {
            const double rc = fmax(0.0, -(C(i, j) + pot[i] - pot[bi]));
            const double nd = best + rc;
            if (nd < dist[i]) {
              dist[i] = nd;
              pred[i] = bi;
            }
          }
        }
      } else {
        const int i = bi;
        for (int j = lane; j < sb; j += 32) {
          const int v = MAXS + j;
          if (!done[v]) {
            const double rc = fmax(0.0, C(i, j) + pot[i] - pot[v]);
            const double nd = best + rc;
            if (nd < dist[v]) {
              dist[v] = nd;
              pred[v] = i;
            }
          }
        }
      }
      __syncwarp();
    }
    if (target < 0) break;  // cannot happen for balanced masses
    const double Dt = dist[target];
    for (int v = lane; v < V; v += 32) {
      const bool exists = v < MAXS ? v < sa : (v - MAXS) < sb;
      if (exists) pot[v] += fmin(dist[v], Dt);
    }
    __syncwarp();
    // ---- augment along the path (lane 0 walks it)
    if (lane == 0) {
      double delta = rem[target];
      int v = target, src = -1;
      while (v >= 0) {
        const int u = pred[v];
        if (u < 0) {
          src = v;
          break;
        }
        if (v < MAXS) delta = fmin(delta, F[v * MAXS + (u - MAXS)]);  // backward arc u=sink -> v=source
        v = u;
      }
      delta = fmin(delta, rem[src]);
      v = target;
      while (true) {
        const int u = pred[v];
        if (u < 0) break;
        if (v >= MAXS) F[u * MAXS + (v - MAXS)] += delta;   // forward arc source u -> sink v
        else F[v * MAXS + (u - MAXS)] -= delta;             // backward: cancel flow on (v, u)
        v = u;
      }
      rem[src] -= delta;
      rem[target] -= delta;
    }
    __syncwarp();
  }
  double tot = 0.0;
  for (int e = lane; e < MAXS * MAXS; e += 32) {
    const int i = e / MAXS, j = e % MAXS;
    if (i < sa && j < sb && F[e] != 0.0) tot += F[e] * C(i, j);
  }
  return warp_sum(tot);
}

template <int MAXS>
__global__ void exact_pairs_kernel(const float* __restrict__ H, int64_t n_dist, int K, const float* __restrict__ cost,
                                   const int32_t* __restrict__ pi, const int32_t* __restrict__ pj, int64_t n_pairs,
                                   double* __restrict__ out, uint8_t* __restrict__ pending, uint32_t* status) {
  extern __shared__ __align__(16) uint8_t exact_smem[];
  constexpr int W = kWarpsPerCta(MAXS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sm = exact_smem + (size_t)warp * Slice<MAXS>::kBytes;
  for (int64_t q = (int64_t)blockIdx.x * W + warp; q < n_pairs; q += (int64_t)gridDim.x * W) {
    if (MAXS > 64 && !pending[q]) continue;   // the 64-bin launch already solved it
    const int i = pi[q], j = pj[q];
    if (i < 0 || j < 0 || i >= n_dist || j >= n_dist) {
      if (lane == 0) out[q] = NAN;
      continue;
    }
    bool ok = true;
    const double d = solve_pair<MAXS>(H + (int64_t)i * K, H + (int64_t)j * K, K, cost, sm, ok);
    if (lane == 0) {
      out[q] = d;
      if (MAXS <= 64) pending[q] = ok ? 0 : 1;
      else if (!ok) atomicOr(status, ASOT_FLAG_EXACT_TOO_LARGE);
    }
  }
}

template <int MAXS>
cudaError_t launch_maxs(const float* H, int64_t n_dist, int K, const float* cost, const int32_t* pi,
                        const int32_t* pj, int64_t n_pairs, double* out, uint8_t* pending, uint32_t* status,
                        int sms, cudaStream_t s) {
  constexpr int W = kWarpsPerCta(MAXS);
  const size_t smem = (size_t)W * Slice<MAXS>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(exact_pairs_kernel<MAXS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int64_t grid = (n_pairs + W - 1) / W;
  if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
  exact_pairs_kernel<MAXS><<<(unsigned)grid, W * 32, smem, s>>>(H, n_dist, K, cost, pi, pj, n_pairs, out,
                                                               pending, status);
  return cudaGetLastError();
}

}  // namespace exact

cudaError_t launch_exact_pairs(const float* H, int64_t n_dist, int K, const float* cost, const int32_t* pi,
                               const int32_t* pj, int64_t n_pairs, double* out, uint8_t* pending,
                               uint32_t* status, int sms, cudaStream_t s) {
  if (n_pairs <= 0) return cudaSuccess;
  cudaError_t e = exact::launch_maxs<64>(H, n_dist, K, cost, pi, pj, n_pairs, out, pending, status, sms, s);
  if (e != cudaSuccess) return e;
  return exact::launch_maxs<128>(H, n_dist, K, cost, pi, pj, n_pairs, out, pending, status, sms, s);
}

}  // namespace asot
