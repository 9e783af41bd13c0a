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
// supports exceed 64 bins run in a second launch with 128-bin slices; above 128 a third launch
// runs one CTA per pair (block-wide arg-min / relaxations, flow matrix in a global scratch).
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

// Exact OT on prefilled supports by successive shortest paths (one warp): sources 0..sa-1 with
// supplies rem[0..sa), sinks 0..sb-1 with demands rem[MAXS..MAXS+sb) (both renormalised to unit
// mass), cost C(i, j) (fp64).  `sm` is the warp's slice (Slice<MAXS> layout).  Returns <F, C>.
template <int MAXS, class CostF>
__device__ double ssp_warp(int sa, int sb, uint8_t* sm, CostF C) {
  constexpr int V = 2 * MAXS;
  const int lane = threadIdx.x & 31;
  double* F = (double*)sm;                                  // [MAXS][MAXS]
  double* dist = F + MAXS * MAXS;                           // [V]
  double* pot = dist + V;                                   // [V]
  double* rem = pot + V;                                    // [V]
  int* pred = (int*)(rem + V);                              // [V]
  int* done = pred + V;                                     // [V]
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
  return ssp_warp<MAXS>(sa, sb, sm, [&](int i, int j) {
    return (double)cost[(int64_t)sidx[i] * K + sidx[MAXS + j]];
  });
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
      pending[q] = ok ? 0 : 1;   // still pending: the next (larger) launch takes it
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

// ---------------------------------------------------------------------------------------------
// Supports above 128 bins (e.g. c5, ~380 of 1024): one CTA per pair, the same successive-shortest-
// path algorithm with block-wide arg-min and relaxations; node arrays in SMEM, the flow matrix
// [sa][sb] f64 in a per-CTA global scratch (L2-resident).
constexpr int kBlockThreads = 256;
constexpr int kBlockMaxS = 1024;

struct BlockSmem {
  double dist[2 * kBlockMaxS], pot[2 * kBlockMaxS], rem[2 * kBlockMaxS];
  int pred[2 * kBlockMaxS], done[2 * kBlockMaxS], sidx[2 * kBlockMaxS];
  double red_v[kBlockThreads / 32];
  int red_i[kBlockThreads / 32];
  int sa, sb, target, cnt;
  double bcast;
};

// Block-wide (value, index) arg-min (lowest index on ties); result in every thread.
__device__ void block_argmin(BlockSmem& S, double& v, int& idx) {
  warp_argmin(v, idx);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) {
    S.red_v[warp] = v;
    S.red_i[warp] = idx;
  }
  __syncthreads();
  v = lane < kBlockThreads / 32 ? S.red_v[lane] : INFINITY;
  idx = lane < kBlockThreads / 32 ? S.red_i[lane] : 0x7fffffff;
  warp_argmin(v, idx);   // every warp reduces the same partials
}

__device__ double block_sum(BlockSmem& S, double v) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) S.red_v[warp] = v;
  __syncthreads();
  v = lane < kBlockThreads / 32 ? S.red_v[lane] : 0.0;
  return warp_sum(v);
}

__global__ void __launch_bounds__(kBlockThreads)
exact_pairs_block_kernel(const float* __restrict__ H, int64_t n_dist, int K, const float* __restrict__ cost,
                         const int32_t* __restrict__ pi, const int32_t* __restrict__ pj, int64_t n_pairs,
                         double* __restrict__ out, const uint8_t* __restrict__ pending, double* __restrict__ flow_all,
                         uint32_t* status) {
  extern __shared__ __align__(16) uint8_t exact_block_smem[];
  BlockSmem& S = *reinterpret_cast<BlockSmem*>(exact_block_smem);
  const int tid = threadIdx.x;
  double* F = flow_all + (size_t)blockIdx.x * K * K;   // [sa][sb] row-major, row stride sb
  for (int64_t q = blockIdx.x; q < n_pairs; q += gridDim.x) {
    if (!pending[q]) continue;
    const int i0 = pi[q], j0 = pj[q];
    if (i0 < 0 || j0 < 0 || i0 >= n_dist || j0 >= n_dist) {
      if (tid == 0) out[q] = NAN;
      continue;
    }
    // ---- supports (order-preserving compaction by warp 0) and fp64 masses
    if (tid < 32) {
      const int lane = tid;
      for (int side = 0; side < 2; ++side) {
        const float* h = H + (int64_t)(side == 0 ? i0 : j0) * K;
        int cnt = 0;
        for (int k0 = 0; k0 < K; k0 += 32) {
          const int k = k0 + lane;
          const float w = k < K ? h[k] : 0.0f;
          const bool nz = w > 0.0f;
          const unsigned m = __ballot_sync(0xffffffffu, nz);
          const int pos = cnt + __popc(m & ((1u << lane) - 1u));
          if (nz && pos < kBlockMaxS) {
            S.sidx[side * kBlockMaxS + pos] = k;
            S.rem[side * kBlockMaxS + pos] = (double)w;
          }
          cnt += __popc(m);
        }
        if (lane == 0) (side == 0 ? S.sa : S.sb) = cnt;
      }
    }
    __syncthreads();
    const int sa = S.sa, sb = S.sb;
    const int M = kBlockMaxS;
    if (sa == 0 || sb == 0) {
      if (tid == 0) out[q] = NAN;
      __syncthreads();
      continue;
    }
    double ma = 0.0, mb = 0.0;
    for (int x = tid; x < sa; x += kBlockThreads) ma += S.rem[x];
    ma = block_sum(S, ma);
    for (int x = tid; x < sb; x += kBlockThreads) mb += S.rem[M + x];
    mb = block_sum(S, mb);
    for (int x = tid; x < sa; x += kBlockThreads) S.rem[x] /= ma;      // renormalise (R#14)
    for (int x = tid; x < sb; x += kBlockThreads) S.rem[M + x] /= mb;
    auto C = [&](int i, int j) { return (double)cost[(int64_t)S.sidx[i] * K + S.sidx[M + j]]; };
    for (int64_t e = tid; e < (int64_t)sa * sb; e += kBlockThreads) F[e] = 0.0;
    for (int i = tid; i < sa; i += kBlockThreads) S.pot[i] = 0.0;
    for (int j = tid; j < sb; j += kBlockThreads) {
      double m = INFINITY;
      for (int i = 0; i < sa; ++i) m = fmin(m, C(i, j));
      S.pot[M + j] = m;
    }
    __syncthreads();
    const int V = 2 * M;
    for (int iter = 0; iter < 4 * (sa + sb) + 16; ++iter) {
      double left = 0.0;
      for (int i = tid; i < sa; i += kBlockThreads) left += S.rem[i];
      left = block_sum(S, left);
      if (left <= 1e-13) break;
      // ---- Dijkstra from every source with remaining supply (node ids: i, M + j)
      for (int v = tid; v < V; v += kBlockThreads) {
        const bool exists = v < M ? v < sa : (v - M) < sb;
        const bool src = v < M && v < sa && S.rem[v] > kMassEps;
        S.dist[v] = src ? 0.0 : INFINITY;
        S.pred[v] = -1;
        S.done[v] = exists ? 0 : 1;
      }
      if (tid == 0) S.target = -1;
      __syncthreads();
      for (int step = 0; step < sa + sb; ++step) {
        double best = INFINITY;
        int bi = 0x7fffffff;
        for (int v = tid; v < V; v += kBlockThreads)
          if (!S.done[v] && S.dist[v] < best) {
            best = S.dist[v];
            bi = v;
          }
        block_argmin(S, best, bi);
        if (best == INFINITY) break;
        __syncthreads();
        if (tid == 0) S.done[bi] = 1;
        if (bi >= M && S.rem[bi] > kMassEps) {   // nearest sink with remaining demand
          if (tid == 0) S.target = bi;
          __syncthreads();
          break;
        }
        if (bi >= M) {
          const int j = bi - M;   // backward arcs j -> i (flow on (i, j))
          for (int i = tid; i < sa; i += kBlockThreads) {
            if (!S.done[i] && F[(int64_t)i * sb + j] > kMassEps) {
              const double nd = best + fmax(0.0, -(C(i, j) + S.pot[i] - S.pot[bi]));
              if (nd < S.dist[i]) {
                S.dist[i] = nd;
                S.pred[i] = bi;
              }
            }
          }
        } else {
          const int i = bi;
          for (int j = tid; j < sb; j += kBlockThreads) {
            const int v = M + j;
            if (!S.done[v]) {
              const double nd = best + fmax(0.0, C(i, j) + S.pot[i] - S.pot[v]);
              if (nd < S.dist[v]) {
                S.dist[v] = nd;
                S.pred[v] = i;
              }
            }
          }
        }
        __syncthreads();
      }
      const int target = S.target;
      if (target < 0) break;  // cannot happen for balanced masses
      const double Dt = S.dist[target];
      for (int v = tid; v < V; v += kBlockThreads) {
        const bool exists = v < M ? v < sa : (v - M) < sb;
        if (exists) S.pot[v] += fmin(S.dist[v], Dt);
      }
      __syncthreads();
      if (tid == 0) {   // augment along the path
        double delta = S.rem[target];
        int v = target, src = -1;
        while (v >= 0) {
          const int u = S.pred[v];
          if (u < 0) {
            src = v;
            break;
          }
          if (v < M) delta = fmin(delta, F[(int64_t)v * sb + (u - M)]);  // backward arc u=sink -> v=source
          v = u;
        }
        delta = fmin(delta, S.rem[src]);
        v = target;
        while (true) {
          const int u = S.pred[v];
          if (u < 0) break;
          if (v >= M) F[(int64_t)u * sb + (v - M)] += delta;   // forward arc source u -> sink v
          else F[(int64_t)v * sb + (u - M)] -= delta;          // backward: cancel flow on (v, u)
          v = u;
        }
        S.rem[src] -= delta;
        S.rem[target] -= delta;
      }
      __syncthreads();
    }
    double tot = 0.0;
    for (int64_t e = tid; e < (int64_t)sa * sb; e += kBlockThreads) {
      const double fe = F[e];
      if (fe != 0.0) tot += fe * C((int)(e / sb), (int)(e % sb));
    }
    tot = block_sum(S, tot);
    if (tid == 0) out[q] = tot;
    __syncthreads();
  }
  (void)status;
}

// ---------------------------------------------------------------------------------------------
// NEXT-3 bound checks: EXACT W_1 on the ORIGINAL point sets (Eq. (1)) with the Euclidean
// ground metric d_E of Prop. 2 (R#7): C(r, c) = ||x_r - y_c||_2 in fp64 from the f32
// points, marginals = the point weights renormalised in fp64 (R#14), solved by the same warp SSP
// on the supports (points with weight > 0, <= 64 per side: graph-sized distributions such as c1 /
// c2).  The n x m cost matrix lives next to the warp's flow matrix in shared memory.
constexpr int kW1MaxS = 64;
constexpr int kW1Warps = 3;
constexpr size_t kW1SliceBytes = Slice<kW1MaxS>::kBytes + (size_t)kW1MaxS * kW1MaxS * 8;

__global__ void w1_points_kernel(const float* __restrict__ points, const int64_t* __restrict__ offsets,
                                 const float* __restrict__ weights, int64_t n_dist, int dim,
                                 const int32_t* __restrict__ pi, const int32_t* __restrict__ pj,
                                 int64_t n_pairs, double* __restrict__ out, uint32_t* status) {
  extern __shared__ __align__(16) uint8_t w1_smem[];
  constexpr int M = kW1MaxS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sm = w1_smem + (size_t)warp * kW1SliceBytes;
  double* rem = (double*)sm + M * M + 2 * (2 * M);            // Slice layout: F, dist, pot, rem
  int* sidx = (int*)(rem + 2 * M) + 2 * (2 * M);              // pred, done, sidx
  double* Cm = (double*)(sm + Slice<M>::kBytes);              // [M][M]
  for (int64_t q = (int64_t)blockIdx.x * kW1Warps + warp; q < n_pairs; q += (int64_t)gridDim.x * kW1Warps) {
    const int i = pi[q], j = pj[q];
    if (i < 0 || j < 0 || i >= n_dist || j >= n_dist) {
      if (lane == 0) {
        out[q] = NAN;
        atomicOr(status, ASOT_FLAG_BAD_INDEX);
      }
      continue;
    }
    // supports: points with weight > 0, in point order (ballot compaction); fp64 masses
    int cnt[2];
    double mass[2] = {0.0, 0.0};
    for (int side = 0; side < 2; ++side) {
      const int64_t d = side == 0 ? i : j;
      const int64_t b = offsets[d], e = offsets[d + 1];
      int c = 0;
      for (int64_t p0 = b; p0 < e; p0 += 32) {
        const int64_t p = p0 + lane;
        const float w = p < e ? weights[p] : 0.0f;
        const unsigned m = __ballot_sync(0xffffffffu, w > 0.0f);
        const int pos = c + __popc(m & ((1u << lane) - 1u));
        if (w > 0.0f && pos < M) {
          sidx[side * M + pos] = (int)(p - b);
          rem[side * M + pos] = (double)w;
        }
        if (w > 0.0f) mass[side] += (double)w;
        c += __popc(m);
      }
      cnt[side] = c;
    }
    const int sa = cnt[0], sb = cnt[1];
    if (sa == 0 || sb == 0 || sa > M || sb > M) {
      if (lane == 0) {
        out[q] = NAN;
        if (sa > M || sb > M) atomicOr(status, ASOT_FLAG_EXACT_TOO_LARGE);
      }
      __syncwarp();
      continue;
    }
    const double ma = warp_sum(mass[0]), mb = warp_sum(mass[1]);
    __syncwarp();
    for (int r = lane; r < sa; r += 32) rem[r] /= ma;            // renormalise (R#14)
    for (int c = lane; c < sb; c += 32) rem[M + c] /= mb;
    const float* X = points + offsets[i] * dim;
    const float* Y = points + offsets[j] * dim;
    for (int e = lane; e < sa * sb; e += 32) {                   // C(r, c) = ||x_r - y_c||_2, fp64
      const int r = e / sb, c = e % sb;
      const float* x = X + (int64_t)sidx[r] * dim;
      const float* y = Y + (int64_t)sidx[M + c] * dim;
      double acc = 0.0;
      for (int k = 0; k < dim; ++k) {
        const double t = (double)x[k] - (double)y[k];
        acc = fma(t, t, acc);
      }
      Cm[r * M + c] = sqrt(acc);
    }
    __syncwarp();
    const double w1 = ssp_warp<M>(sa, sb, sm, [&](int r, int c) { return Cm[r * M + c]; });
    if (lane == 0) out[q] = w1;
    __syncwarp();
  }
}

}  // namespace exact

size_t exact_pairs_workspace_bytes(int64_t n_pairs, int K, int sms) {
  size_t b = ((size_t)(n_pairs > 0 ? n_pairs : 1) + 255) & ~(size_t)255;   // pending flags
  if (K > 128) b += (size_t)sms * K * K * 8;                                 // per-CTA flow matrices
  return b;
}

cudaError_t launch_exact_pairs(const float* H, int64_t n_dist, int K, const float* cost, const int32_t* pi,
                               const int32_t* pj, int64_t n_pairs, double* out, uint8_t* pending,
                               uint32_t* status, int sms, cudaStream_t s) {
  if (n_pairs <= 0) return cudaSuccess;
  cudaError_t e = exact::launch_maxs<64>(H, n_dist, K, cost, pi, pj, n_pairs, out, pending, status, sms, s);
  if (e != cudaSuccess) return e;
  e = exact::launch_maxs<128>(H, n_dist, K, cost, pi, pj, n_pairs, out, pending, status, sms, s);
  if (e != cudaSuccess || K <= 128) return e;
  // supports above 128 bins: one CTA per pair (flow matrices after the pending flags)
  double* flow = (double*)(pending + (((size_t)n_pairs + 255) & ~(size_t)255));
  const size_t smem = sizeof(exact::BlockSmem);
  e = cudaFuncSetAttribute(exact::exact_pairs_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  exact::exact_pairs_block_kernel<<<(unsigned)sms, exact::kBlockThreads, smem, s>>>(
      H, n_dist, K, cost, pi, pj, n_pairs, out, pending, flow, status);
  return cudaGetLastError();
}

cudaError_t launch_w1_points(const float* points, const int64_t* offsets, const float* weights, int64_t n_dist,
                             int dim, const int32_t* pi, const int32_t* pj, int64_t n_pairs, double* out,
                             uint32_t* status, int sms, cudaStream_t s) {
  if (n_pairs <= 0) return cudaSuccess;
  const size_t smem = (size_t)exact::kW1Warps * exact::kW1SliceBytes;
  cudaError_t e = cudaFuncSetAttribute(exact::w1_points_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t grid = (n_pairs + exact::kW1Warps - 1) / exact::kW1Warps;
  if (grid > (int64_t)sms * 4) grid = (int64_t)sms * 4;
  exact::w1_points_kernel<<<(unsigned)grid, exact::kW1Warps * 32, smem, s>>>(points, offsets, weights, n_dist, dim,
                                                                            pi, pj, n_pairs, out, status);
  return cudaGetLastError();
}

}  // namespace asot
