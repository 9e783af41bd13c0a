// asot_soft_map.cu -- SURVEY §8(f) NEXT-1: soft / near-one-hot mappings P (inference) fused with
// the mapped-marginal reduction a' = Z^T a, plus the ASOT-ML Mahalanobis anchor cost.
//
// ASOT-ML (Table 4; readings R#24, R#25): z = |MLP(x)| / || MLP(x) ||_1 with the
//   MLP d -> hidden -> K (ReLU hidden layer); an all-zero row falls back to the uniform row and
//   raises ASOT_FLAG_SOFT_FALLBACK.
// ASOT-DL (Eq. (9), appendix P:500-538 step size 1; Table 4; R#26-R#28):
//   lambda = softplus(MLP(x)) (d -> hidden -> 1), z^(0) = 0, n_layers x
//   z <- max(0, z - W^T (W z - x) - lambda), then z / sum(z) (uniform fallback, flagged).
// Both: H[i, :] = sum_{p in i} w_p z_p (Eq. (5) P:100 with the 1/n factor dropped, R#1), the
//   same N x K layout the Sinkhorn kernels read, so the soft H feeds asot_distance_matrix(hist_in).
//
// Kernel: one CTA per distribution, point tiles of kPT = 16 points staged in shared memory; every
// matrix product runs on CUDA cores in fp32 (one output column per thread for all 16 points of
// the tile, weights read coalesced from L2, activations broadcast from SMEM).  The DL dictionary
// is SMEM-resident when it fits (K (d+1) 4 B <= 100 KB), else streamed through SMEM in 64-row
// chunks every layer.  The per-distribution sum of w_p z_p is accumulated in fp64 in SMEM in
// point order (thread j owns bin j), so H is deterministic.
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "asot_internal.cuh"

namespace asot {
namespace soft {

constexpr int kThreads = 256;
constexpr int kPT = 16;            // points per tile
constexpr int kChunkRows = 64;     // dictionary rows per streamed chunk
constexpr size_t kResidentBytes = 100 * 1024;

struct Params {
  const float* points;
  const int64_t* offsets;
  const float* weights;
  int64_t n_dist;
  int dim;
  int K;
  int hidden;
  // ML mapper (mode 0): W1 [dim, hidden], b1 [hidden], W2 [hidden, K], b2 [K]
  // DL lambda net (mode 1): W1 = V1 [dim, hidden], b1 = c1, W2 = v2 [hidden], b2 = c2 [1]
  const float* W1;
  const float* b1;
  const float* W2;
  const float* b2;
  const float* dict;   // DL: [K, dim] rows = anchors (the paper's W = dict^T)
  int n_layers;
  int wrows;           // dictionary rows per SMEM chunk (K when resident)
  float* H;            // [n_dist, K]
  float* codes;        // [T, K] or null
  uint32_t* status;
};

__device__ __forceinline__ float softplus_f(float t) { return t > 30.0f ? t : log1pf(expf(t)); }

// Hidden layer of either MLP for the tile: Hs[p][c] = relu(b[c] + sum_k Xs[p][k] W[k][c]).
template <int DP>
__device__ __forceinline__ void hidden_layer(const Params& P, const float* Xs, float* Hs) {
  for (int c = threadIdx.x; c < P.hidden; c += kThreads) {
    float a[kPT];
    const float b = P.b1[c];
#pragma unroll
    for (int p = 0; p < kPT; ++p) a[p] = b;
    for (int k = 0; k < P.dim; ++k) {
      const float w = __ldg(P.W1 + (int64_t)k * P.hidden + c);
#pragma unroll
      for (int p = 0; p < kPT; ++p) a[p] = fmaf(Xs[p * DP + k], w, a[p]);
    }
#pragma unroll
    for (int p = 0; p < kPT; ++p) Hs[p * P.hidden + c] = fmaxf(a[p], 0.0f);
  }
}

// Warp w reduces rows p = w, w + 8 of Zs[kPT][K] into rs[p].
__device__ __forceinline__ void row_sums(const float* Zs, int K, float* rs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int p = warp; p < kPT; p += kThreads / 32) {
    float s = 0.0f;
    for (int j = lane; j < K; j += 32) s += Zs[p * K + j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) rs[p] = s;
  }
}

template <int MODE, int DP>
__global__ void __launch_bounds__(kThreads)
soft_map_kernel(Params P) {
  constexpr int WS = DP + 1;  // dictionary row stride in SMEM (odd: conflict-free column reads)
  extern __shared__ double soft_smem[];
  const int K = P.K;
  double* acc = soft_smem;                        // [K] fp64 per-bin sums
  float* Xs = (float*)(acc + K);                  // [kPT][DP]
  float* Rs = Xs + kPT * DP;                      // [kPT][DP] (DL residual)
  float* Hs = Rs + kPT * DP;                      // [kPT][hidden]
  float* Zs = Hs + kPT * P.hidden;                // [kPT][K]
  float* misc = Zs + kPT * K;                     // lam[kPT], rs[kPT], wts[kPT]
  float* lam = misc;
  float* rs = misc + kPT;
  float* wts = misc + 2 * kPT;
  float* Wc = misc + 3 * kPT;                     // [wrows][WS] dictionary chunk (DL)
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t i = blockIdx.x;
  const int64_t s = P.offsets[i], e = P.offsets[i + 1];
  const bool resident = P.wrows >= K;

  for (int j = tid; j < K; j += kThreads) acc[j] = 0.0;
  if (MODE == 1 && resident) {
    for (int x = tid; x < K * DP; x += kThreads) {
      const int j = x / DP, k = x % DP;
      Wc[j * WS + k] = k < P.dim ? P.dict[(int64_t)j * P.dim + k] : 0.0f;
    }
  }
  bool nonfinite = false, negative = false;
  double msum = 0.0;

  for (int64_t t0 = s; t0 < e; t0 += kPT) {
    const int np = (int)min((int64_t)kPT, e - t0);
    __syncthreads();  // previous tile's readers are done
    for (int x = tid; x < kPT * DP; x += kThreads) {
      const int p = x / DP, k = x % DP;
      float v = 0.0f;
      if (p < np && k < P.dim) {
        v = P.points[(t0 + p) * P.dim + k];
        nonfinite |= !isfinite(v);
      }
      Xs[x] = v;
    }
    if (tid < kPT) {
      float w = tid < np ? P.weights[t0 + tid] : 0.0f;
      if (tid < np) {
        nonfinite |= !isfinite(w);
        negative |= w < 0.0f;
        msum += (double)w;
      }
      wts[tid] = w;
    }
    __syncthreads();
    hidden_layer<DP>(P, Xs, Hs);
    __syncthreads();

    if (MODE == 0) {
      // ---- ASOT-ML: output layer, |.|
      for (int j = tid; j < K; j += kThreads) {
        float a[kPT];
        const float b = P.b2[j];
#pragma unroll
        for (int p = 0; p < kPT; ++p) a[p] = b;
        for (int c = 0; c < P.hidden; ++c) {
          const float w = __ldg(P.W2 + (int64_t)c * K + j);
#pragma unroll
          for (int p = 0; p < kPT; ++p) a[p] = fmaf(Hs[p * P.hidden + c], w, a[p]);
        }
#pragma unroll
        for (int p = 0; p < kPT; ++p) Zs[p * K + j] = fabsf(a[p]);
      }
    } else {
      // ---- ASOT-DL: lambda_p = softplus(v2 . h_p + c2), warp per point
      const int warp = tid >> 5;
      for (int p = warp; p < kPT; p += kThreads / 32) {
        float sdot = 0.0f;
        for (int c = lane; c < P.hidden; c += 32) sdot = fmaf(Hs[p * P.hidden + c], __ldg(P.W2 + c), sdot);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
        if (lane == 0) lam[p] = softplus_f(sdot + P.b2[0]);
      }
      for (int x = tid; x < kPT * K; x += kThreads) Zs[x] = 0.0f;   // z^(0) = 0 (R#27)
      __syncthreads();
      // R phase ownership: column k = tid % DP, points p = tid / DP + m * (kThreads / DP)
      constexpr int PG = kThreads / DP > kPT ? kPT : kThreads / DP;   // point groups
      constexpr int M = kPT / PG;                                       // points per thread
      const int rk = tid % DP, rp0 = tid / DP;
      const bool r_active = rp0 < PG;
      for (int layer = 0; layer < P.n_layers; ++layer) {
        // r = W z - x  (W z)_k = sum_j dict[j][k] z_j
        float racc[M];
#pragma unroll
        for (int m = 0; m < M; ++m) racc[m] = 0.0f;
        for (int c0 = 0; c0 < K; c0 += P.wrows) {
          const int nr = min(P.wrows, K - c0);
          if (!resident) {
            __syncthreads();
            for (int x = tid; x < nr * DP; x += kThreads) {
              const int j = x / DP, k = x % DP;
              Wc[j * WS + k] = k < P.dim ? P.dict[(int64_t)(c0 + j) * P.dim + k] : 0.0f;
            }
            __syncthreads();
          }
          if (r_active) {
            for (int j = 0; j < nr; ++j) {
              const float w = Wc[j * WS + rk];
#pragma unroll
              for (int m = 0; m < M; ++m) racc[m] = fmaf(Zs[(rp0 + m * PG) * K + c0 + j], w, racc[m]);
            }
          }
        }
        if (r_active) {
#pragma unroll
          for (int m = 0; m < M; ++m) {
            const int p = rp0 + m * PG;
            Rs[p * DP + rk] = racc[m] - Xs[p * DP + rk];
          }
        }
        __syncthreads();
        // g = W^T r, z <- max(0, z - g - lambda)
        for (int c0 = 0; c0 < K; c0 += P.wrows) {
          const int nr = min(P.wrows, K - c0);
          if (!resident) {
            __syncthreads();
            for (int x = tid; x < nr * DP; x += kThreads) {
              const int j = x / DP, k = x % DP;
              Wc[j * WS + k] = k < P.dim ? P.dict[(int64_t)(c0 + j) * P.dim + k] : 0.0f;
            }
            __syncthreads();
          }
          for (int x = tid; x < nr * (kPT / 4); x += kThreads) {
            const int j = x % nr, p0 = (x / nr) * 4;
            float g[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            for (int k = 0; k < DP; ++k) {
              const float w = Wc[j * WS + k];
#pragma unroll
              for (int q = 0; q < 4; ++q) g[q] = fmaf(Rs[(p0 + q) * DP + k], w, g[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float* z = &Zs[(p0 + q) * K + c0 + j];
              *z = fmaxf(0.0f, (*z - g[q]) - lam[p0 + q]);
            }
          }
        }
        __syncthreads();
      }
    }
    __syncthreads();
    row_sums(Zs, K, rs);
    __syncthreads();
    if (tid < np && !(rs[tid] > 0.0f)) atomicOr(P.status, ASOT_FLAG_SOFT_FALLBACK);
    const float unif = 1.0f / (float)K;
    for (int j = tid; j < K; j += kThreads) {
      double a = acc[j];
      for (int p = 0; p < np; ++p) {  // point order
        const float z = rs[p] > 0.0f ? Zs[p * K + j] / rs[p] : unif;
        if (P.codes) P.codes[(t0 + p) * K + j] = z;
        a += (double)wts[p] * (double)z;
      }
      acc[j] = a;
    }
  }
  __syncthreads();
  for (int j = tid; j < K; j += kThreads) P.H[i * K + j] = (float)acc[j];

  // status: per-thread input checks, then the mass checks of the one-hot histogram kernel
  if (__syncthreads_or(nonfinite) && tid == 0) atomicOr(P.status, ASOT_FLAG_NONFINITE_INPUT);
  if (__syncthreads_or(negative) && tid == 0) atomicOr(P.status, ASOT_FLAG_BAD_MASS);
  if (tid < kPT) {  // threads < kPT hold the weight partial sums
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) msum += __shfl_xor_sync(0x0000ffffu, msum, o, 16);
    if (tid == 0) {
      if (e <= s) atomicOr(P.status, ASOT_FLAG_EMPTY_DIST);
      else if (fabs(msum - 1.0) > 1e-5) atomicOr(P.status, ASOT_FLAG_BAD_MASS);
    }
  }
}

// ------------------------------------------------------------------------------------------
// ASOT-DL, register-tiled (K in {64, 128, 256}, d in {32, 64, 128}, dictionary SMEM-resident):
// a tile of PT = 8192 / K points; per layer two CUDA-core GEMMs with register tiles
//   R[p][k] = sum_j Z[p][j] Wd[j][k] - X[p][k]      thread: TP1 points x 4 dims
//   G[p][j] = sum_k R[p][k] Wd[j][k]; z <- max(0, z - g - lambda_p)   thread: 4 points x 8 codes
// with Z and R stored transposed (Zt[j][p], Rt[k][p]) and the dictionary stored twice
// (Wd[j][k] for GEMM 1, WdT[k][j] for GEMM 2), so every inner step is two or three vector
// shared-memory loads feeding 8-32 FMAs.  Same arithmetic as the generic kernel up to fp32
// summation order.
// ------------------------------------------------------------------------------------------
template <int DP, int K>
struct TiledDL {
  static constexpr int PT = 8192 / K;            // points per tile
  static constexpr int ZS = PT + 4;              // Zt / Rt row stride
  static constexpr int WS = DP + 4;              // Wd row stride
  static constexpr int TS = K + 4;               // WdT row stride
  static constexpr int TP1 = PT * DP / 1024;     // GEMM-1 points per thread
  static constexpr size_t kFloats(int hidden) {
    return (size_t)K * WS + (size_t)DP * TS + (size_t)K * ZS + (size_t)DP * ZS + (size_t)PT * DP +
           (size_t)PT * hidden + 3 * PT;
  }
  static constexpr size_t bytes(int hidden) { return (size_t)K * 8 + kFloats(hidden) * 4; }
};

template <int DP, int K>
__global__ void __launch_bounds__(kThreads)
soft_dl_tiled_kernel(Params P) {
  using T = TiledDL<DP, K>;
  constexpr int PT = T::PT, ZS = T::ZS, WS = T::WS, TS = T::TS, TP1 = T::TP1;
  static_assert(TP1 >= 1 && (PT / 4) * (K / 8) == kThreads, "tile shape");
  extern __shared__ double soft_smem[];
  double* acc = soft_smem;                         // [K]
  float* Wd = (float*)(acc + K);                   // [K][WS]
  float* WdT = Wd + K * WS;                        // [DP][TS]
  float* Zt = WdT + DP * TS;                       // [K][ZS]
  float* Rt = Zt + K * ZS;                         // [DP][ZS]
  float* Xs = Rt + DP * ZS;                        // [PT][DP]
  float* Hs = Xs + PT * DP;                        // [PT][hidden]
  float* lam = Hs + PT * P.hidden;
  float* rs = lam + PT;
  float* wts = rs + PT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i = blockIdx.x;
  const int64_t s = P.offsets[i], e = P.offsets[i + 1];

  for (int j = tid; j < K; j += kThreads) acc[j] = 0.0;
  for (int x = tid; x < K * DP; x += kThreads) {
    const int j = x / DP, k = x % DP;
    const float w = k < P.dim ? P.dict[(int64_t)j * P.dim + k] : 0.0f;
    Wd[j * WS + k] = w;
    WdT[k * TS + j] = w;
  }
  bool nonfinite = false, negative = false;
  double msum = 0.0;
  // GEMM-1 ownership: dims k1..k1+3, points p1..p1+TP1-1
  const int k1 = 4 * (tid % (DP / 4)), p1 = TP1 * (tid / (DP / 4));
  // GEMM-2 ownership: codes j2..j2+7, points p2..p2+3
  const int j2 = 8 * (tid % (K / 8)), p2 = 4 * (tid / (K / 8));

  for (int64_t t0 = s; t0 < e; t0 += PT) {
    const int np = (int)min((int64_t)PT, e - t0);
    __syncthreads();
    for (int x = tid; x < PT * DP; x += kThreads) {
      const int p = x / DP, k = x % DP;
      float v = 0.0f;
      if (p < np && k < P.dim) {
        v = P.points[(t0 + p) * P.dim + k];
        nonfinite |= !isfinite(v);
      }
      Xs[x] = v;
    }
    for (int p = tid; p < PT; p += kThreads) {
      const float w = p < np ? P.weights[t0 + p] : 0.0f;
      if (p < np) {
        nonfinite |= !isfinite(w);
        negative |= w < 0.0f;
        msum += (double)w;
      }
      wts[p] = w;
    }
    for (int x = tid; x < K * ZS; x += kThreads) Zt[x] = 0.0f;    // z^(0) = 0 (R#27)
    __syncthreads();
    // lambda-net hidden layer (thread = one hidden unit for all PT points)
    for (int c = tid; c < P.hidden; c += kThreads) {
      const float b = P.b1[c];
      for (int p0 = 0; p0 < PT; p0 += 16) {
        float a[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) a[q] = b;
        for (int k = 0; k < P.dim; ++k) {
          const float w = __ldg(P.W1 + (int64_t)k * P.hidden + c);
#pragma unroll
          for (int q = 0; q < 16; ++q) a[q] = fmaf(Xs[(p0 + q) * DP + k], w, a[q]);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) Hs[(p0 + q) * P.hidden + c] = fmaxf(a[q], 0.0f);
      }
    }
    __syncthreads();
    for (int p = warp; p < PT; p += kThreads / 32) {
      float sdot = 0.0f;
      for (int c = lane; c < P.hidden; c += 32) sdot = fmaf(Hs[p * P.hidden + c], __ldg(P.W2 + c), sdot);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
      if (lane == 0) lam[p] = softplus_f(sdot + P.b2[0]);
    }
    __syncthreads();

    for (int layer = 0; layer < P.n_layers; ++layer) {
      // ---- GEMM 1: R = Z Wd - X
      float r[TP1][4];
#pragma unroll
      for (int t = 0; t < TP1; ++t)
#pragma unroll
        for (int q = 0; q < 4; ++q) r[t][q] = 0.0f;
#pragma unroll 4
      for (int j = 0; j < K; ++j) {
        const float4 w = *reinterpret_cast<const float4*>(Wd + j * WS + k1);
        float z[TP1];
        if constexpr (TP1 == 4) {
          const float4 z4 = *reinterpret_cast<const float4*>(Zt + j * ZS + p1);
          z[0] = z4.x; z[1] = z4.y; z[2] = z4.z; z[3] = z4.w;
        } else if constexpr (TP1 == 2) {
          const float2 z2 = *reinterpret_cast<const float2*>(Zt + j * ZS + p1);
          z[0] = z2.x; z[1] = z2.y;
        } else {
#pragma unroll
          for (int t = 0; t < TP1; ++t) z[t] = Zt[j * ZS + p1 + t];
        }
#pragma unroll
        for (int t = 0; t < TP1; ++t) {
          r[t][0] = fmaf(z[t], w.x, r[t][0]);
          r[t][1] = fmaf(z[t], w.y, r[t][1]);
          r[t][2] = fmaf(z[t], w.z, r[t][2]);
          r[t][3] = fmaf(z[t], w.w, r[t][3]);
        }
      }
#pragma unroll
      for (int t = 0; t < TP1; ++t)
#pragma unroll
        for (int q = 0; q < 4; ++q) Rt[(k1 + q) * ZS + p1 + t] = r[t][q] - Xs[(p1 + t) * DP + k1 + q];
      __syncthreads();
      // ---- GEMM 2 + update: g = W^T r, z <- max(0, z - g - lambda)
      float g[4][8];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int q = 0; q < 8; ++q) g[t][q] = 0.0f;
#pragma unroll 4
      for (int k = 0; k < DP; ++k) {
        const float4 rv = *reinterpret_cast<const float4*>(Rt + k * ZS + p2);
        const float4 wa = *reinterpret_cast<const float4*>(WdT + k * TS + j2);
        const float4 wb = *reinterpret_cast<const float4*>(WdT + k * TS + j2 + 4);
        const float rr[4] = {rv.x, rv.y, rv.z, rv.w};
        const float ww[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int q = 0; q < 8; ++q) g[t][q] = fmaf(rr[t], ww[q], g[t][q]);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 z4 = *reinterpret_cast<float4*>(Zt + (j2 + q) * ZS + p2);
        z4.x = fmaxf(0.0f, (z4.x - g[0][q]) - lam[p2 + 0]);
        z4.y = fmaxf(0.0f, (z4.y - g[1][q]) - lam[p2 + 1]);
        z4.z = fmaxf(0.0f, (z4.z - g[2][q]) - lam[p2 + 2]);
        z4.w = fmaxf(0.0f, (z4.w - g[3][q]) - lam[p2 + 3]);
        *reinterpret_cast<float4*>(Zt + (j2 + q) * ZS + p2) = z4;
      }
      __syncthreads();
    }
    // ---- row sums (warp per point), normalisation, fp64 point-order accumulation
    for (int p = warp; p < PT; p += kThreads / 32) {
      float sum = 0.0f;
      for (int j = lane; j < K; j += 32) sum += Zt[j * ZS + p];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) rs[p] = sum;
    }
    __syncthreads();
    if (tid < np && !(rs[tid] > 0.0f)) atomicOr(P.status, ASOT_FLAG_SOFT_FALLBACK);
    const float unif = 1.0f / (float)K;
    for (int j = tid; j < K; j += kThreads) {
      double a = acc[j];
      for (int p = 0; p < np; ++p) {
        const float z = rs[p] > 0.0f ? Zt[j * ZS + p] / rs[p] : unif;
        if (P.codes) P.codes[(t0 + p) * K + j] = z;
        a += (double)wts[p] * (double)z;
      }
      acc[j] = a;
    }
  }
  __syncthreads();
  for (int j = tid; j < K; j += kThreads) P.H[i * K + j] = (float)acc[j];
  if (__syncthreads_or(nonfinite) && tid == 0) atomicOr(P.status, ASOT_FLAG_NONFINITE_INPUT);
  if (__syncthreads_or(negative) && tid == 0) atomicOr(P.status, ASOT_FLAG_BAD_MASS);
  // weights were read by threads p < PT: reduce their partial sums through the acc buffer
  __syncthreads();
  if (tid < PT) acc[tid] = msum;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int p = 0; p < PT && p < K; ++p) tot += acc[p];
    if (e <= s) atomicOr(P.status, ASOT_FLAG_EMPTY_DIST);
    else if (fabs(tot - 1.0) > 1e-5) atomicOr(P.status, ASOT_FLAG_BAD_MASS);
  }
}

template <int DP, int K>
cudaError_t launch_tiled_dl(const Params& P, cudaStream_t s, bool& done) {
  const size_t smem = TiledDL<DP, K>::bytes(P.hidden);
  if (smem > 220 * 1024 || TiledDL<DP, K>::PT > K) { done = false; return cudaSuccess; }
  cudaError_t e = cudaFuncSetAttribute(soft_dl_tiled_kernel<DP, K>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  soft_dl_tiled_kernel<DP, K><<<(unsigned)P.n_dist, kThreads, smem, s>>>(P);
  done = true;
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// ASOT-DL, dictionary streamed (d in {64, 128} = DP, K a multiple of 64 that the resident
// kernels cannot hold, e.g. c5: K = 1024, d = 128): same tile of kPT points and the same
// arithmetic order as the generic kernel (bitwise the same codes), but every layer streams the
// dictionary through SMEM in 64-row chunks with 16-byte cp.async copies, double-buffered, and
// both products are register-tiled so each shared-memory load feeds several FMAs:
//   R[p][k] = sum_j Z[p][j] W[j][k] - X[p][k]   warp w: dims [w DP/8, +DP/8), lane: point p =
//                                                lane % 16 x DP/16 dims; Z rows read as float4
//   G[p][j] = sum_k R[p][k] W[j][k]              warp w: chunk rows [8w, 8w+8), lane: point p x
//                                                4 rows; z <- max(0, z - g - lambda_p)
// ------------------------------------------------------------------------------------------
template <int DP>
struct StreamDL {
  static constexpr int CR = 64;          // dictionary rows per chunk
  static constexpr int WS = DP + 4;      // chunk row stride (floats; 16-byte aligned rows)
  static constexpr int RS = DP + 4;      // R row stride
  static constexpr size_t bytes(int K, int hidden) {
    return (size_t)K * 8 + ((size_t)kPT * DP + (size_t)kPT * RS + (size_t)kPT * hidden +
                            (size_t)kPT * (K + 4) + 3 * kPT + 2 * (size_t)CR * WS) * 4 + 16;
  }
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int DP>
__global__ void __launch_bounds__(kThreads, 1)
soft_dl_stream_kernel(Params P) {
  using C = StreamDL<DP>;
  constexpr int CR = C::CR, WS = C::WS, RS = C::RS;
  constexpr int ND = DP / 16;              // GEMM-1 dims per thread
  extern __shared__ double soft_smem[];
  const int K = P.K, ZS = K + 4;
  double* acc = soft_smem;                        // [K] fp64 per-bin sums
  float* Xs = (float*)(acc + K);                  // [kPT][DP]
  float* Rs = Xs + kPT * DP;                      // [kPT][RS]
  float* Hs = Rs + kPT * RS;                      // [kPT][hidden]
  float* Zs = Hs + kPT * P.hidden;                // [kPT][K + 4]
  float* misc = Zs + kPT * ZS;
  float* lam = misc;
  float* rs = misc + kPT;
  float* wts = misc + 2 * kPT;
  float* Wb = (float*)(((uintptr_t)(misc + 3 * kPT) + 15) & ~(uintptr_t)15);   // [2][CR][WS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i = blockIdx.x;
  const int64_t s = P.offsets[i], e = P.offsets[i + 1];
  const int nchunks = K / CR;

  // chunk c of the dictionary -> buffer b (16-byte async copies; rows padded to WS floats)
  auto stage = [&](int c, int b) {
    float* dst = Wb + (size_t)b * CR * WS;
    const float* src = P.dict + (int64_t)c * CR * DP;
    for (int x = tid; x < CR * (DP / 4); x += kThreads) {
      const int r = x / (DP / 4), k4 = x % (DP / 4);
      cp_async16(dst + r * WS + 4 * k4, src + (int64_t)r * DP + 4 * k4);
    }
    cp_async_commit();
  };

  for (int j = tid; j < K; j += kThreads) acc[j] = 0.0;
  bool nonfinite = false, negative = false;
  double msum = 0.0;
  const int p = lane & 15;                         // point of this lane in both products
  const int d0 = warp * (DP / 8) + (lane >> 4) * ND;   // GEMM-1 dims [d0, d0 + ND)
  const int jr0 = warp * 8 + (lane >> 4) * 4;           // GEMM-2 chunk rows [jr0, jr0 + 4)

  for (int64_t t0 = s; t0 < e; t0 += kPT) {
    const int np = (int)min((int64_t)kPT, e - t0);
    __syncthreads();  // previous tile's readers are done
    for (int x = tid; x < kPT * DP; x += kThreads) {
      const int pp = x / DP, k = x % DP;
      float v = 0.0f;
      if (pp < np) {
        v = P.points[(t0 + pp) * DP + k];
        nonfinite |= !isfinite(v);
      }
      Xs[x] = v;
    }
    if (tid < kPT) {
      float w = tid < np ? P.weights[t0 + tid] : 0.0f;
      if (tid < np) {
        nonfinite |= !isfinite(w);
        negative |= w < 0.0f;
        msum += (double)w;
      }
      wts[tid] = w;
    }
    __syncthreads();
    hidden_layer<DP>(P, Xs, Hs);
    __syncthreads();
    // lambda_p = softplus(v2 . h_p + c2), warp per point
    for (int pp = warp; pp < kPT; pp += kThreads / 32) {
      float sdot = 0.0f;
      for (int c = lane; c < P.hidden; c += 32) sdot = fmaf(Hs[pp * P.hidden + c], __ldg(P.W2 + c), sdot);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
      if (lane == 0) lam[pp] = softplus_f(sdot + P.b2[0]);
    }
    for (int x = tid; x < kPT * ZS; x += kThreads) Zs[x] = 0.0f;   // z^(0) = 0 (R#27)
    // the dictionary stream: per layer one pass for R, one for G; chunk sequence number g
    int g = 0;
    stage(0, 0);
    for (int layer = 0; layer < P.n_layers; ++layer) {
      for (int pass = 0; pass < 2; ++pass) {
        float racc[ND];
#pragma unroll
        for (int q = 0; q < ND; ++q) racc[q] = 0.0f;
        for (int c = 0; c < nchunks; ++c, ++g) {
          // prefetch the next chunk of the stream (next pass / layer wraps to chunk 0)
          const bool more = !(layer + 1 == P.n_layers && pass == 1 && c + 1 == nchunks);
          if (more) {
            stage(c + 1 < nchunks ? c + 1 : 0, (g + 1) & 1);
            cp_async_wait<1>();
          } else {
            cp_async_wait<0>();
          }
          __syncthreads();   // chunk g visible; (pass 1) R complete; (pass 0) Z updated
          const float* W = Wb + (size_t)(g & 1) * CR * WS;
          const int c0 = c * CR;
          if (pass == 0) {
            // R[p][d0 + q] += sum_j Z[p][c0 + j] W[j][d0 + q]  (j in order)
            const float* zr = Zs + p * ZS + c0;
#pragma unroll 4
            for (int j = 0; j < CR; j += 4) {
              const float4 z4 = *reinterpret_cast<const float4*>(zr + j);
              const float zz[4] = {z4.x, z4.y, z4.z, z4.w};
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const float* wr = W + (j + jj) * WS + d0;
#pragma unroll
                for (int q4 = 0; q4 < ND; q4 += 4) {
                  const float4 w4 = *reinterpret_cast<const float4*>(wr + q4);
                  racc[q4 + 0] = fmaf(zz[jj], w4.x, racc[q4 + 0]);
                  racc[q4 + 1] = fmaf(zz[jj], w4.y, racc[q4 + 1]);
                  racc[q4 + 2] = fmaf(zz[jj], w4.z, racc[q4 + 2]);
                  racc[q4 + 3] = fmaf(zz[jj], w4.w, racc[q4 + 3]);
                }
              }
            }
          } else {
            // G[p][c0 + jr] = sum_k R[p][k] W[jr][k] (k in order); z update in place
            float gacc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            const float* rr = Rs + p * RS;
#pragma unroll 4
            for (int k = 0; k < DP; k += 4) {
              const float4 r4 = *reinterpret_cast<const float4*>(rr + k);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float4 w4 = *reinterpret_cast<const float4*>(W + (jr0 + q) * WS + k);
                gacc[q] = fmaf(r4.x, w4.x, gacc[q]);
                gacc[q] = fmaf(r4.y, w4.y, gacc[q]);
                gacc[q] = fmaf(r4.z, w4.z, gacc[q]);
                gacc[q] = fmaf(r4.w, w4.w, gacc[q]);
              }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float* z = &Zs[p * ZS + c0 + jr0 + q];
              *z = fmaxf(0.0f, (*z - gacc[q]) - lam[p]);
            }
          }
          __syncthreads();   // buffer g & 1 may be refilled two chunks later
        }
        if (pass == 0) {   // r = W z - x
#pragma unroll
          for (int q = 0; q < ND; ++q) Rs[p * RS + d0 + q] = racc[q] - Xs[p * DP + d0 + q];
        }
      }
    }
    __syncthreads();
    // row sums (warp per point), normalisation, codes, the fp64 point-order H accumulation
    for (int pp = warp; pp < kPT; pp += kThreads / 32) {
      float sm = 0.0f;
      for (int j = lane; j < K; j += 32) sm += Zs[pp * ZS + j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
      if (lane == 0) rs[pp] = sm;
    }
    __syncthreads();
    if (tid < np && !(rs[tid] > 0.0f)) atomicOr(P.status, ASOT_FLAG_SOFT_FALLBACK);
    const float unif = 1.0f / (float)K;
    for (int j = tid; j < K; j += kThreads) {
      double a = acc[j];
      for (int pp = 0; pp < np; ++pp) {  // point order
        const float z = rs[pp] > 0.0f ? Zs[pp * ZS + j] / rs[pp] : unif;
        if (P.codes) P.codes[(t0 + pp) * K + j] = z;
        a += (double)wts[pp] * (double)z;
      }
      acc[j] = a;
    }
  }
  __syncthreads();
  for (int j = tid; j < K; j += kThreads) P.H[i * K + j] = (float)acc[j];
  if (__syncthreads_or(nonfinite) && tid == 0) atomicOr(P.status, ASOT_FLAG_NONFINITE_INPUT);
  if (__syncthreads_or(negative) && tid == 0) atomicOr(P.status, ASOT_FLAG_BAD_MASS);
  if (tid < kPT) {  // threads < kPT hold the weight partial sums
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) msum += __shfl_xor_sync(0x0000ffffu, msum, o, 16);
    if (tid == 0) {
      if (e <= s) atomicOr(P.status, ASOT_FLAG_EMPTY_DIST);
      else if (fabs(msum - 1.0) > 1e-5) atomicOr(P.status, ASOT_FLAG_BAD_MASS);
    }
  }
}

template <int DP>
cudaError_t try_stream_dl(const Params& P, cudaStream_t s, bool& done) {
  done = false;
  const size_t smem = StreamDL<DP>::bytes(P.K, P.hidden);
  if (P.dim != DP || P.K % StreamDL<DP>::CR != 0 || smem > 220 * 1024 ||
      (reinterpret_cast<uintptr_t>(P.dict) & 15u) != 0)
    return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(soft_dl_stream_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  soft_dl_stream_kernel<DP><<<(unsigned)P.n_dist, kThreads, smem, s>>>(P);
  done = true;
  return cudaGetLastError();
}

// Picks the register-tiled DL kernel when (d, K) has an instantiation and it fits SMEM.
template <int DP>
cudaError_t try_tiled_dl(const Params& P, cudaStream_t s, bool& done) {
  done = false;
  if (P.K == 64) return launch_tiled_dl<DP, 64>(P, s, done);
  if (P.K == 128) return launch_tiled_dl<DP, 128>(P, s, done);
  if (P.K == 256) return launch_tiled_dl<DP, 256>(P, s, done);
  return cudaSuccess;
}

size_t smem_bytes(int mode, int dp, int K, int hidden, int wrows) {
  size_t b = (size_t)K * 8 + (size_t)(2 * kPT * dp + kPT * hidden + kPT * K + 3 * kPT) * 4;
  if (mode == 1) b += (size_t)wrows * (dp + 1) * 4;
  return b;
}

template <int MODE, int DP>
cudaError_t launch_dp(Params P, cudaStream_t s) {
  if (MODE == 1) {
    P.wrows = (size_t)P.K * (DP + 1) * 4 <= kResidentBytes ? P.K : kChunkRows;
  } else {
    P.wrows = 0;
  }
  const size_t smem = smem_bytes(MODE, DP, P.K, P.hidden, P.wrows);
  cudaError_t e = cudaFuncSetAttribute(soft_map_kernel<MODE, DP>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  soft_map_kernel<MODE, DP><<<(unsigned)P.n_dist, kThreads, smem, s>>>(P);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_mode(const Params& P, cudaStream_t s) {
  if (P.dim <= 8) return launch_dp<MODE, 8>(P, s);
  if (P.dim <= 16) return launch_dp<MODE, 16>(P, s);
  if (P.dim <= 32) return launch_dp<MODE, 32>(P, s);
  if (P.dim <= 64) return launch_dp<MODE, 64>(P, s);
  return launch_dp<MODE, 128>(P, s);
}

// ---------------------------------------------------------------- Mahalanobis anchor cost
// Y[u][r] = sum_k M[r][k] w_u[k]; C[u][v] = ||Y_u - Y_v||_2.  C[v][u] evaluates the
// negated differences in the same order, so C is bitwise symmetric with an exact zero diagonal.
__global__ void mahalanobis_project_kernel(const float* __restrict__ W, int K, int d,
                                           const float* __restrict__ M, int h, float* __restrict__ Y) {
  const int64_t total = (int64_t)K * h;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(x / h), r = (int)(x % h);
    float a = 0.0f;
    for (int k = 0; k < d; ++k) a = fmaf(M[(int64_t)r * d + k], W[(int64_t)u * d + k], a);
    Y[x] = a;
  }
}

__global__ void mahalanobis_pair_kernel(const float* __restrict__ Y, int K, int h, float* __restrict__ C) {
  const int64_t total = (int64_t)K * K;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(x / K), v = (int)(x % K);
    float a = 0.0f;
    for (int r = 0; r < h; ++r) {
      const float t = Y[(int64_t)u * h + r] - Y[(int64_t)v * h + r];
      a = fmaf(t, t, a);
    }
    C[x] = u == v ? 0.0f : sqrtf(a);
  }
}

// Single CTA: max over C, then C /= max (max entry becomes exactly 1).
__global__ void normalize_by_max_kernel(float* C, int64_t n) {
  __shared__ float red[32];
  float m = 0.0f;
  for (int64_t x = threadIdx.x; x < n; x += blockDim.x) m = fmaxf(m, C[x]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  m = red[0];
  if (m > 0.0f)
    for (int64_t x = threadIdx.x; x < n; x += blockDim.x) C[x] = C[x] / m;
}

}  // namespace soft

cudaError_t launch_soft_map_ml(const float* points, const int64_t* offsets, const float* weights,
                               int64_t n_dist, int dim, int K, int hidden, const float* W1,
                               const float* b1, const float* W2, const float* b2, float* H,
                               float* codes, uint32_t* status, cudaStream_t s) {
  soft::Params P{points, offsets, weights, n_dist, dim, K, hidden, W1, b1, W2, b2,
                 nullptr, 0, 0, H, codes, status};
  return soft::launch_mode<0>(P, s);
}

cudaError_t launch_soft_map_dl(const float* points, const int64_t* offsets, const float* weights,
                               int64_t n_dist, int dim, const float* dict, int K, int n_layers,
                               int hidden, const float* V1, const float* c1, const float* v2,
                               const float* c2, float* H, float* codes, uint32_t* status,
                               cudaStream_t s) {
  soft::Params P{points, offsets, weights, n_dist, dim, K, hidden, V1, c1, v2, c2,
                 dict, n_layers, 0, H, codes, status};
  if (!getenv("ASOT_SOFT_DL_GENERIC") && (dim == 32 || dim == 64 || dim == 128)) {
    bool done = false;
    cudaError_t e = dim == 32 ? soft::try_tiled_dl<32>(P, s, done)
                  : dim == 64 ? soft::try_tiled_dl<64>(P, s, done)
                              : soft::try_tiled_dl<128>(P, s, done);
    if (e != cudaSuccess || done) return e;
    if (dim == 64 || dim == 128) {   // dictionary too large for the resident kernels: streamed
      e = dim == 64 ? soft::try_stream_dl<64>(P, s, done) : soft::try_stream_dl<128>(P, s, done);
      if (e != cudaSuccess || done) return e;
    }
  }
  return soft::launch_mode<1>(P, s);
}

cudaError_t launch_normalize_by_max(float* C, int64_t n, cudaStream_t s) {
  soft::normalize_by_max_kernel<<<1, 1024, 0, s>>>(C, n);
  return cudaGetLastError();
}

cudaError_t launch_mahalanobis_cost(const float* anchors, int K, int d, const float* M, int h,
                                    bool normalize, float* Y, float* C, cudaStream_t s) {
  const int64_t ny = (int64_t)K * h, nc = (int64_t)K * K;
  soft::mahalanobis_project_kernel<<<(unsigned)std::min<int64_t>((ny + 255) / 256, 148 * 16), 256, 0, s>>>(
      anchors, K, d, M, h, Y);
  soft::mahalanobis_pair_kernel<<<(unsigned)std::min<int64_t>((nc + 255) / 256, 148 * 16), 256, 0, s>>>(
      Y, K, h, C);
  if (normalize) soft::normalize_by_max_kernel<<<1, 1024, 0, s>>>(C, nc);
  return cudaGetLastError();
}

}  // namespace asot
