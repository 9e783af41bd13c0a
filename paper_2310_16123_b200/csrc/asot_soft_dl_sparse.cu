// asot_soft_dl_sparse.cu -- SURVEY §8(f) NEXT-1: the ASOT-DL encoder (Eqs. (8)(9),
// appendix P:500-538 step size 1; R#26-R#28) for large dictionaries (d in {64, 128}, K a multiple
// of 64, K >= 256: c3 K = 256, c5 K = 1024), built around the sparsity of the codes.
//
//   lambda_p = softplus(v2 . relu(V1^T x_p + c1) + c2),  z^(0) = 0,
//   n_layers x { r = W z - x;  g = W^T r;  z <- max(0, z - g - lambda) },  then z / sum z
//   (uniform fallback, flagged), H[i] = sum_p w_p z_p in fp64 in point order (Eq. (5), R#1).
//
// The codes are near-one-hot (the point of ASOT-DL): measured with the fp64 oracle, c5 keeps 8-16
// of 1024 entries non-zero at every layer, c3 15-61 of 256.  So the first product, r = W z - x, is
// a sparse gather -- sum over the non-zero z_j of z_j w_j, in increasing j -- and the dense work
// is the second product, the [64 points x d] x [d x K] GEMM g = W^T r, register-blocked like the
// mapping kernel: the tile's residuals and a 64-anchor chunk of the dictionary sit in shared
// memory (the chunk double-buffered with cp.async), thread (warp w, lane l) computes the 4 x 4
// block of points 4 (2w + l/16) + [0, 4) and anchors 16 a + l % 16, two f32x2 FMAs per block
// entry and 4 coordinates.  The codes of the tile live densely in a per-CTA global scratch
// (L2-resident, 64 x K floats) with a bitmap of their non-zeros in shared memory; the epilogue of
// each chunk reads z_old from the scratch, writes z_new and its bit.  fp32 throughout (codes
// within 1e-5 of the fp64 oracle); persistent CTAs loop over distributions.
#include <cfloat>
#include <cmath>

#include "asot_internal.cuh"

namespace asot {
namespace softdl {

constexpr int kThreads = 256;
constexpr int kTP = 64;          // points per tile
constexpr int kCA = 64;          // anchors per dictionary chunk (16 lanes x 4)

struct Args {
  const float* points;
  const int64_t* offsets;
  const float* weights;
  int64_t n_dist;
  int K;
  int hidden;
  const float* V1;   // [d, hidden]
  const float* c1;   // [hidden]
  const float* v2;   // [hidden]
  const float* c2;   // [1]
  const float* dict; // [K, d]
  int n_layers;
  float* H;          // [n_dist, K]
  float* codes;      // [T, K] or null
  float* zbuf;       // [gridDim.x][kTP][K] scratch
  uint32_t* status;
};

template <int DP>
struct Lay {
  static constexpr int RS = DP + 4;   // row stride (floats): 16-byte rows, 16 B apart in bank space
  static size_t bytes(int K, int hidden) {
    return (size_t)K * 8                              // acc (fp64)
           + (size_t)kTP * RS * 4 * 2                 // X, R
           + (size_t)2 * kCA * RS * 4                 // dictionary chunks (double buffer)
           + (size_t)kTP * (K / 32) * 4               // bitmap
           + (size_t)kTP * hidden * 4                 // hidden activations
           + (size_t)kTP * 4 * 3 + 64;                // lambda, weights, row sums
  }
};

__device__ __forceinline__ float softplus_f(float t) { return t > 30.0f ? t : log1pf(expf(t)); }

template <int DP>
__global__ void __launch_bounds__(kThreads, 1)
soft_dl_sparse_kernel(Args A) {
  using L = Lay<DP>;
  constexpr int RS = L::RS;
  extern __shared__ double sdl_smem[];
  const int K = A.K, KW = K / 32;
  double* acc = sdl_smem;                          // [K]
  float* Xs = (float*)(acc + K);                   // [kTP][RS]
  float* Rs = Xs + kTP * RS;                       // [kTP][RS]
  float* Wb = Rs + kTP * RS;                       // [2][kCA][RS]
  uint32_t* bm = (uint32_t*)(Wb + 2 * kCA * RS);   // [kTP][KW] non-zero bitmap of the codes
  float* Hs = (float*)(bm + kTP * KW);             // [kTP][hidden]
  float* lam = Hs + kTP * A.hidden;                // [kTP]
  float* wts = lam + kTP;                          // [kTP]
  float* rsum = wts + kTP;                         // [kTP]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = lane & 15, pg = 2 * warp + (lane >> 4);   // GEMM block: anchors tx + 16a, points 4pg + q
  float* Z = A.zbuf + (size_t)blockIdx.x * kTP * K;         // this CTA's codes (dense, L2)
  const int nchunks = K / kCA;

  auto stage = [&](int c, int b) {   // dictionary rows [c kCA, +kCA) -> buffer b (cp.async 16 B)
    float* dst = Wb + (size_t)b * kCA * RS;
    const float* src = A.dict + (int64_t)c * kCA * DP;
    for (int x = tid; x < kCA * (DP / 4); x += kThreads) {
      const int r = x / (DP / 4), k4 = x % (DP / 4);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + r * RS + 4 * k4)),
                   "l"(src + (int64_t)r * DP + 4 * k4)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  for (int64_t i = blockIdx.x; i < A.n_dist; i += gridDim.x) {
    const int64_t s = A.offsets[i], e = A.offsets[i + 1];
    __syncthreads();   // previous distribution's readers of acc are done
    for (int j = tid; j < K; j += kThreads) acc[j] = 0.0;
    bool nonfinite = false, negative = false;
    double msum = 0.0;
    for (int64_t t0 = s; t0 < e; t0 += kTP) {
      const int np = (int)min((int64_t)kTP, e - t0);
      __syncthreads();   // previous tile's readers are done
      for (int x = tid; x < kTP * DP; x += kThreads) {
        const int p = x / DP, k = x % DP;
        float v = 0.0f;
        if (p < np) {
          v = A.points[(t0 + p) * DP + k];
          nonfinite |= !isfinite(v);
        }
        Xs[p * RS + k] = v;
      }
      if (tid < kTP) {
        const float w = tid < np ? A.weights[t0 + tid] : 0.0f;
        if (tid < np) {
          nonfinite |= !isfinite(w);
          negative |= w < 0.0f;
          msum += (double)w;
        }
        wts[tid] = w;
      }
      for (int x = tid; x < kTP * KW; x += kThreads) bm[x] = 0u;   // z^(0) = 0 (R#27)
      __syncthreads();
      // ---- lambda_p = softplus(v2 . relu(V1^T x_p + c1) + c2)  (R#24, R#26)
      for (int x = tid; x < kTP * A.hidden; x += kThreads) {
        const int p = x / A.hidden, c = x % A.hidden;
        float a = A.c1[c];
        for (int k = 0; k < DP; ++k) a = fmaf(Xs[p * RS + k], __ldg(A.V1 + (int64_t)k * A.hidden + c), a);
        Hs[x] = fmaxf(a, 0.0f);
      }
      __syncthreads();
      for (int p = warp; p < kTP; p += kThreads / 32) {
        float sd = 0.0f;
        for (int c = lane; c < A.hidden; c += 32) sd = fmaf(Hs[p * A.hidden + c], __ldg(A.v2 + c), sd);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
        if (lane == 0) lam[p] = softplus_f(sd + A.c2[0]);
      }
      __syncthreads();

      for (int layer = 0; layer < A.n_layers; ++layer) {
        stage(0, 0);   // first dictionary chunk of this layer's GEMM, under the sparse pass
        // ---- r = W z - x: 4 threads per point, DP/4 dims each; the non-zero z_j in increasing j
        {
          constexpr int DQ = DP / 4;
          const int p = tid >> 2, k0 = (tid & 3) * DQ;
          float r[DQ];
#pragma unroll
          for (int q = 0; q < DQ; ++q) r[q] = 0.0f;
          if (layer > 0) {
            for (int w = 0; w < KW; ++w) {
              uint32_t bits = bm[p * KW + w];
              while (bits) {
                const int j = 32 * w + __ffs(bits) - 1;
                bits &= bits - 1;
                const float zj = Z[(size_t)p * K + j];
                const float4* wr = reinterpret_cast<const float4*>(A.dict + (int64_t)j * DP + k0);
#pragma unroll
                for (int q4 = 0; q4 < DQ / 4; ++q4) {
                  const float4 w4 = __ldg(wr + q4);
                  r[4 * q4] = fmaf(zj, w4.x, r[4 * q4]);
                  r[4 * q4 + 1] = fmaf(zj, w4.y, r[4 * q4 + 1]);
                  r[4 * q4 + 2] = fmaf(zj, w4.z, r[4 * q4 + 2]);
                  r[4 * q4 + 3] = fmaf(zj, w4.w, r[4 * q4 + 3]);
                }
              }
            }
          }
#pragma unroll
          for (int q = 0; q < DQ; ++q) Rs[p * RS + k0 + q] = r[q] - Xs[p * RS + k0 + q];
        }
        __syncthreads();   // R complete; the bitmap is rebuilt by the GEMM epilogue below
        for (int x = tid; x < kTP * KW; x += kThreads) bm[x] = 0u;
        // ---- g = W^T r per 64-anchor chunk; z <- max(0, z - g - lambda)
        const float* rr = Rs + 4 * pg * RS;
        for (int c = 0; c < nchunks; ++c) {
          if (c + 1 < nchunks) {
            stage(c + 1, (c + 1) & 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
          }
          __syncthreads();   // chunk c visible; (c = 0) the bitmap cleared
          const float* wr = Wb + (size_t)(c & 1) * kCA * RS + tx * RS;
          float2 g2[4][4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int a = 0; a < 4; ++a) g2[q][a] = make_float2(0.0f, 0.0f);
#pragma unroll 2
          for (int k = 0; k < DP; k += 4) {
            float4 rv[4], wv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) rv[q] = *reinterpret_cast<const float4*>(rr + q * RS + k);
#pragma unroll
            for (int a = 0; a < 4; ++a) wv[a] = *reinterpret_cast<const float4*>(wr + 16 * a * RS + k);
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                g2[q][a] = ffma2(make_float2(rv[q].x, rv[q].y), make_float2(wv[a].x, wv[a].y), g2[q][a]);
                g2[q][a] = ffma2(make_float2(rv[q].z, rv[q].w), make_float2(wv[a].z, wv[a].w), g2[q][a]);
              }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int p = 4 * pg + q;
            const float lp = lam[p];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const int j = c * kCA + 16 * a + tx;
              float* zp = Z + (size_t)p * K + j;
              const float zo = layer > 0 ? *zp : 0.0f;
              const float zn = fmaxf(0.0f, (zo - (g2[q][a].x + g2[q][a].y)) - lp);
              *zp = zn;
              if (zn > 0.0f) atomicOr(&bm[p * KW + (j >> 5)], 1u << (j & 31));
            }
          }
          __syncthreads();   // buffer c & 1 is refilled by the next iteration's prefetch
        }
      }
      __syncthreads();   // codes and bitmap of the tile complete
      // ---- row sums in increasing j (warp per point, non-zeros only), the uniform fallback
      for (int p = warp; p < kTP; p += kThreads / 32) {
        float sm = 0.0f;
        for (int w = lane; w < KW; w += 32) {
          uint32_t bits = bm[p * KW + w];
          while (bits) {
            const int j = 32 * w + __ffs(bits) - 1;
            bits &= bits - 1;
            sm += Z[(size_t)p * K + j];
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
        if (lane == 0) rsum[p] = sm;
      }
      __syncthreads();
      if (tid < np && !(rsum[tid] > 0.0f)) atomicOr(A.status, ASOT_FLAG_SOFT_FALLBACK);
      // ---- codes (z / sum z) and the fp64 point-order histogram: thread per bin j
      const float unif = 1.0f / (float)K;
      for (int j = tid; j < K; j += kThreads) {
        double a = acc[j];
        for (int p = 0; p < np; ++p) {   // point order
          float z;
          if (!(rsum[p] > 0.0f)) z = unif;
          else z = (bm[p * KW + (j >> 5)] >> (j & 31)) & 1u ? Z[(size_t)p * K + j] / rsum[p] : 0.0f;
          if (A.codes) A.codes[(t0 + p) * K + j] = z;
          a += (double)wts[p] * (double)z;
        }
        acc[j] = a;
      }
    }
    __syncthreads();
    for (int j = tid; j < K; j += kThreads) A.H[i * K + j] = (float)acc[j];
    if (__syncthreads_or(nonfinite) && tid == 0) atomicOr(A.status, ASOT_FLAG_NONFINITE_INPUT);
    if (__syncthreads_or(negative) && tid == 0) atomicOr(A.status, ASOT_FLAG_BAD_MASS);
    if (tid < kTP) {   // threads < kTP hold the weight partial sums
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) msum += __shfl_xor_sync(0xffffffffu, msum, o);
      __syncwarp();
    }
    __shared__ double ms2[2];
    if (tid == 0 || tid == 32) ms2[tid >> 5] = msum;
    __syncthreads();
    if (tid == 0) {
      if (e <= s) atomicOr(A.status, ASOT_FLAG_EMPTY_DIST);
      else if (fabs((ms2[0] + ms2[1]) - 1.0) > 1e-5) atomicOr(A.status, ASOT_FLAG_BAD_MASS);
    }
  }
}

}  // namespace softdl

bool soft_dl_sparse_supported(int dim, int K) { return (dim == 64 || dim == 128) && K >= 256 && K % 64 == 0 && K <= 1024; }

int soft_dl_sparse_grid(int sms) { return sms; }

size_t soft_dl_sparse_workspace_bytes(int K, int sms) { return (size_t)soft_dl_sparse_grid(sms) * softdl::kTP * K * 4; }

cudaError_t launch_soft_dl_sparse(const float* points, const int64_t* offsets, const float* weights, int64_t n_dist,
                                  int dim, const float* dict, int K, int n_layers, int hidden, const float* V1,
                                  const float* c1, const float* v2, const float* c2, float* H, float* codes,
                                  float* zbuf, uint32_t* status, int sms, cudaStream_t s) {
  softdl::Args A{points, offsets, weights, n_dist, K, hidden, V1, c1, v2, c2, dict, n_layers, H, codes, zbuf, status};
  const int grid = (int)(n_dist < soft_dl_sparse_grid(sms) ? n_dist : soft_dl_sparse_grid(sms));
  if (grid < 1) return cudaSuccess;
  if (dim == 64) {
    const size_t smem = softdl::Lay<64>::bytes(K, hidden);
    cudaError_t e = cudaFuncSetAttribute(softdl::soft_dl_sparse_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    softdl::soft_dl_sparse_kernel<64><<<grid, softdl::kThreads, smem, s>>>(A);
  } else {
    const size_t smem = softdl::Lay<128>::bytes(K, hidden);
    cudaError_t e = cudaFuncSetAttribute(softdl::soft_dl_sparse_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    softdl::soft_dl_sparse_kernel<128><<<grid, softdl::kThreads, smem, s>>>(A);
  }
  return cudaGetLastError();
}

}  // namespace asot
