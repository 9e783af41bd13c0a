// asot_sinkhorn_simt.cu -- steps a5 + a6 on CUDA cores in fp32 (ASOT_PREC_FP32 path, any K <= 1024).
//
// Batched Sinkhorn on the shared Gibbs kernel:
//   U = A / (K V),  V = B / (K^T U),  V^(0) = 1 (R#4), exactly L iterations (R#5),
//   0/x = 0 (R#11), denominators below FLT_MIN clamped and flagged (R#12);
// then d = u^T ((K (.) C_s) v) (R#3, R#6).
// One CTA owns 16 pairs.  The scalings of those 16 pairs live in shared memory for all L
// iterations ([K][16] transposed so one LDS.128 feeds 4 pairs).  Each thread owns anchors
// r = tid + 256 m and accumulates (K v)_r for all 16 pairs in registers while streaming the
// symmetric K row-wise (coalesced, L2-resident: every CTA reads the same K x K matrix).
#include <cfloat>

#include "asot_internal.cuh"

namespace asot {

constexpr int kSimtPairs = 16;
constexpr int kSimtThreads = 256;
constexpr int kSimtMaxRows = kMaxAnchors / kSimtThreads;  // 4

// acc[m][p] = sum_c Gm[c, r_m] * X[c][p]  (Gm symmetric: Gm[c, r] = Gm[r, c])
__device__ __forceinline__ void simt_matvec(const float* __restrict__ Gm, const float* X, int K,
                                            float (&acc)[kSimtMaxRows][kSimtPairs]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int m = 0; m < kSimtMaxRows; ++m)
#pragma unroll
    for (int p = 0; p < kSimtPairs; ++p) acc[m][p] = 0.0f;
  for (int c = 0; c < K; ++c) {
    const float4* x4 = reinterpret_cast<const float4*>(X + c * kSimtPairs);
    const float4 xa = x4[0], xb = x4[1], xc = x4[2], xd = x4[3];
    const float xv[kSimtPairs] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w,
                                  xc.x, xc.y, xc.z, xc.w, xd.x, xd.y, xd.z, xd.w};
#pragma unroll
    for (int m = 0; m < kSimtMaxRows; ++m) {
      const int r = tid + m * kSimtThreads;
      if (r < K) {
        const float g = __ldg(Gm + (int64_t)c * K + r);
#pragma unroll
        for (int p = 0; p < kSimtPairs; ++p) acc[m][p] = fmaf(g, xv[p], acc[m][p]);
      }
    }
  }
}

__global__ void __launch_bounds__(kSimtThreads)
sinkhorn_simt_kernel(PairSource ps, PairSink out, const float* __restrict__ H, int K,
                     const float* __restrict__ G, const float* __restrict__ GC, int iters) {
  extern __shared__ float4 simt_smem4[];
  float* Vt = reinterpret_cast<float*>(simt_smem4);  // [K][16]
  float* Ut = Vt + (size_t)K * kSimtPairs;           // [K][16]
  __shared__ int s_i[kSimtPairs], s_j[kSimtPairs];
  __shared__ int s_valid[kSimtPairs];
  __shared__ float s_red[kSimtThreads / 32][kSimtPairs];

  const int tid = threadIdx.x;
  const int64_t slot0 = (int64_t)blockIdx.x * kSimtPairs;
  if (tid < kSimtPairs) {
    int i = 0, j = 0;
    const bool v = decode_slot(ps, slot0 + tid, i, j);
    s_i[tid] = v ? i : 0;
    s_j[tid] = v ? j : 0;
    s_valid[tid] = v;
  }
  for (int e = tid; e < K * kSimtPairs; e += kSimtThreads) Vt[e] = 1.0f;  // v0 = 1
  __syncthreads();

  float acc[kSimtMaxRows][kSimtPairs];
  bool clamped = false;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      const float* X = half == 0 ? Vt : Ut;   // u-update reads v, v-update reads u
      float* Y = half == 0 ? Ut : Vt;
      const int* rows = half == 0 ? s_i : s_j;  // a = H[i] (u side), b = H[j] (v side)
      simt_matvec(G, X, K, acc);  // Y was last read before the previous half's barrier
#pragma unroll
      for (int m = 0; m < kSimtMaxRows; ++m) {
        const int r = tid + m * kSimtThreads;
        if (r < K) {
#pragma unroll
          for (int p = 0; p < kSimtPairs; ++p) {
            const float a = s_valid[p] ? H[(int64_t)rows[p] * K + r] : 0.0f;
            float den = acc[m][p];
            if (!(den >= FLT_MIN)) {
              clamped |= a > 0.0f;
              den = FLT_MIN;
            }
            Y[r * kSimtPairs + p] = a > 0.0f ? a / den : 0.0f;  // IEEE divide, 0/x = 0
          }
        }
      }
      __syncthreads();
    }
  }
  if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);

  // a6: d_p = sum_r u_r (GC v)_r
  simt_matvec(GC, Vt, K, acc);
  float part[kSimtPairs];
#pragma unroll
  for (int p = 0; p < kSimtPairs; ++p) part[p] = 0.0f;
#pragma unroll
  for (int m = 0; m < kSimtMaxRows; ++m) {
    const int r = tid + m * kSimtThreads;
    if (r < K) {
#pragma unroll
      for (int p = 0; p < kSimtPairs; ++p) part[p] = fmaf(Ut[r * kSimtPairs + p], acc[m][p], part[p]);
    }
  }
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int p = 0; p < kSimtPairs; ++p) {
    float v = part[p];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) s_red[warp][p] = v;
  }
  __syncthreads();
  if (tid < kSimtPairs) {
    float d = 0.0f;
#pragma unroll
    for (int w = 0; w < kSimtThreads / 32; ++w) d += s_red[w][tid];
    write_result(out, slot0 + tid, s_valid[tid] != 0, s_i[tid], s_j[tid], d);
  }
}

cudaError_t launch_sinkhorn_simt(const PairSource& ps, const PairSink& out, const float* H, int K,
                                 const float* G, const float* GC, int iters, cudaStream_t s) {
  const int64_t blocks = (ps.n_slots + kSimtPairs - 1) / kSimtPairs;
  if (blocks == 0) return cudaSuccess;
  const size_t smem = 2 * (size_t)K * kSimtPairs * sizeof(float);
  cudaFuncSetAttribute(sinkhorn_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  sinkhorn_simt_kernel<<<(unsigned)blocks, kSimtThreads, smem, s>>>(ps, out, H, K, G, GC, iters);
  return cudaGetLastError();
}

}  // namespace asot
