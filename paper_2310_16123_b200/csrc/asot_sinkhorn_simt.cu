// asot_sinkhorn_simt.cu -- steps a5 + a6 on CUDA cores in fp32 as a batched GEMM: the first fp32
// path, now the independent cross-check of the tensor-core pair-list modes (ASOT_PAIR_KERNEL=simt).
//
// Batched Sinkhorn on the shared Gibbs kernel:
//   U = A / (K V),  V = B / (K^T U),  V^(0) = 1 (R#4), exactly L iterations (R#5),
//   0/x = 0 (R#11), denominators below FLT_MIN clamped and flagged (R#12);
// then d = u^T ((K (.) C_s) v) (R#3, R#6), evaluated as sum_c v_c ((K (.) C_s) u)_c
// (K and C_s symmetric) so the last v-update is fused with the cost (v_L never stored).
//
// Each half-iteration is a CUDA-core GEMM  Y[KP x P] = K[KP x K] X[K x P]  over the CTA's P
// pairs followed by the elementwise divide.  X (the current scaling, [KP][P]) is the only
// shared-memory array (128 KB): every thread keeps its 4 rows x 16 pairs of Y in registers
// until the whole CTA has finished reading X, then overwrites X in place with m / Y.  Per
// reduction step a thread loads one float4 of a K row (coalesced across the warp, L1/L2
// resident: every CTA streams the same K x KP matrix) and four float4 of X (one pair group
// per warp: SMEM broadcasts) for 64 FMAs.  Marginals are read straight from the L2-resident H
// rows of the pair (no staging), so arbitrary pair lists work as well as tiles.
#include <cfloat>

#include "asot_internal.cuh"

namespace asot {
namespace simt {

constexpr int kThreads = 512;
constexpr int kTR = 4;    // rows per thread
constexpr int kTP = 16;   // pairs per thread

template <int KP>
struct Shape {
  static constexpr int P = 32768 / KP;          // pairs per CTA (X = KP x P x 4 B = 128 KB)
  static constexpr int RT = KP / kTR;           // row-threads (>= 32: one pair group per warp)
  static constexpr int PG = P / kTP;            // pair groups
  static_assert(RT * PG == kThreads, "thread shape");
  static_assert(RT % 32 == 0, "a warp must share one pair group");
  static constexpr size_t kSmem = (size_t)KP * P * 4;
};

// acc[rr][q] = sum_{c < K} Gp[c][r0 + rr] * X[c][p0 + q]   (Gp row-padded to KP, symmetric)
template <int KP>
__device__ __forceinline__ void gemm_tile(const float* __restrict__ Gp, const float* X, int K, int r0, int p0,
                                          float (&acc)[kTR][kTP]) {
  constexpr int P = Shape<KP>::P;
#pragma unroll
  for (int rr = 0; rr < kTR; ++rr)
#pragma unroll
    for (int q = 0; q < kTP; ++q) acc[rr][q] = 0.0f;
  const float4* g4 = reinterpret_cast<const float4*>(Gp + r0);
  float4 gn = __ldg(g4);
#pragma unroll 2
  for (int c = 0; c < K; ++c) {
    const float4 g = gn;
    if (c + 1 < K) gn = __ldg(g4 + (size_t)(c + 1) * (KP / 4));   // prefetch the next K row
    const float4* x4 = reinterpret_cast<const float4*>(X + (size_t)c * P + p0);
    float x[kTP];
#pragma unroll
    for (int v = 0; v < kTP / 4; ++v) {
      const float4 t = x4[v];
      x[4 * v] = t.x; x[4 * v + 1] = t.y; x[4 * v + 2] = t.z; x[4 * v + 3] = t.w;
    }
    const float gg[kTR] = {g.x, g.y, g.z, g.w};
#pragma unroll
    for (int rr = 0; rr < kTR; ++rr)
#pragma unroll
      for (int q = 0; q < kTP; ++q) acc[rr][q] = fmaf(gg[rr], x[q], acc[rr][q]);
  }
}

template <int KP>
__global__ void __launch_bounds__(kThreads, 1)
sinkhorn_simt_kernel(PairSource ps, PairSink out, const float* __restrict__ H, int K,
                     const float* __restrict__ Gp, const float* __restrict__ GCp, int iters) {
  if (dense_skipped(out)) return;   // the small-support kernel serves this call (R#36)
  using S = Shape<KP>;
  constexpr int P = S::P;
  extern __shared__ float4 simt_smem4[];
  float* X = reinterpret_cast<float*>(simt_smem4);   // [KP][P]
  __shared__ float red[kThreads / 32][kTP];
  __shared__ int s_i[P], s_j[P];                      // pair rows (-1: invalid slot)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tr = tid % S::RT, pg = tid / S::RT;
  const int r0 = tr * kTR, p0 = pg * kTP;
  const int64_t slot0 = (int64_t)blockIdx.x * P;

  for (int q = tid; q < P; q += kThreads) {   // a = H[i] on the u side, b = H[j]
    int i = 0, j = 0;
    const bool v = decode_slot(ps, slot0 + q, i, j);
    s_i[q] = v ? i : -1;
    s_j[q] = v ? j : -1;
  }
  for (int e = tid; e < KP * P; e += kThreads) X[e] = (e / P) < K ? 1.0f : 0.0f;   // v0 = 1
  __syncthreads();
  auto marg = [&](const int* rows, int q, int r) {
    const int row = rows[p0 + q];
    return (r < K && row >= 0) ? __ldg(H + (int64_t)row * K + r) : 0.0f;
  };

  bool clamped = false;
  float acc[kTR][kTP];
  // the scaling for rows r0..r0+3 from marginal m and denominator den (0/x = 0; clamp + flag)
  auto divide = [&](float m, float den) {
    if (!(den >= FLT_MIN)) {
      clamped |= m > 0.0f;
      den = FLT_MIN;
    }
    return m > 0.0f ? m / den : 0.0f;   // IEEE divide
  };
  for (int it = 0; it < iters; ++it) {
    // ---- u = a / (K v)
    gemm_tile<KP>(Gp, X, K, r0, p0, acc);
    __syncthreads();   // every thread is done reading X: overwrite in place
#pragma unroll
    for (int rr = 0; rr < kTR; ++rr) {
      const int r = r0 + rr;
#pragma unroll
      for (int q = 0; q < kTP; ++q) {
        X[(size_t)r * P + p0 + q] = divide(marg(s_i, q, r), acc[rr][q]);
      }
    }
    __syncthreads();
    if (it + 1 == iters) break;
    // ---- v = b / (K^T u)
    gemm_tile<KP>(Gp, X, K, r0, p0, acc);
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < kTR; ++rr) {
      const int r = r0 + rr;
#pragma unroll
      for (int q = 0; q < kTP; ++q) {
        X[(size_t)r * P + p0 + q] = divide(marg(s_j, q, r), acc[rr][q]);
      }
    }
    __syncthreads();
  }

  // ---- last v-update fused with the cost: d = sum_c v_c ((K (.) C_s) u)_c, v_c = b_c / (K u)_c,
  // in two passes of 8 pairs so both products fit in registers
  float part[kTP];
#pragma unroll
  for (int q = 0; q < kTP; ++q) part[q] = 0.0f;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    float a1[kTR][kTP / 2], a2[kTR][kTP / 2];
#pragma unroll
    for (int rr = 0; rr < kTR; ++rr)
#pragma unroll
      for (int q = 0; q < kTP / 2; ++q) a1[rr][q] = a2[rr][q] = 0.0f;
    const float4* g4 = reinterpret_cast<const float4*>(Gp + r0);
    const float4* gc4 = reinterpret_cast<const float4*>(GCp + r0);
#pragma unroll 2
    for (int c = 0; c < K; ++c) {
      const float4 g = __ldg(g4 + (size_t)c * (KP / 4)), gc = __ldg(gc4 + (size_t)c * (KP / 4));
      const float4* x4 = reinterpret_cast<const float4*>(X + (size_t)c * P + p0 + half * (kTP / 2));
      const float4 xa = x4[0], xb = x4[1];
      const float x[kTP / 2] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
      const float gg[kTR] = {g.x, g.y, g.z, g.w}, gcc[kTR] = {gc.x, gc.y, gc.z, gc.w};
#pragma unroll
      for (int rr = 0; rr < kTR; ++rr)
#pragma unroll
        for (int q = 0; q < kTP / 2; ++q) {
          a1[rr][q] = fmaf(gg[rr], x[q], a1[rr][q]);
          a2[rr][q] = fmaf(gcc[rr], x[q], a2[rr][q]);
        }
    }
#pragma unroll
    for (int rr = 0; rr < kTR; ++rr) {
      const int r = r0 + rr;
#pragma unroll
      for (int q = 0; q < kTP / 2; ++q) {
        const int qq = half * (kTP / 2) + q;
        part[qq] = fmaf(divide(marg(s_j, qq, r), a1[rr][q]), a2[rr][q], part[qq]);
      }
    }
  }
  if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
  // reduce over the RT row-threads of each pair group: warp shuffle, then across warps
#pragma unroll
  for (int q = 0; q < kTP; ++q) {
    float v = part[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    part[q] = v;
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < kTP; ++q) red[warp][q] = part[q];
  }
  __syncthreads();
  constexpr int WPG = S::RT / 32;   // warps per pair group
  if (tid < P) {
    const int g = tid / kTP, q = tid % kTP;
    float d = 0.0f;
    for (int w = 0; w < WPG; ++w) d += red[g * WPG + w][q];
    if (slot0 + tid < ps.n_slots)   // the last CTA's slots past the list / range are not outputs
      write_result(out, slot0 + tid, s_i[tid] >= 0, s_i[tid], s_j[tid], d);
  }
}

// Row-padded fp32 Gibbs kernel and K (.) C_s: Gp[c][r], r < KP (zeros beyond K), c < K.
__global__ void gibbs_prep_simt_kernel(const float* __restrict__ cost, int K, float eps, int kp,
                                       float* __restrict__ Gp, float* __restrict__ GCp) {
  const int64_t total = (int64_t)K * kp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / kp), r = (int)(idx % kp);
    const bool in = r < K;
    const double cv = in ? (double)cost[(int64_t)c * K + r] : 0.0;
    const double g = in ? exp(-cv / (double)eps) : 0.0;   // P:183  K := exp(-C_s / eps)
    Gp[idx] = (float)g;
    GCp[idx] = (float)(g * cv);
  }
}

template <int KP>
cudaError_t launch_kp(const PairSource& ps, const PairSink& out, const float* H, int K, const float* Gp,
                      const float* GCp, int iters, cudaStream_t s) {
  using S = Shape<KP>;
  const int64_t blocks = (ps.n_slots + S::P - 1) / S::P;
  if (blocks == 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(sinkhorn_simt_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)S::kSmem);
  if (e != cudaSuccess) return e;
  sinkhorn_simt_kernel<KP><<<(unsigned)blocks, kThreads, S::kSmem, s>>>(ps, out, H, K, Gp, GCp, iters);
  return cudaGetLastError();
}

}  // namespace simt

int simt_kpad(int K) { return K <= 128 ? 128 : K <= 256 ? 256 : K <= 512 ? 512 : 1024; }

cudaError_t launch_gibbs_prep_simt(const float* cost, int K, float eps, float* Gp, float* GCp, cudaStream_t s) {
  const int kp = simt_kpad(K);
  const int64_t total = (int64_t)K * kp;
  simt::gibbs_prep_simt_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, s>>>(
      cost, K, eps, kp, Gp, GCp);
  return cudaGetLastError();
}

cudaError_t launch_sinkhorn_simt(const PairSource& ps, const PairSink& out, const float* H, int K,
                                 const float* Gp, const float* GCp, int iters, cudaStream_t s) {
  switch (simt_kpad(K)) {
    case 128: return simt::launch_kp<128>(ps, out, H, K, Gp, GCp, iters, s);
    case 256: return simt::launch_kp<256>(ps, out, H, K, Gp, GCp, iters, s);
    case 512: return simt::launch_kp<512>(ps, out, H, K, Gp, GCp, iters, s);
    default: return simt::launch_kp<1024>(ps, out, H, K, Gp, GCp, iters, s);
  }
}

}  // namespace asot
