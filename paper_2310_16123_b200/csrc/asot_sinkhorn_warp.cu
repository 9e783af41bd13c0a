// asot_sinkhorn_warp.cu -- steps a5 + a6 for small anchor sets (K < 32) in fp32 on CUDA cores,
// one group of LP = 8 / 16 / 32 lanes per pair.
//
// Same recurrence and conventions as the fp32 CUDA-core kernel (asot_sinkhorn_simt.cu; P:179-183,
// S:61-62, R#4, R#5, R#11, R#12): v0 = 1, exactly L iterations of u = a / (K v), v = b / (K^T u)
// with 0/x = 0 and denominators clamped into [FLT_MIN, 2^126] and flagged, then
// d = sum_c v_c ((K (.) C_s) u)_c with the last v-update fused (K and C_s symmetric).
//
// Why a separate kernel: at K < 32 one pair's whole state is K floats, so the batched GEMM form
// (tensor-core tiles of 128 pairs, or the CUDA-core kernel's 1024-pair CTAs) leaves c1
// (N = 64: 2,016 pairs = 16 tiles) on 16 SMs running 2L dependent phases of ~3.4k cycles each.
// Here lane r of a pair's group owns anchor r: its column of K and of K (.) C_s sit in registers
// for the whole call, the current scaling is exchanged through LP floats of shared memory
// (one store, LP/4 broadcast float4 loads) and each half-iteration is LP FMAs and one
// reciprocal per lane -- ~260 cycles, with thousands of pairs in flight across all SMs.  The dot
// products run in the CUDA-core kernel's order (c = 0 .. K-1, fmaf from 0); the divide is
// m * rcp.approx(den) (<= 1 ulp, as in the tensor-core epilogues) instead of the IEEE divide,
// which alone took a third of the time at c1.  (Above 2^126 the approximate reciprocal would be
// flushed to 0 where the IEEE divide returns a subnormal: such denominators are clamped to 2^126
// and flagged, as in every tensor-core kernel.)
#include <cfloat>

#include "asot_internal.cuh"

namespace asot {
namespace warp {

constexpr int kThreads = 256;

// (min 1 block per SM: c1's 2,016 pairs x 16 lanes fill fewer than 148 blocks anyway, and the
// default register heuristic spilled the LP = 16 instance at 64 registers)
template <int LP>
__global__ void __launch_bounds__(kThreads, 1)
sinkhorn_warp_kernel(PairSource ps, PairSink out, const float* __restrict__ H, int K,
                     const float* __restrict__ Gp, const float* __restrict__ GCp, int kp, int iters) {
  if (dense_skipped(out)) return;   // the small-support kernel serves this call (R#36)
  __shared__ __align__(16) float xs[2][kThreads];   // double-buffered: one __syncwarp per step
  const int r = threadIdx.x % LP;                                  // anchor owned by this lane
  const int64_t slot = ((int64_t)blockIdx.x * kThreads + threadIdx.x) / LP;
  float* xg0 = &xs[0][threadIdx.x - r];                            // this pair's LP floats
  float* xg1 = &xs[1][threadIdx.x - r];
  const bool in = r < K;

  // columns r of K and K (.) C_s (row-padded images Gp[c][r], c < K; zeros past K)
  float g[LP], gc[LP];
#pragma unroll
  for (int c = 0; c < LP; ++c) {
    g[c] = (c < K && in) ? __ldg(Gp + (size_t)c * kp + r) : 0.0f;
    gc[c] = (c < K && in) ? __ldg(GCp + (size_t)c * kp + r) : 0.0f;
  }
  int i = 0, j = 0;
  const bool live = slot < ps.n_slots;
  const bool valid = live && decode_slot(ps, slot, i, j);          // a = H[i] on the u side
  const float a = (valid && in) ? __ldg(H + (int64_t)i * K + r) : 0.0f;
  const float b = (valid && in) ? __ldg(H + (int64_t)j * K + r) : 0.0f;

  bool clamped = false;
  const bool apos = a > 0.0f, bpos = b > 0.0f;   // loop-invariant: 0/x = 0 (R#11)
  auto divide = [&](float m, bool mpos, float den) {   // clamp + flag (R#12)
    // den clamped into [FLT_MIN, 2^126]: rcp.approx.ftz then never overflows or flushes
    const float q = div_clamped(m, den, clamped);
    return mpos ? q : 0.0f;
  };
  // y = sum_c col[c] * x_c over the group's shared vector, c = 0 .. LP-1 in order
  auto dot = [&](const float* xg, const float (&col)[LP]) {
    float y = 0.0f;
#pragma unroll
    for (int c4 = 0; c4 < LP; c4 += 4) {
      const float4 x = *reinterpret_cast<const float4*>(xg + c4);
      y = fmaf(col[c4], x.x, y);
      y = fmaf(col[c4 + 1], x.y, y);
      y = fmaf(col[c4 + 2], x.z, y);
      y = fmaf(col[c4 + 3], x.w, y);
    }
    return y;
  };

  float v = in ? 1.0f : 0.0f;   // v0 = 1 on real anchors (R#4)
  float u = 0.0f;
  // buffer 0 carries v, buffer 1 carries u: a buffer is rewritten only after the __syncwarp that
  // follows the other buffer's store, which every lane passes after finishing its reads
  for (int it = 0; it < iters; ++it) {
    xg0[r] = v;
    __syncwarp();
    u = divide(a, apos, dot(xg0, g));
    if (it + 1 == iters) break;
    xg1[r] = u;
    __syncwarp();
    v = divide(b, bpos, dot(xg1, g));
  }
  // last v-update fused with the cost: part_r = v_r ((K (.) C_s) u)_r
  xg1[r] = u;
  __syncwarp();
  float part = divide(b, bpos, dot(xg1, g)) * dot(xg1, gc);
#pragma unroll
  for (int o = LP / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
  if (r == 0 && live) write_result(out, slot, valid, i, j, part);
}

template <int LP>
cudaError_t launch_lp(const PairSource& ps, const PairSink& out, const float* H, int K, const float* Gp,
                      const float* GCp, int kp, int iters, cudaStream_t s) {
  const int64_t threads = ps.n_slots * LP;
  const int64_t blocks = (threads + kThreads - 1) / kThreads;
  if (blocks == 0) return cudaSuccess;
  sinkhorn_warp_kernel<LP><<<(unsigned)blocks, kThreads, 0, s>>>(ps, out, H, K, Gp, GCp, kp, iters);
  return cudaGetLastError();
}

}  // namespace warp

bool sinkhorn_warp_supported(int K) { return K >= 1 && K < 32; }

// Gp / GCp: the CUDA-core kernel's row-padded images (launch_gibbs_prep_simt, row stride simt_kpad(K)).
cudaError_t launch_sinkhorn_warp(const PairSource& ps, const PairSink& out, const float* H, int K,
                                 const float* Gp, const float* GCp, int iters, cudaStream_t s) {
  const int kp = simt_kpad(K);
  if (K <= 8) return warp::launch_lp<8>(ps, out, H, K, Gp, GCp, kp, iters, s);
  if (K <= 16) return warp::launch_lp<16>(ps, out, H, K, Gp, GCp, kp, iters, s);
  return warp::launch_lp<32>(ps, out, H, K, Gp, GCp, kp, iters, s);
}

}  // namespace asot
