// asot_sinkhorn_tc.cu -- steps a5 + a6 on the 5th-gen tensor cores (tcgen05, kind::tf32), K <= 128.
//
// Batched Sinkhorn on the shared Gibbs kernel ("GPU parallelization version"):
//   U = A / (K V),  V = B / (K^T U)  with  V^(0) = 1, exactly L iterations (R#4, R#5),
// then d = <diag(u) K diag(v), C_s> = sum_c v_c ((K (.) C_s)^T u)_c  (R#3, R#6).
//
// Layout: pairs are the MMA M dimension.  A pair tile (128 slots, step a4) is one M = 128 MMA:
//   D[p, r] = sum_c X[p, c] * K[c, r]       (X = V^T or U^T, K symmetric)
// with X held in TENSOR MEMORY as the A operand (lane p = pair, column c = anchor, TF32 bits),
// the Gibbs kernel K (and K (.) C_s for the cost) resident in SHARED MEMORY as the B operand
// (K-major SWIZZLE_128B image staged once per CTA by a TMA bulk copy), and the fp32 accumulator
// D in TMEM.  The scalings of a tile never leave the SM for all 2L+1 MMA phases.
//
// Warp roles (512 threads): warps 0-7 own slot 0 and warps 8-15 slot 1 (one pair tile each);
// warp w reads TMEM lane quarter w%4 and the column half (w%8)/4, so each SMSP runs two
// independent instruction streams per slot.  After a slot barrier one elected thread issues
// that slot's tcgen05.mma chain and commits it to the slot's mbarrier.  While the tensor core
// computes one slot's product, the other slot's warps turn their accumulator into the next
// scaling (tcgen05.ld x16, double-buffered -> u = a / D with one MUFU.RCP per two anchors ->
// RNA rounding to TF32 (add half an ulp; the MMA truncates) -> tcgen05.st), so MMA and the elementwise divide overlap (ping-pong).
// Each pair lives in one TMEM lane; its two column halves are reduced in-thread and summed
// through SMEM once per tile.  The cost (a6): the last v-update writes v_L in place into D, two
// N = K/2 MMAs apply K (.) C_s to it (output into the consumed half of A), and the threads
// reduce sum_r u_r ((K (.) C_s) v)_r.
//
// TMEM map (columns): slot s: A at 2s*KP, D at 2s*KP + KP.  SMEM: [K image | KC image |
// marginal rows (8 a-rows, 16 b-rows, 1 dummy row) per slot | partial costs | mbarriers].
#include <cfloat>
#include <cstdlib>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace tc {

// Debug timeline (ASOT_TC_DEBUG_MODE=3): slot, event, phase -> clock64 for CTA 0's first tile.
__device__ long long g_tc_trace[2][4][512];

constexpr int kWarpsPerSlot = 8;
constexpr int kThreads = 2 * kWarpsPerSlot * 32;  // 512

using namespace ::asot::ptx;

// One slot's MMA chain with compile-time TMEM addresses (TMEM base is 0) and descriptors formed
// from the uniform SMEM base plus constant offsets.
//   MODE 0:    D_S = A_S (x) B          (N = KP, B = K image)
//   MODE 1, 2: A_S[:, 0:KP/2] = D_S (x) B[rows (MODE-1)*KP/2 ...]   (N = KP/2, B = K (.) C_s)
template <int KP, int S, int MODE>
__device__ __forceinline__ void issue_chain(uint32_t b_base) {
  constexpr uint32_t a0 = 2u * S * KP, d0 = a0 + KP;
  constexpr uint32_t idesc = make_idesc_tf32(128, MODE == 0 ? KP : KP / 2);
  constexpr uint32_t row0 = MODE == 0 ? 0u : (uint32_t)((MODE - 1) * (KP / 2) * 128);
  const uint64_t desc0 = make_sw128_desc(b_base + row0);
#pragma unroll
  for (int ks = 0; ks < KP / 8; ++ks) {
    const uint64_t desc = desc0 + (uint64_t)(((ks >> 2) * KP * 128 + (ks & 3) * 32) >> 4);
    if (MODE == 0)
      mma1_tf32_ts(d0, a0 + 8 * ks, desc, idesc, ks > 0 ? 1u : 0u);
    else
      mma1_tf32_ts(a0, d0 + 8 * ks, desc, idesc, ks > 0 ? 1u : 0u);
  }
}

template <int KP>
struct Smem {
  static constexpr int kRS = KP + 4;                      // marginal row stride (floats)
  static constexpr int kRows = 8 + 16 + 1;                // a-rows, b-rows, dummy row
  static constexpr size_t kImg = (size_t)KP * KP * 4;     // one operand image
  static constexpr size_t kMarg = (size_t)kRows * kRS * 4;
  static constexpr size_t kOffG = 0;
  static constexpr size_t kOffGC = kImg;
  static constexpr size_t kOffMarg = 2 * kImg;
  static constexpr size_t kOffRed = kOffMarg + 2 * kMarg;     // [2 slots][128] partial costs
  static constexpr size_t kOffBar = kOffRed + 2 * 128 * 4;
  static constexpr size_t kBytes = kOffBar + 64 + 1024;      // + alignment slack
};

// Per-thread view: thread = (slot s, TMEM lane quarter, column half h).  Columns are processed
// in chunks of 16 with the next chunk's tcgen05.ld in flight while the current one is computed.
template <int KP, int DBG>
__global__ void __launch_bounds__(kThreads, 1)
sinkhorn_tc_kernel(int64_t tile_begin, int64_t n_tiles, int64_t n_dist, PairSink out,
                   const float* __restrict__ H, int K, const uint32_t* __restrict__ g_img,
                   const uint32_t* __restrict__ gc_img, int iters) {
  using S = Smem<KP>;
  // All 512 columns: the allocation then necessarily starts at column 0 (one CTA per SM), so
  // every TMEM address below is a compile-time constant per slot and the MMA operands live in
  // uniform registers (no per-instruction R2UR / ELECT loops in the issue path).
  constexpr uint32_t kTmemCols = 512;
  constexpr uint32_t kIdesc = make_idesc_tf32(128, KP);
  constexpr uint32_t kIdescHalf = make_idesc_tf32(128, KP / 2);
  constexpr int kWG = kWarpsPerSlot * 32;
  constexpr int CW = KP / 2;    // columns per thread in the Sinkhorn phases
  constexpr int NC = CW / 16;   // x16 chunks per phase
  constexpr int CQ = KP / 4;    // columns per thread in each cost half
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base derived from smem_raw by pointer arithmetic, so the compiler keeps
  // the shared address space (LDS, not generic loads) for everything carved from it
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* marg = (float*)(smem + S::kOffMarg);
  float* red = (float*)(smem + S::kOffRed);
  uint64_t* bars = (uint64_t*)(smem + S::kOffBar);
  uint32_t* tmem_holder = (uint32_t*)(bars + 6);
  // Tensor-pipe turn token: the two slots issue their MMA chains strictly alternately, so one
  // slot's chain finishes while the other's is still queued and the epilogues interleave with
  // MMAs instead of both slots running in lockstep (issue blocks for about the chain's duration).
  volatile int* turn = (volatile int*)(bars + 7);
  volatile int* slot_done = turn + 1;  // [2]
  const uint32_t bar_g = smem_u32(&bars[0]);
  const uint32_t bar_mma0 = smem_u32(&bars[1]);  // +8*s

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = warp / kWarpsPerSlot;          // slot (pair tile) owned by this warpgroup pair
  const int sub = warp & 3;                    // TMEM lane quarter this warp may access
  const int h = (warp % kWarpsPerSlot) >> 2;   // column half
  const int p = sub * 32 + lane;               // pair slot within the tile == TMEM lane
  const int wg_tid = threadIdx.x - s * kWG;

  if (threadIdx.x == 0) {
    turn[0] = 0;
    slot_done[0] = 0;
    slot_done[1] = 0;
    mbar_init(bar_g, 1);
    mbar_init(bar_mma0, 1);
    mbar_init(bar_mma0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (tmem_base != 0) __trap();  // cannot happen with a full 512-column allocation
  if (threadIdx.x == 0) {  // stage K and K (.) C_s once per CTA (TMA bulk copies)
    mbar_expect_tx(bar_g, (uint32_t)(2 * S::kImg));
    constexpr uint32_t kChunk = 32768;
    for (uint32_t off = 0; off < S::kImg; off += kChunk) {
      const uint32_t n = (uint32_t)((S::kImg - off) < kChunk ? (S::kImg - off) : kChunk);
      bulk_g2s(smem_u32(smem + S::kOffG + off), (const uint8_t*)g_img + off, n, bar_g);
      bulk_g2s(smem_u32(smem + S::kOffGC + off), (const uint8_t*)gc_img + off, n, bar_g);
    }
  }

  float* mrows = marg + (size_t)s * S::kRows * S::kRS;
  const uint32_t lane_off = (uint32_t)(sub * 32) << 16;
  const uint32_t a_col = (uint32_t)(2 * s * KP);
  const uint32_t a_tmem = tmem_base + lane_off + a_col;   // this thread's lane of A
  const uint32_t d_tmem = a_tmem + KP;                    // this thread's lane of D
  const uint32_t bar_mma = bar_mma0 + 8 * s;
  const uint32_t g_base = smem_u32(smem + S::kOffG), gc_base = smem_u32(smem + S::kOffGC);
  uint32_t mma_par = 0;
  bool g_ready = false;

  // Slot barrier, then one elected thread issues this slot's MMA chain and commits it.
  //   mode 0:    D = A K                  (N = KP; A = V^T or U^T in TMEM, K in SMEM)
  //   mode 1, 2: A[:, 0:KP/2] = D (K (.) C_s)[:, half]   (N = KP/2; D holds v_L^T as the
  //              A operand, the output overwrites the half of u_L already consumed)
  auto issue_mma = [&](int mode, int fdbg) {
    tc_fence_before();
    named_bar_sync(1 + s, kWG);
    if (wg_tid < 32) {  // the slot's first warp, converged: one elected lane issues
      if (DBG == 3 && blockIdx.x == 0 && fdbg >= 0 && fdbg < 512 && lane == 0) g_tc_trace[s][3][fdbg] = clock64();
      if (!g_ready) {
        mbar_wait(bar_g, 0);
        g_ready = true;
      }
      while (*turn != s && !slot_done[s ^ 1]) __nanosleep(32);
      __syncwarp();
      if (DBG == 3 && blockIdx.x == 0 && fdbg >= 0 && fdbg < 512 && lane == 0) g_tc_trace[s][1][fdbg] = clock64();
      tc_fence_after();
      if (elect_one()) {
        if (DBG != 2) {
          if (s == 0) {
            if (mode == 0) issue_chain<KP, 0, 0>(g_base);
            else if (mode == 1) issue_chain<KP, 0, 1>(gc_base);
            else issue_chain<KP, 0, 2>(gc_base);
          } else {
            if (mode == 0) issue_chain<KP, 1, 0>(g_base);
            else if (mode == 1) issue_chain<KP, 1, 1>(gc_base);
            else issue_chain<KP, 1, 2>(gc_base);
          }
        }
        mma1_commit(bar_mma);
        *turn = s ^ 1;
      }
      __syncwarp();
    }
  };
  auto wait_mma = [&]() {
    mbar_wait(bar_mma, mma_par);
    mma_par ^= 1u;
    tc_fence_after();
  };

  for (int64_t tk = s;; tk += 2) {
    const int64_t tr = blockIdx.x + tk * (int64_t)gridDim.x;  // tile index within the range
    if (tr >= n_tiles) {
      if (wg_tid == 0) {
        slot_done[s] = 1;
        *turn = s ^ 1;
      }
      break;
    }
    const int64_t t = tile_begin + tr;
    // ---- tile init: marginal rows -> SMEM, V^T = 1 -> TMEM (A operand)
    int64_t bi, bj;
    block_pair_decode(t >> 1, num_blocks(n_dist), bi, bj);
    const int64_t i0 = bi * kBlockDist + (t & 1) * 8, j0 = bj * kBlockDist;
    named_bar_sync(1 + s, kWG);  // previous tile's readers are done with mrows / red
    for (int e = wg_tid; e < S::kRows * KP; e += kWG) {
      const int r = e / KP, c = e % KP;
      const int64_t row = r < 8 ? i0 + r : (r < 24 ? j0 + (r - 8) : n_dist);
      float v = (row < n_dist && c < K) ? H[row * K + c] : 0.0f;
      if (r == 24) v = c < K ? 1.0f / (float)K : 0.0f;  // dummy marginal for invalid slots
      mrows[r * S::kRS + c] = v;
    }
    int ii, jj;
    const bool valid = tile_slot_pair(t, p, n_dist, ii, jj);
    const float* arow = mrows + (valid ? (p >> 4) : 24) * S::kRS + h * CW;
    const float* brow = mrows + (valid ? 8 + (p & 15) : 24) * S::kRS + h * CW;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      uint32_t ones[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) ones[e] = (h * CW + c * 16 + e < K) ? 0x3f800000u : 0u;
      tmem_st16(a_tmem + h * CW + c * 16, ones);
    }
    tmem_wait_st();
    issue_mma(0, -1);  // (its barrier also publishes mrows to the slot's warps)

    for (int f = 0; f < 2 * iters; ++f) {
      wait_mma();
      if (DBG == 3 && blockIdx.x == 0 && tk < 2 && wg_tid == 0 && f < 512) g_tc_trace[s][0][f] = clock64();
      const float* mrow = (f & 1) ? brow : arow;  // u-update: a = H[i]; v-update: b = H[j]
      // u / v scalings go back to A (next MMA operand); the last v_L goes into D in place
      const uint32_t dst = ((f == 2 * iters - 1) ? d_tmem : a_tmem) + h * CW;
      const uint32_t src = d_tmem + h * CW;
      if (DBG == 1) {
        if (f != 2 * iters - 1) issue_mma(0, -1);
        continue;
      }
      uint32_t d[2][16];
      tmem_ld16u(src, d[0]);
      tmem_wait_ld();
      reg_fence16(d[0]);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (c + 1 < NC) tmem_ld16u(src + (c + 1) * 16, d[(c + 1) & 1]);
        const uint32_t* dc = d[c & 1];
        uint32_t o[16];
        const float4* m4 = reinterpret_cast<const float4*>(mrow + c * 16);
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const float4 mq = m4[e >> 2];
          const float m0 = (e & 2) ? mq.z : mq.x, m1 = (e & 2) ? mq.w : mq.y;
          // x = m / D for two anchors with one MUFU: r = 1/(D0 D1), m0/D0 = m0 D1 r, m1/D1 = m1 D0 r.
          // D > 0 by construction (padded K = 1, dummy marginals); m = 0 gives exactly 0 (R#11).
          const float d0 = __uint_as_float(dc[e]), d1 = __uint_as_float(dc[e + 1]);
          const float r = rcp_approx(d0 * d1);
          const float2 x = fmul2(fmul2(make_float2(m0, m1), make_float2(d1, d0)), make_float2(r, r));
          o[e] = tf32_rna_pre(x.x);
          o[e + 1] = tf32_rna_pre(x.y);
          if (DBG == 4) {  // diagnostics: TMEM traffic without the arithmetic
            o[e] = dc[e];
            o[e + 1] = dc[e + 1];
          }
        }
        if (DBG == 5) {  // diagnostics: arithmetic and loads without the TMEM stores
          uint32_t acc5 = 0;
#pragma unroll
          for (int e = 0; e < 16; ++e) acc5 ^= o[e];
          if (acc5 == 0x12345678u && iters < 0) g_tc_trace[0][0][0] = acc5;
        } else {
          tmem_st16(dst + c * 16, o);
        }
        if (c + 1 < NC) {
          tmem_wait_ld();
          reg_fence16(d[(c + 1) & 1]);
        }
      }
      tmem_wait_st();
      if (f != 2 * iters - 1) issue_mma(0, (DBG == 3 && tk < 2) ? f : -1);
      if (DBG == 3 && blockIdx.x == 0 && tk < 2 && wg_tid == 0 && f < 512) g_tc_trace[s][2][f] = clock64();
    }
    // ---- cost (a6): d = sum_r u_r ((K (.) C_s) v)_r with u_L in A and v_L in D, in two halves
    // of N = KP/2 so the product can land in the already-consumed half of A.  Thread half h
    // covers columns [h KP/4, (h+1) KP/4) of each half; the two partials meet in SMEM.
    float ust[CQ];
#pragma unroll
    for (int c = 0; c < CQ / 8; ++c) tmem_ld8(a_tmem + h * CQ + 8 * c, &ust[8 * c]);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < CQ; ++e) ust[e] = tf32_mask(ust[e]);
    issue_mma(1, -1);
    wait_mma();
    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < CQ / 8; ++c) {
      float g[8];
      tmem_ld8(a_tmem + h * CQ + 8 * c, g);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fmaf(ust[8 * c + e], g[e], acc);
    }
    issue_mma(2, -1);
    wait_mma();
#pragma unroll
    for (int c = 0; c < CQ / 8; ++c) {
      float g[8], u[8];
      tmem_ld8(a_tmem + h * CQ + 8 * c, g);
      tmem_ld8(a_tmem + KP / 2 + h * CQ + 8 * c, u);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fmaf(tf32_mask(u[e]), g[e], acc);
    }
    float* rs = red + s * 128;
    if (h == 1) rs[p] = acc;
    named_bar_sync(1 + s, kWG);
    if (h == 0) write_result(out, tr * kTileSlots + p, valid, ii, jj, acc + rs[p]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols)
                 : "memory");
  }
}

template <int KP>
static cudaError_t launch_kp(int64_t tile_begin, int64_t n_tiles, int64_t n_dist, const PairSink& out,
                             const float* H, int K, const uint32_t* g_img, const uint32_t* gc_img,
                             int iters, cudaStream_t s) {
  const size_t smem = Smem<KP>::kBytes;
  static const int dbg = getenv("ASOT_TC_DEBUG_MODE") ? atoi(getenv("ASOT_TC_DEBUG_MODE")) : 0;
  auto kern = dbg == 1 ? sinkhorn_tc_kernel<KP, 1> : dbg == 2 ? sinkhorn_tc_kernel<KP, 2>
            : dbg == 3 ? sinkhorn_tc_kernel<KP, 3> : dbg == 4 ? sinkhorn_tc_kernel<KP, 4>
            : dbg == 5 ? sinkhorn_tc_kernel<KP, 5> : sinkhorn_tc_kernel<KP, 0>;
  cudaError_t e = cudaFuncSetAttribute(kern,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (n_tiles + 1) / 2;
  if (grid > sms) grid = sms;
  if (grid < 1) return cudaSuccess;
  kern<<<(unsigned)grid, kThreads, smem, s>>>(tile_begin, n_tiles, n_dist, out, H, K,
                                                               g_img, gc_img, iters);
  return cudaGetLastError();
}

}  // namespace tc

bool sinkhorn_tc_supported(int K) { return K >= 1 && K <= 128; }

cudaError_t launch_sinkhorn_tc(int64_t tile_begin, int64_t tile_end, int64_t n_dist,
                               const PairSink& out, const float* H, int K, const uint32_t* g_img,
                               const uint32_t* gc_img, int iters, cudaStream_t s) {
  const int64_t n_tiles = tile_end - tile_begin;
  if (n_tiles <= 0) return cudaSuccess;
  switch (kpad32(K)) {
    case 32: return tc::launch_kp<32>(tile_begin, n_tiles, n_dist, out, H, K, g_img, gc_img, iters, s);
    case 64: return tc::launch_kp<64>(tile_begin, n_tiles, n_dist, out, H, K, g_img, gc_img, iters, s);
    case 96: return tc::launch_kp<96>(tile_begin, n_tiles, n_dist, out, H, K, g_img, gc_img, iters, s);
    case 128: return tc::launch_kp<128>(tile_begin, n_tiles, n_dist, out, H, K, g_img, gc_img, iters, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace asot

extern "C" int asot_debug_tc_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, asot::tc::g_tc_trace, sizeof(asot::tc::g_tc_trace));
}
