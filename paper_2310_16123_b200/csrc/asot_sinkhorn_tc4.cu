// asot_sinkhorn_tc4.cu -- steps a5 + a6 for 256 < K <= 1024: the HBM/L2-streamed GEMM form.
//
// Same recurrence as the resident kernels (R#3-R#6, R#11).  At K = 1024 neither the
// Gibbs kernel (4 MB TF32) nor one tile's scalings (128 pairs x 4 KB) fit on chip, so every
// phase is a GEMM  D[256 pairs x 1024] = X[256 x 1024] . K[1024 x 1024]  per CTA pair
// (tcgen05.mma.cta_group::2.kind::tf32, M = 256, N = 256 per instruction, both operands from
// SMEM) with the divide fused into the epilogue:
//   - X (the current scaling, TF32 bits in the no-swizzle K-major operand layout) lives in
//     per-CTA buffers in global memory (L2-resident: a rotation over three half-buffers at
//     K = 1024, see xhalf); K and K (.) C_s live in global
//     images pre-arranged so each (K-chunk, N-half) operand slice is one contiguous block;
//   - a producer warp streams 48 KB stages (A: 128 pairs x 32 anchors of X; B: this CTA's 256
//     output anchors x 32) with TMA bulk copies into a 4-stage mbarrier pipeline; the leader's
//     MMA warp waits for both CTAs' stages (the peer relays its "full" to the leader) and frees
//     them with multicast commits;
//   - each phase is two passes over N (512 anchors each, D = 512 TMEM columns); after a pass the
//     16 epilogue warps compute x = m / D (one MUFU per two anchors), RNA-round to TF32 and
//     write the next X to global; the last phase multiplies by K (.) C_s and reduces
//     sum_r u_r ((K (.) C_s) v)_r against u_L read back from global;
//   - K-chunks made only of padding anchors (K not a multiple of 32 * KC) are neither loaded
//     nor multiplied (x = 0 there).
#include <cfloat>
#include <cstdlib>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace tc4 {

using namespace ::asot::ptx;

// KP = K padded to 512 or 1024: NH = KP/512 passes per phase (N = 512 each), KC = KP/32 chunks
template <int KP>
struct Cfg {
  static constexpr int NH = KP / 512;
  static constexpr int KC = KP / 32;
  static constexpr uint32_t kXBytes = 128u * KP * 4u;             // one X buffer: 128 rows x KP x 4 B
  static constexpr size_t kImgRankBytes = (size_t)KP * KP * 2;    // one rank's half of a K image
};
constexpr int kEpiWarps = 16;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kThreads = kEpiThreads + 64;  // + producer warp + MMA (leader) / relay (peer) warp
constexpr int kStages = 4;
constexpr uint32_t kAChunk = 16384;          // 128 pair rows x 128 B (32 anchors)
constexpr uint32_t kBChunk = 32768;          // 2 N-subs x 128 anchor rows x 128 B
constexpr uint32_t kStageBytes = kAChunk + kBChunk;

struct Smem {
  static constexpr int kMRS = 512 + 4;  // marginal half-row stride (floats), 16-byte shift per row
  static constexpr size_t kOffStage = 0;
  static constexpr size_t kOffMarg = (size_t)kStages * kStageBytes;     // [16 rows][516] floats
  static constexpr size_t kOffRed = kOffMarg;                           // [4][128] floats (aliases marg)
  static constexpr size_t kOffBar = kOffMarg + (size_t)16 * kMRS * 4;
  static constexpr size_t kBytes = kOffBar + 256 + 1024;
  static_assert(kBytes <= 232448, "shared memory budget");
};

__host__ __device__ inline uint32_t sw_rows(uint32_t r, uint32_t kin) {  // [rows][128 B] block
  const uint32_t lin = r * 128u + kin * 4u;
  return lin ^ (((lin >> 7) & 7u) << 4);
}
// X buffer (A operand image) in the no-swizzle K-major core-matrix layout [k/4][128 rows][16 B]:
// a warp (32 consecutive pair rows) writes 512 contiguous bytes per 16-byte store, and each
// 32-anchor K-chunk is one contiguous 16 KB block for the TMA bulk load.  Descriptor: LBO (next
// core matrix along K) = 2048 B, SBO (next 8-row group) = 128 B.
__host__ __device__ inline uint32_t x_offset(uint32_t p, uint32_t k) { return (k >> 2) * 2048u + p * 16u + (k & 3) * 4u; }
__device__ __forceinline__ uint64_t make_noswz_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(2048u >> 4) << 16;  // LBO
  d |= (uint64_t)(128u >> 4) << 32;   // SBO
  d |= (uint64_t)1u << 46;            // version (sm_100); layout type 0 = SWIZZLE_NONE
  return d;
}
// K image of one rank: [nh NH][kc KC][ns 2][128 rows][128 B]; output anchor n = nh*512 + ns*256 + rank*128 + r
template <int KP>
__host__ __device__ inline uint32_t b_offset(uint32_t nh, uint32_t ns, uint32_t r, uint32_t k) {
  return ((nh * (uint32_t)Cfg<KP>::KC + (k >> 5)) * 2u + ns) * 16384u + sw_rows(r, k & 31);
}

// 16 consecutive anchors [k0, k0+16) (k0 % 4 == 0) of pair row p in an X image: four 16-byte chunks
__device__ __forceinline__ void x_load16(const uint8_t* xb, uint32_t p, uint32_t k0, float* v) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float4 q = *reinterpret_cast<const float4*>(xb + x_offset(p, k0 + 4 * c));
    v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
  }
}

// Debug timeline (ASOT_TC_DEBUG_MODE=3): [event][pass] for CTA 0's first tile:
//   0 issuer: first MMA of the pass issued, 1 issuer: last MMA issued,
//   2 epilogue woke (D ready), 3 epilogue done (after the barrier), 4 producer: first load issued
__device__ long long g_tc4_trace[5][256];
__device__ long long g_tc4_clock[4];  // clock_probe: (clock64, globaltimer) at start / end

template <int KP, int DBG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
sinkhorn_tc4_kernel(int64_t tile_begin, int64_t tile_end, int64_t n_dist, PairSink out,
                    const float* __restrict__ Hp, int K, const uint8_t* __restrict__ g_img,
                    const uint8_t* __restrict__ gc_img, uint8_t* __restrict__ xbuf, int iters,
                    const int32_t* __restrict__ units, const int64_t* __restrict__ n_dev) {
  if (dense_skipped(out)) return;   // the small-support kernel serves this call (R#36)
  using S = Smem;
  constexpr int NH = Cfg<KP>::NH, kKC = Cfg<KP>::KC;
  constexpr uint32_t kXBytes = Cfg<KP>::kXBytes;
  constexpr size_t kImgRankBytes = Cfg<KP>::kImgRankBytes;
  constexpr uint32_t kIdesc = make_idesc_tf32(256, 256);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = (uint64_t*)(smem + S::kOffBar);
  // bars: full[S], empty[S], peer_full[S] (leader), mma_done, tmem_free (leader), x_ready
  constexpr int S3 = 3 * kStages;
  static_assert((S3 + 4) * 8 <= 256, "barrier area");
  uint32_t* tmem_holder = (uint32_t*)(bars + S3 + 3);
  const uint32_t bar_full = smem_u32(&bars[0]), bar_empty = smem_u32(&bars[kStages]);
  const uint32_t bar_peer = smem_u32(&bars[2 * kStages]), bar_done = smem_u32(&bars[S3]);
  const uint32_t bar_free = smem_u32(&bars[S3 + 1]), bar_xr = smem_u32(&bars[S3 + 2]);
  const uint32_t stage0 = smem_u32(smem + S::kOffStage);

  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
      mbar_init(bar_peer + 8 * s, 1);
    }
    mbar_init(bar_done, 1);
    mbar_init(bar_free, 2);
    mbar_init(bar_xr, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  clock_probe(g_tc4_clock, 0);
  if (*tmem_holder != 0) __trap();

  uint8_t* xb = xbuf + (size_t)blockIdx.x * (2 * kXBytes);
  const int64_t bp_begin = tile_begin >> 1, bp_end = (tile_end + 1) >> 1;
  // block pairs kb = 0, 1, ... of the range, or (bucketed pair lists, tile mode) of the unit list
  int64_t n_kb = bp_end - bp_begin;
  if (units != nullptr && *n_dev < n_kb) n_kb = *n_dev;
  const int64_t cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int phases = 2 * iters + 1;
  // Where half h (anchors [512 h, 512 h + 512)) of X_f, the input of phase f, lives.  KP = 512:
  // ping-pong of whole buffers.  KP = 1024: a rotation over three half-buffers -- pass 0's
  // epilogue writes X_{f+1} half 0 into the third buffer while pass 1 still reads X_f; pass 1's
  // epilogue (after its MMAs completed) writes X_{f+1} half 1 over X_f half 0 -- so the working
  // set is 3 x 256 KB per CTA (111 MB over 148 CTAs) instead of 4 x 256 KB (148 MB).  The last
  // phase's half 1 goes to a fourth half-buffer: the cost phase reads u_L (X_{2L-1}) next to v_L
  // (X_{2L}).  Measured (ncu, c5 N = 300): DRAM writes 19.3 -> 16.2 GB per launch, reads
  // unchanged at 21.6 GB -- the two-die L2 still does not hold the set (L2 evict_last hints on
  // the X stores / bulk loads changed nothing and were dropped).

  auto xhalf = [&](int f, int h) -> uint8_t* {
    if constexpr (NH == 1) {
      return xb + (f & 1) * kXBytes;
    } else {
      const int idx = (f == phases - 1 && h == 1) ? 3 : (2 * f + h) % 3;
      return xb + (size_t)idx * (kXBytes / 2);
    }
  };
  constexpr int kHalfChunks = kKC / NH;   // 32-anchor chunks per half-buffer
  // 32-anchor input chunks holding real anchors: padded chunks (x = 0 there) are neither loaded
  // nor multiplied (K = 384: 12 of 16, K = 768: 24 of 32)
  const int kcn = (K + 31) / 32 < kKC ? (K + 31) / 32 : kKC;

  if (warp == kEpiWarps) {
    // ------------------------------------------------------------------ producer (TMA)
    if (lane == 0) {
      int64_t it = 0;
      uint32_t xr_par = 0;
      for (int64_t kb = cluster_id; kb < n_kb; kb += n_clusters) {
        const int64_t b = units != nullptr ? (int64_t)units[kb] : bp_begin + kb;
        for (int f = 0; f < phases; ++f) {

          const uint8_t* img = (f < phases - 1 ? g_img : gc_img) + rank * kImgRankBytes;
          mbar_wait(bar_xr, xr_par);  // X_in fully written (previous phase / tile init)
          xr_par ^= 1u;
          fence_proxy_async_global();
          for (int nh = 0; nh < NH; ++nh) {
            for (int kc = 0; kc < kcn; ++kc, ++it) {
              const int s = (int)(it % kStages);
              if (it >= kStages) mbar_wait(bar_empty + 8 * s, (uint32_t)((it / kStages - 1) & 1));
              if (DBG == 3 && blockIdx.x == 0 && b == bp_begin + cluster_id && kc == 0 && 2 * f + nh < 256)
                g_tc4_trace[4][2 * f + nh] = clock64();
              mbar_expect_tx(bar_full + 8 * s, kStageBytes);
              bulk_g2s(stage0 + s * kStageBytes, xhalf(f, kc / kHalfChunks) + (kc % kHalfChunks) * kAChunk, kAChunk,
                       bar_full + 8 * s);
              bulk_g2s(stage0 + s * kStageBytes + kAChunk, img + (size_t)(nh * kKC + kc) * kBChunk, kBChunk,
                       bar_full + 8 * s);
            }
          }
        }
      }
    }
  } else if (warp == kEpiWarps + 1) {
    // ------------------------------------------------------------------ MMA (leader) / relay (peer)
    int64_t it = 0;
    uint32_t free_par = 0;
    bool first = true;
    for (int64_t kb = cluster_id; kb < n_kb; kb += n_clusters) {
        const int64_t b = units != nullptr ? (int64_t)units[kb] : bp_begin + kb;
      for (int f = 0; f < phases; ++f) {
        for (int nh = 0; nh < NH; ++nh) {
          if (rank == 0 && !first) {
            mbar_wait(bar_free, free_par);  // both CTAs drained D of the previous pass
            free_par ^= 1u;
          }
          first = false;
          for (int kc = 0; kc < kcn; ++kc, ++it) {
            const int s = (int)(it % kStages);
            const uint32_t par = (uint32_t)((it / kStages) & 1);
            mbar_wait(bar_full + 8 * s, par);
            if (rank != 0) {
              if (lane == 0) mbar_arrive_cluster(mapa(bar_peer + 8 * s, 0));
              continue;
            }
            mbar_wait(bar_peer + 8 * s, par);
            tc_fence_after();
            if (DBG == 3 && blockIdx.x == 0 && b == bp_begin + cluster_id && lane == 0 && (kc == 0 || kc == kcn - 1) &&
                2 * f + nh < 256)
              g_tc4_trace[kc == 0 ? 0 : 1][2 * f + nh] = clock64();
            if (elect_one()) {
              const uint32_t a_base = stage0 + s * kStageBytes, b_base = a_base + kAChunk;
              const uint64_t a0 = make_noswz_desc(a_base), b0 = make_sw128_desc(b_base);
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
                for (int ns = 0; ns < 2; ++ns) {
                  if (DBG != 2)
                    mma2_tf32_ss((uint32_t)(ns * 256), a0 + (uint64_t)((ks * 4096) >> 4),
                                 b0 + (uint64_t)((ns * 16384 + ks * 32) >> 4), kIdesc, (kc | ks) ? 1u : 0u);
                }
              }
              mma2_commit_mc(bar_empty + 8 * s);
              if (kc == kcn - 1) mma2_commit_mc(bar_done);
            }
            __syncwarp();
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (16 warps)
    const int q = warp & 3, g = warp >> 2;  // TMEM lane quarter, column group (128 of a pass)
    const int p = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t free_remote = mapa(bar_free, 0);
    uint32_t done_par = 0;
    bool clamped = false;   // a denominator left [FLT_MIN, 2^126] on an anchor with mass
    for (int64_t kb = cluster_id; kb < n_kb; kb += n_clusters) {
        const int64_t b = units != nullptr ? (int64_t)units[kb] : bp_begin + kb;
      const int64_t t = 2 * b + rank;
      const bool t_in = units != nullptr || (t >= tile_begin && t < tile_end);
      int ii, jj;
      const bool valid = tile_slot_pair(t, p, n_dist, ii, jj) && t_in;
      // marginal rows of this tile: u side = distributions i0 + [0, 8), v side = j0 + [0, 16)
      int64_t bi, bj;
      block_pair_decode(b, num_blocks(n_dist), bi, bj);
      const int64_t i0 = bi * kBlockDist + rank * 8, j0 = bj * kBlockDist;
      // invalid slots read row 0 of the staged side (finite, discarded: MMA rows are independent)
      const int arow_s = valid ? (p >> 4) : 0, brow_s = valid ? (p & 15) : 0;
      float* marg = (float*)(smem + S::kOffMarg);
      // tile init: X_in of phase 0 = V^T = 1 on real anchors (padding stays 0), my row, anchors
      // [g*256, g*256+256)
      for (int k = g * (KP / 4); k < (g + 1) * (KP / 4); k += 4) {
        uint32_t v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (k + e < K) ? 0x3f800000u : 0u;
        stg128(xhalf(0, k / 512) + x_offset(p, k % 512), v[0], v[1], v[2], v[3]);
      }
      fence_proxy_async_global();
      named_bar_sync(1, kEpiThreads);
      if (threadIdx.x == 0) mbar_arrive_local(bar_xr);
      float acc = 0.0f;
      for (int f = 0; f < phases; ++f) {
        const bool cost_phase = f == phases - 1;

        // u-update: a = H[i] (8 rows); v-update: b = H[j] (16 rows)
        const int nrows = (f & 1) ? 16 : 8;
        const int64_t row0 = (f & 1) ? j0 : i0;
        const float* mrow = marg + ((f & 1) ? brow_s : arow_s) * S::kMRS;
        for (int nh = 0; nh < NH; ++nh) {
          if (!cost_phase) {
            // stage this pass's marginal half-rows (<= 32 KB) while the pass's MMAs run; the
            // previous epilogue's barrier guarantees nobody still reads the buffer
            for (int e = threadIdx.x; e < nrows * 128; e += kEpiThreads) {
              const int r = e >> 7, c4 = (e & 127) * 4;
              const int64_t row = row0 + r < n_dist ? row0 + r : n_dist;
              *reinterpret_cast<float4*>(marg + r * S::kMRS + c4) =
                  *reinterpret_cast<const float4*>(Hp + (size_t)row * KP + nh * 512 + c4);
            }
            named_bar_sync(1, kEpiThreads);
          }
          mbar_wait(bar_done, done_par);
          done_par ^= 1u;
          tc_fence_after();
          if (DBG == 3 && blockIdx.x == 0 && b == bp_begin + cluster_id && threadIdx.x == 0 && 2 * f + nh < 256)
            g_tc4_trace[2][2 * f + nh] = clock64();
          const uint32_t col0 = (uint32_t)(nh * 512 + g * 128);   // global anchor index of my first column
          uint8_t* xout = xhalf(f + 1, nh);                         // half nh of the next X
          const uint8_t* ubuf = xhalf(phases - 2, nh);              // u_L (cost phase only)
          const uint32_t tcol = lane_off + (uint32_t)(g * 128);   // my TMEM columns (N-subs = g>>1)
          if (DBG != 1) {
            uint32_t d[2][16];
            float4 mq[2][4];  // marginals of the next chunk are prefetched with its TMEM load
            tmem_ld16u(tcol, d[0]);
            if (!cost_phase) {
#pragma unroll
              for (int e = 0; e < 4; ++e) mq[0][e] = *reinterpret_cast<const float4*>(mrow + g * 128 + 4 * e);
            }
            tmem_wait_ld();
            reg_fence16(d[0]);
#pragma unroll 2
            for (int c = 0; c < 8; ++c) {
              if (c + 1 < 8) {
                tmem_ld16u(tcol + (c + 1) * 16, d[(c + 1) & 1]);
                if (!cost_phase) {
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    mq[(c + 1) & 1][e] = *reinterpret_cast<const float4*>(mrow + g * 128 + (c + 1) * 16 + 4 * e);
                }
              }
              const uint32_t* dc = d[c & 1];
              const uint32_t k0 = col0 - (uint32_t)(nh * 512) + c * 16;   // anchor within half nh
              if (!cost_phase) {
                float m[16];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float4 q4 = mq[c & 1][e];
                  m[4 * e] = q4.x; m[4 * e + 1] = q4.y; m[4 * e + 2] = q4.z; m[4 * e + 3] = q4.w;
                }
                // x = m / D, one MUFU per two anchors (epi_div_fast; S:62 clamp + flag when a
                // product D0 D1 leaves fp32 range; m = 0 -> exactly 0, R#11)
                uint32_t o[16];
                const bool bad = epi_div_fast<16>(m, *reinterpret_cast<const uint32_t(*)[16]>(dc), o);
                if (__builtin_expect(__any_sync(0xffffffffu, bad), 0)) {   // a product D0 D1 out of fp32 range (rare)
#pragma unroll
                  for (int s8 = 0; s8 < 16; s8 += 8) {
                    uint32_t d8[8];
                    tmem_ld8u(tcol + c * 16 + s8, d8);
                    tmem_wait_ld();
                    if (bad) epi_div_fix8(m + s8, d8, o + s8, clamped);
                  }
                }
#pragma unroll
                for (int e = 0; e < 16; e += 4) stg128(xout + x_offset(p, k0 + e), o[e], o[e + 1], o[e + 2], o[e + 3]);
              } else {
                float u[16];
                x_load16(ubuf, p, k0, u);
#pragma unroll
                for (int e = 0; e < 16; ++e) acc = fmaf(tf32_mask(u[e]), __uint_as_float(dc[e]), acc);
              }
              if (c + 1 < 8) {
                tmem_wait_ld();
                reg_fence16(d[(c + 1) & 1]);
              }
            }
          }
          if (!cost_phase && nh == NH - 1) fence_proxy_async_global();
          tc_fence_before();
          named_bar_sync(1, kEpiThreads);
          if (DBG == 3 && blockIdx.x == 0 && b == bp_begin + cluster_id && threadIdx.x == 0 && 2 * f + nh < 256)
            g_tc4_trace[3][2 * f + nh] = clock64();
          if (threadIdx.x == 0) {
            mbar_arrive_cluster(free_remote);
            if (!cost_phase && nh == NH - 1) mbar_arrive_local(bar_xr);
          }
        }
      }
      float* red = (float*)(smem + S::kOffRed);
      red[g * 128 + p] = acc;
      named_bar_sync(1, kEpiThreads);
      if (g == 0 && t_in)
        write_result(out, (units != nullptr ? 2 * kb + rank : t - tile_begin) * kTileSlots + p, valid, ii, jj,
                     red[p] + red[128 + p] + red[256 + p] + red[384 + p]);
      named_bar_sync(1, kEpiThreads);  // red reused by the next tile
    }
    if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
  }
  tc_fence_before();
  cluster_sync();
  clock_probe(g_tc4_clock, 1);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(0u) : "memory");
}

// ----------------------------------------------------------------------------- prep kernels
template <int KP>
__global__ void gibbs_prep_tc4_kernel(const float* __restrict__ cost, int K, float eps, uint8_t* __restrict__ g_img,
                                      uint8_t* __restrict__ gc_img) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < KP * KP; idx += gridDim.x * blockDim.x) {
    const int n = idx / KP, k = idx % KP;
    const bool in = n < K && k < K;
    const double c = in ? (double)cost[(int64_t)n * K + k] : 0.0;
    const double gv = in ? exp(-c / (double)eps) : 0.0;               // P:183  K := exp(-C_s / eps)
    const uint32_t gb = in ? tf32_rna_bits((float)gv) : 0x3f800000u;  // padding = 1 (R#12)
    const uint32_t gcb = in ? tf32_rna_bits((float)(gv * c)) : 0u;
    const uint32_t nh = n >> 9, ns = (n >> 8) & 1, rk = (n >> 7) & 1, r = n & 127;
    const size_t off = (size_t)rk * Cfg<KP>::kImgRankBytes + b_offset<KP>(nh, ns, r, k);
    *(uint32_t*)(g_img + off) = gb;
    *(uint32_t*)(gc_img + off) = gcb;
  }
}

// Marginal rows padded to 1024 anchors, plus a dummy row (index N) for invalid pair slots.
template <int KP>
__global__ void pad_marginals_kernel(const float* __restrict__ H, int64_t n_dist, int K, float* __restrict__ Hp) {
  const int64_t total = (n_dist + 1) * KP;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / KP;
    const int c = (int)(idx % KP);
    float v = 0.0f;
    if (c < K) v = row < n_dist ? H[row * K + c] : 1.0f / (float)K;
    Hp[idx] = v;
  }
}

}  // namespace tc4

int tc4_kpad(int K) { return K <= 512 ? 512 : 1024; }
bool sinkhorn_tc4_supported(int K) { return K > 256 && K <= 1024; }
size_t sinkhorn_tc4_image_bytes(int K) { const size_t kp = tc4_kpad(K); return kp * kp * 4; }
size_t sinkhorn_tc4_scratch_bytes(int K, int64_t n_dist, int sms) {
  const size_t kp = tc4_kpad(K);
  return (size_t)(n_dist + 1) * kp * 4 + 1024 + (size_t)sms * 2 * 128 * kp * 4;
}

cudaError_t launch_gibbs_prep_tc4(const float* cost, int K, float eps, uint8_t* g_img, uint8_t* gc_img,
                                  cudaStream_t s) {
  if (tc4_kpad(K) == 512) tc4::gibbs_prep_tc4_kernel<512><<<512, 256, 0, s>>>(cost, K, eps, g_img, gc_img);
  else tc4::gibbs_prep_tc4_kernel<1024><<<1024, 256, 0, s>>>(cost, K, eps, g_img, gc_img);
  return cudaGetLastError();
}

namespace tc4 {
template <int KP>
static cudaError_t launch_kp(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                             const float* H, int K, const uint8_t* g_img, const uint8_t* gc_img, uint8_t* scratch,
                             int iters, cudaStream_t s, const int32_t* units, const int64_t* n_dev) {
  float* Hp = (float*)scratch;
  uint8_t* xbuf = scratch + (((size_t)(n_dist + 1) * KP * 4 + 1023) & ~(size_t)1023);
  pad_marginals_kernel<KP><<<512, 256, 0, s>>>(H, n_dist, K, Hp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
#ifdef ASOT_DEBUG_KERNELS   // diagnostic variants (tools/): only in debug builds
  static const int dbg = getenv("ASOT_TC_DEBUG_MODE") ? atoi(getenv("ASOT_TC_DEBUG_MODE")) : 0;
  auto kern = dbg == 1 ? sinkhorn_tc4_kernel<KP, 1> : dbg == 2 ? sinkhorn_tc4_kernel<KP, 2>
            : dbg == 3 ? sinkhorn_tc4_kernel<KP, 3> : sinkhorn_tc4_kernel<KP, 0>;
#else
  auto kern = sinkhorn_tc4_kernel<KP, 0>;
#endif
  const size_t smem = Smem::kBytes;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_bp = ((tile_end + 1) >> 1) - (tile_begin >> 1);
  int64_t clusters = n_bp < sms / 2 ? n_bp : sms / 2;
  if (clusters < 1) clusters = 1;
  kern<<<(unsigned)(2 * clusters), kThreads, smem, s>>>(tile_begin, tile_end, n_dist, out, Hp, K, g_img, gc_img,
                                                        xbuf, iters, units, n_dev);
  return cudaGetLastError();
}
}  // namespace tc4

cudaError_t launch_sinkhorn_tc4(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const float* H, int K, const uint8_t* g_img, const uint8_t* gc_img, uint8_t* scratch,
                                int iters, cudaStream_t s, const int32_t* units, const int64_t* n_dev) {
  if (tile_end <= tile_begin) return cudaSuccess;
  if (tc4_kpad(K) == 512)
    return tc4::launch_kp<512>(tile_begin, tile_end, n_dist, out, H, K, g_img, gc_img, scratch, iters, s, units,
                               n_dev);
  return tc4::launch_kp<1024>(tile_begin, tile_end, n_dist, out, H, K, g_img, gc_img, scratch, iters, s, units,
                              n_dev);
}

}  // namespace asot

extern "C" int asot_debug_tc4_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, asot::tc4::g_tc4_trace, sizeof(asot::tc4::g_tc4_trace));
}

namespace asot {
cudaError_t read_kernel_clock_tc4(long long* host4) {
  return cudaMemcpyFromSymbol(host4, tc4::g_tc4_clock, 4 * sizeof(long long));
}
}  // namespace asot
