// asot_sinkhorn_tc5.cu -- steps a5 + a6 with fp32 accuracy for 128 < K <= 1024: the streamed GEMM
// form (as asot_sinkhorn_tc4.cu) with 3xTF32 operands -- the ASOT_PREC_FP32 path where the
// scalings of a tile do not fit on chip twice (R#22).
//
// Same recurrence (R#3-R#6, R#11): every phase is a GEMM D[256 pairs x KP] =
// X[256 x KP] . K[KP x KP] per CTA pair (tcgen05.mma.cta_group::2.kind::tf32, M = N = 256 per
// instruction, both operands from SMEM) evaluated as X_hi K_hi + X_lo K_hi + X_hi K_lo with
// X_hi = RNA_tf32(x), X_lo = x - X_hi (exact in fp32) and the same split of K (and of K (.) C_s
// for the cost).  Phases are KP/256 passes over N = 256 output anchors (D = 256 TMEM columns);
// a pass streams KP/32 K-chunks through a 3-stage TMA bulk-copy pipeline whose 64 KB stages hold
// [X_hi | X_lo | K_hi | K_lo] chunks (A: this CTA's 128 pair rows x 32 anchors; B: this CTA's 128
// of the pass's 256 output anchors x 32).  The epilogue computes x = m / D (rcp.approx, clamp +
// flag like the fp32 kernel), splits it and writes X_hi / X_lo of the next phase to per-CTA
// ping-pong images in global memory (L2-resident for KP = 256: 0.5 MB per CTA); the last phase
// multiplies v_L by K (.) C_s and reduces against u_L = hi + lo read back from global.
//
// Template variants: SPLIT = 3 (the fp32-accurate path above) or 1 (one TF32 pass: stages [X | K],
// 6 deep; the TF32 path for 256 < K <= 512 without padding to 1024), and EXPLICIT (pairs from an
// explicit (pair_i, pair_j) list -- SPEC batched_sinkhorn_fixed, asot_pairwise_sinkhorn -- with
// the marginals read per thread from the L2-resident padded H rows instead of staged per tile).
#include <cfloat>
#include <cstdlib>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace tc5 {

using namespace ::asot::ptx;

__device__ long long g_tc5_clock[4];  // clock_probe: (clock64, globaltimer) at start / end

constexpr int kEpiWarps = 16;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kThreads = kEpiThreads + 64;   // + producer warp + MMA (leader) / relay (peer) warp
constexpr uint32_t kChunk = 16384;           // 128 rows x 128 B (32 anchors, fp32)
constexpr uint32_t kStageRegion = 196608;    // 192 KB of stages: 3 x [A_hi|A_lo|B_hi|B_lo] or 6 x [A|B]

template <int SPLIT>
struct Pipe {
  static constexpr uint32_t kStageBytes = (SPLIT == 3 ? 4u : 2u) * kChunk;
  static constexpr int kStages = (int)(kStageRegion / kStageBytes);
};

template <int KP>
struct Cfg {
  static constexpr int NP = KP / 256;                       // passes per phase (N = 256 each)
  static constexpr int KC = KP / 32;                        // K-chunks per pass
  static constexpr uint32_t kXBytes = 128u * KP * 4u;       // one X image (hi or lo) of one CTA
  static constexpr size_t kImgRankBytes = (size_t)KP * KP * 2;  // one rank's half of one image
};

struct Smem {
  static constexpr int kMRS = 256 + 4;                                   // marginal row stride
  static constexpr size_t kOffStage = 0;
  static constexpr size_t kOffMarg = kStageRegion;                        // [16 rows][260] floats
  static constexpr size_t kOffRed = kOffMarg;                            // [4][128] (aliases marg)
  static constexpr size_t kOffBar = kOffMarg + (size_t)16 * kMRS * 4;
  static constexpr size_t kBytes = kOffBar + 512 + 1024;
  static_assert(kBytes <= 232448, "shared memory budget");
};

__host__ __device__ inline uint32_t sw_rows(uint32_t r, uint32_t kin) {
  const uint32_t lin = r * 128u + kin * 4u;
  return lin ^ (((lin >> 7) & 7u) << 4);
}
// X image: no-swizzle K-major core-matrix layout [k/4][128 rows][16 B]; each 32-anchor chunk is a
// contiguous 16 KB block (descriptor LBO 2048 B, SBO 128 B) -- as in the TF32 streamed kernel.
__host__ __device__ inline uint32_t x_offset(uint32_t p, uint32_t k) { return (k >> 2) * 2048u + p * 16u + (k & 3) * 4u; }
__device__ __forceinline__ uint64_t make_noswz_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(2048u >> 4) << 16;
  d |= (uint64_t)(128u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  return d;
}
// K image of one rank: [pass][kc][128 rows][128 B]; output anchor n = pass*256 + rank*128 + r.
template <int KP>
__host__ __device__ inline uint32_t b_offset(uint32_t pass, uint32_t r, uint32_t k) {
  return (pass * (uint32_t)Cfg<KP>::KC + (k >> 5)) * kChunk + sw_rows(r, k & 31);
}

template <int KP, int SPLIT, bool EXPLICIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
sinkhorn_tc5_kernel(int64_t tile_begin, int64_t tile_end, int64_t n_dist, PairSink out, PairSource ps,
                    const float* __restrict__ Hp, int K, const uint8_t* __restrict__ g_hi,
                    const uint8_t* __restrict__ g_lo, const uint8_t* __restrict__ gc_hi,
                    const uint8_t* __restrict__ gc_lo, uint8_t* __restrict__ xbuf, int iters) {
  if (dense_skipped(out)) return;   // the small-support kernel serves this call (R#36)
  using S = Smem;
  const int32_t* units = EXPLICIT ? nullptr : ps.units;   // bucketed pair lists (tile mode)
  const int64_t* n_dev = ps.n_dev;
  using C = Cfg<KP>;
  constexpr int kStages = Pipe<SPLIT>::kStages;
  constexpr uint32_t kStageBytes = Pipe<SPLIT>::kStageBytes;
  constexpr uint32_t kIdesc = make_idesc_tf32(256, 256);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = (uint64_t*)(smem + S::kOffBar);
  constexpr int S3 = 3 * kStages;
  static_assert((S3 + 4) * 8 <= 512, "barrier area");
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
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  clock_probe(g_tc5_clock, 0);
  const uint32_t tmem_base = *tmem_holder;

  // per-CTA X images: [side 2][hi, lo]
  uint8_t* xb = xbuf + (size_t)blockIdx.x * (4 * (size_t)C::kXBytes);
  auto ximg = [&](int side, int lo) { return xb + (size_t)(2 * side + lo) * C::kXBytes; };
  if (EXPLICIT && ps.n_dev != nullptr) {   // bucketed pair lists: the list length on the device
    if (*ps.n_dev < ps.n_slots) ps.n_slots = *ps.n_dev;
    const int64_t te = (ps.n_slots + kTileSlots - 1) / kTileSlots;
    if (te < tile_end) tile_end = te;
  }
  const int64_t bp_begin = tile_begin >> 1, bp_end = (tile_end + 1) >> 1;
  // block pairs kb = 0, 1, ... of the range, or (bucketed pair lists, tile mode) of the unit list
  int64_t n_kb = bp_end - bp_begin;
  if (units != nullptr && *n_dev < n_kb) n_kb = *n_dev;
  const int64_t cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int phases = 2 * iters + 1;
  // 32-anchor input chunks holding real anchors: padded chunks (x = 0 there) are skipped
  const int kcn = (K + 31) / 32 < C::KC ? (K + 31) / 32 : C::KC;

  if (warp == kEpiWarps) {
    // ------------------------------------------------------------------ producer (TMA)
    if (lane == 0) {
      int64_t it = 0;
      uint32_t xr_par = 0;
      for (int64_t kb = cluster_id; kb < n_kb; kb += n_clusters) {
        const int64_t b = units != nullptr ? (int64_t)units[kb] : bp_begin + kb;
        for (int f = 0; f < phases; ++f) {
          const uint8_t* xin_hi = ximg(f & 1, 0);
          const uint8_t* xin_lo = ximg(f & 1, 1);
          const bool cost = f == phases - 1;
          const uint8_t* bh = (cost ? gc_hi : g_hi) + rank * C::kImgRankBytes;
          const uint8_t* bl = (cost ? gc_lo : g_lo) + rank * C::kImgRankBytes;
          mbar_wait(bar_xr, xr_par);  // X_in fully written (previous phase / tile init)
          xr_par ^= 1u;
          fence_proxy_async_global();
          for (int pass = 0; pass < C::NP; ++pass) {
            for (int kc = 0; kc < kcn; ++kc, ++it) {
              const int s = (int)(it % kStages);
              if (it >= kStages) mbar_wait(bar_empty + 8 * s, (uint32_t)((it / kStages - 1) & 1));
              const uint32_t st = stage0 + s * kStageBytes;
              const size_t boff = (size_t)(pass * C::KC + kc) * kChunk;
              mbar_expect_tx(bar_full + 8 * s, kStageBytes);
              if (SPLIT == 3) {
                bulk_g2s(st, xin_hi + kc * kChunk, kChunk, bar_full + 8 * s);
                bulk_g2s(st + kChunk, xin_lo + kc * kChunk, kChunk, bar_full + 8 * s);
                bulk_g2s(st + 2 * kChunk, bh + boff, kChunk, bar_full + 8 * s);
                bulk_g2s(st + 3 * kChunk, bl + boff, kChunk, bar_full + 8 * s);
              } else {
                bulk_g2s(st, xin_hi + kc * kChunk, kChunk, bar_full + 8 * s);
                bulk_g2s(st + kChunk, bh + boff, kChunk, bar_full + 8 * s);
              }
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
        for (int pass = 0; pass < C::NP; ++pass) {
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
            if (elect_one()) {
              const uint32_t st = stage0 + s * kStageBytes;
              const uint64_t ahi = make_noswz_desc(st), alo = make_noswz_desc(st + kChunk);
              const uint64_t bhi = make_sw128_desc(st + (SPLIT == 3 ? 2 : 1) * kChunk);
              const uint64_t blo = make_sw128_desc(st + 3 * kChunk);
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
                const uint64_t ao = (uint64_t)((ks * 4096) >> 4), bo = (uint64_t)((ks * 32) >> 4);
                mma2_tf32_ss(tmem_base, ahi + ao, bhi + bo, kIdesc, (kc | ks) ? 1u : 0u);
                if (SPLIT == 3) {
                  mma2_tf32_ss(tmem_base, alo + ao, bhi + bo, kIdesc, 1u);
                  mma2_tf32_ss(tmem_base, ahi + ao, blo + bo, kIdesc, 1u);
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
    const int q = warp & 3, g = warp >> 2;  // TMEM lane quarter, column group (64 of a pass)
    const int p = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t free_remote = mapa(bar_free, 0);
    uint32_t done_par = 0;
    bool clamped = false;
    float* marg = (float*)(smem + S::kOffMarg);
    for (int64_t kb = cluster_id; kb < n_kb; kb += n_clusters) {
        const int64_t b = units != nullptr ? (int64_t)units[kb] : bp_begin + kb;
      const int64_t t = 2 * b + rank;
      const bool t_in = units != nullptr || (t >= tile_begin && t < tile_end);
      int ii = 0, jj = 0;
      bool valid;
      int64_t i0 = 0, j0 = 0;
      if (EXPLICIT) {
        valid = t_in && decode_slot(ps, (t - tile_begin) * kTileSlots + p, ii, jj);
      } else {
        valid = tile_slot_pair(t, p, n_dist, ii, jj) && t_in;
        int64_t bi, bj;
        block_pair_decode(b, num_blocks(n_dist), bi, bj);
        i0 = bi * kBlockDist + rank * 8;
        j0 = bj * kBlockDist;
      }
      // invalid slots read row 0 of the staged side / the dummy row (finite, discarded: MMA rows
      // are independent)
      const int arow_s = valid ? (p >> 4) : 0, brow_s = valid ? (p & 15) : 0;
      const float* ha = Hp + (size_t)(valid ? ii : n_dist) * KP;   // EXPLICIT: padded H rows
      const float* hb = Hp + (size_t)(valid ? jj : n_dist) * KP;
      // tile init: X of phase 0 = v0 = 1 on real anchors (hi = 1, lo = 0), anchors [g*KP/4, ...)
      for (int k = g * (KP / 4); k < (g + 1) * (KP / 4); k += 4) {
        uint32_t v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (k + e < K) ? 0x3f800000u : 0u;
        stg128(ximg(0, 0) + x_offset(p, k), v[0], v[1], v[2], v[3]);
        if (SPLIT == 3) stg128(ximg(0, 1) + x_offset(p, k), 0u, 0u, 0u, 0u);
      }
      fence_proxy_async_global();
      named_bar_sync(1, kEpiThreads);
      if (threadIdx.x == 0) mbar_arrive_local(bar_xr);
      float acc = 0.0f;
      for (int f = 0; f < phases; ++f) {
        const bool cost_phase = f == phases - 1;
        const int nrows = (f & 1) ? 16 : 8;           // u-update: a = H[i] (8 rows); v: b = H[j]
        const int64_t row0 = (f & 1) ? j0 : i0;
        const float* mrow = marg + ((f & 1) ? brow_s : arow_s) * S::kMRS;
        for (int pass = 0; pass < C::NP; ++pass) {
          if (!cost_phase && !EXPLICIT) {
            // stage this pass's 256 marginal columns (<= 16 KB) while the pass's MMAs run
            for (int e = threadIdx.x; e < nrows * 64; e += kEpiThreads) {
              const int r = e >> 6, c4 = (e & 63) * 4;
              const int64_t row = row0 + r < n_dist ? row0 + r : n_dist;
              *reinterpret_cast<float4*>(marg + r * S::kMRS + c4) =
                  *reinterpret_cast<const float4*>(Hp + (size_t)row * KP + pass * 256 + c4);
            }
            named_bar_sync(1, kEpiThreads);
          }
          mbar_wait(bar_done, done_par);
          done_par ^= 1u;
          tc_fence_after();
          const uint32_t tcol = tmem_base + lane_off + (uint32_t)(g * 64);
          const uint32_t col0 = (uint32_t)(pass * 256 + g * 64);   // anchor index of my first column
          uint8_t* xo_hi = ximg((f + 1) & 1, 0);
          uint8_t* xo_lo = ximg((f + 1) & 1, 1);
          const float* hrow = (f & 1) ? hb : ha;   // EXPLICIT marginal row of this phase
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t d[16];
            tmem_ld16u(tcol + c * 16, d);
            tmem_wait_ld();
            reg_fence16(d);
            const uint32_t k0 = col0 + c * 16;
            if (!cost_phase) {
              uint32_t hi[16], lo[16];
#pragma unroll
              for (int e = 0; e < 16; e += 4) {
                const float4 mq = EXPLICIT ? __ldg(reinterpret_cast<const float4*>(hrow + k0 + e))
                                           : *reinterpret_cast<const float4*>(mrow + g * 64 + c * 16 + e);
                const float mm[4] = {mq.x, mq.y, mq.z, mq.w};
                // S:62 clamp into [FLT_MIN, 2^126] + flag; m = 0 -> exactly 0 (R#11); one range
                // test per four anchors (div4_clamped)
                const float dq[4] = {__uint_as_float(d[e]), __uint_as_float(d[e + 1]), __uint_as_float(d[e + 2]),
                                     __uint_as_float(d[e + 3])};
                float xq[4];
                div4_clamped(mm, dq, xq, clamped);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const float x = xq[u];
                  if (SPLIT == 3) {
                    const uint32_t xh = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;   // RNA to TF32
                    hi[e + u] = xh;
                    lo[e + u] = __float_as_uint(x - __uint_as_float(xh));
                  } else {
                    hi[e + u] = tf32_rna_pre(x);   // the MMA truncates: RNA (read back masked)
                    lo[e + u] = 0u;
                  }
                }
              }
#pragma unroll
              for (int e = 0; e < 16; e += 4) {
                stg128(xo_hi + x_offset(p, k0 + e), hi[e], hi[e + 1], hi[e + 2], hi[e + 3]);
                if (SPLIT == 3) stg128(xo_lo + x_offset(p, k0 + e), lo[e], lo[e + 1], lo[e + 2], lo[e + 3]);
              }
            } else {
              // cost: D = v_L (K (.) C_s); u_L (side 1) = hi + lo
#pragma unroll
              for (int e = 0; e < 16; e += 4) {
                const float4 uh = *reinterpret_cast<const float4*>(ximg(1, 0) + x_offset(p, k0 + e));
                float uu[4] = {uh.x, uh.y, uh.z, uh.w};
                if (SPLIT == 3) {
                  const float4 ul = *reinterpret_cast<const float4*>(ximg(1, 1) + x_offset(p, k0 + e));
                  uu[0] += ul.x; uu[1] += ul.y; uu[2] += ul.z; uu[3] += ul.w;
                } else {
#pragma unroll
                  for (int u = 0; u < 4; ++u) uu[u] = tf32_mask(uu[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) acc = fmaf(uu[u], __uint_as_float(d[e + u]), acc);
              }
            }
          }
          if (!cost_phase && pass == C::NP - 1) fence_proxy_async_global();
          tc_fence_before();
          named_bar_sync(1, kEpiThreads);
          if (threadIdx.x == 0) {
            mbar_arrive_cluster(free_remote);
            if (!cost_phase && pass == C::NP - 1) mbar_arrive_local(bar_xr);
          }
        }
      }
      float* red = (float*)(smem + S::kOffRed);
      red[g * 128 + p] = acc;
      named_bar_sync(1, kEpiThreads);
      const int64_t slot = (units != nullptr ? 2 * kb + rank : t - tile_begin) * kTileSlots + p;
      if (g == 0 && t_in && (!EXPLICIT || slot < ps.n_slots))
        write_result(out, slot, valid, ii, jj,
                     (red[p] + red[128 + p]) + (red[256 + p] + red[384 + p]));
      named_bar_sync(1, kEpiThreads);  // red (aliases the marginal rows) reused by the next tile
    }
    if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
  }
  tc_fence_before();
  cluster_sync();
  clock_probe(g_tc5_clock, 1);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem_base) : "memory");
}

// K_hi, K_lo, (K (.) C_s)_hi, (K (.) C_s)_lo images; padding (K < KP): K_hi = 1 (denominators stay
// > 0; padded scalings are exactly 0), everything else 0.
template <int KP>
__global__ void gibbs_prep_tc5_kernel(const float* __restrict__ cost, int K, float eps, uint8_t* __restrict__ ghi,
                                      uint8_t* __restrict__ glo, uint8_t* __restrict__ gchi,
                                      uint8_t* __restrict__ gclo) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < KP * KP; idx += gridDim.x * blockDim.x) {
    const int n = idx / KP, k = idx % KP;
    const bool in = n < K && k < K;
    const double c = in ? (double)cost[(int64_t)n * K + k] : 0.0;
    const double gv = in ? exp(-c / (double)eps) : 1.0;   // P:183  K := exp(-C_s / eps)
    const float g32 = (float)gv, gc32 = in ? (float)(gv * c) : 0.0f;
    const uint32_t gh = tf32_rna_bits(g32), gch = tf32_rna_bits(gc32);
    const uint32_t pass = n >> 8, rk = (n >> 7) & 1, r = n & 127;
    const size_t off = (size_t)rk * Cfg<KP>::kImgRankBytes + b_offset<KP>(pass, r, k);
    *(uint32_t*)(ghi + off) = gh;
    *(uint32_t*)(glo + off) = in ? __float_as_uint(g32 - __uint_as_float(gh)) : 0u;
    *(uint32_t*)(gchi + off) = gch;
    *(uint32_t*)(gclo + off) = __float_as_uint(gc32 - __uint_as_float(gch));
  }
}

// Marginal rows padded to KP anchors, plus a dummy row (index N) for invalid pair slots.
template <int KP>
__global__ void pad_marginals_tc5_kernel(const float* __restrict__ H, int64_t n_dist, int K, float* __restrict__ Hp) {
  const int64_t total = (n_dist + 1) * KP;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / KP;
    const int c = (int)(idx % KP);
    float v = 0.0f;
    if (c < K) v = row < n_dist ? H[row * K + c] : 1.0f / (float)K;
    Hp[idx] = v;
  }
}

template <int KP, int SPLIT, bool EXPLICIT>
cudaError_t launch_kp(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                      const PairSource& ps, const float* H, int K, const uint8_t* img, uint8_t* scratch,
                      int iters, cudaStream_t s) {
  using C = Cfg<KP>;
  float* Hp = (float*)scratch;
  uint8_t* xbuf = scratch + (((size_t)(n_dist + 1) * KP * 4 + 1023) & ~(size_t)1023);
  pad_marginals_tc5_kernel<KP><<<512, 256, 0, s>>>(H, n_dist, K, Hp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = Smem::kBytes;
  e = cudaFuncSetAttribute(sinkhorn_tc5_kernel<KP, SPLIT, EXPLICIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_bp = ((tile_end + 1) >> 1) - (tile_begin >> 1);
  int64_t clusters = n_bp < sms / 2 ? n_bp : sms / 2;
  if (clusters < 1) clusters = 1;
  const size_t img_bytes = 2 * C::kImgRankBytes;
  sinkhorn_tc5_kernel<KP, SPLIT, EXPLICIT><<<(unsigned)(2 * clusters), kThreads, smem, s>>>(
      tile_begin, tile_end, n_dist, out, ps, Hp, K, img, img + img_bytes, img + 2 * img_bytes,
      img + 3 * img_bytes, xbuf, iters);
  return cudaGetLastError();
}

}  // namespace tc5

int tc5_kpad(int K) { return K <= 256 ? 256 : K <= 512 ? 512 : 1024; }
bool sinkhorn_tc5_supported(int K) { return K > 128 && K <= 1024; }
size_t sinkhorn_tc5_image_bytes(int K) {  // all four images
  const size_t kp = (size_t)tc5_kpad(K);
  return 4 * kp * kp * 4;
}
size_t sinkhorn_tc5_scratch_bytes(int K, int64_t n_dist, int sms) {
  const size_t kp = (size_t)tc5_kpad(K);
  return (size_t)(n_dist + 1) * kp * 4 + 1024 + (size_t)sms * 4 * 128 * kp * 4;
}

cudaError_t launch_gibbs_prep_tc5(const float* cost, int K, float eps, uint8_t* img, cudaStream_t s) {
  const size_t quarter = sinkhorn_tc5_image_bytes(K) / 4;
  switch (tc5_kpad(K)) {
    case 256: tc5::gibbs_prep_tc5_kernel<256><<<256, 256, 0, s>>>(cost, K, eps, img, img + quarter, img + 2 * quarter, img + 3 * quarter); break;
    case 512: tc5::gibbs_prep_tc5_kernel<512><<<512, 256, 0, s>>>(cost, K, eps, img, img + quarter, img + 2 * quarter, img + 3 * quarter); break;
    default: tc5::gibbs_prep_tc5_kernel<1024><<<1024, 256, 0, s>>>(cost, K, eps, img, img + quarter, img + 2 * quarter, img + 3 * quarter); break;
  }
  return cudaGetLastError();
}

template <int SPLIT, bool EXPLICIT>
static cudaError_t launch_split(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const PairSource& ps, const float* H, int K, const uint8_t* img,
                                uint8_t* scratch, int iters, cudaStream_t s) {
  switch (tc5_kpad(K)) {
    case 256: return tc5::launch_kp<256, SPLIT, EXPLICIT>(tile_begin, tile_end, n_dist, out, ps, H, K, img, scratch, iters, s);
    case 512: return tc5::launch_kp<512, SPLIT, EXPLICIT>(tile_begin, tile_end, n_dist, out, ps, H, K, img, scratch, iters, s);
    default: return tc5::launch_kp<1024, SPLIT, EXPLICIT>(tile_begin, tile_end, n_dist, out, ps, H, K, img, scratch, iters, s);
  }
}

// Tile mode (ps.pi == nullptr): tiles [tile_begin, tile_end) of the upper triangle.  Explicit mode:
// tiles of 128 consecutive entries of the pair list (tile_begin = 0, tile_end = ceil(n / 128)).
cudaError_t launch_sinkhorn_tc5(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const PairSource& ps, const float* H, int K, const uint8_t* img,
                                uint8_t* scratch, int iters, bool split3, cudaStream_t s) {
  if (tile_end <= tile_begin) return cudaSuccess;
  const bool expl = ps.pi != nullptr;
  if (split3) {
    return expl ? launch_split<3, true>(tile_begin, tile_end, n_dist, out, ps, H, K, img, scratch, iters, s)
                : launch_split<3, false>(tile_begin, tile_end, n_dist, out, ps, H, K, img, scratch, iters, s);
  }
  return expl ? launch_split<1, true>(tile_begin, tile_end, n_dist, out, ps, H, K, img, scratch, iters, s)
              : launch_split<1, false>(tile_begin, tile_end, n_dist, out, ps, H, K, img, scratch, iters, s);
}

}  // namespace asot

namespace asot {
cudaError_t read_kernel_clock_tc5(long long* host4) {
  return cudaMemcpyFromSymbol(host4, tc5::g_tc5_clock, 4 * sizeof(long long));
}
}  // namespace asot
