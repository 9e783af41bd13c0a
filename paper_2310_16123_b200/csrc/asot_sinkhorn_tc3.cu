// asot_sinkhorn_tc3.cu -- steps a5 + a6 with fp32 accuracy on the 5th-gen tensor cores
// (3xTF32, K <= 128): the ASOT_PREC_FP32 path (north star: 1e-4 of the fp64 oracle).
//
// Same recurrence as the TF32 kernels (R#4, R#5, R#11): U = A / (K V), V = B / (K^T U),
// V^(0) = 1, exactly L iterations; d = <diag(u) K diag(v), C_s> (R#3, R#6).
// Every product K x is evaluated as x_hi K_hi + x_lo K_hi + x_hi K_lo (3 tcgen05.mma kind::tf32
// chains, fp32 accumulate), with x_hi = RNA_tf32(x), x_lo = x - x_hi (exact in fp32) and the same
// split of the Gibbs kernel: the dropped x_lo K_lo term and the TF32 truncation of the lo parts
// are O(2^-21) relative, i.e. fp32-level (SURVEY §8(d) precision table: 3xTF32 <= 1e-6 vs 2e-3 for
// one pass; R#22 emulation: a 2-term split without K_lo fails 1e-4 at c2).
//
// Layout: pairs are the MMA M dimension (128 pair slots of a tile = 128 TMEM lanes).  TMEM is two
// regions R0 = [0, 2KP), R1 = [2KP, 4KP) of [x_hi | x_lo] columns; phase f reads A from R(f%2)
// and accumulates D into the hi columns of R((f+1)%2); the epilogue turns D in place into the
// next x_hi and writes x_lo next to it.  K_hi and K_lo are SW128 K-major images in SMEM (TMA bulk
// copies, once per CTA); K (.) C_s is a plain fp32 [KP][KP] SMEM copy for the cost, which runs on
// the CUDA cores (1% of the MMA work) so all of SMEM goes to the two Gibbs images.
//
// One slot per CTA (TMEM holds one tile's hi/lo scalings twice), so the epilogue is overlapped
// with the MMAs of the same tile: each phase is issued in four parts (K-half, N-half) =
// (0,0) (0,1) (1,0) | commit D-half-0 | (1,1) | commit D-half-1.  The epilogue of N-half 0 runs
// during part (1,1); the next phase's parts (0,0) (0,1) need only K-half 0 of the new x and run
// during the N-half-1 epilogue.  Warps 0-15 are epilogue warps (lane quarter w%4, column group
// w/4); warp 16 issues the MMAs.
#include <cfloat>
#include <cstdlib>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace tc3 {

using namespace ptx;

constexpr int kEpiWarps = 16;
constexpr int kEpiThreads = kEpiWarps * 32;   // 512

// Pair tiles (slots) per CTA: TMEM holds 4·KP columns per slot (two [x_hi | x_lo] regions), so
// KP = 64 fits two slots and KP = 32 four; the 16 epilogue warps split evenly over the slots
// and each slot has its own MMA warp.  With short phases the other slots' MMAs hide a slot's
// epilogue latency.
template <int KP> struct Slots {
  static constexpr int NS = KP <= 32 ? 4 : (KP <= 64 ? 2 : 1);
  static constexpr int kWarpsPerSlot = kEpiWarps / NS;
  static constexpr int NCG = kWarpsPerSlot / 4;      // column groups per slot
  static constexpr int kThreads = kEpiThreads + 32 * NS;
};
constexpr uint32_t kTmemCols = 512;

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}

template <int KP>
struct Smem {
  static constexpr int kRS = KP + 4;                       // marginal row stride (floats)
  static constexpr int kRows = 8 + 16 + 1;                 // a-rows, b-rows, dummy row
  static constexpr size_t kImg = (size_t)KP * KP * 4;      // one operand image / the GC copy
  static constexpr size_t kOffGhi = 0;
  static constexpr size_t kOffGlo = kImg;
  static constexpr size_t kOffGC = 2 * kImg;
  static constexpr int NS = Slots<KP>::NS;
  static constexpr size_t kOffMarg = 3 * kImg;                             // [NS][kRows][kRS]
  static constexpr size_t kOffRed = kOffMarg + (size_t)NS * kRows * kRS * 4;   // [NS][NCG][128]
  static constexpr size_t kOffBar = kOffRed + (size_t)NS * Slots<KP>::NCG * 128 * 4;
  static constexpr size_t kBytes = kOffBar + 256 + 1024;
};

// One part of a phase: D[:, nh*KP/2 ...] (+)= sum over K-half kh of
// (A_hi K_hi + A_lo K_hi + A_hi K_lo), N = KP/2.
// (The descriptors are the per-image base descriptor plus a constant offset: the issuing warp
// shares its SM sub-partition with four busy epilogue warps, so its stream is kept short.)
template <int KP>
__device__ __forceinline__ void issue_part(uint32_t a_reg, uint32_t d_reg, uint64_t ghi_desc, uint64_t glo_desc,
                                           int kh, int nh) {
  constexpr int NH = KP / 2;
  constexpr uint32_t idesc = make_idesc_tf32(128, NH);
  const uint32_t d = d_reg + (uint32_t)(nh * NH);
  const uint32_t row0 = (uint32_t)(nh * NH * 128);  // byte offset of row nh*NH inside a k-block
#pragma unroll
  for (int s = 0; s < KP / 16; ++s) {
    const int ks = kh * (KP / 16) + s;  // 8-wide k step
    const uint32_t boff = (uint32_t)((ks >> 2) * KP * 128 + (ks & 3) * 32) + row0;
    const uint64_t dhi = ghi_desc + (uint64_t)(boff >> 4), dlo = glo_desc + (uint64_t)(boff >> 4);
    const uint32_t acc0 = (kh > 0 || s > 0) ? 1u : 0u;
    mma1_tf32_ts(d, a_reg + 8 * ks, dhi, idesc, acc0);         // x_hi K_hi
    mma1_tf32_ts(d, a_reg + KP + 8 * ks, dhi, idesc, 1u);      // x_lo K_hi
    mma1_tf32_ts(d, a_reg + 8 * ks, dlo, idesc, 1u);           // x_hi K_lo
  }
}

// Debug timeline (ASOT_TC_DEBUG_MODE=3, CTA 0's first tile): event, phase -> clock64.
// events: 0 / 1 = epilogue woke for D half 0 / 1, 2 / 3 = its x half 0 / 1 arrive,
// 4 / 5 = issuer passed the x half 0 / 1 gate
__device__ long long g_tc3_trace[6][256];
__device__ long long g_tc3_clock[4];  // clock_probe: (clock64, globaltimer) at start / end

// EX (pair-list mode): tile tr holds list entries [128 tr, 128 tr + 128); each lane's marginal rows
// come from the padded copy Hp [(n_dist + 1)][KP] (row n_dist = uniform, for invalid entries),
// prefetched half a phase ahead into registers, instead of the tile's 25 rows in SMEM.
template <int KP, int DBG, bool EX>
__global__ void __launch_bounds__(Slots<KP>::kThreads, 1)
sinkhorn_tc3_kernel(int64_t tile_begin, int64_t n_tiles, int64_t n_dist, PairSink out,
                    const float* __restrict__ H, int K, const uint32_t* __restrict__ ghi_img,
                    const uint32_t* __restrict__ glo_img, const float* __restrict__ gc_plain, int iters,
                    const int32_t* __restrict__ pair_i, const int32_t* __restrict__ pair_j, int64_t n_pairs,
                    const float* __restrict__ Hp, const int32_t* __restrict__ units,
                    const int64_t* __restrict__ n_dev) {
  if (dense_skipped(out)) return;   // the small-support kernel serves this call (R#36)
  using S = Smem<KP>;
  // device-side counts (bucketed pair lists, asot_pairs_bucket.cu): the host passed upper bounds
  if (n_dev != nullptr) {
    const int64_t c = *n_dev;
    if constexpr (EX) {
      n_pairs = c < n_pairs ? c : n_pairs;
      n_tiles = (n_pairs + kTileSlots - 1) / kTileSlots;
    } else {
      n_tiles = c < n_tiles ? c : n_tiles;
    }
  }
  constexpr int NS = Slots<KP>::NS, NCG = Slots<KP>::NCG;
  constexpr int kWPS = Slots<KP>::kWarpsPerSlot, kWG = kWPS * 32;
  constexpr int NH = KP / 2;          // columns per N-half
  constexpr int CPT = NH / NCG;       // columns per epilogue thread per half
  constexpr int CQ = KP / NCG;        // columns per thread in the cost
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* marg = (float*)(smem + S::kOffMarg);
  float* red = (float*)(smem + S::kOffRed);
  const float* gcs = (const float*)(smem + S::kOffGC);
  uint64_t* bars = (uint64_t*)(smem + S::kOffBar);
  // bars: 0 g_loaded; slot s: 1 + 4s D-half-0 done, +1 D-half-1 done, +2 x-half-0 ready, +3 x-half-1
  uint32_t* tmem_holder = (uint32_t*)(bars + 17);
  volatile int* turn = (volatile int*)(bars + 18);
  volatile int* slot_done = turn + 1;  // [NS]
  const uint32_t bar_g = smem_u32(&bars[0]);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tiles of slot s: tk = s, s+NS, ... with tr = blockIdx.x + tk * gridDim.x < n_tiles
  auto slot_tiles = [&](int slot) -> int64_t {
    const int64_t per = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    return per <= slot ? 0 : (per - slot + NS - 1) / NS;
  };
  if (threadIdx.x == 0) {
    turn[0] = 0;   // slot 0 always has a tile (grid <= n_tiles)
    for (int b = 0; b < NS; ++b) slot_done[b] = slot_tiles(b) == 0 ? 1 : 0;
    mbar_init(bar_g, 1);
    for (int b = 0; b < NS; ++b) {
      const uint32_t sb = smem_u32(&bars[1 + 4 * b]);
      mbar_init(sb, 1);
      mbar_init(sb + 8, 1);
      mbar_init(sb + 16, kWPS);
      mbar_init(sb + 24, kWPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  clock_probe(g_tc3_clock, 0);
  if (*tmem_holder != 0) __trap();  // full allocation starts at column 0 (one CTA per SM)
  if (threadIdx.x == 0) {           // K_hi, K_lo images and the GC copy, once per CTA (TMA bulk)
    mbar_expect_tx(bar_g, (uint32_t)(3 * S::kImg));
    constexpr uint32_t kChunk = 32768;
    for (uint32_t off = 0; off < S::kImg; off += kChunk) {
      const uint32_t n = (uint32_t)((S::kImg - off) < kChunk ? (S::kImg - off) : kChunk);
      bulk_g2s(smem_u32(smem + S::kOffGhi + off), (const uint8_t*)ghi_img + off, n, bar_g);
      bulk_g2s(smem_u32(smem + S::kOffGlo + off), (const uint8_t*)glo_img + off, n, bar_g);
      bulk_g2s(smem_u32(smem + S::kOffGC + off), (const uint8_t*)gc_plain + off, n, bar_g);
    }
  }

  if (warp >= kEpiWarps) {
    // ------------------------------------------------------------------ MMA warps (one per slot)
    // A turn token passed round the active slots orders whole phases of the slots in the tensor
    // pipe; only the holder writes it.
    const int ss = warp - kEpiWarps;
    const uint32_t sb = (uint32_t)(ss * 4 * KP);   // this slot's TMEM columns
    const uint32_t bar_d0 = smem_u32(&bars[1 + 4 * ss]), bar_d1 = bar_d0 + 8;
    const uint32_t bar_x0 = bar_d0 + 16, bar_x1 = bar_d0 + 24;
    auto pass_turn = [&]() {
      for (int k = 1; k <= NS; ++k) {
        const int cand = (ss + k) % NS;
        if (cand == ss || !slot_done[cand]) {
          *turn = cand;
          break;
        }
      }
    };
    const uint64_t ghi = make_sw128_desc(smem_u32(smem + S::kOffGhi));
    const uint64_t glo = make_sw128_desc(smem_u32(smem + S::kOffGlo));
    mbar_wait(bar_g, 0);
    uint32_t xpar = 0;
    const int64_t my_tiles = slot_tiles(ss);
    for (int64_t k2 = 0; k2 < my_tiles; ++k2) {
      const int64_t tr = blockIdx.x + (ss + NS * k2) * (int64_t)gridDim.x;
      for (int f = 0; f < 2 * iters; ++f) {
        const uint32_t a_reg = sb + (uint32_t)((f & 1) * 2 * KP), d_reg = sb + (uint32_t)(((f + 1) & 1) * 2 * KP);
        mbar_wait(bar_x0, xpar);
        if (NS > 1)
          while (*turn != ss) __nanosleep(20);
        __syncwarp();
        tc_fence_after();
        if (DBG == 3 && blockIdx.x == 0 && tr == blockIdx.x && lane == 0 && f < 256) g_tc3_trace[4][f] = clock64();
        if (elect_one()) {
          issue_part<KP>(a_reg, d_reg, ghi, glo, 0, 0);
          issue_part<KP>(a_reg, d_reg, ghi, glo, 0, 1);
        }
        __syncwarp();
        mbar_wait(bar_x1, xpar);
        tc_fence_after();
        if (DBG == 3 && blockIdx.x == 0 && tr == blockIdx.x && lane == 0 && f < 256) g_tc3_trace[5][f] = clock64();
        if (elect_one()) {
          issue_part<KP>(a_reg, d_reg, ghi, glo, 1, 0);
          mma1_commit(bar_d0);
          issue_part<KP>(a_reg, d_reg, ghi, glo, 1, 1);
          mma1_commit(bar_d1);
          if (NS > 1) {
            if (k2 + 1 == my_tiles && f + 1 == 2 * iters) slot_done[ss] = 1;
            pass_turn();
          }
        }
        __syncwarp();
        xpar ^= 1u;
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue warps
    const int s = warp / kWPS;                // slot
    const int q = warp & 3, cg = (warp % kWPS) >> 2;   // TMEM lane quarter, column group
    const int p = q * 32 + lane;              // pair slot == TMEM lane
    const int wg_tid = threadIdx.x - s * kWG;
    const uint32_t lane_off = ((uint32_t)(q * 32) << 16) + (uint32_t)(s * 4 * KP);   // + slot columns
    const uint32_t bar_d0 = smem_u32(&bars[1 + 4 * s]), bar_d1 = bar_d0 + 8;
    const uint32_t bar_x0 = bar_d0 + 16, bar_x1 = bar_d0 + 24;
    marg += (size_t)s * S::kRows * S::kRS;
    red += (size_t)s * NCG * 128;
    uint32_t dpar = 0;
    bool clamped = false;
    const int64_t my_tiles = slot_tiles(s);
    for (int64_t k2 = 0; k2 < my_tiles; ++k2) {
      const int64_t tr = blockIdx.x + (s + NS * k2) * (int64_t)gridDim.x;
      const int64_t t = units != nullptr ? (int64_t)units[tr] : tile_begin + tr;
      named_bar_sync(1 + s, kWG);  // previous tile's cost readers are done (marg, red, R0)
      int ii = 0, jj = 0;
      bool valid;
      const float* arow;
      const float* brow;
      if constexpr (EX) {
        const int64_t q = tr * kTileSlots + p;   // list entry of this lane
        valid = q < n_pairs;
        if (valid) {
          ii = pair_i[q];
          jj = pair_j[q];
          valid = ii >= 0 && jj >= 0 && ii < n_dist && jj < n_dist;
        }
        arow = Hp + (valid ? (int64_t)ii : n_dist) * KP;
        brow = Hp + (valid ? (int64_t)jj : n_dist) * KP;
      } else {
        int64_t bi, bj;
        block_pair_decode(t >> 1, num_blocks(n_dist), bi, bj);
        const int64_t i0 = bi * kBlockDist + (t & 1) * 8, j0 = bj * kBlockDist;
        for (int e = wg_tid; e < S::kRows * KP; e += kWG) {
          const int r = e / KP, c = e % KP;
          const int64_t row = r < 8 ? i0 + r : (r < 24 ? j0 + (r - 8) : n_dist);
          float v = (row < n_dist && c < K) ? H[row * K + c] : 0.0f;
          if (r == 24) v = c < K ? 1.0f / (float)K : 0.0f;  // dummy marginal for invalid slots
          marg[r * S::kRS + c] = v;
        }
        valid = tile_slot_pair(t, p, n_dist, ii, jj);
        arow = marg + (valid ? (p >> 4) : 24) * S::kRS;
        brow = marg + (valid ? 8 + (p & 15) : 24) * S::kRS;
      }
      // (EX) the lane's CPT marginal values of the next half, prefetched from L2
      float mk[EX ? CPT : 1];
      auto load_mk = [&](int f, int h) {
        if constexpr (EX) {
          const float4* m4 = reinterpret_cast<const float4*>(((f & 1) ? brow : arow) + h * NH + cg * CPT);
#pragma unroll
          for (int e = 0; e < CPT / 4; ++e) {
            const float4 mq = __ldg(m4 + e);
            mk[4 * e] = mq.x; mk[4 * e + 1] = mq.y; mk[4 * e + 2] = mq.z; mk[4 * e + 3] = mq.w;
          }
        }
      };
      load_mk(0, 0);
      // x^(0) = v0 = 1 on the real anchors, hi = 1, lo = 0, into R0 (both halves)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int c4 = 0; c4 < CPT; c4 += 4) {
          const int c = h * NH + cg * CPT + c4;
          uint32_t hi[4], lo[4] = {0u, 0u, 0u, 0u};
#pragma unroll
          for (int e = 0; e < 4; ++e) hi[e] = (c + e < K) ? 0x3f800000u : 0u;
          tmem_st4(lane_off + (uint32_t)c, hi);
          tmem_st4(lane_off + (uint32_t)(KP + c), lo);
        }
      }
      tmem_wait_st();
      named_bar_sync(1 + s, kWG);  // marginals visible to every epilogue thread of the slot
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_local(bar_x0);
        mbar_arrive_local(bar_x1);
      }
      for (int f = 0; f < 2 * iters; ++f) {
        const uint32_t d_reg = (uint32_t)(((f + 1) & 1) * 2 * KP);
        const float* mrow = (f & 1) ? brow : arow;   // u-update: a = H[i]; v-update: b = H[j]
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait(h == 0 ? bar_d0 : bar_d1, dpar);
          tc_fence_after();
          if (DBG == 3 && blockIdx.x == 0 && tr == blockIdx.x && threadIdx.x == 0 && f < 256)
            g_tc3_trace[h][f] = clock64();
#pragma unroll
          for (int c4 = 0; c4 < CPT; c4 += 4) {
            const int c = h * NH + cg * CPT + c4;
            uint32_t dv[4], hi[4], lo[4];
            tmem_ld4(lane_off + d_reg + (uint32_t)c, dv);
            tmem_wait_ld();
            float mm[4];
            if constexpr (EX) {
              mm[0] = mk[c4]; mm[1] = mk[c4 + 1]; mm[2] = mk[c4 + 2]; mm[3] = mk[c4 + 3];
            } else {
              const float4 m4 = *reinterpret_cast<const float4*>(mrow + c);
              mm[0] = m4.x; mm[1] = m4.y; mm[2] = m4.z; mm[3] = m4.w;
            }
            // S:62 clamp into [FLT_MIN, 2^126] + flag; m = 0 -> exactly 0 (R#11); one range
            // test per four anchors (div4_clamped)
            float xq[4];
            const float dq[4] = {__uint_as_float(dv[0]), __uint_as_float(dv[1]), __uint_as_float(dv[2]),
                                 __uint_as_float(dv[3])};
            div4_clamped(mm, dq, xq, clamped);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t xh = (__float_as_uint(xq[e]) + 0x1000u) & 0xFFFFE000u;  // RNA to TF32
              hi[e] = xh;
              lo[e] = __float_as_uint(xq[e] - __uint_as_float(xh));
            }
            tmem_st4(lane_off + d_reg + (uint32_t)c, hi);
            tmem_st4(lane_off + d_reg + (uint32_t)(KP + c), lo);
          }
          if (h == 0) load_mk(f, 1);
          else if (f + 1 < 2 * iters) load_mk(f + 1, 0);
          tmem_wait_st();
          if (f + 1 < 2 * iters) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_local(h == 0 ? bar_x0 : bar_x1);
            if (DBG == 3 && blockIdx.x == 0 && tr == blockIdx.x && threadIdx.x == 0 && f < 256)
              g_tc3_trace[2 + h][f] = clock64();
          }
        }
        dpar ^= 1u;
      }
      // ---- cost (a6): u_L in R1, v_L in R0 (hi + lo = the fp32 values).  Thread (p, cg):
      // t_c = sum_r (K (.) C_s)[r][c] u_r for its CQ columns, partial = sum_c v_c t_c.
      // Every thread reads all columns of its lane, written by the other column groups' warps.
      tc_fence_before();
      named_bar_sync(1 + s, kWG);
      tc_fence_after();
      float tacc[CQ];
#pragma unroll
      for (int c = 0; c < CQ; ++c) tacc[c] = 0.0f;
      const uint32_t r1 = lane_off + (uint32_t)(2 * KP);   // (lane_off includes the slot base)
      for (int r0 = 0; r0 < KP; r0 += 4) {
        uint32_t uh[4], ul[4];
        tmem_ld4(r1 + (uint32_t)r0, uh);
        tmem_ld4(r1 + (uint32_t)(KP + r0), ul);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float ur = __uint_as_float(uh[e]) + __uint_as_float(ul[e]);
          const float4* g4 = reinterpret_cast<const float4*>(gcs + (size_t)(r0 + e) * KP + cg * CQ);
#pragma unroll
          for (int c4 = 0; c4 < CQ / 4; ++c4) {
            const float4 g = g4[c4];
            tacc[4 * c4 + 0] = fmaf(g.x, ur, tacc[4 * c4 + 0]);
            tacc[4 * c4 + 1] = fmaf(g.y, ur, tacc[4 * c4 + 1]);
            tacc[4 * c4 + 2] = fmaf(g.z, ur, tacc[4 * c4 + 2]);
            tacc[4 * c4 + 3] = fmaf(g.w, ur, tacc[4 * c4 + 3]);
          }
        }
      }
      float part = 0.0f;
#pragma unroll
      for (int c4 = 0; c4 < CQ; c4 += 4) {
        uint32_t vh[4], vl[4];
        tmem_ld4(lane_off + (uint32_t)(cg * CQ + c4), vh);
        tmem_ld4(lane_off + (uint32_t)(KP + cg * CQ + c4), vl);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 4; ++e)
          part = fmaf(__uint_as_float(vh[e]) + __uint_as_float(vl[e]), tacc[c4 + e], part);
      }
      red[cg * 128 + p] = part;
      named_bar_sync(1 + s, kWG);
      if (cg == 0) {
        float dsum;
        if (NCG == 4) dsum = (red[p] + red[128 + p]) + (red[256 + p] + red[384 + p]);
        else if (NCG == 2) dsum = red[p] + red[128 + p];
        else dsum = red[p];
        if (!EX || tr * kTileSlots + p < n_pairs)   // (pair lists: no slot past the list)
          write_result(out, tr * kTileSlots + p, valid, ii, jj, dsum);
      }
      tc_fence_before();
    }
    if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
  }
  tc_fence_before();
  __syncthreads();
  clock_probe(g_tc3_clock, 1);
  tc_fence_after();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(0u), "r"(kTmemCols) : "memory");
  }
}

// K_hi / K_lo SW128 images and the plain padded K (.) C_s copy.  Padding (K < KP): K_hi = 1,
// K_lo = 0 outside the real block (denominators stay > 0, padded scalings are exactly 0),
// K (.) C_s = 0.
__global__ void gibbs_prep_tc3_kernel(const float* __restrict__ cost, int K, float eps, int kp,
                                      uint32_t* __restrict__ ghi, uint32_t* __restrict__ glo,
                                      float* __restrict__ gc) {
  const int64_t total = (int64_t)kp * kp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(idx / kp), k = (int)(idx % kp);
    const bool in = n < K && k < K;
    const double c = in ? (double)cost[(int64_t)n * K + k] : 0.0;
    const double g = in ? exp(-c / (double)eps) : 1.0;   // P:183 K := exp(-C_s / eps)
    const float g32 = (float)g;
    const uint32_t h = tf32_rna_bits(g32);
    const uint32_t off = sw128_kmajor_offset((uint32_t)n, (uint32_t)k, (uint32_t)kp) >> 2;
    ghi[off] = h;
    glo[off] = in ? __float_as_uint(g32 - __uint_as_float(h)) : 0u;
    gc[idx] = in ? (float)(g * c) : 0.0f;
  }
}

template <int KP>
static cudaError_t launch_kp(int64_t tile_begin, int64_t n_tiles, int64_t n_dist, const PairSink& out,
                             const float* H, int K, const uint32_t* ghi, const uint32_t* glo,
                             const float* gc, int iters, cudaStream_t s, const int32_t* pi = nullptr,
                             const int32_t* pj = nullptr, int64_t n_pairs = 0, const float* Hp = nullptr,
                             const int32_t* units = nullptr, const int64_t* n_dev = nullptr) {
  const size_t smem = Smem<KP>::kBytes;
#ifdef ASOT_DEBUG_KERNELS   // diagnostic variant (tools/): only in debug builds
  static const int dbg = getenv("ASOT_TC_DEBUG_MODE") ? atoi(getenv("ASOT_TC_DEBUG_MODE")) : 0;
  auto kern = pi != nullptr ? sinkhorn_tc3_kernel<KP, 0, true>
            : dbg == 3 ? sinkhorn_tc3_kernel<KP, 3, false> : sinkhorn_tc3_kernel<KP, 0, false>;
#else
  auto kern = pi != nullptr ? sinkhorn_tc3_kernel<KP, 0, true> : sinkhorn_tc3_kernel<KP, 0, false>;
#endif
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (n_tiles + Slots<KP>::NS - 1) / Slots<KP>::NS;
  if (grid > sms) grid = sms;
  if (grid < 1) return cudaSuccess;
  kern<<<(unsigned)grid, Slots<KP>::kThreads, smem, s>>>(tile_begin, n_tiles, n_dist, out, H, K,
                                                                 ghi, glo, gc, iters, pi, pj, n_pairs, Hp,
                                                                 units, n_dev);
  return cudaGetLastError();
}

// Padded marginal rows for the pair-list mode (row n_dist = uniform 1/K, the invalid-entry dummy).
__global__ void pad_marginals_tc3_kernel(const float* __restrict__ H, int64_t n_dist, int K, int kp,
                                         float* __restrict__ Hp) {
  const int64_t total = (n_dist + 1) * kp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / kp;
    const int c = (int)(idx % kp);
    float v = 0.0f;
    if (c < K) v = row < n_dist ? H[row * K + c] : 1.0f / (float)K;
    Hp[idx] = v;
  }
}

}  // namespace tc3

bool sinkhorn_tc3_supported(int K) { return K >= 1 && K <= 128; }

size_t sinkhorn_tc3_image_bytes(int K) {
  const size_t kp = (size_t)kpad32(K);
  return kp * kp * 4;
}

cudaError_t launch_gibbs_prep_tc3(const float* cost, int K, float eps, uint32_t* ghi, uint32_t* glo,
                                  float* gc, cudaStream_t s) {
  const int kp = kpad32(K);
  const int64_t total = (int64_t)kp * kp;
  tc3::gibbs_prep_tc3_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(cost, K, eps, kp, ghi, glo, gc);
  return cudaGetLastError();
}

cudaError_t launch_sinkhorn_tc3(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const float* H, int K, const uint32_t* ghi, const uint32_t* glo,
                                const float* gc, int iters, cudaStream_t s, const int32_t* units,
                                const int64_t* n_dev) {
  const int64_t n_tiles = tile_end - tile_begin;
  if (n_tiles <= 0) return cudaSuccess;
  switch (kpad32(K)) {
#define ASOT_TC3_CASE(KP)                                                                              \
    case KP: return tc3::launch_kp<KP>(tile_begin, n_tiles, n_dist, out, H, K, ghi, glo, gc, iters, s, \
                                       nullptr, nullptr, 0, nullptr, units, n_dev);
    ASOT_TC3_CASE(32)
    ASOT_TC3_CASE(64)
    ASOT_TC3_CASE(96)
    ASOT_TC3_CASE(128)
#undef ASOT_TC3_CASE
    default: return cudaErrorNotSupported;
  }
}

}  // namespace asot

namespace asot {
size_t sinkhorn_tc3_pairs_scratch_bytes(int64_t n_dist, int K) { return (size_t)(n_dist + 1) * kpad32(K) * 4; }

cudaError_t launch_sinkhorn_tc3_pairs(const int32_t* pi, const int32_t* pj, int64_t n_pairs, int64_t n_dist,
                                      const PairSink& out, const float* H, int K, const uint32_t* ghi,
                                      const uint32_t* glo, const float* gc, float* Hp, int iters, cudaStream_t s,
                                      const int64_t* n_dev) {
  if (n_pairs <= 0) return cudaSuccess;
  const int kp = kpad32(K);
  tc3::pad_marginals_tc3_kernel<<<512, 256, 0, s>>>(H, n_dist, K, kp, Hp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t n_tiles = (n_pairs + kTileSlots - 1) / kTileSlots;
  switch (kp) {
#define ASOT_TC3_CASE(KP)                                                                                \
    case KP: return tc3::launch_kp<KP>(0, n_tiles, n_dist, out, H, K, ghi, glo, gc, iters, s, pi, pj, \
                                       n_pairs, Hp, nullptr, n_dev);
    ASOT_TC3_CASE(32)
    ASOT_TC3_CASE(64)
    ASOT_TC3_CASE(96)
    ASOT_TC3_CASE(128)
#undef ASOT_TC3_CASE
    default: return cudaErrorNotSupported;
  }
}
}  // namespace asot

extern "C" int asot_debug_tc3_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, asot::tc3::g_tc3_trace, sizeof(asot::tc3::g_tc3_trace));
}

namespace asot {
cudaError_t read_kernel_clock_tc3(long long* host4) {
  return cudaMemcpyFromSymbol(host4, tc3::g_tc3_clock, 4 * sizeof(long long));
}
}  // namespace asot
