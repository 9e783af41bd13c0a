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
// Two pair tiles (slots) per CTA -- four for KP <= 64 -- keep the tensor pipe busy: while it
// runs one slot's product ("chain"), the other slots' warps turn their accumulators into the
// next scalings.  Each slot has
// two TMEM regions of KP columns; phase f reads A from R[f%2] and writes D into R[(f+1)%2], and
// the epilogue writes the new scaling IN PLACE over D, so the roles swap every phase.  The
// input anchors are cut into two chunks of CH = KP/2: a chain is issued as two halves of N = KP
// MMAs (k-steps of chunk 0, then chunk 1), each gated by the epilogue of that chunk of the
// previous phase, so the next chain of a slot waits only for the epilogue of chunk 0 -- which
// hides behind the other slot's chain -- instead of the whole epilogue.  (Also splitting N into
// parts with early output chunks measured slower: 2380 vs 2324 cycles per two chains.)
//
// Warp roles (576 threads; 640 with four slots): warps 0-7 slot 0, warps 8-15 slot 1 (warp w
// reads TMEM lane quarter w%4 and the column half (w%8)/4 of every chunk; four slots: 4 warps
// each, whole chunks); warp 16 + s issues the MMAs of slot s,
// alternating chains through a turn token, gated per (slot, chunk) by mbarriers the epilogue arrives
// on, and commits once per chain.  Epilogue: tcgen05.ld -> u = a / D with one MUFU.RCP per
// two anchors -> RNA rounding to TF32 (add half an ulp; the MMA truncates) -> tcgen05.st.
// Cost (a6): the last v-update leaves v_L in place in R0 (u_L in R1); two N = KP/2 chains apply
// K (.) C_s to it (output into the consumed half of R1), and the threads reduce
// sum_r u_r ((K (.) C_s) v)_r; the two column halves meet in SMEM once per tile.
//
// TMEM map (columns): slot s: R0 at 2s*KP, R1 at 2s*KP + KP.  SMEM: [K image | KC image |
// marginal rows (8 a-rows, 16 b-rows, 1 dummy row) per slot | partial costs | mbarriers].
#include <cfloat>
#include <cstdlib>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace tc {

// Debug timeline (ASOT_TC_DEBUG_MODE=3): slot, event, phase -> clock64 for CTA 0's first tile.
// events: 0 / 1 = epilogue woke for chunk 0 / 1, 2 / 3 = MMA warp passed the chunk 0 / 1 gate
__device__ long long g_tc_trace[2][4][512];
__device__ long long g_tc_clock[4];  // clock_probe: (clock64, globaltimer) at start / end

constexpr int kEpiWarps = 16;
constexpr int kThreads = kEpiWarps * 32;  // epilogue threads

// Pair tiles (slots) per CTA: two for KP > 64, four for KP <= 64 (TMEM holds 2·KP columns per
// slot; with short chains more slots are needed to hide the epilogue latency).  The 16 epilogue
// warps split evenly over the slots; each slot has its own MMA warp.
template <int KP> struct Slots {
  static constexpr int NS = KP <= 64 ? 4 : 2;
  static constexpr int kWarpsPerSlot = kEpiWarps / NS;   // 8 or 4
  static constexpr int NG = kWarpsPerSlot / 4;           // column groups per slot: 2 or 1
  static constexpr int kAllThreads = kThreads + 32 * NS;
};

using namespace ::asot::ptx;

template <int KP>
struct Smem {
  static constexpr int NS = Slots<KP>::NS;
  static constexpr int kRS = KP + 4;                      // marginal row stride (floats)
  static constexpr int kRows = 8 + 16 + 1;                // a-rows, b-rows, dummy row
  static constexpr size_t kImg = (size_t)KP * KP * 4;     // one operand image
  static constexpr size_t kMarg = (size_t)kRows * kRS * 4;
  static constexpr size_t kOffG = 0;
  static constexpr size_t kOffGC = kImg;
  static constexpr size_t kOffMarg = 2 * kImg;
  static constexpr size_t kOffRed = kOffMarg + NS * kMarg;    // [NS slots][128] partial costs
  static constexpr size_t kOffBar = kOffRed + NS * 128 * 4;
  static constexpr size_t kBytes = kOffBar + 256 + 1024;     // + alignment slack
};

// Loads / stores of W columns (W = 8, 16, 24 or 32) of one TMEM lane quarter.
template <int W>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[W]) {
  static_assert(W % 8 == 0, "width");
  if constexpr (W % 16 == 0) {
#pragma unroll
    for (int c = 0; c < W / 16; ++c) tmem_ld16u(taddr + 16 * c, *reinterpret_cast<uint32_t(*)[16]>(&r[16 * c]));
  } else {
#pragma unroll
    for (int c = 0; c < W / 8; ++c) {
      float v[8];
      tmem_ld8(taddr + 8 * c, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) r[8 * c + e] = __float_as_uint(v[e]);
    }
  }
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
template <int W>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t (&r)[W]) {
  if constexpr (W % 16 == 0) {
#pragma unroll
    for (int c = 0; c < W / 16; ++c) tmem_st16(taddr + 16 * c, *reinterpret_cast<const uint32_t(*)[16]>(&r[16 * c]));
  } else {
#pragma unroll
    for (int c = 0; c < W / 8; ++c) tmem_st8(taddr + 8 * c, &r[8 * c]);
  }
}

// EX (pair-list mode, asot_pairwise_sinkhorn): tile tr holds list entries [128 tr, 128 tr + 128);
// each slot's marginal rows come straight from the padded copy Hp [(n_dist + 1)][KP] (row n_dist
// = uniform, for invalid entries), prefetched a chunk ahead into registers, instead of the
// tile's 25 shared rows in SMEM.
template <int KP, int DBG, bool EX>
__global__ void __launch_bounds__(Slots<KP>::kAllThreads, 1)
sinkhorn_tc_kernel(int64_t tile_begin, int64_t n_tiles, int64_t n_dist, PairSink out,
                   const float* __restrict__ H, int K, const uint32_t* __restrict__ g_img,
                   const uint32_t* __restrict__ gc_img, int iters, const int32_t* __restrict__ pair_i,
                   const int32_t* __restrict__ pair_j, int64_t n_pairs, const float* __restrict__ Hp,
                   const int32_t* __restrict__ units, const int64_t* __restrict__ n_dev) {
  if (dense_skipped(out)) return;   // the small-support kernel serves this call (R#36)
  using S = Smem<KP>;
  // device-side counts (bucketed pair lists): the host passed upper bounds
  if (n_dev != nullptr) {
    const int64_t c = *n_dev;
    if constexpr (EX) {
      n_pairs = c < n_pairs ? c : n_pairs;
      n_tiles = (n_pairs + kTileSlots - 1) / kTileSlots;
    } else {
      n_tiles = c < n_tiles ? c : n_tiles;
    }
  }
  // All 512 columns: the allocation then necessarily starts at column 0 (one CTA per SM), so
  // every TMEM address below is a compile-time constant per slot.
  constexpr uint32_t kTmemCols = 512;
  constexpr int NS = Slots<KP>::NS, NG = Slots<KP>::NG;
  constexpr int kWarpsPerSlot = Slots<KP>::kWarpsPerSlot;
  constexpr int CH = KP / 2;         // anchors per chunk
  constexpr int W = CH / NG;         // columns per thread per chunk
  constexpr int SB = NG == 2 ? W : 16;       // TMEM ld/st sub-block (columns)
  constexpr int CQ = KP / 2 / NG;    // columns per thread in each cost half
  constexpr int kWG = kWarpsPerSlot * 32;
  constexpr uint32_t kIdesc = make_idesc_tf32(128, KP);
  constexpr uint32_t kIdescHalf = make_idesc_tf32(128, KP / 2);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* marg = (float*)(smem + S::kOffMarg);
  float* red = (float*)(smem + S::kOffRed);
  uint64_t* bars = (uint64_t*)(smem + S::kOffBar);
  // bars: 0 g_loaded, 1 + 2s + c mma_done[s][c], 9 + 2s + c go[s][c]
  uint32_t* tmem_holder = (uint32_t*)(bars + 17);
  volatile int* turn = (volatile int*)(bars + 18);
  volatile int* slot_done = turn + 1;  // [NS]
  const uint32_t bar_g = smem_u32(&bars[0]);
  const uint32_t bar_mma0 = smem_u32(&bars[1]);
  const uint32_t bar_go0 = smem_u32(&bars[9]);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = warp / kWarpsPerSlot;          // slot (pair tile) of an epilogue warp; NS = MMA warps
  const int sub = warp & 3;                    // TMEM lane quarter this warp may access
  const int h = (warp % kWarpsPerSlot) >> 2;   // column group of every chunk (0 .. NG-1)
  const int p = sub * 32 + lane;               // pair slot within the tile == TMEM lane
  const int wg_tid = threadIdx.x - s * kWG;

  // tiles of slot s: tk = s, s+NS, ... with tr = blockIdx.x + tk * gridDim.x < n_tiles
  auto slot_tiles = [&](int slot) -> int64_t {
    const int64_t per = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tk = 0..per-1
    return per <= slot ? 0 : (per - slot + NS - 1) / NS;
  };
  if (threadIdx.x == 0) {
    turn[0] = 0;   // slot 0 always has a tile (grid <= n_tiles)
    for (int b = 0; b < NS; ++b) slot_done[b] = slot_tiles(b) == 0 ? 1 : 0;
    mbar_init(bar_g, 1);
    for (int b = 0; b < 2 * NS; ++b) {
      mbar_init(bar_mma0 + 8 * b, 1);
      mbar_init(bar_go0 + 8 * b, 1);
    }
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
  clock_probe(g_tc_clock, 0);
  if (*tmem_holder != 0) __trap();  // cannot happen with a full 512-column allocation
  if (threadIdx.x == 0) {  // stage K and K (.) C_s once per CTA (TMA bulk copies)
    mbar_expect_tx(bar_g, (uint32_t)(2 * S::kImg));
    constexpr uint32_t kChunkBytes = 32768;
    for (uint32_t off = 0; off < S::kImg; off += kChunkBytes) {
      const uint32_t n = (uint32_t)((S::kImg - off) < kChunkBytes ? (S::kImg - off) : kChunkBytes);
      bulk_g2s(smem_u32(smem + S::kOffG + off), (const uint8_t*)g_img + off, n, bar_g);
      bulk_g2s(smem_u32(smem + S::kOffGC + off), (const uint8_t*)gc_img + off, n, bar_g);
    }
  }
  const int chains_per_tile = 2 * iters + 2;   // 2L Sinkhorn phases + 2 cost halves

  if (warp >= kEpiWarps) {
    // ------------------------------------------------------------------------ MMA warps
    // One per slot; a turn token passed round the active slots makes their chains alternate in
    // the tensor pipe, and the waiting warps already spin on it while the holder issues, so the
    // handoff overlaps the MMAs still queued.  Only the holder writes the token.
    const int ss = warp - kEpiWarps;
    auto pass_turn = [&]() {
      for (int k = 1; k <= NS; ++k) {
        const int cand = (ss + k) % NS;
        if (cand == ss || !slot_done[cand]) {
          *turn = cand;
          break;
        }
      }
    };
    const uint32_t g_base = smem_u32(smem + S::kOffG), gc_base = smem_u32(smem + S::kOffGC);
    const uint64_t gdesc0 = make_sw128_desc(g_base);
    const uint32_t r0 = (uint32_t)(2 * ss * KP);
    const uint32_t go = bar_go0 + 16 * ss, mma = bar_mma0 + 16 * ss;
    const int64_t n_chains = slot_tiles(ss) * chains_per_tile;
    uint32_t go_par = 0;
    int f = 0;   // chain index within the current tile
    mbar_wait(bar_g, 0);
    for (int64_t j = 0; j < n_chains; ++j) {
      if (f < 2 * iters) {
        // Sinkhorn phase f: A = R[f%2], D = R[(f+1)%2]; two halves of the k-steps
        const uint32_t ra = r0 + (uint32_t)((f & 1) * KP), rd = r0 + (uint32_t)(((f + 1) & 1) * KP);
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          mbar_wait(go + 8 * kc, go_par);
          if (kc == 0)
            while (*turn != ss) __nanosleep(20);
          __syncwarp();
          tc_fence_after();
          if (DBG >= 3 && blockIdx.x == 0 && ss < 2 && j < chains_per_tile && lane == 0 && f < 512)
            g_tc_trace[ss][2 + kc][f] = clock64();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < CH / 8; ++kk) {
              const int ks = kc * (CH / 8) + kk;
              const uint64_t desc = gdesc0 + (uint64_t)((((ks >> 2) * KP * 128) + (ks & 3) * 32) >> 4);
              if (DBG != 2) mma1_tf32_ts(rd, ra + 8 * ks, desc, kIdesc, (kc > 0 || kk > 0) ? 1u : 0u);
            }
            if (kc == 1) {
              mma1_commit(mma);
              mma1_commit(mma + 8);
              if (j + 1 == n_chains) slot_done[ss] = 1;   // last chain of this slot
              pass_turn();
            }
          }
          __syncwarp();
        }
      } else {
        // cost half m = f - 2L: R1[:, 0:KP/2] = R0 (v_L) x (K (.) C_s)[rows m*KP/2 ...]
        const int m = f - 2 * iters;
        mbar_wait(go, go_par);
        mbar_wait(go + 8, go_par);
        while (*turn != ss) __nanosleep(20);
        __syncwarp();
        tc_fence_after();
        if (elect_one()) {
          const uint64_t desc0 = make_sw128_desc(gc_base + (uint32_t)(m * (KP / 2) * 128));
#pragma unroll
          for (int ks = 0; ks < KP / 8; ++ks) {
            const uint64_t desc = desc0 + (uint64_t)(((ks >> 2) * KP * 128 + (ks & 3) * 32) >> 4);
            mma1_tf32_ts(r0 + KP, r0 + 8 * ks, desc, kIdescHalf, ks > 0 ? 1u : 0u);
          }
          mma1_commit(mma);
          mma1_commit(mma + 8);
          if (j + 1 == n_chains) slot_done[ss] = 1;
          pass_turn();
        }
        __syncwarp();
      }
      go_par ^= 1u;
      f = f + 1 == chains_per_tile ? 0 : f + 1;
    }
  } else {
    // ------------------------------------------------------------------------ epilogue warps
    float* mrows = marg + (size_t)s * S::kRows * S::kRS;
    const uint32_t lane_off = (uint32_t)(sub * 32) << 16;
    const uint32_t r0 = lane_off + (uint32_t)(2 * s * KP);   // this thread's lane of R0; R1 = r0 + KP
    const uint32_t bar_mma = bar_mma0 + 16 * s, bar_go = bar_go0 + 16 * s;
    uint32_t mma_par = 0;
    bool clamped = false;   // a denominator left [FLT_MIN, 2^126] on an anchor with mass
    // chunk c of this slot's columns is ready: every thread of the slot stored its part
    auto go = [&](int c) {
      tmem_wait_st();
      tc_fence_before();
      named_bar_sync(1 + s, kWG);
      if (wg_tid == 0) mbar_arrive_local(bar_go + 8 * c);
    };
    const int64_t my_tiles = slot_tiles(s);
    for (int64_t tk2 = 0; tk2 < my_tiles; ++tk2) {
      const int64_t tk = s + NS * tk2;
      const int64_t tr = blockIdx.x + tk * (int64_t)gridDim.x;  // tile index within the range
      const int64_t t = units != nullptr ? (int64_t)units[tr] : tile_begin + tr;
      // ---- tile init: marginal rows -> SMEM, V^T = 1 -> R0 (phase 0's A operand)
      named_bar_sync(1 + s, kWG);  // previous tile's readers are done with mrows / red
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
        arow = Hp + (valid ? (int64_t)ii : n_dist) * KP + h * W;
        brow = Hp + (valid ? (int64_t)jj : n_dist) * KP + h * W;
      } else {
        int64_t bi, bj;
        block_pair_decode(t >> 1, num_blocks(n_dist), bi, bj);
        const int64_t i0 = bi * kBlockDist + (t & 1) * 8, j0 = bj * kBlockDist;
        for (int e = wg_tid; e < S::kRows * KP; e += kWG) {
          const int r = e / KP, c = e % KP;
          const int64_t row = r < 8 ? i0 + r : (r < 24 ? j0 + (r - 8) : n_dist);
          float v = (row < n_dist && c < K) ? H[row * K + c] : 0.0f;
          if (r == 24) v = c < K ? 1.0f / (float)K : 0.0f;  // dummy marginal for invalid slots
          mrows[r * S::kRS + c] = v;
        }
        valid = tile_slot_pair(t, p, n_dist, ii, jj);
        arow = mrows + (valid ? (p >> 4) : 24) * S::kRS + h * W;
        brow = mrows + (valid ? 8 + (p & 15) : 24) * S::kRS + h * W;
      }
      // (EX) marginal values of the current chunk, prefetched from L2 one chunk ahead
      float mk[EX ? W : 1];
      auto load_mk = [&](int f, int c) {
        if constexpr (EX) {
          const float4* m4 = reinterpret_cast<const float4*>(((f & 1) ? brow : arow) + c * CH);
#pragma unroll
          for (int e = 0; e < W / 4; ++e) {
            const float4 mq = __ldg(m4 + e);
            mk[4 * e] = mq.x; mk[4 * e + 1] = mq.y; mk[4 * e + 2] = mq.z; mk[4 * e + 3] = mq.w;
          }
        }
      };
      load_mk(0, 0);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t ones[W];
#pragma unroll
        for (int e = 0; e < W; ++e) ones[e] = (c * CH + h * W + e < K) ? 0x3f800000u : 0u;
        tmem_st_cols<W>(r0 + c * CH + h * W, ones);
      }
      go(0);  // (its barrier also publishes mrows to the slot's warps)
      if (wg_tid == 0) mbar_arrive_local(bar_go + 8);

      for (int f = 0; f < 2 * iters; ++f) {
        const float* mrow = (f & 1) ? brow : arow;  // u-update: a = H[i]; v-update: b = H[j]
        const uint32_t rd = r0 + (uint32_t)(((f + 1) & 1) * KP) + h * W;
        const bool last = f + 1 == 2 * iters;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          mbar_wait(bar_mma + 8 * c, mma_par);
          tc_fence_after();
          if (DBG >= 3 && blockIdx.x == 0 && tk < 2 && wg_tid == 0 && f < 512) g_tc_trace[s][c][f] = clock64();
          if (DBG != 1 && DBG != 4) {
            // the thread's W columns of chunk c in sub-blocks of SB (live registers stay small
            // when one column group covers a whole chunk)
#pragma unroll
            for (int b0 = 0; b0 < W; b0 += SB) {
              uint32_t d[SB];
              tmem_ld_cols<SB>(rd + c * CH + b0, d);
              float m[SB];
              if constexpr (EX) {
#pragma unroll
                for (int e = 0; e < SB; ++e) m[e] = mk[b0 + e];
              } else {
                const float4* m4 = reinterpret_cast<const float4*>(mrow + c * CH + b0);
#pragma unroll
                for (int e = 0; e < SB / 4; ++e) {
                  const float4 mq = m4[e];
                  m[4 * e] = mq.x; m[4 * e + 1] = mq.y; m[4 * e + 2] = mq.z; m[4 * e + 3] = mq.w;
                }
              }
              tmem_wait_ld();
              // x = m / D, one MUFU per two anchors while the sub-block's D lie in
              // [2^-62, 2^62], else one clamped reciprocal each (S:62 clamp + flag); m = 0 gives
              // exactly 0 (R#11).
              uint32_t o[SB];
              const bool bad = epi_div_fast<SB>(m, d, o);
              if (__builtin_expect(__any_sync(0xffffffffu, bad), 0)) {   // a product D0 D1 out of fp32 range (rare)
#pragma unroll
                for (int s8 = 0; s8 < SB; s8 += 8) {
                  uint32_t d8[8];
                  tmem_ld8u(rd + c * CH + b0 + s8, d8);
                  tmem_wait_ld();
                  if (bad) epi_div_fix8(m + s8, d8, o + s8, clamped);
                }
              }
              tmem_st_cols<SB>(rd + c * CH + b0, o);  // in place: the new scaling replaces D
            }
            if (c == 0) load_mk(f, 1);
            else if (!last) load_mk(f + 1, 0);
          }
          if (!last) go(c);
        }
        mma_par ^= 1u;
        if (last) tmem_wait_st();
      }
      // ---- cost (a6): u_L in R1, v_L in R0.  Thread half h covers columns [h KP/4, (h+1) KP/4)
      // of each cost half; the two partials meet in SMEM.
      const uint32_t r1 = r0 + KP;
      float ust[CQ];
#pragma unroll
      for (int c = 0; c < CQ / 8; ++c) tmem_ld8(r1 + h * CQ + 8 * c, &ust[8 * c]);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < CQ; ++e) ust[e] = tf32_mask(ust[e]);
      go(0);
      if (wg_tid == 0) mbar_arrive_local(bar_go + 8);
      mbar_wait(bar_mma, mma_par);
      mbar_wait(bar_mma + 8, mma_par);
      mma_par ^= 1u;
      tc_fence_after();
      float acc = 0.0f;
#pragma unroll
      for (int c = 0; c < CQ / 8; ++c) {
        float g[8];
        tmem_ld8(r1 + h * CQ + 8 * c, g);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(ust[8 * c + e], g[e], acc);
      }
      tc_fence_before();
      named_bar_sync(1 + s, kWG);   // everyone consumed the first half's product
      if (wg_tid == 0) {
        mbar_arrive_local(bar_go);
        mbar_arrive_local(bar_go + 8);
      }
      mbar_wait(bar_mma, mma_par);
      mbar_wait(bar_mma + 8, mma_par);
      mma_par ^= 1u;
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < CQ / 8; ++c) {
        float g[8], u[8];
        tmem_ld8(r1 + h * CQ + 8 * c, g);
        tmem_ld8(r1 + KP / 2 + h * CQ + 8 * c, u);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(tf32_mask(u[e]), g[e], acc);
      }
      float* rs = red + s * 128;
      if (NG == 1) {
        tc_fence_before();
        named_bar_sync(1 + s, kWG);   // R1 reads done before the next tile's phase-0 MMA
        if (!EX || tr * kTileSlots + p < n_pairs)   // (pair lists: no slot past the list)
          write_result(out, tr * kTileSlots + p, valid, ii, jj, acc);
        continue;
      }
      if (h == 1) rs[p] = acc;
      tc_fence_before();
      named_bar_sync(1 + s, kWG);   // (also: R1 reads done before the next tile's phase-0 MMA)
      if (h == 0 && (!EX || tr * kTileSlots + p < n_pairs))
        write_result(out, tr * kTileSlots + p, valid, ii, jj, acc + rs[p]);
    }
    if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
  }
  tc_fence_before();
  __syncthreads();
  clock_probe(g_tc_clock, 1);
  tc_fence_after();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(0u), "r"(kTmemCols)
                 : "memory");
  }
}

template <int KP>
static cudaError_t launch_kp(int64_t tile_begin, int64_t n_tiles, int64_t n_dist, const PairSink& out,
                             const float* H, int K, const uint32_t* g_img, const uint32_t* gc_img,
                             int iters, cudaStream_t s, const int32_t* pi = nullptr,
                             const int32_t* pj = nullptr, int64_t n_pairs = 0, const float* Hp = nullptr,
                             const int32_t* units = nullptr, const int64_t* n_dev = nullptr) {
  const size_t smem = Smem<KP>::kBytes;
#ifdef ASOT_DEBUG_KERNELS   // diagnostic variants (tools/): only in debug builds
  static const int dbg = getenv("ASOT_TC_DEBUG_MODE") ? atoi(getenv("ASOT_TC_DEBUG_MODE")) : 0;
  auto kern = pi != nullptr ? sinkhorn_tc_kernel<KP, 0, true>
            : dbg == 1 ? sinkhorn_tc_kernel<KP, 1, false> : dbg == 2 ? sinkhorn_tc_kernel<KP, 2, false>
            : dbg == 3 ? sinkhorn_tc_kernel<KP, 3, false> : dbg == 4 ? sinkhorn_tc_kernel<KP, 4, false>
            : sinkhorn_tc_kernel<KP, 0, false>;
#else
  auto kern = pi != nullptr ? sinkhorn_tc_kernel<KP, 0, true> : sinkhorn_tc_kernel<KP, 0, false>;
#endif
  cudaError_t e = cudaFuncSetAttribute(kern,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (n_tiles + Slots<KP>::NS - 1) / Slots<KP>::NS;
  if (grid > sms) grid = sms;
  if (grid < 1) return cudaSuccess;
  kern<<<(unsigned)grid, Slots<KP>::kAllThreads, smem, s>>>(tile_begin, n_tiles, n_dist, out, H, K,
                                                               g_img, gc_img, iters, pi, pj, n_pairs, Hp,
                                                               units, n_dev);
  return cudaGetLastError();
}

// Padded marginal rows for the pair-list mode: Hp[r][c] = H[r][c] (c < K), 0 (K <= c < KP);
// row n_dist = uniform 1/K (the dummy for invalid list entries).
__global__ void pad_marginals_tc_kernel(const float* __restrict__ H, int64_t n_dist, int K, int kp,
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

}  // namespace tc

bool sinkhorn_tc_supported(int K) { return K >= 1 && K <= 128; }

cudaError_t launch_sinkhorn_tc(int64_t tile_begin, int64_t tile_end, int64_t n_dist,
                               const PairSink& out, const float* H, int K, const uint32_t* g_img,
                               const uint32_t* gc_img, int iters, cudaStream_t s, const int32_t* units,
                               const int64_t* n_dev) {
  const int64_t n_tiles = tile_end - tile_begin;
  if (n_tiles <= 0) return cudaSuccess;
  switch (kpad32(K)) {
#define ASOT_TC_CASE(KP)                                                                               \
    case KP: return tc::launch_kp<KP>(tile_begin, n_tiles, n_dist, out, H, K, g_img, gc_img, iters, s, \
                                      nullptr, nullptr, 0, nullptr, units, n_dev);
    ASOT_TC_CASE(32)
    ASOT_TC_CASE(64)
    ASOT_TC_CASE(96)
    ASOT_TC_CASE(128)
#undef ASOT_TC_CASE
    default: return cudaErrorNotSupported;
  }
}

size_t sinkhorn_tc_pairs_scratch_bytes(int64_t n_dist, int K) {
  return (size_t)(n_dist + 1) * kpad32(K) * 4;
}

cudaError_t launch_sinkhorn_tc_pairs(const int32_t* pi, const int32_t* pj, int64_t n_pairs, int64_t n_dist,
                                     const PairSink& out, const float* H, int K, const uint32_t* g_img,
                                     const uint32_t* gc_img, float* Hp, int iters, cudaStream_t s,
                                     const int64_t* n_dev) {
  if (n_pairs <= 0) return cudaSuccess;
  const int kp = kpad32(K);
  tc::pad_marginals_tc_kernel<<<512, 256, 0, s>>>(H, n_dist, K, kp, Hp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t n_tiles = (n_pairs + kTileSlots - 1) / kTileSlots;
  switch (kp) {
#define ASOT_TC_CASE(KP)                                                                                \
    case KP: return tc::launch_kp<KP>(0, n_tiles, n_dist, out, H, K, g_img, gc_img, iters, s, pi, pj, \
                                      n_pairs, Hp, nullptr, n_dev);
    ASOT_TC_CASE(32)
    ASOT_TC_CASE(64)
    ASOT_TC_CASE(96)
    ASOT_TC_CASE(128)
#undef ASOT_TC_CASE
    default: return cudaErrorNotSupported;
  }
}

}  // namespace asot

extern "C" int asot_debug_tc_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, asot::tc::g_tc_trace, sizeof(asot::tc::g_tc_trace));
}

namespace asot {
cudaError_t read_kernel_clock_tc(long long* host4) {
  return cudaMemcpyFromSymbol(host4, tc::g_tc_clock, 4 * sizeof(long long));
}
}  // namespace asot
