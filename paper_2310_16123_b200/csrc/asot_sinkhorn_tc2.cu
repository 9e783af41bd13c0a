// asot_sinkhorn_tc2.cu -- steps a5 + a6 for 128 < K <= 256 on a CTA pair (tcgen05 cta_group::2).
//
// Same recurrence as asot_sinkhorn_tc.cu (R#3-R#6, R#11): U = A/(K V), V = B/(K^T U),
// v0 = 1, L iterations, d = sum_r u_r ((K (.) C_s) v)_r.  K (256 x 256 TF32 = 256 KB) does not fit
// one SM's shared memory, so a cluster of two CTAs computes M = 256 pairs per MMA
// (tcgen05.mma.cta_group::2.kind::tf32, A from TMEM): CTA c owns the 128-slot tile 2b+c of block
// pair b, keeps its 128 pairs' scalings in its own TMEM, and holds rows {nc*64 + c*32 + [0,32)}
// (nc = 0..3) of K in its SMEM (the B operand is split N-wise across the pair).  A dedicated MMA
// warp of the leader CTA issues every MMA for both CTAs; commits multicast to both CTAs'
// mbarriers; epilogue completion is reported to the leader by remote mbarrier arrives.
//
// TMEM (per CTA, 512 columns): R0 = [0,256), R1 = [256,512).  Phase f reads A from R[f%2] and
// writes D into R[(f+1)%2]; the epilogue writes the new scaling IN PLACE over D, so the roles
// swap every phase.  The anchors are cut into four 64-wide chunks.  A phase is issued as 16 parts
// (kc, nc) = (input chunk, output chunk), kc-major, each 8 MMAs of M=256 x N=64 x k=8: the parts
// of input chunk kc wait only for the epilogue of chunk kc of the previous phase, and output
// chunk nc is complete (commit) after part (3, nc).  So the next phase's first parts wait for the
// epilogue of ONE chunk (all 16 epilogue warps, 16 anchors per thread) that starts three parts
// (~780 cycles) before the tensor pipe runs dry: the epilogue latency is hidden, not just
// overlapped with half a phase.  For K <= 192 the all-padding fourth chunk is skipped (9 parts).
//
// Cost (a6): v_L is written in place into D; u_L stays in A.  K (.) C_s is streamed through a
// 32 KB SMEM staging buffer in four (N-half, K-half) sub-parts (once per tile: < 1% of a tile),
// the products land in the consumed half of A, and each thread reduces its 32 anchors.
#include <cfloat>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace tc2 {

constexpr int kKP = 256;
constexpr int kChunk = 64;                  // anchors per epilogue chunk / MMA part
constexpr int kNChunks = kKP / kChunk;
constexpr int kWarps = 16;                  // epilogue warps
constexpr int kThreads = kWarps * 32;
constexpr int kAllThreads = kThreads + 32;  // + the MMA warp

using namespace ::asot::ptx;

// ----------------------------------------------------------------------------- SMEM layout
struct Smem {
  static constexpr int kRS = kKP + 4;
  static constexpr int kRows = 25;
  static constexpr size_t kOffG = 0;                          // 128 KB: [kb 8][nc 4][32 rows][128 B]
  static constexpr size_t kOffStage = 128 * 1024;             // 32 KB:  [kb_in 4][64 rows][128 B]
  static constexpr size_t kOffMarg = kOffStage + 32 * 1024;   // 25 x 260 floats
  static constexpr size_t kOffRed = kOffMarg + (size_t)kRows * kRS * 4;  // [4][128] floats
  static constexpr size_t kOffBar = kOffRed + 4 * 128 * 4;
  static constexpr size_t kBytes = kOffBar + 128 + 1024;
};

// Global image offsets (bytes) within one rank's image; element (output anchor n, k), n and k in
// [0, 256).  K (the Sinkhorn B operand): n = nc*64 + rank*32 + r, blocks [kb 8][nc 4][32 rows][128 B]
// (an N = 64 part of chunk nc takes 32 rows from each CTA).  K (.) C_s (the cost B operand, N = 128
// sub-parts): n = Nh*128 + rank*64 + r, blocks [Nh 2][kb 8][64 rows][128 B].
__host__ __device__ inline uint32_t sw_block(uint32_t r, uint32_t kin) {  // [rows][128 B], SW128
  const uint32_t lin = r * 128u + kin * 4u;
  return lin ^ (((lin >> 7) & 7u) << 4);
}
__host__ __device__ inline uint32_t g_image_offset(uint32_t nc, uint32_t r, uint32_t k) {
  return (k >> 5) * 16384u + nc * 4096u + sw_block(r, k & 31);
}
__host__ __device__ inline uint32_t gc_image_offset(uint32_t nh, uint32_t r, uint32_t k) {
  const uint32_t kb = k >> 5;
  return nh * 65536u + (kb >> 2) * 32768u + (kb & 3) * 8192u + sw_block(r, k & 31);
}

__device__ long long g_tc2_trace[4][256];
__device__ long long g_tc2_clock[4];  // clock_probe: (clock64, globaltimer) at start / end

template <int DBG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kAllThreads, 1)
sinkhorn_tc2_kernel(int64_t tile_begin, int64_t tile_end, int64_t n_dist, PairSink out,
                    const float* __restrict__ H, int K, const uint8_t* __restrict__ g_img,
                    const uint8_t* __restrict__ gc_img, int iters, const int32_t* __restrict__ units,
                    const int64_t* __restrict__ n_dev) {
  if (dense_skipped(out)) return;   // the small-support kernel serves this call (R#36)
  using S = Smem;
  constexpr uint32_t kIdescPart = make_idesc_tf32(256, kChunk);   // Sinkhorn parts: N = 64
  constexpr uint32_t kIdescCost = make_idesc_tf32(256, 128);      // cost sub-parts: N = 128
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* mrows = (float*)(smem + S::kOffMarg);
  float* red = (float*)(smem + S::kOffRed);
  uint64_t* bars = (uint64_t*)(smem + S::kOffBar);
  // bars: 0 g_loaded, 1-4 mma_done[c] (D chunk c complete), 5-8 epi_done[c] (leader only used:
  // scaling chunk c written by both CTAs), 9 cost_done
  uint32_t* tmem_holder = (uint32_t*)(bars + 12);
  const uint32_t bar_g = smem_u32(&bars[0]);
  const uint32_t bar_mma0 = smem_u32(&bars[1]);
  const uint32_t bar_epi0 = smem_u32(&bars[5]);
  const uint32_t bar_cost = smem_u32(&bars[9]);
  static_assert(Smem::kOffBar % 8 == 0, "barrier alignment");

  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool epi_warp = warp < kWarps;
  const int q = warp & 3;            // TMEM lane quarter
  const int cq = (warp >> 2) & 3;    // column group: 16 columns of every 64-anchor chunk
  const int p = q * 32 + lane;       // pair slot within this CTA's tile == TMEM lane

  if (threadIdx.x == 0) {
    mbar_init(bar_g, 1);
    for (int c = 0; c < kNChunks; ++c) {
      mbar_init(bar_mma0 + 8 * c, 1);
      mbar_init(bar_epi0 + 8 * c, 2);
    }
    mbar_init(bar_cost, 1);
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
  clock_probe(g_tc2_clock, 0);
  if (*tmem_holder != 0) __trap();  // full 512-column allocation starts at column 0
  if (threadIdx.x == 0) {          // this CTA's half of K, once (TMA bulk copies)
    const uint8_t* src = g_img + (size_t)rank * (128 * 1024);
    mbar_expect_tx(bar_g, 128 * 1024);
    for (uint32_t off = 0; off < 128 * 1024; off += 32768)
      bulk_g2s(smem_u32(smem + S::kOffG + off), src + off, 32768, bar_g);
  }
  const uint32_t g_base = smem_u32(smem + S::kOffG);
  const uint32_t st_base = smem_u32(smem + S::kOffStage);
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  const uint32_t epi_remote0 = mapa(bar_epi0, 0);  // leader's epi_done[0] (cluster address)
  const bool leader = rank == 0;
  const bool issuer = leader && warp == kWarps;    // the MMA warp (Sinkhorn parts and cost)
  // 64-anchor chunks holding real anchors: K <= 192 skips the all-padding fourth chunk in every
  // Sinkhorn phase (9 of the 16 parts); the padded scalings stay exactly 0 there
  const int NCH = (K + kChunk - 1) / kChunk;

  uint32_t mma_par = 0, epi_par = 0, cost_par = 0;   // one parity bit per barrier family (all
                                                     // chunks of a family complete once per phase)
  bool g_ready = false;

  // Part (kc, nc) of phase f: D(R_d)[:, nc*64 +: 64] (+)= A(R_a)[:, kc*64 +: 64] x K[kc, nc]
  // The MMA warp's per-part instruction stream is kept minimal (it shares its SM sub-partition
  // with four busy epilogue warps): one descriptor base per input chunk, constant offsets.
  const uint64_t gdesc0 = make_sw128_desc(g_base);
  auto issue_part = [&](uint32_t a_col, uint32_t d_col, uint64_t desc, uint32_t acc0) {
#pragma unroll
    for (int ks = 0; ks < kChunk / 8; ++ks)
      mma2_tf32_ts(d_col, a_col + 8 * ks, desc + (uint64_t)((((ks >> 2) * 16384) + (ks & 3) * 32) >> 4), kIdescPart,
                   ks > 0 ? 1u : acc0);
  };
  // End of an epilogue chunk: every epilogue thread of this CTA stored its part of chunk c;
  // report to the leader's epi_done[c].
  auto chunk_done = [&](int c) {
    tmem_wait_st();
    tc_fence_before();
    named_bar_sync(1, kThreads);
    if (threadIdx.x == 0) mbar_arrive_cluster(epi_remote0 + 8 * c);
  };

  bool clamped = false;   // a denominator left [FLT_MIN, 2^126] on an anchor with mass
  // block pairs kb = 0, 1, ... of the range, or (bucketed pair lists) of the unit list
  int64_t n_kb = ((tile_end + 1) >> 1) - (tile_begin >> 1);
  if (units != nullptr && *n_dev < n_kb) n_kb = *n_dev;
  for (int64_t kb = blockIdx.x >> 1; kb < n_kb; kb += gridDim.x >> 1) {
    const int64_t b = units != nullptr ? (int64_t)units[kb] : (tile_begin >> 1) + kb;
    const int64_t t = 2 * b + rank;          // this CTA's tile
    const bool t_in = units != nullptr || (t >= tile_begin && t < tile_end);
    // ---- tile init
    int64_t bi, bj;
    block_pair_decode(b, num_blocks(n_dist), bi, bj);
    const int64_t i0 = bi * kBlockDist + rank * 8, j0 = bj * kBlockDist;
    __syncthreads();  // previous tile's readers are done with mrows / red
    for (int e = threadIdx.x; e < S::kRows * kKP; e += kAllThreads) {
      const int r = e / kKP, c = e % kKP;
      const int64_t row = r < 8 ? i0 + r : (r < 24 ? j0 + (r - 8) : n_dist);
      float v = (row < n_dist && c < K) ? H[row * K + c] : 0.0f;
      if (r == 24) v = c < K ? 1.0f / (float)K : 0.0f;  // dummy marginal for invalid slots
      mrows[r * S::kRS + c] = v;
    }
    int ii, jj;
    // TMEM lane p holds tile slot ps: a warp's 32 lanes then touch 8 distinct i-rows and 4
    // distinct j-rows of the marginals (one SMEM wavefront per 16-byte load, not two)
    const int ps = ((p & 7) << 4) | (p >> 3);
    const bool valid = tile_slot_pair(t, ps, n_dist, ii, jj) && t_in;
    const float* arow = mrows + (valid ? (ps >> 4) : 24) * S::kRS + cq * 16;
    const float* brow = mrows + (valid ? 8 + (ps & 15) : 24) * S::kRS + cq * 16;
    if (!g_ready) {
      mbar_wait(bar_g, 0);
      g_ready = true;
    }
    if (epi_warp) {
#pragma unroll
      for (int c = 0; c < kNChunks; ++c) {  // V^T = 1 into R0 (phase 0's A operand)
        uint32_t ones[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) ones[e] = (c * kChunk + cq * 16 + e < K) ? 0x3f800000u : 0u;
        tmem_st16(lane_off + c * kChunk + cq * 16, ones);
        if (c >= NCH) {   // skipped chunk: R1's copy is read by the cost, so it must be 0 too
          uint32_t zeros[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) zeros[e] = 0u;
          tmem_st16(lane_off + 256 + c * kChunk + cq * 16, zeros);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      named_bar_sync(1, kThreads);
      if (threadIdx.x == 0)
        for (int c = 0; c < kNChunks; ++c) mbar_arrive_cluster(epi_remote0 + 8 * c);

      // marginal values of the next chunk are prefetched into registers right after the
      // current chunk's stores, so the SMEM reads stay off the chunk's critical path
      float mk[16];
      auto load_m = [&](int f, int c) {
        const float4* m4 = reinterpret_cast<const float4*>(((f & 1) ? brow : arow) + c * kChunk);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4 mq = m4[e];
          mk[4 * e] = mq.x; mk[4 * e + 1] = mq.y; mk[4 * e + 2] = mq.z; mk[4 * e + 3] = mq.w;
        }
      };
      load_m(0, 0);
      for (int f = 0; f < 2 * iters; ++f) {
        const uint32_t rd = lane_off + (uint32_t)(((f + 1) & 1) * 256) + cq * 16;
        const bool last = f + 1 == 2 * iters;
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          mbar_wait(bar_mma0 + 8 * c, mma_par);
          tc_fence_after();
          if (DBG >= 3 && blockIdx.x == 0 && kb == 0 && threadIdx.x == 0 && f < 64)
            g_tc2_trace[0][f * 4 + c] = clock64();
          if (DBG != 1 && DBG != 4) {
            uint32_t d[16];
            tmem_ld16u(rd + c * kChunk, d);
            tmem_wait_ld();
            reg_fence16(d);
            // x = m / D, one MUFU per two anchors; a product D0 D1 out of fp32 range (rare):
            // reload D, per-anchor clamped reciprocals on that thread (S:62 clamp + flag)
            uint32_t o[16];
            const bool bad = epi_div_fast<16>(mk, d, o);
            if (__builtin_expect(__any_sync(0xffffffffu, bad), 0)) {   // a product D0 D1 out of fp32 range (rare)
#pragma unroll
              for (int s8 = 0; s8 < 16; s8 += 8) {
                uint32_t d8[8];
                tmem_ld8u(rd + c * kChunk + s8, d8);
                tmem_wait_ld();
                if (bad) epi_div_fix8(mk + s8, d8, o + s8, clamped);
              }
            }
            tmem_st16(rd + c * kChunk, o);  // in place: the new scaling replaces D
            if (c + 1 < NCH) load_m(f, c + 1);
            else if (!last) load_m(f + 1, 0);
          }
          if (DBG >= 3 && blockIdx.x == 0 && kb == 0 && threadIdx.x == 0 && f < 64)
            g_tc2_trace[1][f * 4 + c] = clock64();
          if (!last) chunk_done(c);
        }
        mma_par ^= 1u;
        if (last) tmem_wait_st();
      }
    } else if (issuer) {
      // Issue order: input chunks 0 .. NCH-3 for every output chunk; then (NCH-2, 0),
      // (NCH-2, 1), (NCH-1, 0), (NCH-2, 2), (NCH-2, 3), (NCH-1, 1), (NCH-1, 2), (NCH-1, 3): output
      // chunk 0 completes five parts before the phase ends (kc-major: three), so its epilogue --
      // the one the next phase's first parts wait for -- has more cover.  Each output chunk still
      // accumulates its input chunks in order.
      auto part = [&](int f, int kc, int nc) {
        const uint32_t a_col = (uint32_t)((f & 1) * 256 + kc * kChunk);
        const uint32_t d_col = (uint32_t)(((f + 1) & 1) * 256);
        const uint64_t desc = gdesc0 + (uint64_t)((kc * 2 * 16384 + nc * 4096) >> 4);
        if (DBG != 2) issue_part(a_col, d_col + nc * kChunk, desc, kc > 0 ? 1u : 0u);
        if (kc == NCH - 1) mma2_commit_mc(bar_mma0 + 8 * nc);
      };
      auto gate = [&](int f, int kc) {
        mbar_wait(bar_epi0 + 8 * kc, epi_par);
        tc_fence_after();
        if (DBG >= 3 && blockIdx.x == 0 && kb == 0 && lane == 0 && f < 64)
          g_tc2_trace[2][f * 4 + kc] = clock64();
      };
      for (int f = 0; f < 2 * iters; ++f) {
#pragma unroll 1
        for (int kc = 0; kc < NCH - 2; ++kc) {
          gate(f, kc);
          if (elect_one()) {
            for (int nc = 0; nc < NCH; ++nc) part(f, kc, nc);
          }
          __syncwarp();
        }
        const int a = NCH - 2, z = NCH - 1;
        gate(f, a);
        if (elect_one()) { part(f, a, 0); part(f, a, 1); }
        __syncwarp();
        gate(f, z);
        if (elect_one()) {
          part(f, z, 0);
          for (int nc = 2; nc < NCH; ++nc) part(f, a, nc);
          for (int nc = 1; nc < NCH; ++nc) part(f, z, nc);
        }
        __syncwarp();
        epi_par ^= 1u;
      }
    }  // (the peer's MMA warp idles until the cost)

    long long t_cost0 = 0;
    if (DBG >= 3) t_cost0 = clock64();
    // ---- cost: u_L in R_a = R[(2L-1)%2] = R1, v_L in R_d = R0 (both as RNA-pre bits)
    const uint32_t ra = lane_off + 256, rdv = 0;  // A-operand (v_L) region base = R0
    float ust[32];
    if (epi_warp) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld8(ra + cq * 32 + 8 * c, &ust[8 * c]);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) ust[e] = tf32_mask(ust[e]);
    }
    float acc = 0.0f;
    for (int sp = 0; sp < 4; ++sp) {  // sub-parts (Nh, Kh) = (sp >> 1, sp & 1)
      const int nh = sp >> 1, kh = sp & 1;
      // stage this CTA's K (.) C_s sub-block (32 KB, contiguous in its image) into SMEM
      const float4* src = reinterpret_cast<const float4*>(gc_img + (size_t)rank * (128 * 1024) +
                                                          (size_t)nh * 65536 + (size_t)kh * 32768);
      float4* dst = reinterpret_cast<float4*>(smem + S::kOffStage);
      for (int e = threadIdx.x; e < 32768 / 16; e += kAllThreads) dst[e] = src[e];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      cluster_sync();
      tc_fence_after();
      if (issuer && elect_one()) {
        const uint64_t desc0 = make_sw128_desc(st_base);
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          const uint64_t desc = desc0 + (uint64_t)(((ks >> 2) * 8192 + (ks & 3) * 32) >> 4);
          mma2_tf32_ts(256, rdv + kh * 128 + 8 * ks, desc, kIdescCost, (kh > 0 || ks > 0) ? 1u : 0u);
        }
        mma2_commit_mc(bar_cost);
      }
      __syncwarp();
      mbar_wait(bar_cost, cost_par);
      cost_par ^= 1u;
      tc_fence_after();
      if (kh == 1 && epi_warp) {
        // (K (.) C_s) v for anchors [nh*128, nh*128+128) now sits in R1 columns [0, 128)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float g[8], u[8];
          tmem_ld8(ra + cq * 32 + 8 * c, g);
          if (nh == 1) tmem_ld8(ra + 128 + cq * 32 + 8 * c, u);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float uu = nh == 0 ? ust[8 * c + e] : tf32_mask(u[e]);
            acc = fmaf(uu, g[e], acc);
          }
        }
      }
      tc_fence_before();
      cluster_sync();  // staging buffer and R1 columns free for the next sub-part / tile
      tc_fence_after();
    }
    if (DBG >= 3 && blockIdx.x == 0 && threadIdx.x == 0) {
      const int64_t k = kb / (gridDim.x >> 1);
      if (k < 64) g_tc2_trace[3][k] = clock64() - t_cost0;
    }
    if (epi_warp) red[cq * 128 + p] = acc;
    __syncthreads();
    if (warp < 4 && t_in)
      write_result(out, (units != nullptr ? 2 * kb + rank : t - tile_begin) * kTileSlots + ps, valid, ii, jj,
                   red[p] + red[128 + p] + red[256 + p] + red[384 + p]);
  }
  if (clamped) atomicOr(out.status, ASOT_FLAG_DENOM_CLAMPED);
  tc_fence_before();
  cluster_sync();
  clock_probe(g_tc2_clock, 1);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(0u) : "memory");
}

// ----------------------------------------------------------------------------- image prep
__global__ void gibbs_prep_tc2_kernel(const float* __restrict__ cost, int K, float eps, uint8_t* __restrict__ g_img,
                                      uint8_t* __restrict__ gc_img) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < kKP * kKP; idx += gridDim.x * blockDim.x) {
    const int n = idx / kKP, k = idx % kKP;
    const bool in = n < K && k < K;
    const double c = in ? (double)cost[(int64_t)n * K + k] : 0.0;
    const double g = in ? exp(-c / (double)eps) : 0.0;  // P:183  K := exp(-C_s / eps)
    const uint32_t gb = in ? tf32_rna_bits((float)g) : 0x3f800000u;  // padding = 1 (R#12)
    const uint32_t gcb = in ? tf32_rna_bits((float)(g * c)) : 0u;
    const uint32_t nc = n >> 6, rg = (n >> 5) & 1, r32 = n & 31;
    *(uint32_t*)(g_img + (size_t)rg * (128 * 1024) + g_image_offset(nc, r32, k)) = gb;
    const uint32_t nh = n >> 7, within = n & 127, rk = within >> 6, r = within & 63;
    *(uint32_t*)(gc_img + (size_t)rk * (128 * 1024) + gc_image_offset(nh, r, k)) = gcb;
  }
}

}  // namespace tc2

bool sinkhorn_tc2_supported(int K) { return K > 128 && K <= 256; }
size_t sinkhorn_tc2_image_bytes() { return 2 * 128 * 1024; }

cudaError_t launch_gibbs_prep_tc2(const float* cost, int K, float eps, uint8_t* g_img, uint8_t* gc_img,
                                  cudaStream_t s) {
  tc2::gibbs_prep_tc2_kernel<<<256, 256, 0, s>>>(cost, K, eps, g_img, gc_img);
  return cudaGetLastError();
}

cudaError_t launch_sinkhorn_tc2(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const float* H, int K, const uint8_t* g_img, const uint8_t* gc_img, int iters,
                                cudaStream_t s, const int32_t* units, const int64_t* n_dev) {
  if (tile_end <= tile_begin) return cudaSuccess;
#ifdef ASOT_DEBUG_KERNELS   // diagnostic variants (tools/): only in debug builds
  static const int dbg = getenv("ASOT_TC_DEBUG_MODE") ? atoi(getenv("ASOT_TC_DEBUG_MODE")) : 0;
  auto kern = dbg == 1 ? tc2::sinkhorn_tc2_kernel<1> : dbg == 2 ? tc2::sinkhorn_tc2_kernel<2>
            : dbg == 3 ? tc2::sinkhorn_tc2_kernel<3> : dbg == 4 ? tc2::sinkhorn_tc2_kernel<4>
            : tc2::sinkhorn_tc2_kernel<0>;
#else
  auto kern = tc2::sinkhorn_tc2_kernel<0>;
#endif
  const size_t smem = tc2::Smem::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_bp = ((tile_end + 1) >> 1) - (tile_begin >> 1);
  int64_t clusters = n_bp < sms / 2 ? n_bp : sms / 2;
  if (clusters < 1) clusters = 1;
  kern<<<(unsigned)(2 * clusters), tc2::kAllThreads, smem, s>>>(tile_begin, tile_end, n_dist, out, H, K, g_img,
                                                             gc_img, iters, units, n_dev);
  return cudaGetLastError();
}

}  // namespace asot

extern "C" int asot_debug_tc2_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, asot::tc2::g_tc2_trace, sizeof(asot::tc2::g_tc2_trace));
}

namespace asot {
cudaError_t read_kernel_clock_tc2(long long* host4) {
  return cudaMemcpyFromSymbol(host4, tc2::g_tc2_clock, 4 * sizeof(long long));
}
}  // namespace asot
