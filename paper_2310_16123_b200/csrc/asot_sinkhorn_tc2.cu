// asot_sinkhorn_tc2.cu -- steps a5 + a6 for 128 < K <= 256 on a CTA pair (tcgen05 cta_group::2).
//
// Same recurrence as asot_sinkhorn_tc.cu (R#3-R#6, R#11): U = A/(K V), V = B/(K^T U),
// v0 = 1, L iterations, d = sum_r u_r ((K (.) C_s) v)_r.  K (256 x 256 TF32 = 256 KB) does not fit
// one SM's shared memory, so a cluster of two CTAs computes M = 256 pairs per MMA
// (tcgen05.mma.cta_group::2.kind::tf32, A from TMEM): CTA c owns the 128-slot tile 2b+c of block
// pair b, keeps its 128 pairs' scalings in its own TMEM, and holds the output-anchor half
// {Nh*128 + c*64 + [0,64)} (Nh = 0, 1) of K in its SMEM (the B operand is split N-wise across
// the pair).  Two warps of the leader CTA issue every MMA for both CTAs (see issue_p12/p34);
// commits multicast to both CTAs' mbarriers; epilogue completion is reported to the leader by
// remote mbarrier arrives.
//
// TMEM (per CTA, 512 columns): R0 = [0,256), R1 = [256,512).  Phase f reads A from R[f%2] and
// writes D into R[(f+1)%2]; the epilogue writes the new scaling IN PLACE over D, so the roles
// swap every phase.  Each phase's product is issued as four parts (K-half, N-half) in the order
// (0,0), (0,1), (1,0), (1,1): N-half 0 of D is complete after part 3, so the epilogue of anchor
// half 0 overlaps part 4, and the next phase's parts 1-2 (which only need K-half 0 of the new
// scaling) overlap the epilogue of anchor half 1.  The tensor pipe never waits for a whole
// epilogue.
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
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kHalfThreads = kThreads / 2;

using namespace ::asot::ptx;

// ----------------------------------------------------------------------------- SMEM layout
struct Smem {
  static constexpr int kRS = kKP + 4;
  static constexpr int kRows = 25;
  static constexpr size_t kOffG = 0;                          // 128 KB: [kb 8][Nh 2][64 rows][128 B]
  static constexpr size_t kOffStage = 128 * 1024;             // 32 KB:  [kb_in 4][64 rows][128 B]
  static constexpr size_t kOffMarg = kOffStage + 32 * 1024;   // 25 x 260 floats
  static constexpr size_t kOffRed = kOffMarg + (size_t)kRows * kRS * 4;  // [4][128] floats
  static constexpr size_t kOffBar = kOffRed + 4 * 128 * 4;
  static constexpr size_t kBytes = kOffBar + 128 + 1024;
};

// Global image offsets (bytes) within one rank's image; element (output anchor n, k), n and k in
// [0, 256).  Output anchors are split as n = Nh*128 + rank*64 + r.
__host__ __device__ inline uint32_t sw_block(uint32_t r, uint32_t kin) {  // [64 or 128 rows][128 B]
  const uint32_t lin = r * 128u + kin * 4u;
  return lin ^ (((lin >> 7) & 7u) << 4);
}
__host__ __device__ inline uint32_t g_image_offset(uint32_t nh, uint32_t r, uint32_t k) {
  return (k >> 5) * 16384u + nh * 8192u + sw_block(r, k & 31);
}
__host__ __device__ inline uint32_t gc_image_offset(uint32_t nh, uint32_t r, uint32_t k) {
  const uint32_t kb = k >> 5;
  return nh * 65536u + (kb >> 2) * 32768u + (kb & 3) * 8192u + sw_block(r, k & 31);
}

__device__ long long g_tc2_trace[18][256];

template <int DBG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
sinkhorn_tc2_kernel(int64_t tile_begin, int64_t tile_end, int64_t n_dist, PairSink out,
                    const float* __restrict__ H, int K, const uint8_t* __restrict__ g_img,
                    const uint8_t* __restrict__ gc_img, int iters) {
  using S = Smem;
  constexpr uint32_t kIdescPart = make_idesc_tf32(256, 128);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* mrows = (float*)(smem + S::kOffMarg);
  float* red = (float*)(smem + S::kOffRed);
  uint64_t* bars = (uint64_t*)(smem + S::kOffBar);
  // bars: 0 g_loaded, 1-2 mma_done[h], 3-4 epi_done[h] (leader only used), 5 cost_done
  uint32_t* tmem_holder = (uint32_t*)(bars + 8);
  volatile long long* p12_token = (volatile long long*)(bars + 9);  // last phase whose parts 1-2 are issued
  const uint32_t bar_g = smem_u32(&bars[0]);
  const uint32_t bar_mma0 = smem_u32(&bars[1]);
  const uint32_t bar_epi0 = smem_u32(&bars[3]);
  const uint32_t bar_cost = smem_u32(&bars[5]);
  static_assert(Smem::kOffBar % 8 == 0, "barrier alignment");

  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;            // TMEM lane quarter
  const int cq = warp >> 2;          // anchor (column) quarter: columns [cq*64, cq*64+64)
  const int h = cq >> 1;             // anchor half handled by this warp in the Sinkhorn phases
  const int p = q * 32 + lane;       // pair slot within this CTA's tile == TMEM lane
  const int htid = threadIdx.x - h * kHalfThreads;  // 0..255 within the half's warps

  if (threadIdx.x == 0) {
    *p12_token = -1;
    mbar_init(bar_g, 1);
    mbar_init(bar_mma0, 1);
    mbar_init(bar_mma0 + 8, 1);
    mbar_init(bar_epi0, 2);
    mbar_init(bar_epi0 + 8, 2);
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
  const bool issuer = leader && warp == 0;  // also issues the cost MMAs
  int64_t gphase = 0;                        // phases issued before this tile (token namespace)

  uint32_t mma_par[2] = {0, 0}, epi_par[2] = {0, 0}, cost_par = 0;
  bool g_ready = false;

  // Issue one part (Kh, Nh) of phase f: D(R_d)[:, Nh] (+)= A(R_a)[:, Kh] x K[Kh, Nh]
  auto issue_part = [&](int f, int kh, int nh) {
    const uint32_t ra = (uint32_t)((f & 1) * 256), rd = (uint32_t)(((f + 1) & 1) * 256);
    const uint64_t desc0 = make_sw128_desc(g_base + (uint32_t)(kh * 4 * 16384 + nh * 8192));
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
      const uint64_t desc = desc0 + (uint64_t)(((ks >> 2) * 16384 + (ks & 3) * 32) >> 4);
      mma2_tf32_ts(rd + nh * 128, ra + kh * 128 + 8 * ks, desc, kIdescPart, (kh > 0 || ks > 0) ? 1u : 0u);
    }
  };
  // Two issuers in the leader CTA.  Warp 0 (anchor half 0) issues parts 1-2 of phase f as soon
  // as both CTAs finished epilogue half 0 (they only need K-half 0 of the new scaling); warp 8
  // (anchor half 1) issues parts 3-4 after epilogue half 1 and after parts 1-2 are in the queue
  // (token), then commits "D half 0 ready" and "D half 1 ready" to both CTAs.  Each issuer's
  // blocking issue ends before its own next epilogue half is due.
  auto issue_p12 = [&](int f, int64_t gph) {
    if (DBG >= 3 && blockIdx.x == 0 && f < 256 && gph == f && lane == 0) g_tc2_trace[16][f] = clock64();
    if (DBG == 7 || DBG == 8) mbar_wait_poll(bar_epi0, epi_par[0]);
    else mbar_wait(bar_epi0, epi_par[0]);
    if (DBG >= 3 && blockIdx.x == 0 && f < 256 && gph == f && lane == 0) g_tc2_trace[17][f] = clock64();
    epi_par[0] ^= 1u;
    tc_fence_after();
    if (elect_one()) {
      if (DBG >= 3 && blockIdx.x == 0 && f < 256 && gph == f) g_tc2_trace[4][f] = clock64();
      if (DBG != 2) {
        issue_part(f, 0, 0);
        issue_part(f, 0, 1);
      }
      if (DBG >= 3 && blockIdx.x == 0 && f < 256 && gph == f) g_tc2_trace[5][f] = clock64();
      *p12_token = gph;
    }
    __syncwarp();
  };
  auto issue_p34 = [&](int f, int64_t gph) {
    if (DBG == 7 || DBG == 8) mbar_wait_poll(bar_epi0 + 8, epi_par[1]);
    else mbar_wait(bar_epi0 + 8, epi_par[1]);
    epi_par[1] ^= 1u;
    while (*p12_token < gph) __nanosleep(20);
    __syncwarp();
    tc_fence_after();
    if (elect_one()) {
      if (DBG >= 3 && blockIdx.x == 0 && f < 256 && gph == f) g_tc2_trace[6][f] = clock64();
      if (DBG != 2) issue_part(f, 1, 0);
      mma2_commit_mc(bar_mma0);
      if (DBG != 2) issue_part(f, 1, 1);
      mma2_commit_mc(bar_mma0 + 8);
      if (DBG >= 3 && blockIdx.x == 0 && f < 256 && gph == f) g_tc2_trace[7][f] = clock64();
    }
    __syncwarp();
  };
  auto issue_phase = [&](int f, int64_t gph) {
    if (leader && warp == 0) issue_p12(f, gph);
    if (leader && warp == 8) issue_p34(f, gph);
  };
  // End of an epilogue half: all of the half's threads stored to TMEM; report to the leader.
  long long t_wake = 0;
  int trace_f = -1;
  auto half_done = [&]() {
    tmem_wait_st();
    tc_fence_before();
    named_bar_sync(1 + h, kHalfThreads);
    if (DBG >= 3 && blockIdx.x < 2 && htid == 0 && trace_f >= 0 && trace_f < 256)
      g_tc2_trace[8 + 2 * h + blockIdx.x][trace_f] = clock64() - t_wake;
    if (htid == 0) {
      if (DBG == 9 && leader) mbar_arrive_local(bar_epi0 + 8 * h);
      else mbar_arrive_cluster(epi_remote0 + 8 * h);
    }
  };

  const int64_t n_bp_total = num_blocks(n_dist) * (num_blocks(n_dist) + 1) / 2;
  const int64_t bp_begin = tile_begin >> 1, bp_end = (tile_end + 1) >> 1;
  const int64_t cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  (void)n_bp_total;

  for (int64_t b = bp_begin + cluster_id; b < bp_end; b += n_clusters) {
    const int64_t t = 2 * b + rank;          // this CTA's tile
    const bool t_in = t >= tile_begin && t < tile_end;
    // ---- tile init
    int64_t bi, bj;
    block_pair_decode(b, num_blocks(n_dist), bi, bj);
    const int64_t i0 = bi * kBlockDist + rank * 8, j0 = bj * kBlockDist;
    __syncthreads();  // previous tile's readers are done with mrows / red
    for (int e = threadIdx.x; e < S::kRows * kKP; e += kThreads) {
      const int r = e / kKP, c = e % kKP;
      const int64_t row = r < 8 ? i0 + r : (r < 24 ? j0 + (r - 8) : n_dist);
      float v = (row < n_dist && c < K) ? H[row * K + c] : 0.0f;
      if (r == 24) v = c < K ? 1.0f / (float)K : 0.0f;  // dummy marginal for invalid slots
      mrows[r * S::kRS + c] = v;
    }
    int ii, jj;
    const bool valid = tile_slot_pair(t, p, n_dist, ii, jj) && t_in;
    const float* arow = mrows + (valid ? (p >> 4) : 24) * S::kRS + cq * 64;
    const float* brow = mrows + (valid ? 8 + (p & 15) : 24) * S::kRS + cq * 64;
#pragma unroll
    for (int c = 0; c < 4; ++c) {  // V^T = 1 into R0 (phase 0's A operand)
      uint32_t ones[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) ones[e] = (cq * 64 + c * 16 + e < K) ? 0x3f800000u : 0u;
      tmem_st16(lane_off + cq * 64 + c * 16, ones);
    }
    if (!g_ready) {
      mbar_wait(bar_g, 0);  // (the leader's first issue depends on both CTAs' arrivals below)
      g_ready = true;
    }
    half_done();
    issue_phase(0, gphase);

    for (int f = 0; f < 2 * iters; ++f) {
      mbar_wait(bar_mma0 + 8 * h, mma_par[h]);
      mma_par[h] ^= 1u;
      tc_fence_after();
      if (DBG >= 3 && blockIdx.x == 0 && b == bp_begin && htid == 0 && f < 256) g_tc2_trace[h][f] = clock64();
      if (DBG >= 3) {
        t_wake = clock64();
        trace_f = b == bp_begin ? f : -1;
        if (blockIdx.x < 2 && htid == 0 && trace_f >= 0 && trace_f < 256) {
          long long gt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
          g_tc2_trace[12 + 2 * h + blockIdx.x][trace_f] = gt;
        }
      }
      const float* mrow = (f & 1) ? brow : arow;
      const uint32_t rd = lane_off + (uint32_t)(((f + 1) & 1) * 256) + cq * 64;
      if (DBG != 1 && DBG != 6 && DBG != 8) {
        uint32_t d[2][16];
        if (DBG == 5) {  // timing experiment: math without TMEM traffic
#pragma unroll
          for (int e = 0; e < 16; ++e) d[0][e] = d[1][e] = 0x3f800000u + (uint32_t)(lane * 16 + e + f);
        } else {
          tmem_ld16u(rd, d[0]);
          tmem_wait_ld();
        }
        reg_fence16(d[0]);
        uint32_t dummy = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c + 1 < 4 && DBG != 5) tmem_ld16u(rd + (c + 1) * 16, d[(c + 1) & 1]);
          const uint32_t* dc = d[c & 1];
          uint32_t o[16];
          const float4* m4 = reinterpret_cast<const float4*>(mrow + c * 16);
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float4 mq = m4[e >> 2];
            const float m0 = (e & 2) ? mq.z : mq.x, m1 = (e & 2) ? mq.w : mq.y;
            const float d0 = __uint_as_float(dc[e]), d1 = __uint_as_float(dc[e + 1]);
            const float r = rcp_approx(d0 * d1);
            const float2 x = fmul2(fmul2(make_float2(m0, m1), make_float2(d1, d0)), make_float2(r, r));
            o[e] = tf32_rna_pre(x.x);
            o[e + 1] = tf32_rna_pre(x.y);
            if (DBG == 4) {  // timing experiment: TMEM traffic without math
              o[e] = dc[e];
              o[e + 1] = dc[e + 1];
            }
          }
          if (DBG == 5) {
#pragma unroll
            for (int e = 0; e < 16; ++e) dummy ^= o[e];
          } else {
            tmem_st16(rd + c * 16, o);  // in place: the new scaling replaces D
          }
          if (c + 1 < 4 && DBG != 5) {
            tmem_wait_ld();
            reg_fence16(d[(c + 1) & 1]);
          }
        }
        if (DBG == 5 && dummy == 0x12345u) g_tc2_trace[0][255] = dummy;
      }
      if (DBG >= 3 && blockIdx.x == 0 && b == bp_begin && htid == 0 && f < 256) g_tc2_trace[2 + h][f] = clock64();
      if (f + 1 < 2 * iters) {
        half_done();
        issue_phase(f + 1, gphase + f + 1);
      } else {
        tmem_wait_st();
      }
    }

    // ---- cost: u_L in R_a = R[(2L-1)%2] = R1, v_L in R_d = R0 (both as RNA-pre bits)
    const uint32_t ra = lane_off + 256, rdv = 256 - 256;  // A-operand (v_L) region base = R0
    float ust[32];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld8(ra + cq * 32 + 8 * c, &ust[8 * c]);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 32; ++e) ust[e] = tf32_mask(ust[e]);
    float acc = 0.0f;
    for (int sp = 0; sp < 4; ++sp) {  // sub-parts (Nh, Kh) = (sp >> 1, sp & 1)
      const int nh = sp >> 1, kh = sp & 1;
      // stage this CTA's K (.) C_s sub-block (32 KB, contiguous in its image) into SMEM
      const float4* src = reinterpret_cast<const float4*>(gc_img + (size_t)rank * (128 * 1024) +
                                                          (size_t)nh * 65536 + (size_t)kh * 32768);
      float4* dst = reinterpret_cast<float4*>(smem + S::kOffStage);
      for (int e = threadIdx.x; e < 32768 / 16; e += kThreads) dst[e] = src[e];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      cluster_sync();
      tc_fence_after();
      if (issuer && elect_one()) {
        const uint64_t desc0 = make_sw128_desc(st_base);
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          const uint64_t desc = desc0 + (uint64_t)(((ks >> 2) * 8192 + (ks & 3) * 32) >> 4);
          mma2_tf32_ts(256, rdv + kh * 128 + 8 * ks, desc, kIdescPart, (kh > 0 || ks > 0) ? 1u : 0u);
        }
        mma2_commit_mc(bar_cost);
      }
      __syncwarp();
      mbar_wait(bar_cost, cost_par);
      cost_par ^= 1u;
      tc_fence_after();
      if (kh == 1) {
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
    gphase += 2 * iters;
    red[cq * 128 + p] = acc;
    __syncthreads();
    if (cq == 0 && t_in)
      write_result(out, (t - tile_begin) * kTileSlots + p, valid, ii, jj,
                   red[p] + red[128 + p] + red[256 + p] + red[384 + p]);
  }
  tc_fence_before();
  cluster_sync();
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
    const uint32_t nh = n >> 7, within = n & 127, rk = within >> 6, r = within & 63;
    *(uint32_t*)(g_img + (size_t)rk * (128 * 1024) + g_image_offset(nh, r, k)) = gb;
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
                                cudaStream_t s) {
  if (tile_end <= tile_begin) return cudaSuccess;
  static const int dbg = getenv("ASOT_TC_DEBUG_MODE") ? atoi(getenv("ASOT_TC_DEBUG_MODE")) : 0;
  auto kern = dbg == 1 ? tc2::sinkhorn_tc2_kernel<1> : dbg == 2 ? tc2::sinkhorn_tc2_kernel<2>
            : dbg == 3 ? tc2::sinkhorn_tc2_kernel<3> : dbg == 4 ? tc2::sinkhorn_tc2_kernel<4>
            : dbg == 5 ? tc2::sinkhorn_tc2_kernel<5> : dbg == 6 ? tc2::sinkhorn_tc2_kernel<6>
            : dbg == 7 ? tc2::sinkhorn_tc2_kernel<7> : dbg == 8 ? tc2::sinkhorn_tc2_kernel<8>
            : dbg == 9 ? tc2::sinkhorn_tc2_kernel<9> : tc2::sinkhorn_tc2_kernel<0>;
  const size_t smem = tc2::Smem::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_bp = ((tile_end + 1) >> 1) - (tile_begin >> 1);
  int64_t clusters = n_bp < sms / 2 ? n_bp : sms / 2;
  if (clusters < 1) clusters = 1;
  kern<<<(unsigned)(2 * clusters), tc2::kThreads, smem, s>>>(tile_begin, tile_end, n_dist, out, H, K, g_img,
                                                             gc_img, iters);
  return cudaGetLastError();
}

}  // namespace asot

extern "C" int asot_debug_tc2_trace(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, asot::tc2::g_tc2_trace, sizeof(asot::tc2::g_tc2_trace));
}
