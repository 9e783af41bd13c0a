// asot_sinkhorn_tc6.cu -- steps a5 + a6, fp32-accurate (ASOT_PREC_FP32), 128 < K <= 256, RESIDENT on
// a CTA pair with BF16x3 split operands (tcgen05 kind::f16, cta_group::2).
//
// Same recurrence as every Sinkhorn kernel (R#3-R#6, R#11): U = A/(K V), V = B/(K^T U),
// v0 = 1, L iterations, d = sum_r u_r ((K (.) C_s) v)_r.  The fp32-accuracy reading (R#22) is met
// here by splitting both operands into two BF16 terms, x = x_hi + x_lo, K = K_hi + K_lo
// (x_hi = RN_bf16(x), x_lo = RN_bf16(x - x_hi): ~16 significant bits), and forming
//   K x ~ x_hi K_hi + x_lo K_hi + x_hi K_lo
// with FP32 accumulation (each BF16 x BF16 product is exact in fp32; the dropped x_lo K_lo term is
// ~2^-16 relative).  SURVEY §8(d)'s emulation: bf16x3 <= 2.2e-5 on c3, inside the 1e-4 bar.
// BF16 MMAs run at twice the TF32 rate, so a phase costs 1.5x a one-pass TF32 phase -- against
// 3x for the streamed 3xTF32 kernel (tc5) this replaces at 128 < K <= 256 -- and the split
// scalings fit on chip: a 16-bit operand packs two anchors per TMEM column, so [x_hi | x_lo] of a
// pair takes the same 256 columns as its fp32 D.
//
// Layout (the schedule is the CTA-pair TF32 kernel's, asot_sinkhorn_tc2.cu):
//   TMEM per CTA: R0 = [0, 256), R1 = [256, 512); phase f reads A from R[f%2] and writes D into
//     R[(f+1)%2]; the epilogue converts D in place.  Within a region, anchor group j (16 anchors,
//     j = 0..15) owns columns [16 j, 16 j + 16): fp32 D of its 16 anchors, or, as a scaling,
//     x_hi in [16 j, 16 j + 8) and x_lo in [16 j + 8, 16 j + 16) (column c packs anchors
//     (2c, 2c+1) of the group, the even anchor in the low half).  A thread's 16 D columns of a
//     chunk are exactly the 16 columns its split scaling goes to: the conversion is in place per
//     thread, with no cross-thread hazard.
//   SMEM per CTA: K_hi and K_lo images (BF16, SW128 K-major, [kb 4][nc 4][32 rows][128 B], 64 KB
//     each: this CTA's 128 of the 256 output anchors, n = nc*64 + rank*32 + r), a 32 KB staging
//     buffer for K (.) C_s in the cost, marginal rows, partial costs, mbarriers.
//   A phase = 16 parts (kc, nc), kc-major, each 4 k-steps of 16 anchors x 3 MMAs (M = 256, N = 64,
//     K = 16): (x_hi, K_hi), (x_lo, K_hi), (x_hi, K_lo).  Output chunk nc is committed after part
//     (3, nc); parts of input chunk kc wait only for the epilogue of chunk kc of the previous phase.
//   Epilogue (16 warps, 16 anchors per thread per chunk): x = m / D with one MUFU per two anchors
//     (epi_div4: the product range check of the TF32 kernels, S:62 clamp + flag on the rare
//     out-of-range chunk), then the BF16 split packed with cvt.rn.bf16x2.
//   Cost (a6): v_L (R0, split) against K (.) C_s, also split and streamed in four (N-half, K-half)
//     sub-parts of [hi | lo] x 64 rows x 128 anchors (32 KB); the fp32 products land in the
//     consumed half of R1 and each thread reduces them against u_L = hi + lo of its 32 anchors.
#include <cuda_bf16.h>

#include <cfloat>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace tc6 {

constexpr int kKP = 256;
constexpr int kChunk = 64;                  // anchors per epilogue chunk / MMA part
constexpr int kNChunks = kKP / kChunk;
constexpr int kWarps = 16;                  // epilogue warps
constexpr int kThreads = kWarps * 32;
constexpr int kAllThreads = kThreads + 32;  // + the MMA warp
constexpr uint32_t kImg = 64 * 1024;        // one BF16 image half (this CTA's 128 output rows)

using namespace ::asot::ptx;

struct Smem {
  static constexpr int kRS = kKP + 4;
  static constexpr int kRows = 25;
  static constexpr size_t kOffG = 0;                          // K_hi 64 KB | K_lo 64 KB
  static constexpr size_t kOffStage = 128 * 1024;             // 32 KB: (K (.) C_s)_hi | _lo sub-block
  static constexpr size_t kOffMarg = kOffStage + 32 * 1024;   // 25 x 260 floats
  static constexpr size_t kOffRed = kOffMarg + (size_t)kRows * kRS * 4;  // [4][128] floats
  static constexpr size_t kOffBar = kOffRed + 4 * 128 * 4;
  static constexpr size_t kBytes = kOffBar + 128 + 1024;
};

// [rows][128 B] SW128 block, element (r, kin) of 16-bit data (kin in [0, 64))
__host__ __device__ inline uint32_t sw_block16(uint32_t r, uint32_t kin) {
  const uint32_t lin = r * 128u + kin * 2u;
  return lin ^ (((lin >> 7) & 7u) << 4);
}
// Sinkhorn B image (one rank, one of hi / lo): element (n, k), n = nc*64 + rank*32 + r
__host__ __device__ inline uint32_t g_image_offset(uint32_t nc, uint32_t r, uint32_t k) {
  return (k >> 6) * 16384u + nc * 4096u + sw_block16(r, k & 63);
}
// Cost B image (one rank): [nh 2][kh 2][hi/lo 2][kb 2][64 rows][128 B]; n = nh*128 + rank*64 + r,
// k = kh*128 + kb*64 + kin
__host__ __device__ inline uint32_t gc_image_offset(uint32_t nh, uint32_t lo, uint32_t r, uint32_t k) {
  const uint32_t kh = k >> 7, kb = (k >> 6) & 1;
  return ((nh * 2 + kh) * 2 + lo) * 16384u + kb * 8192u + sw_block16(r, k & 63);
}

__device__ __forceinline__ uint32_t cvt_bf16x2(float hi_elem, float lo_elem) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
  return r;
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// x = m / D for a thread's 16 anchors (fp32; one MUFU per two anchors and the product range check
// of the TF32 kernels, epi_div4), then the BF16 split:
// o[0..8) = x_hi pairs, o[8..16) = x_lo pairs.  Returns true if a product D0 D1 left
// [2^-126, 2^126) -- the caller then redoes the thread's values with clamped reciprocals.
__device__ __forceinline__ bool epi_split_fast(const float* m, const uint32_t (&d)[16], float (&x)[16]) {
  float2 t = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int e = 0; e < 16; e += 4)
    epi_div4(m + e, __uint_as_float(d[e]), __uint_as_float(d[e + 1]), __uint_as_float(d[e + 2]),
             __uint_as_float(d[e + 3]), x + e, t);
  return epi_div_bad(t, 16);
}
__device__ __forceinline__ void split16(const float (&x)[16], uint32_t (&o)[16]) {
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    const uint32_t h = cvt_bf16x2(x[e + 1], x[e]);
    const float2 r = fsub2(make_float2(x[e], x[e + 1]), make_float2(bf16_lo(h), bf16_hi(h)));
    o[e >> 1] = h;
    o[8 + (e >> 1)] = cvt_bf16x2(r.y, r.x);
  }
}

__device__ long long g_tc6_clock[4];  // clock_probe: (clock64, globaltimer) at start / end

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kAllThreads, 1)
sinkhorn_tc6_kernel(int64_t tile_begin, int64_t tile_end, int64_t n_dist, PairSink out,
                    const float* __restrict__ H, int K, const uint8_t* __restrict__ g_img,
                    const uint8_t* __restrict__ gc_img, int iters, const int32_t* __restrict__ units,
                    const int64_t* __restrict__ n_dev) {
  if (dense_skipped(out)) return;   // the small-support kernel serves this call (R#36)
  using S = Smem;
  constexpr uint32_t kIdescPart = make_idesc_bf16(256, kChunk);   // Sinkhorn parts: N = 64
  constexpr uint32_t kIdescCost = make_idesc_bf16(256, 128);      // cost sub-parts: N = 128
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* mrows = (float*)(smem + S::kOffMarg);
  float* red = (float*)(smem + S::kOffRed);
  uint64_t* bars = (uint64_t*)(smem + S::kOffBar);
  // bars: 0 g_loaded, 1-4 mma_done[c], 5-8 epi_done[c] (leader), 9 cost_done
  uint32_t* tmem_holder = (uint32_t*)(bars + 12);
  const uint32_t bar_g = smem_u32(&bars[0]);
  const uint32_t bar_mma0 = smem_u32(&bars[1]);
  const uint32_t bar_epi0 = smem_u32(&bars[5]);
  const uint32_t bar_cost = smem_u32(&bars[9]);

  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool epi_warp = warp < kWarps;
  const int q = warp & 3;            // TMEM lane quarter
  const int cq = (warp >> 2) & 3;    // column group: anchor group 4c + cq of every chunk c
  const int p = q * 32 + lane;       // TMEM lane

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
  clock_probe(g_tc6_clock, 0);
  if (*tmem_holder != 0) __trap();
  if (threadIdx.x == 0) {          // this CTA's K_hi | K_lo images, once (TMA bulk copies)
    const uint8_t* src = g_img + (size_t)rank * (2 * kImg);
    mbar_expect_tx(bar_g, 2 * kImg);
    for (uint32_t off = 0; off < 2 * kImg; off += 32768)
      bulk_g2s(smem_u32(smem + S::kOffG + off), src + off, 32768, bar_g);
  }
  const uint32_t g_base = smem_u32(smem + S::kOffG);
  const uint32_t st_base = smem_u32(smem + S::kOffStage);
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  const uint32_t epi_remote0 = mapa(bar_epi0, 0);
  const bool leader = rank == 0;
  const bool issuer = leader && warp == kWarps;
  const int NCH = (K + kChunk - 1) / kChunk;   // K <= 192: the all-padding fourth chunk is skipped

  uint32_t mma_par = 0, epi_par = 0, cost_par = 0;
  bool g_ready = false;

  // Part (kc, nc): D(R_d)[:, nc*64 +: 64] (+)= sum over the 4 anchor groups j = 4kc + ks of
  // x_hi,j K_hi + x_lo,j K_hi + x_hi,j K_lo
  const uint64_t ghi0 = make_sw128_desc(g_base), glo0 = make_sw128_desc(g_base + kImg);
  auto issue_part = [&](uint32_t a_col, uint32_t d_col, uint32_t boff, uint32_t acc0) {
#pragma unroll
    for (int ks = 0; ks < kChunk / 16; ++ks) {
      const uint64_t o = (uint64_t)((boff + ks * 32) >> 4);
      const uint32_t ah = a_col + 16 * ks;
      mma2_bf16_ts(d_col, ah, ghi0 + o, kIdescPart, ks > 0 ? 1u : acc0);
      mma2_bf16_ts(d_col, ah + 8, ghi0 + o, kIdescPart, 1u);
      mma2_bf16_ts(d_col, ah, glo0 + o, kIdescPart, 1u);
    }
  };
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
    const int64_t t = 2 * b + rank;
    const bool t_in = units != nullptr || (t >= tile_begin && t < tile_end);
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
    const int ps = ((p & 7) << 4) | (p >> 3);   // TMEM lane p holds tile slot ps (see tc2)
    const bool valid = tile_slot_pair(t, ps, n_dist, ii, jj) && t_in;
    const float* arow = mrows + (valid ? (ps >> 4) : 24) * S::kRS + cq * 16;
    const float* brow = mrows + (valid ? 8 + (ps & 15) : 24) * S::kRS + cq * 16;
    if (!g_ready) {
      mbar_wait(bar_g, 0);
      g_ready = true;
    }
    if (epi_warp) {
#pragma unroll
      for (int c = 0; c < kNChunks; ++c) {  // V^T = 1 (hi = 1, lo = 0) into R0
        const int a0 = c * kChunk + cq * 16;
        uint32_t ones[16];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t lo16 = a0 + 2 * e < K ? 0x3F80u : 0u, hi16 = a0 + 2 * e + 1 < K ? 0x3F80u : 0u;
          ones[e] = lo16 | (hi16 << 16);
          ones[8 + e] = 0u;
        }
        tmem_st16(lane_off + a0, ones);
        if (c >= NCH) {   // skipped chunk: R1's copy is read by the cost, so it must be 0 too
          uint32_t zeros[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) zeros[e] = 0u;
          tmem_st16(lane_off + 256 + a0, zeros);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      named_bar_sync(1, kThreads);
      if (threadIdx.x == 0)
        for (int c = 0; c < kNChunks; ++c) mbar_arrive_cluster(epi_remote0 + 8 * c);

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
          uint32_t d[16];
          tmem_ld16u(rd + c * kChunk, d);
          tmem_wait_ld();
          reg_fence16(d);
          float x[16];
          const bool bad = epi_split_fast(mk, d, x);
          if (__any_sync(0xffffffffu, bad)) {   // a product D0 D1 out of fp32 range (rare): reload D
#pragma unroll
            for (int s8 = 0; s8 < 16; s8 += 8) {
              uint32_t d8[8];
              tmem_ld8u(rd + c * kChunk + s8, d8);
              tmem_wait_ld();
              if (bad) {
#pragma unroll
                for (int e = 0; e < 8; ++e) x[s8 + e] = div_clamped(mk[s8 + e], __uint_as_float(d8[e]), clamped);
              }
            }
          }
          uint32_t o[16];
          split16(x, o);
          tmem_st16(rd + c * kChunk, o);  // in place: [x_hi | x_lo] of the group replaces its D
          if (c + 1 < NCH) load_m(f, c + 1);
          else if (!last) load_m(f + 1, 0);
          if (!last) chunk_done(c);
        }
        mma_par ^= 1u;
        if (last) tmem_wait_st();
      }
    } else if (issuer) {
      for (int f = 0; f < 2 * iters; ++f) {
#pragma unroll 1
        for (int kc = 0; kc < NCH; ++kc) {
          mbar_wait(bar_epi0 + 8 * kc, epi_par);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a_col = (uint32_t)((f & 1) * 256 + kc * kChunk);
            const uint32_t d_col = (uint32_t)(((f + 1) & 1) * 256);
            const uint32_t acc0 = kc > 0 ? 1u : 0u;
#pragma unroll
            for (int nc = 0; nc < kNChunks; ++nc) {
              if (nc < NCH) {
                issue_part(a_col, d_col + nc * kChunk, (uint32_t)(kc * 16384 + nc * 4096), acc0);
                if (kc == NCH - 1) mma2_commit_mc(bar_mma0 + 8 * nc);
              }
            }
          }
          __syncwarp();
        }
        epi_par ^= 1u;
      }
    }

    // ---- cost: u_L in R1 (split), v_L in R0 (split; the cost MMAs' A operand)
    const uint32_t ra = lane_off + 256;
    float ust[32];   // u_L of anchors cq*32 + [0, 32) (their R1 columns get the first D sub-part)
    if (epi_warp) {
      uint32_t w[32];
      tmem_ld16u(ra + cq * 32, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
      tmem_ld16u(ra + cq * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
      tmem_wait_ld();
#pragma unroll
      for (int g = 0; g < 2; ++g)      // anchor group 2cq + g: hi words w[16g + 0..8), lo w[16g + 8..16)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t h = w[16 * g + e], l = w[16 * g + 8 + e];
          ust[16 * g + 2 * e] = bf16_lo(h) + bf16_lo(l);
          ust[16 * g + 2 * e + 1] = bf16_hi(h) + bf16_hi(l);
        }
    }
    float acc = 0.0f;
    for (int sp = 0; sp < 4; ++sp) {  // sub-parts (Nh, Kh) = (sp >> 1, sp & 1)
      const int nh = sp >> 1, kh = sp & 1;
      const float4* src = reinterpret_cast<const float4*>(gc_img + (size_t)rank * (128 * 1024) +
                                                          (size_t)(nh * 2 + kh) * 32768);
      float4* dst = reinterpret_cast<float4*>(smem + S::kOffStage);
      for (int e = threadIdx.x; e < 32768 / 16; e += kAllThreads) dst[e] = src[e];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      cluster_sync();
      tc_fence_after();
      if (issuer && elect_one()) {
        const uint64_t dhi = make_sw128_desc(st_base), dlo = make_sw128_desc(st_base + 16384);
#pragma unroll
        for (int js = 0; js < 8; ++js) {   // anchor groups kh*8 + js of v_L (R0)
          const uint64_t o = (uint64_t)(((js >> 2) * 8192 + (js & 3) * 32) >> 4);
          const uint32_t ah = (uint32_t)(kh * 128 + 16 * js);
          mma2_bf16_ts(256, ah, dhi + o, kIdescCost, (kh > 0 || js > 0) ? 1u : 0u);
          mma2_bf16_ts(256, ah + 8, dhi + o, kIdescCost, 1u);
          mma2_bf16_ts(256, ah, dlo + o, kIdescCost, 1u);
        }
        mma2_commit_mc(bar_cost);
      }
      __syncwarp();
      mbar_wait(bar_cost, cost_par);
      cost_par ^= 1u;
      tc_fence_after();
      if (kh == 1 && epi_warp) {
        // (K (.) C_s) v for anchors nh*128 + [0, 128) now sits (fp32) in R1 columns [0, 128); this
        // thread reduces anchors nh*128 + cq*32 + [0, 32) in blocks of 8
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t g[8];
          tmem_ld8u(ra + cq * 32 + 8 * c, g);
          uint32_t wh[4], wl[4];   // nh = 1: u_L hi / lo words of these 8 anchors (R1, untouched)
          if (nh == 1) {
            const uint32_t col = ra + 128 + 16 * (2 * cq + (c >> 1)) + 4 * (c & 1);
            tmem_ld4u(col, wh);
            tmem_ld4u(col + 8, wl);
          }
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float u0, u1;
            if (nh == 0) {
              u0 = ust[8 * c + 2 * e];
              u1 = ust[8 * c + 2 * e + 1];
            } else {
              u0 = bf16_lo(wh[e]) + bf16_lo(wl[e]);
              u1 = bf16_hi(wh[e]) + bf16_hi(wl[e]);
            }
            acc = fmaf(u0, __uint_as_float(g[2 * e]), acc);
            acc = fmaf(u1, __uint_as_float(g[2 * e + 1]), acc);
          }
        }
      }
      tc_fence_before();
      cluster_sync();  // staging buffer and R1 columns free for the next sub-part / tile
      tc_fence_after();
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
  clock_probe(g_tc6_clock, 1);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(0u) : "memory");
}

// ----------------------------------------------------------------------------- image prep
// K = exp(-C_s / eps) in fp64, rounded to fp32, split into BF16 hi + lo; padding: K = 1
// (hi = 1, lo = 0: every padded denominator stays > 0, R#12), K (.) C_s = 0.
__global__ void gibbs_prep_tc6_kernel(const float* __restrict__ cost, int K, float eps, uint8_t* __restrict__ g_img,
                                      uint8_t* __restrict__ gc_img) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < kKP * kKP; idx += gridDim.x * blockDim.x) {
    const int n = idx / kKP, k = idx % kKP;
    const bool in = n < K && k < K;
    const double c = in ? (double)cost[(int64_t)n * K + k] : 0.0;
    const double g = in ? exp(-c / (double)eps) : 1.0;
    const float g32 = (float)g, gc32 = in ? (float)(g * c) : 0.0f;
    const __nv_bfloat16 ghi = __float2bfloat16_rn(g32);
    const __nv_bfloat16 glo = __float2bfloat16_rn(g32 - __bfloat162float(ghi));
    const __nv_bfloat16 chi = __float2bfloat16_rn(gc32);
    const __nv_bfloat16 clo = __float2bfloat16_rn(gc32 - __bfloat162float(chi));
    // Sinkhorn image: n = nc*64 + rank*32 + r
    const uint32_t nc = n >> 6, rg = (n >> 5) & 1, r32 = n & 31;
    uint8_t* gi = g_img + (size_t)rg * (2 * kImg);
    *(__nv_bfloat16*)(gi + g_image_offset(nc, r32, k)) = ghi;
    *(__nv_bfloat16*)(gi + kImg + g_image_offset(nc, r32, k)) = glo;
    // cost image: n = nh*128 + rank*64 + r
    const uint32_t nh = n >> 7, within = n & 127, rk = within >> 6, r = within & 63;
    uint8_t* ci = gc_img + (size_t)rk * (128 * 1024);
    *(__nv_bfloat16*)(ci + gc_image_offset(nh, 0, r, k)) = chi;
    *(__nv_bfloat16*)(ci + gc_image_offset(nh, 1, r, k)) = clo;
  }
}

}  // namespace tc6

bool sinkhorn_tc6_supported(int K) { return K > 128 && K <= 256; }
size_t sinkhorn_tc6_image_bytes() { return 2 * 2 * tc6::kImg; }   // (hi + lo) x 2 ranks

cudaError_t launch_gibbs_prep_tc6(const float* cost, int K, float eps, uint8_t* g_img, uint8_t* gc_img,
                                  cudaStream_t s) {
  tc6::gibbs_prep_tc6_kernel<<<256, 256, 0, s>>>(cost, K, eps, g_img, gc_img);
  return cudaGetLastError();
}

cudaError_t launch_sinkhorn_tc6(int64_t tile_begin, int64_t tile_end, int64_t n_dist, const PairSink& out,
                                const float* H, int K, const uint8_t* g_img, const uint8_t* gc_img, int iters,
                                cudaStream_t s, const int32_t* units, const int64_t* n_dev) {
  if (tile_end <= tile_begin) return cudaSuccess;
  const size_t smem = tc6::Smem::kBytes;
  cudaError_t e = cudaFuncSetAttribute(tc6::sinkhorn_tc6_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_bp = ((tile_end + 1) >> 1) - (tile_begin >> 1);
  int64_t clusters = n_bp < sms / 2 ? n_bp : sms / 2;
  if (clusters < 1) clusters = 1;
  tc6::sinkhorn_tc6_kernel<<<(unsigned)(2 * clusters), tc6::kAllThreads, smem, s>>>(tile_begin, tile_end, n_dist, out,
                                                                                  H, K, g_img, gc_img, iters,
                                                                                  units, n_dev);
  return cudaGetLastError();
}

cudaError_t read_kernel_clock_tc6(long long* host4) {
  return cudaMemcpyFromSymbol(host4, tc6::g_tc6_clock, 4 * sizeof(long long));
}

}  // namespace asot
