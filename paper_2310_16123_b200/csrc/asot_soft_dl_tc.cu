// asot_soft_dl_tc.cu -- SURVEY §8(f) NEXT-1 on the tensor cores: the ASOT-DL encoder (P:262-272
// Eqs. (8)(9), appendix P:500-538 step size 1; R#26-R#28) with its dense product on tcgen05.
//
//   lambda_p = softplus(v2 . relu(V1^T x_p + c1) + c2),  z^(0) = 0,
//   n_layers x { r = W z - x;  g = W^T r;  z <- max(0, z - g - lambda) },  then z / sum z
//   (uniform fallback, flagged), H[i] = sum_p w_p z_p in fp64 in point order (Eq. (5), R#1).
//
// Per CTA a tile of 128 points of one distribution (persistent CTAs loop over distributions):
//   * r = W z - x is a gather over the non-zero codes (near-one-hot: 8-16 of 1024 at c5, 15-61 of
//     256 at c3; asot_soft_dl_sparse.cu) on the CUDA cores: warp per point, its non-zeros decoded
//     lane-parallel from the bitmap, 32 / (d / 32) coalesced dictionary rows in flight, the row
//     r - x staged in SMEM; then split x = x_hi + x_lo with x_hi = RNA_tf32(x) (3xTF32,
//     fp32-accurate: R#22's split) and stored into TMEM as the MMA's A operand by thread p of
//     warp w (lane quarter w % 4), which owns point p = TMEM lane p;
//   * g = W^T r, [128 points x d] x [d x K], is `tcgen05.mma.cta_group::1.kind::tf32` with
//     A = R from TMEM and B = 64-anchor chunks of the dictionary (pre-split K_hi / K_lo images,
//     SW128 K-major, streamed by a TMA producer warp through a double-buffered SMEM ring), three
//     MMAs per 8-wide k-step (r_hi W_hi, r_lo W_hi, r_hi W_lo), fp32 accumulators in two TMEM
//     buffers of 64 columns so the epilogue of chunk c overlaps the MMAs of chunk c + 1;
//   * epilogue (8 warps: lane quarter x column half): z <- max(0, z_old - g - lambda) with the
//     dense codes of the tile in a per-CTA global scratch (L2) and a bitmap of their non-zeros
//     in shared memory (each thread owns one bitmap word per chunk: no atomics).
// TMEM: A_hi [0, d), A_lo [d, 2d), D0 [256, 320), D1 [320, 384).
#include <cfloat>
#include <cmath>

#include "asot_internal.cuh"
#include "asot_tcgen05.cuh"

namespace asot {
namespace dltc {

using namespace ::asot::ptx;

constexpr int kTP = 128;                 // points per tile (MMA M)
constexpr int kCN = 64;                  // anchors per chunk (MMA N)
constexpr int kCompWarps = 16;
constexpr int kThreads = kCompWarps * 32 + 64;   // + MMA warp + TMA producer warp
constexpr int kStages = 2;

template <int DP>
struct Cfg {
  static constexpr uint32_t kImgBytes = (uint32_t)kCN * DP * 4;        // one chunk, one of hi / lo
  static constexpr uint32_t kStageBytes = 2 * kImgBytes;               // hi | lo
  static constexpr uint32_t kDCol0 = 256;                              // D buffers
};
template <int DP>
constexpr int kStgOf = DP + 4;           // staging row stride (floats): conflict-free LDS.128 by lane = point

struct Args {
  const float* points;
  const int64_t* offsets;
  const float* weights;
  int64_t n_dist;
  int K;
  int hidden;
  const float* V1;
  const float* c1;
  const float* v2;
  const float* c2;
  const float* dict;        // [K, d] fp32
  const uint8_t* img;       // [K / 64 chunks][hi | lo][d / 32 kb][64 rows][128 B]
  const float* lam;         // [T] lambda per point (dl_lambda_kernel)
  int n_layers;
  float* H;
  float* codes;
  float* zbuf;              // [gridDim.x][kTP][K]
  uint32_t* status;
};

__device__ __forceinline__ float softplus_f(float t) { return t > 30.0f ? t : log1pf(expf(t)); }

template <int DP>
__global__ void __launch_bounds__(kThreads, 1)
soft_dl_tc_kernel(Args A) {
  using C = Cfg<DP>;
  constexpr int kStg = kStgOf<DP>;
  constexpr uint32_t kIdesc = make_idesc_tf32(kTP, kCN);
  extern __shared__ uint8_t dl_smem_raw[];
  uint8_t* smem = dl_smem_raw + ((1024u - (smem_u32(dl_smem_raw) & 1023u)) & 1023u);
  const int K = A.K, KW = K / 32, nchunks = K / kCN;
  uint8_t* stage_base = smem;                                        // kStages x kStageBytes
  double* acc = (double*)(smem + kStages * C::kStageBytes);          // [K]
  uint32_t* bm = (uint32_t*)(acc + K);                               // [kTP][KW]
  float* lam = (float*)(bm + kTP * KW);                              // [kTP]
  float* wts = lam + kTP;                                            // [kTP]
  float* rsum = wts + kTP;                                           // [kTP]
  float* stg = rsum + kTP;                                           // [kTP][kStg]: r - x rows
  uint64_t* bars = (uint64_t*)(((uintptr_t)(stg + kTP * kStg) + 7) & ~(uintptr_t)7);
  // bars: full[2], empty[2], dfull[2], dfree[2], a_ready
  const uint32_t bar_full = smem_u32(&bars[0]), bar_empty = smem_u32(&bars[2]);
  const uint32_t bar_dfull = smem_u32(&bars[4]), bar_dfree = smem_u32(&bars[6]);
  const uint32_t bar_a = smem_u32(&bars[8]);
  uint32_t* tmem_holder = (uint32_t*)&bars[10];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* Z = A.zbuf + (size_t)blockIdx.x * kTP * K;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
      mbar_init(bar_dfull + 8 * s, 1);
      mbar_init(bar_dfree + 8 * s, kCompWarps / 2);   // the 8 warps of D[s]'s epilogue group
    }
    mbar_init(bar_a, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_holder != 0) __trap();

  // the work sequence every role walks: distributions i = blockIdx.x + k gridDim.x, their
  // 128-point tiles, n_layers layers, nchunks chunks
  auto n_tiles_of = [&](int64_t i) -> int { return (int)((A.offsets[i + 1] - A.offsets[i] + kTP - 1) / kTP); };

  if (warp == kCompWarps + 1) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t i = blockIdx.x; i < A.n_dist; i += gridDim.x) {
        const int nt = n_tiles_of(i);
        for (int t = 0; t < nt * A.n_layers; ++t)
          for (int c = 0; c < nchunks; ++c, ++it) {
            const uint32_t s = it % kStages;
            if (it >= kStages) mbar_wait(bar_empty + 8 * s, ((it / kStages) - 1) & 1);
            mbar_expect_tx(bar_full + 8 * s, C::kStageBytes);
            bulk_g2s(smem_u32(stage_base + s * C::kStageBytes), A.img + (size_t)c * C::kStageBytes, C::kStageBytes,
                     bar_full + 8 * s);
          }
      }
    }
  } else if (warp == kCompWarps) {
    // ------------------------------------------------------------------ MMA issuer
    uint32_t it = 0, a_par = 0;
    for (int64_t i = blockIdx.x; i < A.n_dist; i += gridDim.x) {
      const int nt = n_tiles_of(i);
      for (int t = 0; t < nt * A.n_layers; ++t) {
        mbar_wait(bar_a, a_par);   // R (A operand) of this layer is in TMEM
        a_par ^= 1u;
        for (int c = 0; c < nchunks; ++c, ++it) {
          const uint32_t s = it % kStages, db = it & 1;
          mbar_wait(bar_full + 8 * s, (it / kStages) & 1);
          if (it >= 2) mbar_wait(bar_dfree + 8 * db, ((it >> 1) - 1) & 1);   // epilogue drained D[db]
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sb = smem_u32(stage_base + s * C::kStageBytes);
            const uint64_t bhi = make_sw128_desc(sb), blo = make_sw128_desc(sb + C::kImgBytes);
            const uint32_t dcol = C::kDCol0 + kCN * db;
#pragma unroll
            for (int ks = 0; ks < DP / 8; ++ks) {
              const uint64_t o = (uint64_t)(((ks >> 2) * (kCN * 128) + (ks & 3) * 32) >> 4);
              mma1_tf32_ts(dcol, (uint32_t)(8 * ks), bhi + o, kIdesc, ks > 0 ? 1u : 0u);
              mma1_tf32_ts(dcol, (uint32_t)(DP + 8 * ks), bhi + o, kIdesc, 1u);
              mma1_tf32_ts(dcol, (uint32_t)(8 * ks), blo + o, kIdesc, 1u);
            }
            mma1_commit(bar_empty + 8 * s);   // the stage can be refilled
            mma1_commit(bar_dfull + 8 * db);  // D[db] ready for the epilogue
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ compute warps (0..15)
    // warp w: TMEM lane quarter q = w % 4 (point p = 32 q + lane), group g = w / 4.  r gather:
    // warp w owns points w + 16 s; TMEM store: the four threads of a point own d/4 dims each.
    // Epilogue: group g handles the chunks that land
    // in D[g / 2] (so two chunks are drained at once), 32 of their 64 columns (g % 2) = one
    // bitmap word per thread and chunk.
    const int q = warp & 3, g = warp >> 2;
    const int p = q * 32 + lane;                       // TMEM lane == point of the tile
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    constexpr int RD = DP / 4;
    constexpr int kCT = kCompWarps * 32;
    const int my_db = g >> 1, half = g & 1;
    uint32_t it = 0;
    for (int64_t i = blockIdx.x; i < A.n_dist; i += gridDim.x) {
      const int64_t s0 = A.offsets[i], e0 = A.offsets[i + 1];
      named_bar_sync(1, kCT);
      for (int j = tid; j < K; j += kCT) acc[j] = 0.0;
      bool nonfinite = false, negative = false;
      double msum = 0.0;
      for (int64_t t0 = s0; t0 < e0; t0 += kTP) {
        const int np = (int)min((int64_t)kTP, e0 - t0);
        const bool pv = p < np;
        const float* xp = A.points + (t0 + (pv ? p : 0)) * DP;
        named_bar_sync(1, kCT);   // previous tile's final pass is done
        for (int x = tid; x < kTP * KW; x += kCT) bm[x] = 0u;   // z^(0) = 0 (R#27)
        if (g == 0) {
          const float w = pv ? A.weights[t0 + p] : 0.0f;
          if (pv) {
            nonfinite |= !isfinite(w);
            negative |= w < 0.0f;
            msum += (double)w;
          }
          wts[p] = w;
          lam[p] = pv ? A.lam[t0 + p] : 0.0f;
        }
        {
          bool nf = false;
          for (int k = g * RD; k < (g + 1) * RD; ++k) nf |= pv && !isfinite(__ldg(xp + k));
          nonfinite |= nf;
        }
        named_bar_sync(1, kCT);
        const float lp = lam[p];
        for (int layer = 0; layer < A.n_layers; ++layer) {
          // ---- r = W z - x (non-zero z_j in increasing j).  Warp w owns the kPW points
          // pp = w + 16 s: their non-zeros form one warp-uniform stream (point-major, j increasing)
          // of which kGB dictionary rows are in flight at a time; each lane owns DP / 32 dims, so a
          // row is one coalesced 512 B (256 B) read.  The rows are staged through SMEM; the thread
          // owning TMEM lane p then splits its d/4 slice into TF32 hi / lo for the A operand.
          {
            constexpr int VEC = DP / 32;
            constexpr int kPW = kTP / kCompWarps;
            constexpr int kGB = 32 / VEC;
            auto row_of = [&](int sl) { return stg + (warp + kCompWarps * sl) * kStg + lane * VEC; };
            auto store_row = [&](int sl, const float (&v)[VEC]) {
              float* sr = row_of(sl);
              if constexpr (VEC == 4) *reinterpret_cast<float4*>(sr) = make_float4(v[0], v[1], v[2], v[3]);
              else *reinterpret_cast<float2*>(sr) = make_float2(v[0], v[1]);
            };
            {
              const float zero[VEC] = {};
#pragma unroll
              for (int sl = 0; sl < kPW; ++sl) store_row(sl, zero);
            }
            if (layer > 0) {
              for (int sl = 0; sl < kPW; ++sl) {
                const int pp = warp + kCompWarps * sl;
                if (pp >= np) break;
                // decode the point's non-zeros lane-parallel: lane l holds bitmap word l; entry t of
                // the (increasing-j) list is found by a shuffle binary search over the inclusive
                // popcount scan, then __fns picks its bit
                const uint32_t word = lane < KW ? bm[pp * KW + lane] : 0u;
                const int cnt = __popc(word);
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                  const int t = __shfl_up_sync(0xffffffffu, incl, o);
                  if (lane >= o) incl += t;
                }
                const int n = __shfl_sync(0xffffffffu, incl, 31);
                if (n == 0) continue;
                float ra[VEC] = {};
                const float* zrow = Z + (size_t)pp * K;
                for (int base = 0; base < n; base += 32) {
                  const int t = base + lane;
                  int own = 0;
#pragma unroll
                  for (int st = 16; st >= 1; st >>= 1) {
                    const int v = __shfl_sync(0xffffffffu, incl, own + st - 1);
                    if (v <= t) own += st;
                  }
                  const uint32_t ow = __shfl_sync(0xffffffffu, word, own);
                  const int oe = __shfl_sync(0xffffffffu, incl - cnt, own);
                  int jl = 0;
                  float zl = 0.0f;
                  if (t < n) {
                    jl = 32 * own + (int)__fns(ow, 0u, t - oe + 1);
                    zl = zrow[jl];
                  }
                  const int m = min(32, n - base);
                  for (int u0 = 0; u0 < m; u0 += kGB) {
                    float rv[kGB][VEC];
#pragma unroll
                    for (int u = 0; u < kGB; ++u) {
                      const int j = __shfl_sync(0xffffffffu, jl, (u0 + u) & 31);
                      if (u0 + u < m) {
                        const float* wr = A.dict + (int64_t)j * DP + lane * VEC;
                        if constexpr (VEC == 4) {
                          const float4 q4 = __ldg(reinterpret_cast<const float4*>(wr));
                          rv[u][0] = q4.x; rv[u][1] = q4.y; rv[u][2] = q4.z; rv[u][3] = q4.w;
                        } else {
                          const float2 q2 = __ldg(reinterpret_cast<const float2*>(wr));
                          rv[u][0] = q2.x; rv[u][1] = q2.y;
                        }
                      }
                    }
#pragma unroll
                    for (int u = 0; u < kGB; ++u) {
                      const float zu = __shfl_sync(0xffffffffu, zl, (u0 + u) & 31);   // after the row loads
                      if (u0 + u < m) {
#pragma unroll
                        for (int k = 0; k < VEC; ++k) ra[k] = fmaf(zu, rv[u][k], ra[k]);
                      }
                    }
                  }
                }
                store_row(sl, ra);
              }
            }
            // r - x for the warp's valid points (the x rows are coalesced reads, all in flight)
            {
              float xv[kPW][VEC];
#pragma unroll
              for (int sl = 0; sl < kPW; ++sl) {
                const int pp = warp + kCompWarps * sl;
                const float* xr = A.points + (t0 + (pp < np ? pp : 0)) * DP + lane * VEC;
                if constexpr (VEC == 4) {
                  const float4 t = __ldg(reinterpret_cast<const float4*>(xr));
                  xv[sl][0] = t.x; xv[sl][1] = t.y; xv[sl][2] = t.z; xv[sl][3] = t.w;
                } else {
                  const float2 t = __ldg(reinterpret_cast<const float2*>(xr));
                  xv[sl][0] = t.x; xv[sl][1] = t.y;
                }
              }
#pragma unroll
              for (int sl = 0; sl < kPW; ++sl) {
                if (warp + kCompWarps * sl >= np) continue;
                float* sr = row_of(sl);
                float v[VEC];
#pragma unroll
                for (int k = 0; k < VEC; ++k) v[k] = sr[k] - xv[sl][k];
                store_row(sl, v);
              }
            }
            named_bar_sync(1, kCT);
#pragma unroll
            for (int b = 0; b < RD; b += 16) {
              uint32_t hi[16], lo[16];
              const float4* sp = reinterpret_cast<const float4*>(stg + p * kStg + g * RD + b);
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4) {
                const float4 v4 = sp[k4];
                const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const uint32_t h = (__float_as_uint(vv[e]) + 0x1000u) & 0xFFFFE000u;   // RNA to TF32
                  hi[4 * k4 + e] = h;
                  lo[4 * k4 + e] = __float_as_uint(vv[e] - __uint_as_float(h));
                }
              }
              tmem_st16(lane_off + (uint32_t)(g * RD + b), hi);
              tmem_st16(lane_off + (uint32_t)(DP + g * RD + b), lo);
            }
            tmem_wait_st();
            tc_fence_before();
            named_bar_sync(1, kCT);   // (also: the bitmap / staging reads above are done)
            if (tid == 0) mbar_arrive_local(bar_a);
          }
          // ---- chunks: z <- max(0, z - g - lambda); each thread rewrites bitmap word 2c + half
          // of its point.  Codes are stored only for words with a non-zero and read only for
          // words that had one (the rest are exactly 0).
          for (int c = 0; c < nchunks; ++c, ++it) {
            const uint32_t db = it & 1;
            if ((int)db != my_db) continue;
            mbar_wait(bar_dfull + 8 * db, (it >> 1) & 1);
            tc_fence_after();
            uint32_t gv[32];
            const uint32_t dcol = C::kDCol0 + kCN * db + 32 * half;
            tmem_ld16u(lane_off + dcol, *reinterpret_cast<uint32_t(*)[16]>(&gv[0]));
            tmem_ld16u(lane_off + dcol + 16, *reinterpret_cast<uint32_t(*)[16]>(&gv[16]));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_local(bar_dfree + 8 * db);   // D[db] may be overwritten
            const int j0 = c * kCN + 32 * half;
            const int wi = p * KW + (j0 >> 5);
            const uint32_t old = layer > 0 ? bm[wi] : 0u;
            float4* zp = reinterpret_cast<float4*>(Z + (size_t)p * K + j0);
            float zn[32];
            uint32_t mask = 0u;
#pragma unroll
            for (int e4 = 0; e4 < 8; ++e4) {
              const float4 zo = old ? zp[e4] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
              const float zz[4] = {zo.x, zo.y, zo.z, zo.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float v = fmaxf(0.0f, (zz[u] - __uint_as_float(gv[4 * e4 + u])) - lp);
                zn[4 * e4 + u] = v;
                if (v > 0.0f) mask |= 1u << (4 * e4 + u);
              }
            }
            if (!pv) mask = 0u;
            if (mask) {
#pragma unroll
              for (int e4 = 0; e4 < 8; ++e4) zp[e4] = make_float4(zn[4 * e4], zn[4 * e4 + 1], zn[4 * e4 + 2], zn[4 * e4 + 3]);
            }
            bm[wi] = mask;
          }
          named_bar_sync(1, kCT);   // codes + bitmap of this layer complete
        }
        // ---- row sums in increasing j (non-zeros only), the uniform fallback
        if (g == 0) {
          float sm = 0.0f;
          for (int w = 0; w < KW; ++w) {
            uint32_t bits = bm[p * KW + w];
            while (bits) {
              const int j = 32 * w + __ffs(bits) - 1;
              bits &= bits - 1;
              sm += Z[(size_t)p * K + j];
            }
          }
          rsum[p] = sm;
          if (pv && !(sm > 0.0f)) atomicOr(A.status, ASOT_FLAG_SOFT_FALLBACK);
        }
        named_bar_sync(1, kCT);
        // ---- codes (z / sum z) and the fp64 point-order histogram: thread per bin j
        const float unif = 1.0f / (float)K;
        for (int j = tid; j < K; j += kCT) {
          double a = acc[j];
          for (int pp = 0; pp < np; ++pp) {
            float z;
            if (!(rsum[pp] > 0.0f)) z = unif;
            else z = (bm[pp * KW + (j >> 5)] >> (j & 31)) & 1u ? Z[(size_t)pp * K + j] / rsum[pp] : 0.0f;
            if (A.codes) A.codes[(t0 + pp) * K + j] = z;
            a += (double)wts[pp] * (double)z;
          }
          acc[j] = a;
        }
      }
      named_bar_sync(1, kCT);
      for (int j = tid; j < K; j += kCT) A.H[i * K + j] = (float)acc[j];
      // flags: every compute thread reports its own; the weight sums live in group 0
      if (nonfinite) atomicOr(A.status, ASOT_FLAG_NONFINITE_INPUT);
      if (negative) atomicOr(A.status, ASOT_FLAG_BAD_MASS);
      __shared__ double msh[kTP];
      if (g == 0) msh[p] = msum;
      named_bar_sync(1, kCT);
      if (tid == 0) {
        double m = 0.0;
        for (int x = 0; x < kTP; ++x) m += msh[x];
        if (e0 <= s0) atomicOr(A.status, ASOT_FLAG_EMPTY_DIST);
        else if (fabs(m - 1.0) > 1e-5) atomicOr(A.status, ASOT_FLAG_BAD_MASS);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(0u) : "memory");
}

// lambda_p = softplus(v2 . relu(V1^T x_p + c1) + c2) for every point (R#24, R#26): thread per
// point, hidden units in order, V1 reads broadcast across the warp
template <int DP>
__global__ void dl_lambda_kernel(const float* __restrict__ points, int64_t T, const float* __restrict__ V1,
                                 const float* __restrict__ c1, const float* __restrict__ v2,
                                 const float* __restrict__ c2, int hidden, float* __restrict__ lam) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < T; p += (int64_t)gridDim.x * blockDim.x) {
    float x[DP];
#pragma unroll
    for (int k4 = 0; k4 < DP / 4; ++k4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(points + p * DP) + k4);
      x[4 * k4] = v.x; x[4 * k4 + 1] = v.y; x[4 * k4 + 2] = v.z; x[4 * k4 + 3] = v.w;
    }
    float lsum = 0.0f;
    for (int c = 0; c < hidden; ++c) {
      float a = __ldg(c1 + c);
#pragma unroll
      for (int k = 0; k < DP; ++k) a = fmaf(x[k], __ldg(V1 + (int64_t)k * hidden + c), a);
      lsum = fmaf(fmaxf(a, 0.0f), __ldg(v2 + c), lsum);
    }
    lam[p] = softplus_f(lsum + c2[0]);
  }
}

// Dictionary [K, d] -> per 64-anchor chunk [hi | lo] images, each [kb = d/32][64 rows][128 B] SW128
// K-major (TF32 RNA hi, fp32 remainder lo: the MMA reads its TF32 truncation).
template <int DP>
__global__ void dl_image_kernel(const float* __restrict__ dict, int K, uint8_t* __restrict__ img) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < K * DP; idx += gridDim.x * blockDim.x) {
    const int n = idx / DP, k = idx % DP;
    const float v = dict[idx];
    const uint32_t h = (__float_as_uint(v) + 0x1000u) & 0xFFFFE000u;
    const float lo = v - __uint_as_float(h);
    const uint32_t c = n / kCN, r = n % kCN;
    const uint32_t lin = (uint32_t)(k >> 5) * (kCN * 128) + r * 128u + (uint32_t)(k & 31) * 4u;
    const uint32_t off = lin ^ (((lin >> 7) & 7u) << 4);
    uint8_t* base = img + (size_t)c * Cfg<DP>::kStageBytes;
    *(uint32_t*)(base + off) = h;
    *(float*)(base + Cfg<DP>::kImgBytes + off) = lo;
  }
}

template <int DP>
size_t smem_bytes(int K) {
  return 1024 + kStages * Cfg<DP>::kStageBytes + (size_t)K * 8 + (size_t)kTP * (K / 32) * 4 + 3 * kTP * 4 +
         (size_t)kTP * kStgOf<DP> * 4 + 128;
}

}  // namespace dltc

bool soft_dl_tc_supported(int dim, int K) { return (dim == 64 || dim == 128) && K >= 256 && K % 64 == 0 && K <= 1024; }

size_t soft_dl_tc_workspace_bytes(int dim, int K, int sms, int64_t T) {
  // codes scratch + images + lambda per point
  return (size_t)sms * dltc::kTP * K * 4 + (size_t)K * dim * 8 + 1024 + (size_t)(T > 0 ? T : 1) * 4 + 256;
}

cudaError_t launch_soft_dl_tc(const float* points, const int64_t* offsets, const float* weights, int64_t n_dist, int dim,
                              const float* dict, int K, int n_layers, int hidden, const float* V1, const float* c1,
                              const float* v2, const float* c2, float* H, float* codes, uint8_t* ws, uint32_t* status,
                              int sms, int64_t T, cudaStream_t s) {
  const int grid = (int)(n_dist < sms ? n_dist : sms);
  if (grid < 1) return cudaSuccess;
  float* zbuf = (float*)ws;
  uint8_t* img = (uint8_t*)(((uintptr_t)(ws + (size_t)sms * dltc::kTP * K * 4) + 1023) & ~(uintptr_t)1023);
  float* lam = (float*)(img + (size_t)K * dim * 8);
  dltc::Args A{points, offsets, weights, n_dist, K, hidden, V1, c1, v2, c2, dict, img, lam, n_layers, H, codes, zbuf,
               status};
  const int lblocks = (int)((T + 255) / 256 < 4 * sms ? (T + 255) / 256 : 4 * sms);
  cudaError_t e;
  if (dim == 64) {
    if (T > 0) dltc::dl_lambda_kernel<64><<<lblocks, 256, 0, s>>>(points, T, V1, c1, v2, c2, hidden, lam);
    dltc::dl_image_kernel<64><<<256, 256, 0, s>>>(dict, K, img);
    const size_t smem = dltc::smem_bytes<64>(K);
    e = cudaFuncSetAttribute(dltc::soft_dl_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dltc::soft_dl_tc_kernel<64><<<grid, dltc::kThreads, smem, s>>>(A);
  } else {
    if (T > 0) dltc::dl_lambda_kernel<128><<<lblocks, 256, 0, s>>>(points, T, V1, c1, v2, c2, hidden, lam);
    dltc::dl_image_kernel<128><<<256, 256, 0, s>>>(dict, K, img);
    const size_t smem = dltc::smem_bytes<128>(K);
    e = cudaFuncSetAttribute(dltc::soft_dl_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dltc::soft_dl_tc_kernel<128><<<grid, dltc::kThreads, smem, s>>>(A);
  }
  return cudaGetLastError();
}

}  // namespace asot
