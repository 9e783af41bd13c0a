// asot_api.cu -- the C ABI (include/asot.h): argument checks, workspace carving, dispatch.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "asot_internal.cuh"

namespace {

thread_local std::string g_last_error;
thread_local int32_t g_launches = 0;

asot_status fail(asot_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

#define ASOT_CHECK_ARG(cond, msg) \
  do {                            \
    if (!(cond)) return fail(ASOT_ERR_INVALID_ARGUMENT, msg); \
  } while (0)

#define ASOT_CUDA(call)                                                                        \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return fail(ASOT_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)

#define ASOT_LAUNCH(call)   \
  do {                      \
    ++g_launches;           \
    ASOT_CUDA(call);        \
  } while (0)

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

// Bump allocator over the caller's workspace.
struct Carver {
  char* base;
  size_t cap;
  size_t used = 0;
  bool overflow = false;
  void* take(size_t bytes) {
    void* p = base ? base + used : nullptr;
    used += align_up(bytes);
    if (used > cap) overflow = true;
    return p;
  }
};

asot_status check_common(int64_t n_dist, int32_t n_anchors, float eps, int32_t iters, float cost_max) {
  ASOT_CHECK_ARG(n_dist >= 1, "n_dist must be >= 1");
  ASOT_CHECK_ARG(n_anchors >= 1, "n_anchors must be >= 1");
  if (n_anchors > asot::kMaxAnchors)
    return fail(ASOT_ERR_UNSUPPORTED, "n_anchors > 1024 is not supported by this build");
  ASOT_CHECK_ARG(std::isfinite(eps) && eps > 0.0f, "eps must be finite and > 0");
  ASOT_CHECK_ARG(iters >= 1, "iters must be >= 1");
  ASOT_CHECK_ARG(std::isfinite(cost_max) && cost_max >= 0.0f, "cost_max must be finite and >= 0");
  ASOT_CHECK_ARG((double)cost_max / (double)eps <= 80.0,
                 "max(C_s)/eps > 80: the fp32 Gibbs kernel would underflow (R#12)");
  return ASOT_OK;
}

// Sinkhorn kernel selection: 0 = the fp32 CUDA-core GEMM kernel (only via ASOT_PAIR_KERNEL=simt),
// 1 = single-CTA resident TF32 (32 <= K <= 128), 2 = CTA-pair resident TF32 (128 < K <= 256),
// 4 = CTA-pair streamed TF32 (256 < K <= 1024), 3 = single-CTA resident 3xTF32 (fp32-accurate
// requests with 32 <= K <= 128), 5 = CTA-pair streamed 3xTF32 for fp32-accurate requests
// (128 < K <= 1024; also explicit fp32 pair lists), 6 = CTA-pair streamed one-pass TF32 in
// pair-list mode (explicit TF32 pair lists), 9 = fp32 lane-per-anchor kernel (every request with
// K < 32, tiles and pair lists).
// K < 32 never uses one-pass TF32: the per-iteration TF32 rounding of u / v dominates the TF32
// error (R#23) and a dot product over fewer than 32 anchors barely averages it out
// (K = 7: 2.3e-3 > the 2e-3 bar), so those requests run in fp32.
constexpr int32_t kMinTcAnchors = 32;
int tc_kind(int32_t K, asot_precision prec) {
  // K < 32: fp32 for both requests -- TF32 rounding is not accurate enough there (R#23) -- on
  // the lane-per-anchor kernel: a pair's state is < 32 floats, so one lane group per pair keeps
  // every SM busy where 128-pair tensor-core tiles leave c1 on 16 SMs (latency-bound)
  if (K < kMinTcAnchors) return K >= 1 && (prec == ASOT_PREC_FP32 || prec == ASOT_PREC_TF32) ? 9 : 0;
  if (prec == ASOT_PREC_FP32)
    return asot::sinkhorn_tc3_supported(K) ? 3 : asot::sinkhorn_tc6_supported(K) ? 10
         : asot::sinkhorn_tc5_supported(K) ? 5 : 0;
  if (prec != ASOT_PREC_TF32) return 0;
  if (asot::sinkhorn_tc_supported(K)) return 1;
  if (asot::sinkhorn_tc2_supported(K)) return 2;
  if (asot::sinkhorn_tc4_supported(K)) return 4;
  return 0;
}
// Explicit pair lists (asot_pairwise_sinkhorn): K <= 128 -> the resident 1-SM kernels in
// pair-list mode (TF32: 7; fp32 requests: 3xTF32, 8; K < 32: the lane-per-anchor kernel, 9); above, the streamed
// kernel in pair-list mode (3xTF32 for fp32 requests, one TF32 pass otherwise).
int pair_kind(int32_t K, asot_precision prec) {
  if (K < 1 || K > asot::kMaxAnchors) return 0;
  // ASOT_PAIR_KERNEL=simt: the fp32 CUDA-core kernel for pair lists (cross-checks of the tensor-core
  // pair-list modes against an independent fp32 implementation)
  static const bool simt = getenv("ASOT_PAIR_KERNEL") && std::string(getenv("ASOT_PAIR_KERNEL")) == "simt";
  if (simt) return 0;
  if (K < kMinTcAnchors) return 9;   // fp32 lane-per-anchor kernel (as tile requests, R#23)
  if (asot::sinkhorn_tc_supported(K)) return prec == ASOT_PREC_FP32 ? 8 : 7;
  return prec == ASOT_PREC_FP32 ? 5 : 6;
}
bool use_tc(int32_t K, asot_precision prec) { return tc_kind(K, prec) != 0; }
constexpr int32_t kMinSparseAnchors = 64;   // the small-support path (R#36) from this K up
// Bucketed pair lists (asot_pairs_bucket.cu): the tile kernel that serves the fully covered tiles
// of a list of pair_kind `lk` (TF32: 7 -> the 1-SM kernel's tile mode, 6 -> the CTA-pair kernel
// for K <= 256, else the streamed one; fp32: 8 -> the 1-SM 3xTF32 kernel, 5 -> the BF16x3
// CTA-pair kernel for K <= 256, else the streamed 3xTF32 kernel's tile mode), its unit (1: tiles,
// 2: block pairs); 0 = the list runs as it is.
int bucket_tile_kind(int32_t K, asot_precision prec) {
  static const bool off = getenv("ASOT_PAIR_BUCKET") && std::string(getenv("ASOT_PAIR_BUCKET")) == "0";
  if (off) return 0;
  const int lk = pair_kind(K, prec);
  if (lk == 7) return 1;
  if (lk == 8) return 3;
  if (lk == 6) return asot::sinkhorn_tc2_supported(K) ? 2 : 4;
  if (lk == 5) return asot::sinkhorn_tc6_supported(K) ? 10 : 5;
  return 0;
}
int bucket_upt(int tk) { return tk == 1 || tk == 3 ? 1 : 2; }
constexpr int64_t kMinBucketPairs = 1024;

int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Gibbs buffers: plain G / GC (SIMT) or swizzled TF32 operand images (tensor-core kernels), plus
// the streamed kernel's scratch (padded marginals, per-CTA scaling buffers).
struct GibbsBufs {
  int kind = 0;
  float* G = nullptr;
  float* GC = nullptr;
  uint32_t* g_img = nullptr;
  uint32_t* gc_img = nullptr;
  uint8_t* scratch = nullptr;
  asot::SparseBufs sp;   // the small-support path (R#36), every kind
};

GibbsBufs carve_gibbs(Carver& cv, int32_t K, int kind, int64_t n_dist) {
  GibbsBufs b;
  b.kind = kind;
  if (kind == 5 || kind == 6) {  // K_hi, K_lo, (K (.) C_s)_hi, _lo images + marginals / X scratch
    b.g_img = (uint32_t*)cv.take(asot::sinkhorn_tc5_image_bytes(K));
    b.scratch = (uint8_t*)cv.take(asot::sinkhorn_tc5_scratch_bytes(K, n_dist, device_sms()) + 1024);
  } else if (kind == 4) {
    b.g_img = (uint32_t*)cv.take(asot::sinkhorn_tc4_image_bytes(K));
    b.gc_img = (uint32_t*)cv.take(asot::sinkhorn_tc4_image_bytes(K));
    b.scratch = (uint8_t*)cv.take(asot::sinkhorn_tc4_scratch_bytes(K, n_dist, device_sms()) + 1024);
  } else if (kind == 2) {
    b.g_img = (uint32_t*)cv.take(asot::sinkhorn_tc2_image_bytes());
    b.gc_img = (uint32_t*)cv.take(asot::sinkhorn_tc2_image_bytes());
  } else if (kind == 10) {   // BF16 hi / lo images of K and K (.) C_s, both ranks
    b.g_img = (uint32_t*)cv.take(asot::sinkhorn_tc6_image_bytes());
    b.gc_img = (uint32_t*)cv.take(asot::sinkhorn_tc6_image_bytes());
  } else if (kind == 1 || kind == 7) {
    const size_t kp = (size_t)asot::kpad32(K);
    b.g_img = (uint32_t*)cv.take(kp * kp * 4);
    b.gc_img = (uint32_t*)cv.take(kp * kp * 4);
    if (kind == 7) b.scratch = (uint8_t*)cv.take(asot::sinkhorn_tc_pairs_scratch_bytes(n_dist, K));
  } else if (kind == 3 || kind == 8) {  // K_hi image, K_lo image, plain K (.) C_s (+ padded H)
    b.g_img = (uint32_t*)cv.take(asot::sinkhorn_tc3_image_bytes(K));
    b.gc_img = (uint32_t*)cv.take(asot::sinkhorn_tc3_image_bytes(K));
    b.GC = (float*)cv.take(asot::sinkhorn_tc3_image_bytes(K));
    if (kind == 8) b.scratch = (uint8_t*)cv.take(asot::sinkhorn_tc3_pairs_scratch_bytes(n_dist, K));
  } else {  // CUDA-core kernel: row-padded fp32 K and K (.) C_s [K][simt_kpad(K)]
    b.G = (float*)cv.take((size_t)K * asot::simt_kpad(K) * 4);
    b.GC = (float*)cv.take((size_t)K * asot::simt_kpad(K) * 4);
  }
  uint8_t* spb = (uint8_t*)cv.take(asot::sparse_bytes(n_dist, K));
  if (spb != nullptr) b.sp = asot::carve_sparse(spb, n_dist, K);
  return b;
}

// ASOT_SPARSE=0 (diagnostic, read per call: the GPU tests of the dense kernels set it; bench.py
// refuses it) keeps every call on the dense kernels
bool sparse_path_enabled() {
  const char* e = getenv("ASOT_SPARSE");
  return !(e && std::string(e) == "0");
}

// NVTX ranges per hot-path phase (SURVEY §5 tracing): host-side push/pop around each phase's
// launches, visible in Nsight Systems / ncu --nvtx; no cost without an attached tool.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

// Profiling (asot_profile_*): event pairs recorded around each launch of the Sinkhorn kernel
// (ASOT_PROF_SINKHORN) and of the mapping kernel (ASOT_PROF_MAP).
thread_local bool g_prof_on = false;
struct ProfList {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
  size_t used = 0;
};
thread_local ProfList g_prof[2];

std::pair<cudaEvent_t, cudaEvent_t> prof_pair(int which) {
  ProfList& l = g_prof[which];
  if (l.used == l.events.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    l.events.emplace_back(a, b);
  }
  return l.events[l.used++];
}

// Records the start event now and the stop event when the scope ends (after the launch).
struct ProfScope {
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  cudaStream_t s;
  ProfScope(int which, cudaStream_t st) : s(st) {
    if (g_prof_on) {
      ev = prof_pair(which);
      cudaEventRecord(ev.first, s);
    }
  }
  ~ProfScope() {
    if (ev.second) cudaEventRecord(ev.second, s);
  }
};

asot_status run_sinkhorn(const asot::PairSource& ps, const asot::PairSink& sink, const float* H,
                         const float* cost, float eps, int32_t K, int32_t iters,
                         const GibbsBufs& gb, int64_t tile_begin, int64_t tile_end,
                         cudaStream_t s, bool ordered = false) {
  const int kind = gb.kind;
  {
  Nvtx range("asot a1 gibbs_prep");
  if (kind == 5 || kind == 6) {
    ASOT_LAUNCH(asot::launch_gibbs_prep_tc5(cost, K, eps, (uint8_t*)gb.g_img, s));
  } else if (kind == 4) {
    ASOT_LAUNCH(asot::launch_gibbs_prep_tc4(cost, K, eps, (uint8_t*)gb.g_img, (uint8_t*)gb.gc_img, s));
  } else if (kind == 2) {
    ASOT_LAUNCH(asot::launch_gibbs_prep_tc2(cost, K, eps, (uint8_t*)gb.g_img, (uint8_t*)gb.gc_img, s));
  } else if (kind == 10) {
    ASOT_LAUNCH(asot::launch_gibbs_prep_tc6(cost, K, eps, (uint8_t*)gb.g_img, (uint8_t*)gb.gc_img, s));
  } else if (kind == 3 || kind == 8) {
    ASOT_LAUNCH(asot::launch_gibbs_prep_tc3(cost, K, eps, gb.g_img, gb.gc_img, gb.GC, s));
  } else if (kind == 1 || kind == 7) {
    ASOT_LAUNCH(asot::launch_gibbs_prep(cost, K, eps, nullptr, nullptr, gb.g_img, gb.gc_img,
                                        asot::kpad32(K), s));
  } else {
    ASOT_LAUNCH(asot::launch_gibbs_prep_simt(cost, K, eps, gb.G, gb.GC, s));
  }
  }
  Nvtx range("asot a5+a6 sinkhorn+cost");
  ProfScope prof(ASOT_PROF_SINKHORN, s);
  // Small supports (R#36): the sparse kernel serves the call when every distribution has at most
  // kSparseCap non-zero bins, decided on the device; the dense kernel below then returns at once
  // (sink.dense_if), and vice versa.
  asot::PairSink sinkd = sink;
  // K < 64 stays on the dense kernels: a 16-bin support there saves at most 16x of K^2 <= 4096
  // products per half-iteration, against the lane-per-anchor / 1-SM kernels' full occupancy
  if (sparse_path_enabled() && gb.sp.flag != nullptr && K >= kMinSparseAnchors) {
    ASOT_LAUNCH(asot::launch_sparse_prep(H, ps.n_dist, K, cost, eps, gb.sp, s));
    const bool units = ps.units != nullptr && ps.pi == nullptr;
    const int upt = units ? bucket_upt(kind) : 1;
    const int64_t max_slots = units ? (tile_end - tile_begin) * asot::kTileSlots : ps.n_slots;
    ASOT_LAUNCH(asot::launch_sinkhorn_sparse(ps, sink, K, gb.sp, iters, upt, max_slots, device_sms(), s, ordered));
    sinkd.dense_if = gb.sp.flag;
  }
  const asot::PairSink& sink_dense = sinkd;
  if (kind == 5 || kind == 6) {
    const bool expl = ps.pi != nullptr;   // pair-list mode: tiles of 128 list entries
    ASOT_LAUNCH(asot::launch_sinkhorn_tc5(expl ? 0 : tile_begin,
                                          expl ? (ps.n_slots + asot::kTileSlots - 1) / asot::kTileSlots : tile_end,
                                          ps.n_dist, sink_dense, ps, H, K, (const uint8_t*)gb.g_img,
                                          (uint8_t*)(((uintptr_t)gb.scratch + 1023) & ~(uintptr_t)1023), iters,
                                          kind == 5, s));
  } else if (kind == 4) {
    ASOT_LAUNCH(asot::launch_sinkhorn_tc4(tile_begin, tile_end, ps.n_dist, sink_dense, H, K,
                                          (const uint8_t*)gb.g_img, (const uint8_t*)gb.gc_img,
                                          (uint8_t*)(((uintptr_t)gb.scratch + 1023) & ~(uintptr_t)1023), iters, s,
                                          ps.units, ps.n_dev));
  } else if (kind == 2) {
    ASOT_LAUNCH(asot::launch_sinkhorn_tc2(tile_begin, tile_end, ps.n_dist, sink_dense, H, K,
                                          (const uint8_t*)gb.g_img, (const uint8_t*)gb.gc_img, iters, s,
                                          ps.units, ps.n_dev));
  } else if (kind == 10) {
    ASOT_LAUNCH(asot::launch_sinkhorn_tc6(tile_begin, tile_end, ps.n_dist, sink_dense, H, K,
                                          (const uint8_t*)gb.g_img, (const uint8_t*)gb.gc_img, iters, s,
                                          ps.units, ps.n_dev));
  } else if (kind == 1) {
    ASOT_LAUNCH(asot::launch_sinkhorn_tc(tile_begin, tile_end, ps.n_dist, sink_dense, H, K, gb.g_img,
                                         gb.gc_img, iters, s, ps.units, ps.n_dev));
  } else if (kind == 7) {
    ASOT_LAUNCH(asot::launch_sinkhorn_tc_pairs(ps.pi, ps.pj, ps.n_slots, ps.n_dist, sink_dense, H, K, gb.g_img,
                                               gb.gc_img, (float*)gb.scratch, iters, s, ps.n_dev));
  } else if (kind == 3) {
    ASOT_LAUNCH(asot::launch_sinkhorn_tc3(tile_begin, tile_end, ps.n_dist, sink_dense, H, K, gb.g_img,
                                          gb.gc_img, gb.GC, iters, s, ps.units, ps.n_dev));
  } else if (kind == 8) {
    ASOT_LAUNCH(asot::launch_sinkhorn_tc3_pairs(ps.pi, ps.pj, ps.n_slots, ps.n_dist, sink_dense, H, K, gb.g_img,
                                                gb.gc_img, gb.GC, (float*)gb.scratch, iters, s, ps.n_dev));
  } else if (kind == 9) {
    ASOT_LAUNCH(asot::launch_sinkhorn_warp(ps, sink_dense, H, K, gb.G, gb.GC, iters, s));
  } else {
    ASOT_LAUNCH(asot::launch_sinkhorn_simt(ps, sink_dense, H, K, gb.G, gb.GC, iters, s));
  }
  return ASOT_OK;
}

// the bucketed layout after the list kind's buffers: the tile kind's Gibbs images (kind 1 shares
// kind 7's), then the bucket arrays
struct BucketLayout {
  GibbsBufs gbt;
  uint8_t* base = nullptr;
};
BucketLayout carve_bucketed(Carver& cv, const GibbsBufs& gbl, int32_t K, int tk, int64_t n_dist, int64_t n_pairs) {
  BucketLayout L;
  if (tk == 1 || tk == 3 || tk == 5) {   // the pair-list kinds 7 / 8 / 5 carve the same images
    L.gbt = gbl;
    L.gbt.kind = tk;
  } else {
    L.gbt = carve_gibbs(cv, K, tk, n_dist);
  }
  L.base = (uint8_t*)cv.take(asot::pair_bucket_bytes(n_dist, n_pairs, bucket_upt(tk)));
  return L;
}
bool bucketed(int32_t K, asot_precision prec, int64_t n_dist, int64_t n_pairs) {
  return bucket_tile_kind(K, prec) != 0 && n_pairs >= kMinBucketPairs && asot::pair_bucket_supported(n_dist);
}
}  // namespace

extern "C" {

int32_t asot_abi_version(void) { return ASOT_ABI_VERSION; }
const char* asot_last_error(void) { return g_last_error.c_str(); }
int32_t asot_last_launch_count(void) { return g_launches; }

asot_status asot_profile_enable(int32_t on) {
  g_prof_on = on != 0;
  return ASOT_OK;
}

asot_status asot_profile_read_kernel(int32_t which, double* ms_out, int64_t* launches,
                                     int32_t reset) {
  ASOT_CHECK_ARG(ms_out && launches, "null pointer argument");
  ASOT_CHECK_ARG(which == ASOT_PROF_SINKHORN || which == ASOT_PROF_MAP, "unknown kernel id");
  ProfList& l = g_prof[which];
  double total = 0.0;
  for (size_t k = 0; k < l.used; ++k) {
    ASOT_CUDA(cudaEventSynchronize(l.events[k].second));
    float ms = 0.0f;
    ASOT_CUDA(cudaEventElapsedTime(&ms, l.events[k].first, l.events[k].second));
    total += ms;
  }
  *ms_out = total;
  *launches = (int64_t)l.used;
  if (reset) l.used = 0;
  return ASOT_OK;
}

asot_status asot_profile_read(double* sinkhorn_ms, int64_t* launches, int32_t reset) {
  return asot_profile_read_kernel(ASOT_PROF_SINKHORN, sinkhorn_ms, launches, reset);
}
asot_status asot_profile_clock(int32_t kind, double* sm_mhz) {
  ASOT_CHECK_ARG(sm_mhz, "null pointer argument");
  long long c[4] = {0, 0, 0, 0};
  cudaError_t e;
  switch (kind) {
    case 1: case 7: e = asot::read_kernel_clock_tc(c); break;
    case 2: e = asot::read_kernel_clock_tc2(c); break;
    case 3: case 8: e = asot::read_kernel_clock_tc3(c); break;
    case 4: e = asot::read_kernel_clock_tc4(c); break;
    case 5: case 6: e = asot::read_kernel_clock_tc5(c); break;
    case 10: e = asot::read_kernel_clock_tc6(c); break;
    default: return fail(ASOT_ERR_INVALID_ARGUMENT, "no clock probe for this kernel kind");
  }
  ASOT_CUDA(e);
  if (c[3] <= c[1] || c[2] <= c[0]) return fail(ASOT_ERR_INVALID_ARGUMENT, "kernel kind not launched yet");
  *sm_mhz = (double)(c[2] - c[0]) / (double)(c[3] - c[1]) * 1000.0;
  return ASOT_OK;
}
int64_t asot_num_tiles(int64_t n_dist) { return n_dist < 1 ? 0 : asot::num_tiles(n_dist); }

int32_t asot_sinkhorn_kernel_kind(int32_t n_anchors, asot_precision requested) {
  return tc_kind(n_anchors, requested);
}

int32_t asot_sinkhorn_path_kind(int32_t n_anchors, asot_precision requested, int32_t max_support) {
  if (sparse_path_enabled() && n_anchors >= kMinSparseAnchors && n_anchors <= asot::kMaxAnchors &&
      max_support <= asot::kSparseCap)
    return 11;
  return tc_kind(n_anchors, requested);
}

asot_precision asot_effective_precision(int32_t n_anchors, asot_precision requested) {
  const int kind = tc_kind(n_anchors, requested);
  return kind == 0 || kind == 3 || kind == 5 || kind == 9 || kind == 10 ? ASOT_PREC_FP32
                                                                        : ASOT_PREC_TF32;   // (6: TF32)
}

static asot_status map_impl(const float* points, const int64_t* offsets, const int64_t* offsets_host,
                            const float* weights, int64_t n_dist, int32_t dim, const float* anchors,
                            int32_t n_anchors, int32_t* assign_out, float* hist_out, uint32_t* status,
                            void* stream, float* const* peers, int32_t n_peers, int64_t row_base,
                            uint8_t* tc_ws);

asot_status asot_map_to_anchors(const float* points, const int64_t* offsets,
                                const int64_t* offsets_host, const float* weights,
                                int64_t n_dist, int32_t dim, const float* anchors,
                                int32_t n_anchors, int32_t* assign_out, float* hist_out,
                                uint32_t* status, void* stream) {
  return map_impl(points, offsets, offsets_host, weights, n_dist, dim, anchors, n_anchors, assign_out,
                  hist_out, status, stream, nullptr, 0, 0, nullptr);
}

asot_status asot_map_to_anchors_bcast(const float* points, const int64_t* offsets,
                                      const int64_t* offsets_host, const float* weights,
                                      int64_t n_dist, int32_t dim, const float* anchors,
                                      int32_t n_anchors, int32_t* assign_out, float* hist_out,
                                      float* const* hist_peers, int32_t n_peers, int64_t row_base,
                                      uint32_t* status, void* stream) {
  ASOT_CHECK_ARG(n_peers >= 0 && (n_peers == 0 || hist_peers), "hist_peers required when n_peers > 0");
  ASOT_CHECK_ARG(row_base >= 0, "row_base must be >= 0");
  return map_impl(points, offsets, offsets_host, weights, n_dist, dim, anchors, n_anchors, assign_out,
                  hist_out, status, stream, hist_peers, n_peers, row_base, nullptr);
}

size_t asot_map_workspace_bytes(int64_t n_points, int32_t n_anchors) {
  return align_up(asot::map_tc_workspace_bytes(n_points, n_anchors));
}

asot_status asot_map_to_anchors_ws(const float* points, const int64_t* offsets,
                                   const int64_t* offsets_host, const float* weights,
                                   int64_t n_dist, int32_t dim, const float* anchors,
                                   int32_t n_anchors, int32_t* assign_out, float* hist_out,
                                   float* const* hist_peers, int32_t n_peers, int64_t row_base,
                                   uint32_t* status, void* workspace, size_t workspace_bytes,
                                   void* stream) {
  ASOT_CHECK_ARG(n_peers >= 0 && (n_peers == 0 || hist_peers), "hist_peers required when n_peers > 0");
  ASOT_CHECK_ARG(row_base >= 0, "row_base must be >= 0");
  ASOT_CHECK_ARG(offsets_host && n_dist >= 1, "offsets_host required, n_dist must be >= 1");
  if (!workspace || ((uintptr_t)workspace & 255u) != 0 ||
      workspace_bytes < asot_map_workspace_bytes(offsets_host[n_dist], n_anchors))
    return fail(ASOT_ERR_WORKSPACE, "workspace too small or not 256-byte aligned (asot_map_workspace_bytes)");
  return map_impl(points, offsets, offsets_host, weights, n_dist, dim, anchors, n_anchors, assign_out,
                  hist_out, status, stream, hist_peers, n_peers, row_base, (uint8_t*)workspace);
}

static asot_status map_impl(const float* points, const int64_t* offsets, const int64_t* offsets_host,
                            const float* weights, int64_t n_dist, int32_t dim, const float* anchors,
                            int32_t n_anchors, int32_t* assign_out, float* hist_out, uint32_t* status,
                            void* stream, float* const* peers, int32_t n_peers, int64_t row_base,
                            uint8_t* tc_ws) {
  g_launches = 0;
  ASOT_CHECK_ARG(points && offsets && offsets_host && weights && anchors && assign_out &&
                     hist_out && status,
                 "null pointer argument");
  ASOT_CHECK_ARG(n_dist >= 1, "n_dist must be >= 1");
  ASOT_CHECK_ARG(dim >= 1, "dim must be >= 1");
  if (dim > asot::kMaxDim) return fail(ASOT_ERR_UNSUPPORTED, "dim > 128 is not supported");
  ASOT_CHECK_ARG(n_anchors >= 1, "n_anchors must be >= 1");
  if (n_anchors > asot::kMaxAnchors) return fail(ASOT_ERR_UNSUPPORTED, "n_anchors > 1024");
  ASOT_CHECK_ARG(offsets_host[0] == 0, "offsets[0] must be 0");
  for (int64_t i = 0; i < n_dist; ++i)
    ASOT_CHECK_ARG(offsets_host[i + 1] >= offsets_host[i], "offsets must be non-decreasing");
  const int64_t T = offsets_host[n_dist];
  cudaStream_t s = (cudaStream_t)stream;
  if (T > 0) {
    Nvtx range("asot a2 map_assign");
    ProfScope prof(ASOT_PROF_MAP, s);
    // with a workspace (asot_distance_matrix): the products on the tensor cores and the exact
    // kernel on the points they cannot decide (R#37); else the exact kernel on every point
    if (tc_ws != nullptr && asot::map_tc_supported(dim, n_anchors) && ((uintptr_t)points & 15u) == 0) {
      ASOT_LAUNCH(asot::launch_map_tc(points, T, dim, anchors, n_anchors, assign_out, status, tc_ws,
                                      device_sms(), s));
    } else {
      ASOT_LAUNCH(asot::launch_map_assign(points, T, dim, anchors, n_anchors, assign_out, status, s));
    }
  }
  Nvtx range("asot a3 histograms");
  ASOT_LAUNCH(asot::launch_histograms(assign_out, weights, offsets, n_dist, n_anchors, hist_out, status, s,
                                      peers, n_peers, row_base));
  return ASOT_OK;
}

// Shared argument checks of the soft mappings (NEXT-1).
static asot_status check_soft(const float* points, const int64_t* offsets, const int64_t* offsets_host,
                              const float* weights, int64_t n_dist, int32_t dim, int32_t n_anchors,
                              int32_t hidden, const float* hist_out, const uint32_t* status) {
  ASOT_CHECK_ARG(points && offsets && offsets_host && weights && hist_out && status,
                 "null pointer argument");
  ASOT_CHECK_ARG(n_dist >= 1 && dim >= 1 && n_anchors >= 1 && hidden >= 1, "sizes must be >= 1");
  if (dim > asot::kMaxDim) return fail(ASOT_ERR_UNSUPPORTED, "dim > 128 is not supported");
  if (n_anchors > asot::kMaxAnchors) return fail(ASOT_ERR_UNSUPPORTED, "n_anchors > 1024");
  if (hidden > 256) return fail(ASOT_ERR_UNSUPPORTED, "hidden > 256 is not supported");
  ASOT_CHECK_ARG(offsets_host[0] == 0, "offsets[0] must be 0");
  for (int64_t i = 0; i < n_dist; ++i)
    ASOT_CHECK_ARG(offsets_host[i + 1] >= offsets_host[i], "offsets must be non-decreasing");
  return ASOT_OK;
}

asot_status asot_map_soft_ml(const float* points, const int64_t* offsets,
                             const int64_t* offsets_host, const float* weights, int64_t n_dist,
                             int32_t dim, int32_t n_anchors, int32_t hidden, const float* W1,
                             const float* b1, const float* W2, const float* b2, float* hist_out,
                             float* codes_out, uint32_t* status, void* workspace,
                             size_t workspace_bytes, void* stream) {
  g_launches = 0;
  asot_status st = check_soft(points, offsets, offsets_host, weights, n_dist, dim, n_anchors,
                              hidden, hist_out, status);
  if (st != ASOT_OK) return st;
  ASOT_CHECK_ARG(W1 && b1 && W2 && b2, "null pointer argument");
  cudaStream_t s = (cudaStream_t)stream;
  Nvtx range("asot next1 map_soft_ml");
  ProfScope prof(ASOT_PROF_MAP, s);
  // both MLP layers on tcgen05 (BF16x3) when the shapes allow and the workspace is given;
  // otherwise the CUDA-core kernel (also the cross-check implementation)
  const size_t need = asot_map_soft_ml_workspace_bytes(dim, hidden, n_anchors);
  if (need > 0 && workspace && workspace_bytes >= need && ((uintptr_t)points & 15u) == 0) {
    ASOT_LAUNCH(asot::launch_soft_ml_tc(points, offsets, weights, n_dist, dim, hidden, n_anchors, W1, b1,
                                        W2, b2, hist_out, codes_out, (uint8_t*)workspace, status,
                                        device_sms(), s));
    return ASOT_OK;
  }
  ASOT_LAUNCH(asot::launch_soft_map_ml(points, offsets, weights, n_dist, dim, n_anchors, hidden,
                                       W1, b1, W2, b2, hist_out, codes_out, status, s));
  return ASOT_OK;
}

asot_status asot_map_soft_dl(const float* points, const int64_t* offsets,
                             const int64_t* offsets_host, const float* weights, int64_t n_dist,
                             int32_t dim, const float* dictionary, int32_t n_anchors,
                             int32_t n_layers, int32_t hidden, const float* V1, const float* c1,
                             const float* v2, const float* c2, float* hist_out, float* codes_out,
                             uint32_t* status, void* workspace, size_t workspace_bytes,
                             void* stream) {
  g_launches = 0;
  asot_status st = check_soft(points, offsets, offsets_host, weights, n_dist, dim, n_anchors,
                              hidden, hist_out, status);
  if (st != ASOT_OK) return st;
  ASOT_CHECK_ARG(dictionary && V1 && c1 && v2 && c2, "null pointer argument");
  ASOT_CHECK_ARG(n_layers >= 1, "n_layers must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  Nvtx range("asot next1 map_soft_dl");
  ProfScope prof(ASOT_PROF_MAP, s);
  const size_t need = asot_map_soft_dl_workspace_bytes(dim, n_anchors, offsets_host[n_dist]);
  const bool aligned = ((uintptr_t)points & 15u) == 0 && ((uintptr_t)dictionary & 15u) == 0;
  // large dictionaries: the tensor-core kernel (default) or, for cross-checks
  // (ASOT_SOFT_DL_GENERIC=sparse), the sparse-code CUDA-core kernel; otherwise / without a
  // workspace the resident, tiled or streamed CUDA-core kernels
  const char* gen = getenv("ASOT_SOFT_DL_GENERIC");
  if (need > 0 && workspace && workspace_bytes >= need && aligned) {
    if (!gen) {
      ASOT_LAUNCH(asot::launch_soft_dl_tc(points, offsets, weights, n_dist, dim, dictionary, n_anchors,
                                          n_layers, hidden, V1, c1, v2, c2, hist_out, codes_out,
                                          (uint8_t*)workspace, status, device_sms(), offsets_host[n_dist], s));
      return ASOT_OK;
    }
    if (std::string(gen) == "sparse") {
      ASOT_LAUNCH(asot::launch_soft_dl_sparse(points, offsets, weights, n_dist, dim, dictionary, n_anchors,
                                              n_layers, hidden, V1, c1, v2, c2, hist_out, codes_out,
                                              (float*)workspace, status, device_sms(), s));
      return ASOT_OK;
    }
  }
  ASOT_LAUNCH(asot::launch_soft_map_dl(points, offsets, weights, n_dist, dim, dictionary, n_anchors,
                                       n_layers, hidden, V1, c1, v2, c2, hist_out, codes_out,
                                       status, s));
  return ASOT_OK;
}

size_t asot_map_soft_ml_workspace_bytes(int32_t dim, int32_t hidden, int32_t n_anchors) {
  if (!asot::soft_ml_tc_supported(dim, hidden, n_anchors)) return 0;
  return asot::soft_ml_tc_workspace_bytes(dim, hidden, n_anchors, device_sms());
}

size_t asot_map_soft_dl_workspace_bytes(int32_t dim, int32_t n_anchors, int64_t n_points) {
  if (!asot::soft_dl_tc_supported(dim, n_anchors)) return 0;
  const size_t a = asot::soft_dl_tc_workspace_bytes(dim, n_anchors, device_sms(), n_points);
  const size_t b = asot::soft_dl_sparse_workspace_bytes(n_anchors, device_sms());
  return a > b ? a : b;
}

size_t asot_mahalanobis_workspace_bytes(int32_t n_anchors, int32_t h) {
  return n_anchors < 1 || h < 1 ? 0 : (size_t)n_anchors * h * 4;
}

asot_status asot_mahalanobis_cost(const float* anchors, int32_t n_anchors, int32_t dim,
                                  const float* M, int32_t h, int32_t normalize, float* cost_out,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(anchors && M && cost_out, "null pointer argument");
  ASOT_CHECK_ARG(n_anchors >= 1 && dim >= 1 && h >= 1, "sizes must be >= 1");
  if (n_anchors > asot::kMaxAnchors) return fail(ASOT_ERR_UNSUPPORTED, "n_anchors > 1024");
  if (!workspace || workspace_bytes < asot_mahalanobis_workspace_bytes(n_anchors, h))
    return fail(ASOT_ERR_WORKSPACE, "workspace too small");
  ASOT_LAUNCH(asot::launch_mahalanobis_cost(anchors, n_anchors, dim, M, h, normalize != 0,
                                            (float*)workspace, cost_out, (cudaStream_t)stream));
  return ASOT_OK;
}

asot_status asot_kmeans_minibatch(const float* points, int64_t n_points, int32_t dim,
                                  int32_t n_anchors, const int64_t* batch_idx, int32_t batch,
                                  int32_t iters, double* centers, int64_t* counts,
                                  float* anchors_out, int32_t* assign_ws, uint32_t* status,
                                  void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(points && (batch_idx || iters == 0) && centers && counts && anchors_out &&
                     (assign_ws || iters == 0) && status,
                 "null pointer argument");
  ASOT_CHECK_ARG(n_points >= 1 && dim >= 1 && n_anchors >= 1 && batch >= 1 && iters >= 0,
                 "sizes must be >= 1 (iters >= 0)");
  if (dim > asot::kMaxDim) return fail(ASOT_ERR_UNSUPPORTED, "dim > 128 is not supported");
  if (n_anchors > asot::kMaxAnchors) return fail(ASOT_ERR_UNSUPPORTED, "n_anchors > 1024");
  cudaStream_t s = (cudaStream_t)stream;
  ASOT_LAUNCH(asot::launch_kmeans_prepare(centers, n_anchors, dim, anchors_out, s));
  for (int32_t t = 0; t < iters; ++t) {
    const int64_t* bt = batch_idx + (int64_t)t * batch;
    ASOT_LAUNCH(asot::launch_map_assign(points, batch, dim, anchors_out, n_anchors, assign_ws,
                                        status, s, bt));
    ASOT_LAUNCH(asot::launch_kmeans_update(points, dim, bt, batch, assign_ws, n_anchors, centers,
                                           anchors_out, counts, s));
  }
  return ASOT_OK;
}

asot_status asot_sqeuclid_cost(const float* anchors, int32_t n_anchors, int32_t dim,
                               int32_t normalize, float* cost_out, void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(anchors && cost_out, "null pointer argument");
  ASOT_CHECK_ARG(n_anchors >= 1 && dim >= 1, "sizes must be >= 1");
  if (n_anchors > asot::kMaxAnchors) return fail(ASOT_ERR_UNSUPPORTED, "n_anchors > 1024");
  ASOT_LAUNCH(asot::launch_sqeuclid_cost(anchors, n_anchors, dim, normalize != 0, cost_out,
                                         (cudaStream_t)stream));
  return ASOT_OK;
}

static int64_t max_dist_size(int64_t n_dist, const int64_t* offsets_host) {
  int64_t m = 0;
  for (int64_t i = 0; i < n_dist; ++i) m = std::max<int64_t>(m, offsets_host[i + 1] - offsets_host[i]);
  return m;
}

size_t asot_eot_workspace_bytes(int64_t n_dist, const int64_t* offsets_host, int64_t n_pairs) {
  if (!offsets_host || n_dist < 1 || n_pairs < 1) return 0;
  return asot::eot_slot_floats(max_dist_size(n_dist, offsets_host)) * 4 *
         (size_t)asot::eot_grid(n_pairs, device_sms());
}

asot_status asot_eot_pairs(const float* points, const int64_t* offsets, const int64_t* offsets_host,
                           const float* weights, int64_t n_dist, int32_t dim, float cost_scale,
                           float eps, int32_t iters, const int32_t* pair_i, const int32_t* pair_j,
                           int64_t n_pairs, float* dist_out, uint32_t* status, void* workspace,
                           size_t workspace_bytes, void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(points && offsets && offsets_host && weights && pair_i && pair_j && dist_out && status,
                 "null pointer argument");
  ASOT_CHECK_ARG(n_dist >= 1 && dim >= 1 && iters >= 1 && n_pairs >= 0, "bad sizes");
  ASOT_CHECK_ARG(std::isfinite(eps) && eps > 0.0f && std::isfinite(cost_scale) && cost_scale >= 0.0f,
                 "eps must be > 0 and cost_scale >= 0, finite");
  const int64_t mx = max_dist_size(n_dist, offsets_host);
  if (!asot::eot_supported(mx)) return fail(ASOT_ERR_UNSUPPORTED, "a distribution has > 16384 points");
  if (n_pairs == 0) return ASOT_OK;
  const size_t need = asot_eot_workspace_bytes(n_dist, offsets_host, n_pairs);
  if (need > 0 && (!workspace || workspace_bytes < need)) return fail(ASOT_ERR_WORKSPACE, "workspace too small");
  const int grid = asot::eot_grid(n_pairs, device_sms());
  ASOT_LAUNCH(asot::launch_eot_pairs(points, offsets, weights, dim, cost_scale, eps, iters, pair_i,
                                     pair_j, n_pairs, dist_out, (float*)workspace,
                                     (int64_t)asot::eot_slot_floats(mx), grid, (int)mx, status,
                                     (cudaStream_t)stream));
  return ASOT_OK;
}

asot_status asot_exact_w1_points(const float* points, const int64_t* offsets, const float* weights,
                                 int64_t n_dist, int32_t dim, const int32_t* pair_i,
                                 const int32_t* pair_j, int64_t n_pairs, double* dist_out,
                                 uint32_t* status, void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(n_pairs >= 0 && n_dist >= 1 && dim >= 1, "bad sizes");
  ASOT_CHECK_ARG(points && offsets && weights && status && (n_pairs == 0 || (pair_i && pair_j && dist_out)),
                 "null pointer argument");
  if (n_pairs == 0) return ASOT_OK;
  Nvtx range("asot next3 exact_w1_points");
  ASOT_LAUNCH(asot::launch_w1_points(points, offsets, weights, n_dist, dim, pair_i, pair_j, n_pairs, dist_out,
                                     status, device_sms(), (cudaStream_t)stream));
  return ASOT_OK;
}

asot_status asot_bound_terms(const float* points, const int64_t* offsets, int64_t n_dist, int32_t dim,
                             const float* anchors, int32_t n_anchors, const int32_t* assign,
                             const float* cost, const int32_t* pair_i, const int32_t* pair_j,
                             int64_t n_pairs, double* prop1_l1, double* prop1_max, double* prop2,
                             uint32_t* status, void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(n_pairs >= 0 && n_dist >= 1 && n_anchors >= 1, "bad sizes");
  ASOT_CHECK_ARG(dim >= 1, "dim must be >= 1");
  if (dim > asot::kMaxDim) return fail(ASOT_ERR_UNSUPPORTED, "dim > 128 is not supported");
  ASOT_CHECK_ARG(points && offsets && anchors && assign && cost && status &&
                     (n_pairs == 0 || (pair_i && pair_j && prop1_l1 && prop1_max && prop2)),
                 "null pointer argument");
  if (n_pairs == 0) return ASOT_OK;
  Nvtx range("asot next3 bound_terms");
  ASOT_LAUNCH(asot::launch_bound_terms(points, offsets, n_dist, dim, anchors, n_anchors, assign, cost, pair_i,
                                       pair_j, n_pairs, prop1_l1, prop1_max, prop2, status, device_sms(),
                                       (cudaStream_t)stream));
  return ASOT_OK;
}

size_t asot_exact_asot_workspace_bytes(int64_t n_pairs, int32_t n_anchors) {
  return asot::exact_pairs_workspace_bytes(n_pairs, n_anchors, device_sms());
}

asot_status asot_exact_asot_pairs(const float* hist, int64_t n_dist, int32_t n_anchors, const float* cost,
                                  const int32_t* pair_i, const int32_t* pair_j, int64_t n_pairs,
                                  double* dist_out, uint32_t* status, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(hist && cost && pair_i && pair_j && dist_out && status, "null pointer argument");
  ASOT_CHECK_ARG(n_dist >= 1 && n_anchors >= 1 && n_pairs >= 0, "bad sizes");
  if (n_anchors > asot::kMaxAnchors) return fail(ASOT_ERR_UNSUPPORTED, "n_anchors > 1024");
  if (n_pairs == 0) return ASOT_OK;
  if (!workspace || workspace_bytes < asot::exact_pairs_workspace_bytes(n_pairs, n_anchors, device_sms()))
    return fail(ASOT_ERR_WORKSPACE, "workspace too small (asot_exact_asot_workspace_bytes)");
  ASOT_LAUNCH(asot::launch_exact_pairs(hist, n_dist, n_anchors, cost, pair_i, pair_j, n_pairs, dist_out,
                                       (uint8_t*)workspace, status, device_sms(), (cudaStream_t)stream));
  return ASOT_OK;
}

size_t asot_pairwise_workspace_bytes(int64_t n_dist, int32_t n_anchors, asot_precision prec) {
  Carver cv{nullptr, 0};
  carve_gibbs(cv, n_anchors, pair_kind(n_anchors, prec), n_dist);
  return cv.used;
}


size_t asot_pairwise_list_workspace_bytes(int64_t n_dist, int32_t n_anchors, asot_precision prec,
                                          int64_t n_pairs) {
  Carver cv{nullptr, 0};
  const GibbsBufs gbl = carve_gibbs(cv, n_anchors, pair_kind(n_anchors, prec), n_dist);
  if (bucketed(n_anchors, prec, n_dist, n_pairs))
    carve_bucketed(cv, gbl, n_anchors, bucket_tile_kind(n_anchors, prec), n_dist, n_pairs);
  return cv.used;
}

asot_status asot_pairwise_sinkhorn(const float* hist, int64_t n_dist, int32_t n_anchors,
                                   const float* cost, float cost_max, float eps, int32_t iters,
                                   asot_precision prec, const int32_t* pair_i,
                                   const int32_t* pair_j, int64_t n_pairs, float* dist_out,
                                   uint32_t* status, void* workspace, size_t workspace_bytes,
                                   void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(n_pairs >= 0, "n_pairs must be >= 0");
  ASOT_CHECK_ARG(hist && cost && status && (n_pairs == 0 || (pair_i && pair_j && dist_out)),
                 "null pointer argument");
  asot_status st = check_common(n_dist, n_anchors, eps, iters, cost_max);
  if (st != ASOT_OK) return st;
  if (n_pairs == 0) return ASOT_OK;   // (pair_i, pair_j, dist_out may be null)
  Carver cv{(char*)workspace, workspace_bytes};
  GibbsBufs gb = carve_gibbs(cv, n_anchors, pair_kind(n_anchors, prec), n_dist);
  if (!workspace || cv.overflow) return fail(ASOT_ERR_WORKSPACE, "workspace too small");
  const cudaStream_t s = (cudaStream_t)stream;
  if (bucketed(n_anchors, prec, n_dist, n_pairs)) {
    // the workspace of asot_pairwise_list_workspace_bytes: whole tiles on the tile path (the
    // smaller asot_pairwise_workspace_bytes runs the list as it is)
    Carver cvb = cv;
    const int tk = bucket_tile_kind(n_anchors, prec), upt = bucket_upt(tk);
    const BucketLayout L = carve_bucketed(cvb, gb, n_anchors, tk, n_dist, n_pairs);
    if (!cvb.overflow) {
      const int sms = device_sms();
      const asot::PairBuckets w = asot::carve_pair_buckets(L.base, n_dist, n_pairs, upt);
      ASOT_LAUNCH(asot::launch_pair_buckets(w, pair_i, pair_j, n_pairs, n_dist, sms, s));
      const int64_t* n_units = (const int64_t*)&w.cnt[0];
      const int64_t* n_left = (const int64_t*)&w.cnt[1];
      asot::PairSource pt{nullptr, nullptr, 0, 0, n_dist};
      pt.units = w.units;
      pt.n_dev = n_units;
      asot::PairSink rt{w.R, nullptr, n_dist, status, 0};
      asot_status st = run_sinkhorn(pt, rt, hist, cost, eps, n_anchors, iters, L.gbt, 0, w.cap * upt, s);
      if (st != ASOT_OK) return st;
      asot::PairSource pl{w.li, w.lj, n_pairs, 0, n_dist};
      pl.n_dev = n_left;
      asot::PairSink rl{dist_out, nullptr, n_dist, status, 1};
      rl.idx = w.lidx;
      st = run_sinkhorn(pl, rl, hist, cost, eps, n_anchors, iters, gb, 0, 0, s);
      if (st != ASOT_OK) return st;
      ASOT_LAUNCH(asot::launch_pair_gather(w, pair_i, pair_j, n_pairs, n_dist, dist_out, sms, s));
      return ASOT_OK;
    }
  }
  asot::PairSource ps{pair_i, pair_j, n_pairs, 0, n_dist};
  asot::PairSink sink{dist_out, nullptr, n_dist, status, 1};
  return run_sinkhorn(ps, sink, hist, cost, eps, n_anchors, iters, gb, 0, 0, s);
}

size_t asot_distance_matrix_workspace_bytes(int64_t n_dist, int64_t n_points, int32_t n_anchors,
                                            asot_precision prec) {
  Carver cv{nullptr, 0};
  cv.take((size_t)n_dist * n_anchors * 4);   // H
  cv.take((size_t)n_points * 4);             // assign scratch
  carve_gibbs(cv, n_anchors, tc_kind(n_anchors, prec), n_dist);
  cv.take(asot::map_tc_workspace_bytes(n_points, n_anchors));   // tensor-core mapping (R#37)
  return cv.used;
}

asot_status asot_distance_matrix(const float* points, const int64_t* offsets,
                                 const int64_t* offsets_host, const float* weights,
                                 int64_t n_dist, int32_t dim, const float* anchors,
                                 int32_t n_anchors, const float* cost, float cost_max, float eps,
                                 int32_t iters, asot_precision prec, const float* hist_in,
                                 int64_t tile_begin, int64_t tile_end, float* dist_out,
                                 float* packed_out, int32_t* assign_out, float* hist_out,
                                 uint32_t* status, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(cost && status, "null pointer argument");
  asot_status st = check_common(n_dist, n_anchors, eps, iters, cost_max);
  if (st != ASOT_OK) return st;
  const int64_t n_tiles = asot::num_tiles(n_dist);
  ASOT_CHECK_ARG(0 <= tile_begin && tile_begin <= tile_end && tile_end <= n_tiles,
                 "tile range outside [0, asot_num_tiles(n_dist)]");
  ASOT_CHECK_ARG(dist_out || packed_out, "need dist_out and/or packed_out");
  cudaStream_t s = (cudaStream_t)stream;
  const bool tc = use_tc(n_anchors, prec);

  int64_t T = 0;
  if (!hist_in) {
    ASOT_CHECK_ARG(points && offsets && offsets_host && weights && anchors,
                   "mapping inputs required when hist_in is NULL");
    T = offsets_host[n_dist];
  }
  Carver cv{(char*)workspace, workspace_bytes};
  float* H = (float*)cv.take((size_t)n_dist * n_anchors * 4);
  int32_t* assign = (int32_t*)cv.take((size_t)T * 4);
  GibbsBufs gb = carve_gibbs(cv, n_anchors, tc_kind(n_anchors, prec), n_dist);
  uint8_t* map_ws = (uint8_t*)cv.take(asot::map_tc_workspace_bytes(T, n_anchors));
  if (!workspace || cv.overflow) return fail(ASOT_ERR_WORKSPACE, "workspace too small");

  const float* Huse = hist_in;
  if (!hist_in) {
    int32_t* asg = assign_out ? assign_out : assign;
    float* Hw = hist_out ? hist_out : H;
    const int32_t launches_before = g_launches;
    st = map_impl(points, offsets, offsets_host, weights, n_dist, dim, anchors, n_anchors, asg, Hw,
                  status, stream, nullptr, 0, 0, map_ws);
    g_launches += launches_before;
    if (st != ASOT_OK) return st;
    Huse = Hw;
  }
  asot::PairSource ps{nullptr, nullptr, (tile_end - tile_begin) * asot::kTileSlots, tile_begin, n_dist};
  asot::PairSink sink{packed_out, dist_out, n_dist, status, 0};
  st = run_sinkhorn(ps, sink, Huse, cost, eps, n_anchors, iters, gb, tile_begin, tile_end, s);
  if (st != ASOT_OK) return st;
  if (dist_out && tile_begin == 0 && tile_end == n_tiles) {
    Nvtx range("asot a6 zero_diag");
    ASOT_LAUNCH(asot::launch_zero_diag(dist_out, n_dist, s));
  }
  return ASOT_OK;
}

asot_status asot_distance_matrix_partition(const float* hist, int64_t n_dist, int32_t n_anchors,
                                           const float* cost, float cost_max, float eps, int32_t iters,
                                           asot_precision prec, int64_t part_begin, int64_t part_end,
                                           float* dist_out, uint32_t* status, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(hist && cost && dist_out && status, "null pointer argument");
  asot_status st = check_common(n_dist, n_anchors, eps, iters, cost_max);
  if (st != ASOT_OK) return st;
  const int64_t n_tiles = asot::num_tiles(n_dist);
  ASOT_CHECK_ARG(0 <= part_begin && part_begin <= part_end && part_end <= n_tiles,
                 "part range outside [0, asot_num_tiles(n_dist)]");
  Carver cv{(char*)workspace, workspace_bytes};
  cv.take((size_t)n_dist * n_anchors * 4);   // (the asot_distance_matrix layout)
  GibbsBufs gb = carve_gibbs(cv, n_anchors, tc_kind(n_anchors, prec), n_dist);
  if (!workspace || cv.overflow) return fail(ASOT_ERR_WORKSPACE, "workspace too small");
  asot::PairSource ps{nullptr, nullptr, (part_end - part_begin) * asot::kTileSlots, part_begin, n_dist};
  asot::PairSink sink{nullptr, dist_out, n_dist, status, 0};
  st = run_sinkhorn(ps, sink, hist, cost, eps, n_anchors, iters, gb, part_begin, part_end,
                    (cudaStream_t)stream, /*ordered=*/true);
  if (st != ASOT_OK) return st;
  if (part_begin == 0 && part_end == n_tiles) {
    Nvtx range("asot a6 zero_diag");
    ASOT_LAUNCH(asot::launch_zero_diag(dist_out, n_dist, (cudaStream_t)stream));
  }
  return ASOT_OK;
}

size_t asot_distance_matrix_host_workspace_bytes(int64_t n_dist, int64_t n_points, int32_t dim,
                                                 int32_t n_anchors, asot_precision prec) {
  Carver cv{nullptr, 0};
  cv.take((size_t)n_points * dim * 4);          // points
  cv.take((size_t)(n_dist + 1) * 8);            // offsets
  cv.take((size_t)n_points * 4);                // weights
  cv.take((size_t)n_anchors * dim * 4);         // anchors
  cv.take((size_t)n_anchors * n_anchors * 4);   // cost
  cv.take((size_t)n_dist * n_dist * 4);         // D
  cv.take(4);                                   // status
  return cv.used + asot_distance_matrix_workspace_bytes(n_dist, n_points, n_anchors, prec);
}

asot_status asot_distance_matrix_host(const float* points_host, const int64_t* offsets_host,
                                      const float* weights_host, int64_t n_dist, int32_t dim,
                                      const float* anchors_host, int32_t n_anchors,
                                      const float* cost_host, float eps, int32_t iters,
                                      asot_precision prec, float* dist_host,
                                      uint32_t* status_host, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  ASOT_CHECK_ARG(points_host && offsets_host && weights_host && anchors_host && cost_host &&
                     dist_host && status_host,
                 "null pointer argument");
  ASOT_CHECK_ARG(n_dist >= 1 && dim >= 1 && n_anchors >= 1, "sizes must be >= 1");
  const int64_t T = offsets_host[n_dist];
  float cmax = 0.0f;
  for (int64_t e = 0; e < (int64_t)n_anchors * n_anchors; ++e) cmax = fmaxf(cmax, cost_host[e]);
  cudaStream_t s = (cudaStream_t)stream;
  Carver cv{(char*)workspace, workspace_bytes};
  float* d_points = (float*)cv.take((size_t)T * dim * 4);
  int64_t* d_offsets = (int64_t*)cv.take((size_t)(n_dist + 1) * 8);
  float* d_weights = (float*)cv.take((size_t)T * 4);
  float* d_anchors = (float*)cv.take((size_t)n_anchors * dim * 4);
  float* d_cost = (float*)cv.take((size_t)n_anchors * n_anchors * 4);
  float* d_D = (float*)cv.take((size_t)n_dist * n_dist * 4);
  uint32_t* d_status = (uint32_t*)cv.take(4);
  if (!workspace || cv.overflow) return fail(ASOT_ERR_WORKSPACE, "workspace too small");
  char* rest = (char*)workspace + cv.used;
  const size_t rest_bytes = workspace_bytes - cv.used;

  // one cudaMemcpyAsync per buffer (no batched-copy APIs)
  {
  Nvtx range("asot e2e h2d");
  ASOT_CUDA(cudaMemcpyAsync(d_points, points_host, (size_t)T * dim * 4, cudaMemcpyHostToDevice, s));
  ASOT_CUDA(cudaMemcpyAsync(d_offsets, offsets_host, (size_t)(n_dist + 1) * 8, cudaMemcpyHostToDevice, s));
  ASOT_CUDA(cudaMemcpyAsync(d_weights, weights_host, (size_t)T * 4, cudaMemcpyHostToDevice, s));
  ASOT_CUDA(cudaMemcpyAsync(d_anchors, anchors_host, (size_t)n_anchors * dim * 4, cudaMemcpyHostToDevice, s));
  ASOT_CUDA(cudaMemcpyAsync(d_cost, cost_host, (size_t)n_anchors * n_anchors * 4, cudaMemcpyHostToDevice, s));
  ASOT_CUDA(cudaMemsetAsync(d_status, 0, 4, s));
  }
  asot_status st = asot_distance_matrix(d_points, d_offsets, offsets_host, d_weights, n_dist, dim,
                                        d_anchors, n_anchors, d_cost, cmax, eps, iters, prec,
                                        nullptr, 0, asot::num_tiles(n_dist), d_D, nullptr,
                                        nullptr, nullptr, d_status, rest, rest_bytes, stream);
  if (st != ASOT_OK) return st;
  Nvtx range("asot e2e d2h");
  ASOT_CUDA(cudaMemcpyAsync(dist_host, d_D, (size_t)n_dist * n_dist * 4, cudaMemcpyDeviceToHost, s));
  ASOT_CUDA(cudaMemcpyAsync(status_host, d_status, 4, cudaMemcpyDeviceToHost, s));
  ASOT_CUDA(cudaStreamSynchronize(s));
  return ASOT_OK;
}

asot_status asot_tile_pairs_host(int64_t n_dist, int64_t tile_begin, int64_t tile_end,
                                 int32_t* i_out, int32_t* j_out, uint8_t* valid_out) {
  ASOT_CHECK_ARG(i_out && j_out && valid_out, "null pointer argument");
  ASOT_CHECK_ARG(n_dist >= 1, "n_dist must be >= 1");
  ASOT_CHECK_ARG(0 <= tile_begin && tile_begin <= tile_end && tile_end <= asot::num_tiles(n_dist),
                 "bad tile range");
  int64_t s = 0;
  for (int64_t t = tile_begin; t < tile_end; ++t)
    for (int lane = 0; lane < asot::kTileSlots; ++lane, ++s) {
      int i, j;
      valid_out[s] = asot::tile_slot_pair(t, lane, n_dist, i, j) ? 1 : 0;
      i_out[s] = i;
      j_out[s] = j;
    }
  return ASOT_OK;
}

asot_status asot_unpack_tiles(const float* packed, int64_t n_dist, int64_t tile_begin,
                              int64_t tile_end, float* dist_out, int32_t zero_diag, void* stream) {
  g_launches = 0;
  ASOT_CHECK_ARG(packed && dist_out, "null pointer argument");
  ASOT_CHECK_ARG(n_dist >= 1, "n_dist must be >= 1");
  ASOT_CHECK_ARG(0 <= tile_begin && tile_begin <= tile_end && tile_end <= asot::num_tiles(n_dist),
                 "bad tile range");
  cudaStream_t s = (cudaStream_t)stream;
  ASOT_LAUNCH(asot::launch_unpack_tiles(packed, n_dist, tile_begin, tile_end, dist_out, s));
  if (zero_diag) ASOT_LAUNCH(asot::launch_zero_diag(dist_out, n_dist, s));
  return ASOT_OK;
}

}  // extern "C"
