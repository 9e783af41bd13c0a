/*
 * asot.h -- C ABI of the B200-native ASOT pairwise-distance library (libasot.so).
 *
 * The hot path of Anchor Space Optimal Transport (arXiv 2310.16123, PAPER.md):
 *   a1  Gibbs kernel      K := exp(-C_s / eps)
 *   a2  mapping P_o       j*(p) = argmin_j ||x_p - w_j||^2, lowest j
 *   a3  mapped marginals  a' = Z^T a (one-hot => histogram; 1/n dropped) P:100
 *   a4  pair set          all i < j (Def. 1, i != j), upper-triangular tiles
 *   a5  batched Sinkhorn  U = A / (K V), V = B / (K^T U), v0 = 1, exactly L iterations
 *   a6  cost              d_ij = <diag(u) K diag(v), C_s> = u^T ((K (.) C_s) v), mirrored,
 *                         zero diagonal
 * Readings of the paper where it is silent or garbled are listed in DESIGN.md ("Readings").
 *
 * Conventions (all entry points):
 *   - Every buffer is caller-owned.  Pointers documented "device" must be device memory of the
 *     current CUDA device; "host" pointers are ordinary host memory (pinned recommended).
 *   - The library keeps no global device state and never allocates device memory: scratch
 *     space is the caller's `workspace` (device, 256-byte aligned), sized by the matching
 *     *_workspace_bytes query.
 *   - Calls only ENQUEUE work on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *     default stream) and return without synchronising, except the *_host variant, which
 *     synchronises `stream` before returning.
 *   - Host-checkable argument errors return synchronously (status codes below) and enqueue
 *     nothing.  Data-dependent conditions are OR-ed by the kernels into the caller's device
 *     word `status` (ASOT_FLAG_* bits); the caller reads it after synchronising.
 *   - asot_last_error() returns a thread-local message for the last non-OK return.
 *   - Floating point: inputs are fp32.  Mapping decisions are taken in fp64 wherever fp32
 *     cannot decide them (bit-exact against the fp64 definition); histograms are accumulated in
 *     fp64 in point order and rounded to fp32; Sinkhorn runs on tcgen05 tensor cores with fp32
 *     accumulation, either fp32-accurate (ASOT_PREC_FP32: 3xTF32 split operands, target 1e-4)
 *     or with one TF32 pass (ASOT_PREC_TF32, target 2e-3); K < 32 runs in fp32 on CUDA cores
 *     (one lane per anchor) for both requests; and when every histogram row has at most 16
 *     non-zero bins (K >= 64) the calls run the exact recurrence on each pair's support block
 *     in fp32 on CUDA cores for both requests (R#36, asot_sinkhorn_path_kind).
 *
 * Beyond the hot path: soft mappings ASOT-ML / ASOT-DL (NEXT-1), mini-batch
 * k-means anchors (NEXT-2), exact anchor-space OT per pair (NEXT-3), entropic OT on the original
 * point sets as the comparison baseline (NEXT-4), and a multi-GPU broadcast form of the mapping.
 */
#ifndef ASOT_H_
#define ASOT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASOT_ABI_VERSION 1

typedef enum {
  ASOT_OK = 0,
  ASOT_ERR_INVALID_ARGUMENT = 1, /* null pointer, size < 1, eps <= 0 / non-finite, iters < 1,
                                    max(C_s)/eps > 80 (fp32 Gibbs underflow guard), bad range */
  ASOT_ERR_INFEASIBLE_MASS = 2,  /* reserved for callers mapping ASOT_FLAG_EMPTY_DIST/BAD_MASS */
  ASOT_ERR_NUMERIC = 3,          /* reserved for callers mapping ASOT_FLAG_NONFINITE_* */
  ASOT_ERR_CUDA = 4,             /* a CUDA runtime call or launch failed (message in last_error) */
  ASOT_ERR_UNSUPPORTED = 5,      /* size outside what this build implements (e.g. K > 1024) */
  ASOT_ERR_WORKSPACE = 6         /* workspace NULL or smaller than the query returned */
} asot_status;

typedef enum {
  ASOT_PREC_FP32 = 0, /* fp32-accurate: 3xTF32 tcgen05 for 32 <= K <= 128 and 256 < K <= 1024,
                         BF16x3 tcgen05 for 128 < K <= 256 (tile path), fp32 CUDA cores
                         (lane per anchor) for K < 32; target rel. err <= 1e-4              */
  ASOT_PREC_TF32 = 1  /* tcgen05 kind::tf32 MMA (RNA-rounded G and U/V, fp32 accumulate):
                         target rel. err <= 2e-3; 32 <= K <= 1024 runs on tcgen05
                         (resident kernels for K <= 256, streamed above); K < 32 runs in
                         fp32 (TF32 rounding of u/v over < 32 terms can exceed 2e-3;
                         reported by asot_effective_precision)                              */
} asot_precision;

/* Bits OR-ed into the caller's device status word. */
#define ASOT_FLAG_EMPTY_DIST       1u  /* a distribution with n_i = 0 (S:24 requires n >= 1)      */
#define ASOT_FLAG_BAD_MASS         2u  /* negative weight or |sum w - 1| > 1e-5 (fp32)     */
#define ASOT_FLAG_NONFINITE_INPUT  4u  /* NaN/Inf in points, weights or anchors                  */
#define ASOT_FLAG_DENOM_CLAMPED    8u  /* a Sinkhorn denominator on an anchor with mass left
                                          [FLT_MIN, 2^126] and was clamped into it (
                                          a warning: the distance is that of the clamped run) */
#define ASOT_FLAG_NONFINITE_OUTPUT 16u /* a distance came out NaN/Inf                            */
#define ASOT_FLAG_SOFT_FALLBACK    32u /* a soft code was all zero -> uniform row (warning) */
#define ASOT_FLAG_EXACT_TOO_LARGE  64u /* asot_exact_w1_points: a support above 64 points (NaN out);
                                          exact ASOT itself solves every support              */
#define ASOT_FLAG_BAD_INDEX       128u /* an explicit pair-list entry had i or j outside [0, n_dist):
                                          its output is NaN (asot_pairwise_sinkhorn)             */

/* Distance-matrix tiling (step a4).  Distributions are grouped in blocks of 16; block pairs
 * (bi <= bj) are enumerated row-major over the upper triangle of the block grid; each block
 * pair is two tiles of 8 x 16 = 128 pair slots (tile 2b+h holds rows 16bi+8h .. +7 against
 * columns 16bj .. +15).  Slot `lane` of a tile is the pair (i, j) = (16bi+8h+lane/16,
 * 16bj+lane%16), valid iff i < j < N.  Multi-GPU callers split [0, asot_num_tiles(N)). */
#define ASOT_TILE_SLOTS 128
int64_t asot_num_tiles(int64_t n_dist);

/* Step a2 + a3: one-hot nearest-anchor mapping and the N x K mapped-marginal histograms.
 *   points   [T, dim] f32 row-major, device;  T = offsets[n_dist] (read from host copy below)
 *   offsets  [n_dist+1] i64, device, offsets[0] = 0, non-decreasing
 *   offsets_host  the same array in host memory (sizes are needed for launch shapes)
 *   weights  [T] f32, device; per distribution >= 0 and summing to 1 +- 1e-5 (not renormalised)
 *   anchors  [n_anchors, dim] f32 row-major, device; 1 <= n_anchors <= 1024, 1 <= dim <= 128
 *   assign_out [T] i32, device: j*(p) (bit-exact vs the fp64 definition, lowest index on ties)
 *   hist_out [n_dist, n_anchors] f32 row-major, device: H[i, j] = sum of w_p over points p of
 *            distribution i with j*(p) = j, accumulated in fp64 in point order, rounded to f32
 *   status   device u32, OR-ed with ASOT_FLAG_EMPTY_DIST / BAD_MASS / NONFINITE_INPUT */
asot_status asot_map_to_anchors(const float* points, const int64_t* offsets,
                                const int64_t* offsets_host, const float* weights,
                                int64_t n_dist, int32_t dim, const float* anchors,
                                int32_t n_anchors, int32_t* assign_out, float* hist_out,
                                uint32_t* status, void* stream);

/* Multi-GPU form of asot_map_to_anchors: additionally stores every histogram row i of this
 * call into each of the n_peers full [N_total, n_anchors] matrices hist_peers[d] (a device array
 * of device pointers -- e.g. every rank's symmetric-memory H, so the rows travel as NVLink stores
 * and the all-gather of H is fused into the histogram kernel) at row row_base + i.  The caller
 * synchronises and barriers before reading the peers' matrices. */
asot_status asot_map_to_anchors_bcast(const float* points, const int64_t* offsets,
                                      const int64_t* offsets_host, const float* weights,
                                      int64_t n_dist, int32_t dim, const float* anchors,
                                      int32_t n_anchors, int32_t* assign_out, float* hist_out,
                                      float* const* hist_peers, int32_t n_peers, int64_t row_base,
                                      uint32_t* status, void* stream);

/* Workspace form of the two calls above (a2 + a3): with the caller's
 * device workspace the score products x.w_j run on the tensor cores (3xTF32 tcgen05) and only the
 * points whose two best scores lie within the rigorous error bound go through the exact kernel
 * (DESIGN R#37), so assign_out and hist_out are bit-identical to asot_map_to_anchors.  The
 * tensor-core pass needs dim in {32, 64, 128}, n_anchors a multiple of 64 and points 16-byte
 * aligned; other shapes run the exact kernel on every point (the workspace is still required).
 * hist_peers / n_peers / row_base as in asot_map_to_anchors_bcast (n_peers = 0: no peer stores).
 * workspace: device, 256-byte aligned, >= asot_map_workspace_bytes(offsets_host[n_dist],
 * n_anchors) bytes, owned by the caller, free for reuse once the stream has passed the call;
 * too small / misaligned -> ASOT_ERR_WORKSPACE, nothing launched. */
size_t asot_map_workspace_bytes(int64_t n_points, int32_t n_anchors);
asot_status asot_map_to_anchors_ws(const float* points, const int64_t* offsets,
                                   const int64_t* offsets_host, const float* weights,
                                   int64_t n_dist, int32_t dim, const float* anchors,
                                   int32_t n_anchors, int32_t* assign_out, float* hist_out,
                                   float* const* hist_peers, int32_t n_peers, int64_t row_base,
                                   uint32_t* status, void* workspace, size_t workspace_bytes,
                                   void* stream);

/* Steps a1 + a5 + a6 on an explicit pair list (SPEC batched_sinkhorn_fixed).
 * 32 <= K <= 128: the resident 1-SM tcgen05 kernels in pair-list mode (ASOT_PREC_TF32: TF32;
 * ASOT_PREC_FP32: 3xTF32), bitwise the values of the tile path; K < 32: the fp32 lane-per-anchor
 * kernel (the tile path's kernel, which takes pair lists natively); K > 128:
 * the streamed tcgen05 kernel in pair-list mode (TF32: one pass; FP32: 3xTF32).  All take tiles
 * of 128 consecutive list entries and read each entry's marginal rows from a padded copy of H in
 * the workspace (L2-resident).  (Environment ASOT_PAIR_KERNEL=simt selects the fp32 CUDA-core
 * kernel instead, for cross-checks.)  Invalid entries (an index outside [0, n_dist)) give NaN
 * and raise ASOT_FLAG_BAD_INDEX.  n_pairs = 0 returns ASOT_OK at once (pair_i, pair_j and
 * dist_out may then be NULL).  Workspace: asot_pairwise_workspace_bytes(n_dist, n_anchors, prec)
 * runs the list as it is; the larger asot_pairwise_list_workspace_bytes(n_dist, n_anchors, prec,
 * n_pairs) lets requests with 32 <= K <= 256 (n_pairs >= 1024, n_dist <= ~2.9e4) serve every
 * tile of the upper triangle whose 8 x 16 block of i < j pairs the list covers COMPLETELY through
 * the tile kernels (marginal rows staged in SMEM once per tile; asot_pairs_bucket.cu), the other
 * entries (i >= j, repeats, partly covered tiles, invalid indices) through the pair-list mode --
 * stream-ordered, no host synchronisation; the values are those of the tile path (K <= 128:
 * bitwise the pair-list mode's; 128 < K <= 256: another kernel -- TF32: the CTA-pair kernel,
 * FP32: the BF16x3 one -- within the precision's tolerance, like the pair-list mode's).
 * (ASOT_PAIR_BUCKET=0 disables it.)  Status: the call's flags are OR-ed into ONE word for the whole list (DESIGN R#33:
 * no per-pair flag array; a flagged run is re-run on a sub-list to locate pairs).  Arguments:
 *   hist     [n_dist, n_anchors] f32 device (rows are a' / b')
 *   cost     [n_anchors, n_anchors] f32 device: C_s symmetric, >= 0, zero diagonal
 *   eps > 0 (max(C_s)/eps <= 80 is checked against cost_max, a host value the caller supplies:
 *            the library does not read device memory synchronously), iters >= 1
 *   pair_i, pair_j [n_pairs] i32 device, 0 <= i, j < n_dist (i != j expected, not required)
 *   dist_out [n_pairs] f32 device: d(pair_i[p], pair_j[p]) with a = H[pair_i] on the u side */
asot_status asot_pairwise_sinkhorn(const float* hist, int64_t n_dist, int32_t n_anchors,
                                   const float* cost, float cost_max, float eps, int32_t iters,
                                   asot_precision prec, const int32_t* pair_i,
                                   const int32_t* pair_j, int64_t n_pairs, float* dist_out,
                                   uint32_t* status, void* workspace, size_t workspace_bytes,
                                   void* stream);
size_t asot_pairwise_workspace_bytes(int64_t n_dist, int32_t n_anchors, asot_precision prec);
size_t asot_pairwise_list_workspace_bytes(int64_t n_dist, int32_t n_anchors, asot_precision prec,
                                          int64_t n_pairs);

/* Full pipeline a1-a6 on the tile range [tile_begin, tile_end) (device buffers):
 *   hist_in  NULL: map + histogram all distributions into the workspace first (needs points,
 *            offsets, offsets_host, weights, anchors, dim); non-NULL: use this [n_dist,
 *            n_anchors] histogram (multi-GPU passes the all-gathered H) and skip mapping
 *   dist_out [n_dist, n_dist] f32 or NULL: D[i,j] = D[j,i] = d_ij for the range's pairs; when
 *            the range is the whole triangle the diagonal is set to 0 as well
 *   packed_out [(tile_end - tile_begin) * 128] f32 or NULL: slot-ordered results (0 for
 *            invalid slots) -- the unit multi-GPU ranks gather
 *   assign_out [T] i32 or NULL, hist_out [n_dist, n_anchors] f32 or NULL: optional copies of
 *            the mapping results (only when hist_in == NULL) */
asot_status asot_distance_matrix(const float* points, const int64_t* offsets,
                                 const int64_t* offsets_host, const float* weights,
                                 int64_t n_dist, int32_t dim, const float* anchors,
                                 int32_t n_anchors, const float* cost, float cost_max, float eps,
                                 int32_t iters, asot_precision prec, const float* hist_in,
                                 int64_t tile_begin, int64_t tile_end, float* dist_out,
                                 float* packed_out, int32_t* assign_out, float* hist_out,
                                 uint32_t* status, void* workspace, size_t workspace_bytes,
                                 void* stream);
size_t asot_distance_matrix_workspace_bytes(int64_t n_dist, int64_t n_points, int32_t n_anchors,
                                            asot_precision prec);

/* Steps a1, a5, a6 on part [part_begin, part_end) of the pair enumeration the call picks (the
 * multi-GPU unit when results go straight into one matrix): on the small-support path (R#36)
 * the tiles of the distributions ordered by support size -- homogeneous warps, as the whole
 * triangle runs there -- otherwise the a4 tiles, exactly as asot_distance_matrix's tile range.
 * Either way a partition of [0, asot_num_tiles(n_dist)) over calls with the same hist covers
 * every pair i < j exactly once (each pair keeps its orientation, R#10).  hist [n_dist,
 * n_anchors] f32 device (e.g. the all-gathered H); dist_out [n_dist, n_dist] f32 device (may be
 * a peer GPU's memory): D[i,j] = D[j,i] for the part's pairs, the diagonal zeroed when the part
 * is the whole range.  Workspace: asot_distance_matrix_workspace_bytes(n_dist, 0, n_anchors,
 * prec). */
asot_status asot_distance_matrix_partition(const float* hist, int64_t n_dist, int32_t n_anchors,
                                           const float* cost, float cost_max, float eps, int32_t iters,
                                           asot_precision prec, int64_t part_begin, int64_t part_end,
                                           float* dist_out, uint32_t* status, void* workspace,
                                           size_t workspace_bytes, void* stream);

/* Same pipeline end to end from HOST buffers (the e2e entry point): copies points, offsets,
 * weights, anchors and cost host->device on `stream`, runs the whole triangle, copies the
 * N x N matrix (and status) back to `dist_host` / `status_host`, and synchronises `stream`.
 * All scratch (inputs, H, G images, D) lives in the caller's device `workspace`. */
asot_status asot_distance_matrix_host(const float* points_host, const int64_t* offsets_host,
                                      const float* weights_host, int64_t n_dist, int32_t dim,
                                      const float* anchors_host, int32_t n_anchors,
                                      const float* cost_host, float eps, int32_t iters,
                                      asot_precision prec, float* dist_host,
                                      uint32_t* status_host, void* workspace,
                                      size_t workspace_bytes, void* stream);
size_t asot_distance_matrix_host_workspace_bytes(int64_t n_dist, int64_t n_points, int32_t dim,
                                                 int32_t n_anchors, asot_precision prec);

/* KN6: scatter packed tile results [(tile_end - tile_begin) * 128] into the N x N matrix
 * (both triangles).  Zeroes the diagonal when zero_diag != 0. */
asot_status asot_unpack_tiles(const float* packed, int64_t n_dist, int64_t tile_begin,
                              int64_t tile_end, float* dist_out, int32_t zero_diag, void* stream);

/* Host-side enumeration of tile slots (no device work): for s in [0, (tile_end-tile_begin)*128)
 * writes pair (i_out[s], j_out[s]) and valid_out[s] (1 iff i < j < n_dist).  Host pointers. */
asot_status asot_tile_pairs_host(int64_t n_dist, int64_t tile_begin, int64_t tile_end,
                                 int32_t* i_out, int32_t* j_out, uint8_t* valid_out);

/* ---- soft / near-one-hot mappings (inference; parameters are inputs) ----
 * Both compute a code z_p on the simplex for every point and the mapped marginals
 * H[i, :] = sum_{p in i} w_p z_p (Eq. (5), 1/n dropped: R#1), accumulated in fp64 in point
 * order and rounded to f32 -- the same [n_dist, n_anchors] layout asot_distance_matrix takes as
 * hist_in.  points / offsets / offsets_host / weights / status as in asot_map_to_anchors;
 * 1 <= dim <= 128, 1 <= n_anchors <= 1024, 1 <= hidden <= 256.  codes_out [T, n_anchors] f32 or
 * NULL receives every z_p.  An all-zero code falls back to the uniform row 1/K and ORs
 * ASOT_FLAG_SOFT_FALLBACK.  All pointers are device pointers owned by the caller.
 *
 * ASOT-ML (Table 4): z = |o| / ||o||_1, o = relu(x W1 + b1) W2 + b2 with
 *   W1 [dim, hidden], b1 [hidden], W2 [hidden, n_anchors], b2 [n_anchors] (row-major f32). */
asot_status asot_map_soft_ml(const float* points, const int64_t* offsets,
                             const int64_t* offsets_host, const float* weights, int64_t n_dist,
                             int32_t dim, int32_t n_anchors, int32_t hidden, const float* W1,
                             const float* b1, const float* W2, const float* b2, float* hist_out,
                             float* codes_out, uint32_t* status, void* workspace,
                             size_t workspace_bytes, void* stream);
/* Device workspace for asot_map_soft_ml: dim in {32, 64, 128} (points 16-byte aligned), hidden a
 * multiple of 64 up to 256 and n_anchors a multiple of 64 in [64, 1024] run both MLP layers on
 * the tensor cores (asot_soft_ml_tc.cu: tcgen05 kind::f16 with BF16 hi + lo split operands,
 * three MMAs per k-step; R#35), which keep their split weight images (BF16 hi + lo of W1 and
 * W2, 4 (dim' hidden + hidden n_anchors) bytes, dim' = dim rounded up to 64) here; 0 for other
 * shapes.  A smaller workspace (or NULL) selects the CUDA-core kernel. */
size_t asot_map_soft_ml_workspace_bytes(int32_t dim, int32_t hidden, int32_t n_anchors);

/* ASOT-DL near-one-hot encoder (Eqs. (8)(9); appendix; Table 4):
 *   lambda_p = softplus(relu(x V1 + c1) . v2 + c2[0]); z^(0) = 0; n_layers times
 *   z <- max(0, z - W^T (W z - x) - lambda_p) with W = dictionary^T (dictionary [n_anchors, dim]
 *   row-major: row u = anchor w_u); finally z / sum(z).  Step size 1 presumes
 *   ||W||_2 <= 1 (R#28); the library does not rescale.  V1 [dim, hidden], c1 [hidden],
 *   v2 [hidden], c2 [1]; n_layers >= 1. */
asot_status asot_map_soft_dl(const float* points, const int64_t* offsets,
                             const int64_t* offsets_host, const float* weights, int64_t n_dist,
                             int32_t dim, const float* dictionary, int32_t n_anchors,
                             int32_t n_layers, int32_t hidden, const float* V1, const float* c1,
                             const float* v2, const float* c2, float* hist_out, float* codes_out,
                             uint32_t* status, void* workspace, size_t workspace_bytes,
                             void* stream);
/* Device workspace for asot_map_soft_dl: dim in {64, 128} with 256 <= n_anchors <= 1024
 * (n_anchors % 64 == 0) runs the tensor-core encoder (asot_soft_dl_tc.cu: the dense product
 * g = W^T r on tcgen05 3xTF32, the sparse r = W z - x on CUDA cores), which keeps each CTA's tile
 * of codes in this scratch (#SMs x 128 x n_anchors floats, L2-resident) next to the split
 * dictionary images and lambda per point (n_points = offsets_host[n_dist]); 0 otherwise.  A smaller workspace (or NULL) selects the CUDA-core kernels. */
size_t asot_map_soft_dl_workspace_bytes(int32_t dim, int32_t n_anchors, int64_t n_points);

/* ASOT-ML anchor cost: C_s[u, v] = ||M w_u - M w_v||_2, M [h, dim] row-major, anchors
 * [n_anchors, dim]; bitwise symmetric, zero diagonal.  normalize != 0 divides by the max entry
 * (R#29; the max becomes exactly 1).  cost_out [n_anchors, n_anchors] f32 device; workspace of
 * asot_mahalanobis_workspace_bytes(n_anchors, h) device bytes. */
asot_status asot_mahalanobis_cost(const float* anchors, int32_t n_anchors, int32_t dim,
                                  const float* M, int32_t h, int32_t normalize, float* cost_out,
                                  void* workspace, size_t workspace_bytes, void* stream);
size_t asot_mahalanobis_workspace_bytes(int32_t n_anchors, int32_t h);

/* ---- ASOT-k anchor learning (mini-batch k-means; Table 4) ----
 * Runs `iters` iterations; iteration t uses the `batch` point indices batch_idx[t * batch ...]
 * (device i64, 0 <= idx < n_points; the random draws are inputs):
 *   assignment j*(x) against the f32 anchors (bit-exact vs the fp64 definition, lowest index on
 *   ties, R#8); per-center batch sums in batch order in fp64; c_j <- (v_j c_j + S_j) / (v_j + m_j),
 *   v_j <- v_j + m_j (Sculley's 1/v learning rate, R#31) in explicitly rounded fp64.
 *   points     [n_points, dim] f32 device
 *   centers    [n_anchors, dim] f64 device, in/out (initial centers in, learned centers out)
 *   counts     [n_anchors] i64 device, in/out (0 for a fresh run)
 *   anchors_out [n_anchors, dim] f32 device: the f32 copy of the centers (what P_o then uses)
 *   assign_ws  [batch] i32 device scratch; status as in asot_map_to_anchors.
 * Centers and counts are bit-identical to the oracle's for the same inputs. */
asot_status asot_kmeans_minibatch(const float* points, int64_t n_points, int32_t dim,
                                  int32_t n_anchors, const int64_t* batch_idx, int32_t batch,
                                  int32_t iters, double* centers, int64_t* counts,
                                  float* anchors_out, int32_t* assign_ws, uint32_t* status,
                                  void* stream);

/* Squared-Euclidean anchor cost of (learned) anchors: C_s[u, v] = ||w_u - w_v||^2 in fp32
 * (bitwise symmetric, zero diagonal), divided by its max when normalize != 0 (R#7). */
asot_status asot_sqeuclid_cost(const float* anchors, int32_t n_anchors, int32_t dim,
                               int32_t normalize, float* cost_out, void* stream);

/* ---- comparison baseline -- entropic OT on the ORIGINAL point sets ----
 * For each pair p: C[r][c] = cost_scale * ||x_r - y_c||^2 over the n_i x n_j points of
 * distributions i = pair_i[p], j = pair_j[p] (device i32), K = exp(-C / eps), v0 = 1, exactly
 * `iters` Sinkhorn iterations with a = w_i, b = w_j, dist_out[p] = <diag(u) K diag(v), C>
 * (fp32 arithmetic, fp64 final reduction).  This is the per-pair cost instantiation ASOT avoids
 * (Table 2 eOT / BDS-eOT rows P:333-334).  Every distribution must have
 * n_i <= 16384 points.  Denominators below FLT_MIN are clamped and flagged (DENOM_CLAMPED).
 * workspace: asot_eot_workspace_bytes(n_dist, offsets_host, n_pairs) device bytes (per-CTA slots
 * for kernels larger than the 160 KB kept in shared memory). */
asot_status asot_eot_pairs(const float* points, const int64_t* offsets, const int64_t* offsets_host,
                           const float* weights, int64_t n_dist, int32_t dim, float cost_scale,
                           float eps, int32_t iters, const int32_t* pair_i, const int32_t* pair_j,
                           int64_t n_pairs, float* dist_out, uint32_t* status, void* workspace,
                           size_t workspace_bytes, void* stream);
size_t asot_eot_workspace_bytes(int64_t n_dist, const int64_t* offsets_host, int64_t n_pairs);

/* ---- EXACT anchor-space OT per pair (Def. 3 / Eq. (4)) ----
 * dist_out[p] = min <T, C_s> over T in U(a', b'), a' = hist[pair_i[p]], b' = hist[pair_j[p]]
 * renormalised to unit mass in fp64 (R#14), solved exactly (successive-shortest-path min-cost flow
 * on the two histogram supports, fp64) -- the eps -> 0 limit of asot_pairwise_sinkhorn.  Supports
 * of up to 128 bins per side run one warp per pair, larger ones (n_anchors > 128) one CTA per
 * pair with the flow matrix in the workspace.  Invalid indices or an empty support give NaN.
 * hist [n_dist, n_anchors] f32, cost [n_anchors, n_anchors] f32, pair_i / pair_j [n_pairs] i32,
 * dist_out [n_pairs] f64: device pointers; workspace: asot_exact_asot_workspace_bytes(n_pairs,
 * n_anchors) device bytes (n_pairs flags, plus #SMs x n_anchors^2 f64 when n_anchors > 128). */
size_t asot_exact_asot_workspace_bytes(int64_t n_pairs, int32_t n_anchors);
asot_status asot_exact_asot_pairs(const float* hist, int64_t n_dist, int32_t n_anchors, const float* cost,
                                  const int32_t* pair_i, const int32_t* pair_j, int64_t n_pairs,
                                  double* dist_out, uint32_t* status, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* ---- NEXT-3 bound checks at scale: the paper's guarantees per pair ------------
 * asot_exact_w1_points: EXACT W_1 on the ORIGINAL point sets (Eq. (1)) with the Euclidean
 * ground metric of Prop. 2 (R#7): dist_out[p] = min <T, C> over T in U(a, b), C(r, c) =
 * ||x_r - y_c||_2 in fp64 from the f32 points, a / b = the point weights of distributions
 * pair_i[p] / pair_j[p] renormalised in fp64 (R#14); successive-shortest-path min-cost flow on the
 * supports (points with weight > 0), one warp per pair, supports of up to 64 points per side
 * (graph-sized distributions, c1 / c2).  Larger supports: NaN and ASOT_FLAG_EXACT_TOO_LARGE;
 * invalid indices: NaN and ASOT_FLAG_BAD_INDEX.  points [T, dim] f32, offsets [n_dist+1] i64,
 * weights [T] f32, pair_i / pair_j [n_pairs] i32, dist_out [n_pairs] f64: device pointers.
 *
 * asot_bound_terms: per pair the right-hand sides of Prop. 1 (Eq. (7)) and
 * Prop. 2 for the one-hot mapping P_o:
 *   prop1_l1[p]   = sum_{r,c} |C_hat(r, c) - C(r, c)|, C_hat(r, c) = cost[u_r][v_c] (Z_x C_s Z_y^T
 *                   for one-hot Z), C(r, c) = ||x_r - y_c||_2;
 *   prop1_max[p]  = max_{r,c} |C_hat(r, c) - C(r, c)| (the tighter bound the proof gives, R#16);
 *   prop2[p]      = m sum_r ||w_{u_r} - x_r||_2 + n sum_c ||w_{v_c} - y_c||_2 (n, m = point counts).
 * u = assign (the mapping's output, asot_map_to_anchors), cost = the C_s the caller's W_AS used
 * (Euclidean anchor distances for Prop. 2: asot_mahalanobis_cost with M = I, normalize = 0).
 * All terms accumulate in fp64.  anchors [n_anchors, dim] f32, assign [T] i32, cost
 * [n_anchors, n_anchors] f32, outputs [n_pairs] f64: device pointers.  One CTA per pair. */
asot_status asot_exact_w1_points(const float* points, const int64_t* offsets, const float* weights,
                                 int64_t n_dist, int32_t dim, const int32_t* pair_i,
                                 const int32_t* pair_j, int64_t n_pairs, double* dist_out,
                                 uint32_t* status, void* stream);
asot_status asot_bound_terms(const float* points, const int64_t* offsets, int64_t n_dist, int32_t dim,
                             const float* anchors, int32_t n_anchors, const int32_t* assign,
                             const float* cost, const int32_t* pair_i, const int32_t* pair_j,
                             int64_t n_pairs, double* prop1_l1, double* prop1_max, double* prop2,
                             uint32_t* status, void* stream);

/* Precision actually used for a given K and request (TF32 covers 32 <= K <= 1024). */
asot_precision asot_effective_precision(int32_t n_anchors, asot_precision requested);

/* Which Sinkhorn kernel asot_distance_matrix runs for (K, request): 0 = fp32 CUDA-core kernel,
 * 1 = TF32 1-SM resident (K <= 128), 2 = TF32 CTA pair (K <= 256), 3 = 3xTF32 fp32-accurate
 * 1-SM resident (ASOT_PREC_FP32 with 32 <= K <= 128), 4 = TF32 CTA-pair
 * streamed (256 < K <= 1024, K padded to 512 or 1024),
 * 5 = 3xTF32 fp32-accurate CTA-pair streamed (ASOT_PREC_FP32, 256 < K <= 1024),
 * 9 = fp32 lane-per-anchor CUDA-core kernel (every request with K < 32),
 * 10 = BF16x3 fp32-accurate CTA-pair resident (ASOT_PREC_FP32, 128 < K <= 256).
 * (Pair lists: K <= 128 the 1-SM kernels' pair-list modes, else the streamed kernel's.) */
int32_t asot_sinkhorn_kernel_kind(int32_t n_anchors, asot_precision requested);
/* The kernel a distance-matrix / pair-list call runs once the histograms are known: 11 = the
 * small-support fp32 kernel (asot_sinkhorn_sparse.cu, DESIGN R#36) when n_anchors >= 64 and every
 * histogram row has at most 16 non-zero bins (max_support = the largest count of non-zero bins
 * in a row), for both precision requests; otherwise asot_sinkhorn_kernel_kind.  The calls take
 * this decision on the device (no host synchronisation); this host function states the rule.
 * Environment ASOT_SPARSE=0 (diagnostic) disables the small-support kernel. */
int32_t asot_sinkhorn_path_kind(int32_t n_anchors, asot_precision requested, int32_t max_support);

/* Optional kernel timing (bench.py's roofline): while enabled on this thread, the library records
 * a CUDA event pair on the launch stream immediately around every Sinkhorn kernel launch
 * (ASOT_PROF_SINKHORN, steps a5+a6) and every mapping kernel launch (ASOT_PROF_MAP, step a2).
 * asot_profile_read_kernel synchronises on the recorded events of one kernel and returns the
 * summed kernel milliseconds and launch count since its last reset; asot_profile_read is the
 * Sinkhorn shorthand.  Host-side only; never on by default. */
#define ASOT_PROF_SINKHORN 0
#define ASOT_PROF_MAP 1
asot_status asot_profile_enable(int32_t on);
asot_status asot_profile_read_kernel(int32_t which, double* ms_out, int64_t* launches, int32_t reset);
asot_status asot_profile_read(double* sinkhorn_ms, int64_t* launches, int32_t reset);
/* Effective SM clock (MHz) of the most recent launch of tensor-core Sinkhorn kernel `kind`
 * (asot_sinkhorn_kernel_kind's numbering, 1..8): CTA 0 records %clock64 and %globaltimer after
 * its setup and at its end, and the clock is their ratio -- the clock the kernel ran at under
 * power capping, for the roofline's nominal peak at clock.  Synchronises the device.
 * ASOT_ERR_INVALID_ARGUMENT for kind 0 (CUDA cores) or a kind not launched yet. */
asot_status asot_profile_clock(int32_t kind, double* sm_mhz);

/* Number of kernel launches the last distance_matrix / pairwise call on this thread issued. */
int32_t asot_last_launch_count(void);

const char* asot_last_error(void);
int32_t asot_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ASOT_H_ */
