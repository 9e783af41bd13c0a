// asot_pairs_bucket.cu -- explicit pair lists (asot_pairwise_sinkhorn; SPEC batched_sinkhorn_fixed,
// S:114-122) served by the tile kernels where the list covers whole tiles.
//
// Step a4 enumerates the upper triangle in tiles of 8 x 16 pairs (asot_internal.cuh): a tile
// stages its 24 marginal rows in SMEM once, where the pair-list mode reads two rows per pair from
// L2.  Here each list entry with i < j is put in the tile it falls in (one bit per slot, atomicOr);
// every unit -- a tile for the 1-SM kernels, a block pair (two tiles) for the CTA-pair kernels --
// whose valid slots are ALL present runs through the tile path into a compact buffer R, and its
// entries are gathered from R into list order.  Every other entry (i > j, i == j, a repeat of an
// entry already counted, an index outside [0, n_dist), a partly covered tile) is compacted into a
// sub-list that runs through the pair-list mode, its results stored at their list positions
// (PairSink::idx).  The unit and sub-list counts never leave the device: the kernels read them
// (PairSource::n_dev), so the call stays asynchronous.
//
// Results: the tile path and the pair-list mode evaluate the same per-pair recurrence (bitwise
// the same at K <= 128, where both are the 1-SM kernel; tc2 vs the streamed kernel's one-pass
// mode at 128 < K <= 256, each within the TF32 tolerance of the oracle).
#include "asot_internal.cuh"

namespace asot {
namespace pb {

// tile of pair (i, j), i < j, and its slot: the inverse of tile_slot_pair
__device__ __forceinline__ int64_t tile_of(int i, int j, int64_t nb, int& slot) {
  const int64_t bi = i / kBlockDist, bj = j / kBlockDist;
  const int h = (i % kBlockDist) >> 3;
  const int64_t b = bi * nb - bi * (bi - 1) / 2 + (bj - bi);   // row-major over bi <= bj
  slot = ((i & 7) << 4) | (j % kBlockDist);
  return 2 * b + h;
}

// pass 1: one bit per (tile, slot) present; code[s] = tile, or -1 (not tile-servable or a repeat)
__global__ void mark_kernel(const int32_t* __restrict__ pi, const int32_t* __restrict__ pj, int64_t n,
                            int64_t n_dist, uint32_t* __restrict__ mask, int32_t* __restrict__ code) {
  const int64_t nb = num_blocks(n_dist);
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const int i = pi[s], j = pj[s];
    int32_t c = -1;
    if (i >= 0 && i < j && j < n_dist) {
      int slot;
      const int64_t t = tile_of(i, j, nb, slot);
      const uint32_t bit = 1u << (slot & 31);
      if (!(atomicOr(&mask[4 * t + (slot >> 5)], bit) & bit)) c = (int32_t)t;
    }
    code[s] = c;
  }
}

// number of valid slots (i < j < n) of tile t
__device__ __forceinline__ int tile_valid_slots(int64_t t, int64_t n_dist) {
  int64_t bi, bj;
  block_pair_decode(t >> 1, num_blocks(n_dist), bi, bj);
  const int64_t i0 = bi * kBlockDist + (t & 1) * 8, j0 = bj * kBlockDist;
  const int64_t jhi = j0 + kBlockDist < n_dist ? j0 + kBlockDist : n_dist;
  int c = 0;
  for (int r = 0; r < 8; ++r) {
    const int64_t lo = i0 + r + 1 > j0 ? i0 + r + 1 : j0;
    if (jhi > lo) c += (int)(jhi - lo);
  }
  return c;
}

// pass 2: units whose valid slots are all present (and non-empty) get a position in R
__global__ void select_kernel(const uint32_t* __restrict__ mask, int64_t n_units, int upt, int64_t n_dist,
                              int64_t cap, int32_t* __restrict__ pos, int32_t* __restrict__ units,
                              unsigned long long* __restrict__ cnt) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n_units;
       u += (int64_t)gridDim.x * blockDim.x) {
    bool full = true;
    int have = 0;
    for (int h = 0; h < upt; ++h) {
      const int64_t t = u * upt + h;
      const int c = __popc(mask[4 * t]) + __popc(mask[4 * t + 1]) + __popc(mask[4 * t + 2]) + __popc(mask[4 * t + 3]);
      full &= c == tile_valid_slots(t, n_dist);
      have += c;
    }
    int32_t k = -1;
    if (full && have > 0) {
      const unsigned long long q = atomicAdd(&cnt[0], 1ull);
      if ((int64_t)q < cap) {
        k = (int32_t)q;
        units[k] = (int32_t)u;
      }
    }
    pos[u] = k;
  }
}

// pass 3: the entries no tile serves -> the sub-list (li, lj) with their list positions
__global__ void route_kernel(const int32_t* __restrict__ pi, const int32_t* __restrict__ pj, int64_t n,
                             const int32_t* __restrict__ code, const int32_t* __restrict__ pos, int upt,
                             int32_t* __restrict__ li, int32_t* __restrict__ lj, int32_t* __restrict__ lidx,
                             unsigned long long* __restrict__ cnt) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = code[s];
    if (c >= 0 && pos[c / upt] >= 0) continue;
    const unsigned long long k = atomicAdd(&cnt[1], 1ull);
    li[k] = pi[s];
    lj[k] = pj[s];
    lidx[k] = (int32_t)s;
  }
}

// pass 4 (after the tile run): tile-served entries take their slot of R
__global__ void gather_kernel(const int32_t* __restrict__ pi, const int32_t* __restrict__ pj, int64_t n,
                              int64_t n_dist, const int32_t* __restrict__ code, const int32_t* __restrict__ pos,
                              int upt, const float* __restrict__ R, float* __restrict__ dist) {
  const int64_t nb = num_blocks(n_dist);
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = code[s];
    if (c < 0) continue;
    const int32_t k = pos[c / upt];
    if (k < 0) continue;
    int slot;
    tile_of(pi[s], pj[s], nb, slot);
    dist[s] = R[((int64_t)k * upt + c % upt) * kTileSlots + slot];
  }
}

}  // namespace pb

// Capacity of R in units: a full unit consumes all its valid slots from the list, and only the
// O(nb) diagonal / last-column tiles have fewer than 16 of them.
int64_t pair_bucket_cap(int64_t n_dist, int64_t n_pairs, int upt) {
  const int64_t n_units = num_tiles(n_dist) / upt;
  const int64_t cap = n_pairs / 16 + 2 * num_blocks(n_dist) + 8;
  return cap < n_units ? cap : n_units;
}

// Usable when the per-tile bitmask stays small (<= 64 MB: n_dist up to ~2.9e4) and tiles fit int32.
bool pair_bucket_supported(int64_t n_dist) {
  return n_dist >= 2 && num_tiles(n_dist) <= ((int64_t)1 << 22);
}

size_t pair_bucket_bytes(int64_t n_dist, int64_t n_pairs, int upt) {
  const int64_t nt = num_tiles(n_dist), cap = pair_bucket_cap(n_dist, n_pairs, upt);
  size_t b = 0;
  auto take = [&](size_t x) { b += (x + 255) & ~(size_t)255; };
  take((size_t)nt * 16);              // mask
  take((size_t)(nt / upt) * 4);       // pos
  take(16);                           // counters
  take((size_t)cap * 4);              // units
  take((size_t)n_pairs * 4 * 4);      // code, li, lj, lidx
  take((size_t)cap * upt * kTileSlots * 4);   // R
  return b;
}

PairBuckets carve_pair_buckets(uint8_t* base, int64_t n_dist, int64_t n_pairs, int upt) {
  PairBuckets w;
  const int64_t nt = num_tiles(n_dist);
  w.upt = upt;
  w.n_units = nt / upt;
  w.cap = pair_bucket_cap(n_dist, n_pairs, upt);
  size_t off = 0;
  auto take = [&](size_t x) {
    uint8_t* p = base + off;
    off += (x + 255) & ~(size_t)255;
    return p;
  };
  w.mask = (uint32_t*)take((size_t)nt * 16);
  w.pos = (int32_t*)take((size_t)w.n_units * 4);
  w.cnt = (unsigned long long*)take(16);
  w.units = (int32_t*)take((size_t)w.cap * 4);
  w.code = (int32_t*)take((size_t)n_pairs * 4);
  w.li = (int32_t*)take((size_t)n_pairs * 4);
  w.lj = (int32_t*)take((size_t)n_pairs * 4);
  w.lidx = (int32_t*)take((size_t)n_pairs * 4);
  w.R = (float*)take((size_t)w.cap * upt * kTileSlots * 4);
  return w;
}

static int grid_for(int64_t n, int sms) {
  const int64_t g = (n + 255) / 256;
  return (int)(g < 8 * sms ? (g > 0 ? g : 1) : 8 * sms);
}

cudaError_t launch_pair_buckets(const PairBuckets& w, const int32_t* pi, const int32_t* pj, int64_t n_pairs,
                                int64_t n_dist, int sms, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(w.mask, 0, (size_t)w.n_units * w.upt * 16, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(w.cnt, 0, 16, s);
  if (e != cudaSuccess) return e;
  pb::mark_kernel<<<grid_for(n_pairs, sms), 256, 0, s>>>(pi, pj, n_pairs, n_dist, w.mask, w.code);
  pb::select_kernel<<<grid_for(w.n_units, sms), 256, 0, s>>>(w.mask, w.n_units, w.upt, n_dist, w.cap, w.pos,
                                                             w.units, w.cnt);
  pb::route_kernel<<<grid_for(n_pairs, sms), 256, 0, s>>>(pi, pj, n_pairs, w.code, w.pos, w.upt, w.li, w.lj,
                                                          w.lidx, w.cnt);
  return cudaGetLastError();
}

cudaError_t launch_pair_gather(const PairBuckets& w, const int32_t* pi, const int32_t* pj, int64_t n_pairs,
                               int64_t n_dist, float* dist, int sms, cudaStream_t s) {
  pb::gather_kernel<<<grid_for(n_pairs, sms), 256, 0, s>>>(pi, pj, n_pairs, n_dist, w.code, w.pos, w.upt, w.R,
                                                           dist);
  return cudaGetLastError();
}

}  // namespace asot
