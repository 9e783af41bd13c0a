// cg2_probe.cu -- verify tcgen05.mma.cta_group::2.kind::tf32 (A from TMEM) operand layouts:
//   A [256 x K]: CTA c's TMEM lane l holds row 128c + l (columns = k)
//   B [K x N] K-major SW128 image: CTA c's SMEM holds output columns [c N/2, (c+1) N/2)
//   D [256 x N]: CTA c's TMEM lane l holds row 128c + l, all N columns
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cg2_probe tools/cg2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

constexpr int KK = 32, NN = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__host__ __device__ inline uint32_t sw(uint32_t n, uint32_t k, uint32_t rows) {
  const uint32_t kb = k >> 5, kin = k & 31;
  const uint32_t lin = kb * rows * 128u + n * 128u + kin * 4u;
  return lin ^ (((lin >> 7) & 7u) << 4);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) uint8_t sm[NN / 2 * KK * 4];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B image: this CTA holds output columns [rank*64, rank*64+64), all K
  for (int e = threadIdx.x; e < NN / 2 * KK; e += blockDim.x) {
    const int n = e / KK, k = e % KK;
    const float v = B[(size_t)k * NN + rank * (NN / 2) + n];
    *(float*)(sm + sw(n, k, NN / 2)) = v;
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  asm volatile("fence.mbarrier_init.release.cluster;");
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = holder;
  // A: lane (32*warp + lane) row 128*rank + that, columns k
  {
    const int row = rank * 128 + warp * 32 + lane;
    uint32_t r[KK];
    for (int k = 0; k < KK; ++k) {
      uint32_t bits = __float_as_uint(A[(size_t)row * KK + k]);
      r[k] = bits;
    }
    const uint32_t ta = tb + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                 "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
                 "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
                 "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (rank == 0 && warp == 0 && lane == 0) {
    const uint32_t b0 = smem_u32(sm);
    for (int ks = 0; ks < KK / 8; ++ks) {
      const uint32_t b_addr = b0 + (uint32_t)((ks >> 2) * (NN / 2) * 128 + (ks & 3) * 32);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb + 256),
                   "r"(tb + 8 * ks), "l"(make_sw128_desc(b_addr)), "r"(idesc(256, NN)), "r"(ks > 0 ? 1 : 0));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)3));
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const int row = rank * 128 + warp * 32 + lane;
    const uint32_t td = tb + 256 + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < NN; c += 32) {
      uint32_t r[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                     "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                     "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(td + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int e = 0; e < 32; ++e) D[(size_t)row * NN + c + e] = __uint_as_float(r[e]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
  const int M = 256;
  float *hA = (float*)malloc(M * KK * 4), *hB = (float*)malloc(KK * NN * 4), *hD = (float*)malloc(M * NN * 4);
  srand(1);
  // values exactly representable in TF32 so the product is exact-ish
  for (int i = 0; i < M * KK; ++i) hA[i] = (float)((rand() % 17) - 8) / 8.0f;
  for (int i = 0; i < KK * NN; ++i) hB[i] = (float)((rand() % 13) - 6) / 4.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, M * KK * 4); cudaMalloc(&dB, KK * NN * 4); cudaMalloc(&dD, M * NN * 4);
  cudaMemcpy(dA, hA, M * KK * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, KK * NN * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * NN * 4);
  probe<<<2, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(hD, dD, M * NN * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0; int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NN; ++n) {
      double ref = 0;
      for (int k = 0; k < KK; ++k) ref += (double)hA[m * KK + k] * hB[k * NN + n];
      double err = fabs(ref - hD[m * NN + n]);
      if (err > 1e-3 && bad < 5) { printf("mismatch m=%d n=%d got %f want %f\n", m, n, hD[m * NN + n], ref); ++bad; }
      if (err > maxerr) maxerr = err;
    }
  printf("cta_group::2 tf32 M=256 N=%d K=%d: max abs err %g\n", NN, KK, maxerr);
  return 0;
}
