// tmem_probe.cu -- microbenchmark: does tcgen05.ld/st latency depend on a concurrently running
// tcgen05.mma (kind::tf32, A from TMEM) issued by another warp on a different TMEM region?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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

// mode bit0: run MMAs, bit1: run TMEM loads, bit2: loads are stores instead
__global__ void __launch_bounds__(256, 1) probe(int mode, int n_mma, int n_ld, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float*)sm)[i] = 0.0f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = holder;
  long long t0 = clock64();
  if (warp == 0 && (mode & 1)) {
    if (lane == 0) {
      const uint32_t b0 = smem_u32(sm);
      for (int i = 0; i < n_mma; ++i) {
        const int ks = i & 15;
        const uint32_t b_addr = b0 + (uint32_t)((ks >> 2) * 128 * 128 + (ks & 3) * 32);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb + 128),
                     "r"(tb + 8 * ks), "l"(make_sw128_desc(b_addr)), "r"(idesc(128, 128)), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      uint32_t ok = 0;
      while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)));
      }
      out[0] = clock64() - t0;
    }
  }
  if (warp >= 4 && (mode & 2)) {
    const uint32_t addr = tb + ((uint32_t)((warp & 3) * 32) << 16) + 256;
    long long s = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < n_ld; ++i) {
      uint32_t r[16];
      if (mode & 4) {
        for (int e = 0; e < 16; ++e) r[e] = i + e;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(addr + (i & 7) * 16), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                     "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(addr + (i & 7) * 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int e = 0; e < 16; ++e) acc += r[e];
      }
    }
    long long e = clock64() - s;
    if (lane == 0) out[1 + (warp - 4)] = e;
    if (acc == 0x12345678) out[7] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
  long long* d_out;
  cudaMalloc(&d_out, 8 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int n_mma = 1600, n_ld = 2000;
  const char* names[] = {"", "mma only", "ld only", "mma + ld", "", "", "st only", "mma + st"};
  for (int mode : {1, 2, 3, 6, 7}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d_out, 0, 8 * sizeof(long long));
      probe<<<148, 256, 64 * 1024>>>(mode, n_mma, n_ld, d_out);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[8];
      cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
      if (rep == 1)
        printf("%-10s err=%d  mma: %lld cyc (%.1f cyc/instr, ideal 64)  ld/st warp4: %lld cyc (%.1f cyc/op)\n",
               names[mode], (int)e, h[0], n_mma ? (double)h[0] / n_mma : 0.0, h[1], (double)h[1] / n_ld);
    }
  }
  return 0;
}
