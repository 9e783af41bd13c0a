// tc2_chain.cu -- microbenchmark: the CTA-pair resident kernel's (asot_sinkhorn_tc2.cu) MMA
// schedule without its epilogue.  Per phase 4 parts of 16 MMAs (M=256, N=128, k=8) into
// D = R_{1-f%2} with A read from TMEM R_{f%2}; commit after part 3 (D half 0 complete) and after
// part 4 (D half 1).  Variants:
//   0  all phases issued back to back, A from a fixed region (no TMEM read-after-write)
//   1  as the kernel: A of phase f+1 = D of phase f, still issued back to back
//   2  as 1, but parts 1,2 of phase f+1 wait for phase f's half-0 commit and parts 3,4 for its
//      half-1 commit (the kernel's dependency structure with a zero-time epilogue)
//   3  as 2, plus DELAY cycles between each commit landing and the dependent issue (an
//      epilogue of that latency)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc2_chain tools/tc2_chain.cu
#include <cstdint>
#include <cstdio>
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
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(bar), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void spin(int cycles) {
  const long long t = clock64();
  while (clock64() - t < cycles) {
  }
}

template <int VAR>
__global__ void __cluster_dims__(2, 1, 1) chain_kernel(int phases, int delay, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bars[2];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[b])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c000000u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = holder;
  const uint32_t b0 = smem_u32(&bars[0]), b1 = smem_u32(&bars[1]);
  if (rank == 0 && warp == 0) {
    constexpr uint32_t id = idesc(256, 128);
    const uint64_t bd0 = make_sw128_desc(smem_u32(smem));
    const long long t0 = clock64();
    for (int f = 0; f < phases; ++f) {
      const uint32_t ra = VAR == 0 ? tm : tm + 256u * (f & 1), rd = VAR == 0 ? tm + 256 : tm + 256u * ((f + 1) & 1);
      for (int part = 0; part < 4; ++part) {
        const int kc = part >> 1, nh = part & 1;
        if (VAR >= 2 && f > 0 && (part == 0 || part == 2)) {
          wait(part == 0 ? b0 : b1, (f - 1) & 1);
          if (VAR == 3) spin(delay);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        __syncwarp();
        if (threadIdx.x == 0) {
          for (int k = 0; k < 16; ++k)
            mma(rd + nh * 128, ra + kc * 128 + k * 8, bd0 + (uint64_t)(((k & 3) * 32 + nh * 8192) >> 4), id,
                (uint32_t)(kc > 0 || k > 0));
          if (part == 2) commit(b0);
          if (part == 3) commit(b1);
        }
        __syncwarp();
      }
    }
    wait(b1, (phases - 1) & 1);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  } else if (rank == 1 && warp == 0) {
    wait(b1, (phases - 1) & 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int VAR>
void run(long long* d, int delay) {
  const int phases = 64;
  auto k = chain_kernel<VAR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  long long h = 0;
  for (int rep = 0; rep < 3; ++rep) {
    k<<<2, 128, 70 * 1024>>>(phases, delay, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return;
    }
  }
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("variant %d delay %4d: %7.1f cycles/phase (64 MMAs; ideal 4141), %5.1f cycles/MMA\n", VAR, delay,
         (double)h / phases, (double)h / phases / 64);
}


// cta_group::1 variants of the 1-SM kernel's chains (asot_sinkhorn_tc.cu): per chain either
// 4 parts of 8 MMAs (M=128, N=64) with commits after parts 3 and 4 (VAR 10), the same with both
// commits at the end (VAR 11), or 16 MMAs of N=128 and one commit (VAR 12); 13-18 are N=64
// operand-pattern variants.  Back to back, issued by elect.sync in a converged warp (issuing
// from `if (threadIdx.x == 0)` instead makes ptxas wrap every MMA in an ELECT loop: ~50 cycles
// per MMA, which once read here as "N = 64 MMAs are slow").
__device__ __forceinline__ void mma1(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit1(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool elect1() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\telect.sync rx|px, %1;\n\t@px mov.s32 %0, 1;\n\t}"
               : "+r"(pred) : "r"(0xffffffffu));
  return pred != 0;
}
template <int VAR>
__global__ void chain1_kernel(int chains, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bars[2];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[b])) : "memory");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c000000u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = holder;
  const uint32_t b0 = smem_u32(&bars[0]), b1 = smem_u32(&bars[1]);
  if (warp == 0) {
    const uint64_t bd0 = make_sw128_desc(smem_u32(smem));
    const long long t0 = clock64();
    for (int c = 0; c < chains; ++c) {
      const uint32_t base = tm + 256u * (c & 1);
      const uint32_t ra = base + 128u * ((c >> 1) & 1), rd = base + 128u * (1 - ((c >> 1) & 1));
      if (elect1()) {  // converged warp + elect.sync: no per-MMA ELECT/R2UR loop
        if (VAR == 13) {         // N = 64, one D range, A marching over 32 k-steps
          for (int k = 0; k < 32; ++k)
            mma1(rd, base + 8 * (k & 15), bd0 + (uint64_t)((((k >> 2) & 3) * 16384 + (k & 3) * 32) >> 4), idesc(128, 64), k > 0);
          commit1(b0);
        } else if (VAR == 14) {  // N = 64, D alternating between two column ranges every 8 MMAs
          for (int part = 0; part < 4; ++part)
            for (int k = 0; k < 8; ++k)
              mma1(rd + 64 * (part & 1), base + 8 * k, bd0 + (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4),
                   idesc(128, 64), part > 1 || k > 0);
          commit1(b0);
        } else if (VAR == 15) {  // N = 64, D alternating every MMA
          for (int k = 0; k < 32; ++k)
            mma1(rd + 64 * (k & 1), base + 8 * (k >> 1 & 7), bd0 + (uint64_t)((((k >> 1) >> 2 & 1) * 16384 + ((k >> 1) & 3) * 32) >> 4),
                 idesc(128, 64), k > 1);
          commit1(b0);
        } else if (VAR == 16) {  // cg2_rate's pattern: fixed D, A = tm+256+8(k&15), B in one 16 KB block
          for (int k = 0; k < 32; ++k)
            mma1(tm, tm + 256 + 8 * (k & 15), bd0 + (uint64_t)(((k & 3) * 32) >> 4), idesc(128, 64), k > 0);
          commit1(b0);
        } else if (VAR == 17) {  // as 16, B marching over 4 blocks of 16 KB like the kernels
          for (int k = 0; k < 32; ++k)
            mma1(tm, tm + 256 + 8 * (k & 15), bd0 + (uint64_t)((((k >> 2) & 3) * 16384 + (k & 3) * 32) >> 4),
                 idesc(128, 64), k > 0);
          commit1(b0);
        } else if (VAR == 18) {  // as 16 but D alternating between two tiles every chain (c)
          for (int k = 0; k < 32; ++k)
            mma1(tm + 128 * (c & 1), tm + 256 + 8 * (k & 15), bd0 + (uint64_t)(((k & 3) * 32) >> 4), idesc(128, 64), k > 0);
          commit1(b0);
        } else if (VAR == 12) {
          for (int k = 0; k < 16; ++k)
            mma1(rd, ra + 8 * k, bd0 + (uint64_t)(((k >> 2) * 16384 + (k & 3) * 32) >> 4), idesc(128, 128), k > 0);
          commit1(b0);
        } else {
          for (int part = 0; part < 4; ++part) {
            const int kc = part >> 1, nc = part & 1;
            for (int k = 0; k < 8; ++k)
              mma1(rd + 64 * nc, ra + 64 * kc + 8 * k,
                   bd0 + (uint64_t)((((kc * 8 + k) >> 2) * 16384 + nc * 8192 + (k & 3) * 32) >> 4), idesc(128, 64),
                   (kc > 0 || k > 0));
            if (VAR == 10 && part >= 2) commit1(part == 2 ? b0 : b1);
          }
          if (VAR == 11) {
            commit1(b0);
            commit1(b1);
          }
        }
      }
      __syncwarp();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int VAR>
void run1(long long* d) {
  const int chains = 256;
  auto k = chain1_kernel<VAR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  long long h = 0;
  for (int rep = 0; rep < 3; ++rep) {
    k<<<1, 128, 70 * 1024>>>(chains, d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return; }
  }
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("1-SM variant %d: %7.1f issue cycles/chain (ideal 1034 at 64.6 per N=128 MMA)\n", VAR, (double)h / chains);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<0>(d, 0);
  run<1>(d, 0);
  run<2>(d, 0);
  for (int delay : {200, 400, 600, 800, 1000, 1200}) run<3>(d, delay);
  run1<10>(d);
  run1<11>(d);
  run1<12>(d);
  run1<13>(d);
  run1<14>(d);
  run1<15>(d);
  run1<16>(d);
  run1<17>(d);
  run1<18>(d);
  return 0;
}
