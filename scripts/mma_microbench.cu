// Microbenchmark (profiling aid, not part of the library): tcgen05.mma issue/execution rate
// for the M=128 shapes the attention kernel uses.  One CTA; warp 1 issues 64 MMAs (fully
// unrolled, descriptors = base + immediates, elect.sync inside a warp-uniform loop), repeated
// REP times; then one commit; clock64 before issue, after issue and after completion.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_microbench scripts/mma_microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

template <int N, bool TS, int NACC>
__global__ void k_bench(unsigned long long* out, int rep) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((TS ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((128u >> 4) << 24);
  if (warp == 1) {
    const uint32_t sb = smem_u32(smem);
    const uint64_t a0 = sdesc(sb, 16, 1024), b0 = sdesc(sb + 65536, TS ? 8192 : 16, 1024);
    unsigned long long t0 = clock64();
    for (int r = 0; r < rep; ++r) {
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const uint32_t d = tm + (TS ? 256 : 0) + ((k % NACC) * (N <= 128 ? 128 : 256)) % 512;
        if (TS)
          asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1; }"
                       ::"r"(d), "r"(tm + (k & 7) * 8), "l"(b0 + (uint64_t)((k & 7) * 128)), "n"(IDESC));
        else
          asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1; }"
                       ::"r"(d), "l"(a0 + (uint64_t)((k & 3) * 2)), "l"(b0 + (uint64_t)((k & 3) * 2)), "n"(IDESC));
      }
    }
    unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(&bar)));
      unsigned long long t2 = clock64();
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// The attention kernel's per-KV-tile MMA mix for one Q tile: QK (SS, K-major Q and K, N=128,
// 8 x K16) into S, then PV (TS, A = P from TMEM, B = V MN-major, N=128, 8 x K16) into O;
// alternating two Q tiles (A, B) as the paired kernel does.  Per "unit" = 16 MMAs.
__global__ void k_mix(unsigned long long* out, int rep) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  constexpr uint32_t IQK = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  constexpr uint32_t IPV = IQK | (1u << 16);
  if (warp == 1) {
    const uint32_t sb = smem_u32(smem);
    // Q_A at 0, Q_B at 32K, K at 64K, V at 96K (each 32 KB: two 16 KB column blocks)
    const uint64_t dqa = sdesc(sb, 16, 1024), dqb = sdesc(sb + 32768, 16, 1024), dk = sdesc(sb + 65536, 16, 1024),
                   dv = sdesc(sb + 98304, 16384, 1024);
    unsigned long long t0 = clock64();
    for (int r = 0; r < rep; ++r) {
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const uint32_t s_t = tm + 128 * x, o_t = tm + 256 + 128 * x;
        const uint64_t dq = x ? dqb : dqa;
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k)
          asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1; }"
                       ::"r"(s_t), "l"(dq + (uint64_t)((((k >> 2) * 16384) + (k & 3) * 32) >> 4)),
                       "l"(dk + (uint64_t)((((k >> 2) * 16384) + (k & 3) * 32) >> 4)), "n"(IQK));
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k)
          asm volatile("{ .reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1; }"
                       ::"r"(o_t), "r"(s_t + 8 * k), "l"(dv + (uint64_t)((k * 2048) >> 4)), "n"(IPV));
      }
    }
    unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(&bar)));
      out[0] = t1 - t0;
      out[1] = clock64() - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, bool TS, int NACC>
void run(unsigned long long* d, const char* name) {
  auto k = k_bench<N, TS, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int rep : {1, 8}) {
    unsigned long long h[2] = {0, 0};
    for (int w = 0; w < 3; ++w) {
      k<<<1, 128, 160 * 1024>>>(d, rep);
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    }
    const int n = 64 * rep;
    printf("%-30s acc=%d n=%4d issue %6.1f cyc/mma  complete %6.1f cyc/mma  %5.0f MAC/clk\n", name, NACC, n,
           (double)h[0] / n, (double)h[1] / n, 128.0 * N * 16 * n / (double)h[1]);
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  run<64, false, 1>(d, "SS M128 N64  (QK 64-key)");
  run<64, false, 2>(d, "SS M128 N64  (QK 64-key)");
  run<128, false, 1>(d, "SS M128 N128 (QK 128-key)");
  run<128, false, 2>(d, "SS M128 N128 (QK 128-key)");
  run<128, true, 1>(d, "TS M128 N128 (PV)");
  run<128, true, 2>(d, "TS M128 N128 (PV)");
  run<256, false, 1>(d, "SS M128 N256");
  run<256, false, 2>(d, "SS M128 N256");
  {
    cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    for (int grid : {1, 148}) {
      unsigned long long h[2] = {0, 0};
      for (int w = 0; w < 3; ++w) {
        k_mix<<<grid, 128, 160 * 1024>>>(d, 16);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      }
      printf("attention MMA mix (QK SS + PV TS, 2 Q tiles) grid %3d: %6.0f cyc per 128x128x128 unit (ideal 1024)\n", grid,
             (double)h[1] / (16 * 2));
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
