// Microbenchmark (profiling aid, not part of the library): tcgen05.ld / tcgen05.st throughput
// per SM for the shapes the softmax uses.  W warps per CTA (warp w reads TMEM lanes
// 32*(w%4)..+31), each warp moves 128 fp32 columns per round (x32 / x64 / x128 loads), REP rounds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tmem_microbench scripts/tmem_microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int REP = 256;

template <int X>
__device__ __forceinline__ void ld(uint32_t a, uint32_t (&r)[128]);
template <>
__device__ __forceinline__ void ld<32>(uint32_t a, uint32_t (&r)[128]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[32 * q + 0]), "=r"(r[32 * q + 1]), "=r"(r[32 * q + 2]), "=r"(r[32 * q + 3]), "=r"(r[32 * q + 4]),
          "=r"(r[32 * q + 5]), "=r"(r[32 * q + 6]), "=r"(r[32 * q + 7]), "=r"(r[32 * q + 8]), "=r"(r[32 * q + 9]),
          "=r"(r[32 * q + 10]), "=r"(r[32 * q + 11]), "=r"(r[32 * q + 12]), "=r"(r[32 * q + 13]), "=r"(r[32 * q + 14]),
          "=r"(r[32 * q + 15]), "=r"(r[32 * q + 16]), "=r"(r[32 * q + 17]), "=r"(r[32 * q + 18]), "=r"(r[32 * q + 19]),
          "=r"(r[32 * q + 20]), "=r"(r[32 * q + 21]), "=r"(r[32 * q + 22]), "=r"(r[32 * q + 23]), "=r"(r[32 * q + 24]),
          "=r"(r[32 * q + 25]), "=r"(r[32 * q + 26]), "=r"(r[32 * q + 27]), "=r"(r[32 * q + 28]), "=r"(r[32 * q + 29]),
          "=r"(r[32 * q + 30]), "=r"(r[32 * q + 31])
        : "r"(a + 32 * q));
}
template <>
__device__ __forceinline__ void ld<16>(uint32_t a, uint32_t (&r)[128]) {
  // 16x256b shape: 16 lanes x 256 bits per call, .x16 -> 16 x 64 columns? (kept simple: x8 of 16x64b)
#pragma unroll
  for (int q = 0; q < 16; ++q)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[8 * q + 0]), "=r"(r[8 * q + 1]), "=r"(r[8 * q + 2]), "=r"(r[8 * q + 3]), "=r"(r[8 * q + 4]),
                   "=r"(r[8 * q + 5]), "=r"(r[8 * q + 6]), "=r"(r[8 * q + 7])
                 : "r"(a + 8 * q));
}

template <int X, bool ST>
__global__ void k_tm(unsigned long long* out) {
  __shared__ uint32_t tslot;
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot + (((32 * (warp & 3)) << 16)) + 128 * ((warp >> 2) & 3);
  uint32_t r[128];
#pragma unroll
  for (int j = 0; j < 128; ++j) r[j] = j;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < REP; ++i) {
    if (ST) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm + 32 * q),
            "r"(r[32 * q + 0]), "r"(r[32 * q + 1]), "r"(r[32 * q + 2]), "r"(r[32 * q + 3]), "r"(r[32 * q + 4]),
            "r"(r[32 * q + 5]), "r"(r[32 * q + 6]), "r"(r[32 * q + 7]), "r"(r[32 * q + 8]), "r"(r[32 * q + 9]),
            "r"(r[32 * q + 10]), "r"(r[32 * q + 11]), "r"(r[32 * q + 12]), "r"(r[32 * q + 13]), "r"(r[32 * q + 14]),
            "r"(r[32 * q + 15]), "r"(r[32 * q + 16]), "r"(r[32 * q + 17]), "r"(r[32 * q + 18]), "r"(r[32 * q + 19]),
            "r"(r[32 * q + 20]), "r"(r[32 * q + 21]), "r"(r[32 * q + 22]), "r"(r[32 * q + 23]), "r"(r[32 * q + 24]),
            "r"(r[32 * q + 25]), "r"(r[32 * q + 26]), "r"(r[32 * q + 27]), "r"(r[32 * q + 28]), "r"(r[32 * q + 29]),
            "r"(r[32 * q + 30]), "r"(r[32 * q + 31]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
    } else {
      ld<X>(tm, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int j = 0; j < 128; j += 16) acc += r[j];
    }
  }
  const unsigned long long t1 = clock64();
  if (acc == 0x9999) out[1] = acc;
  if ((threadIdx.x & 31) == 0) atomicMax(&out[0], t1 - t0);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

template <int X, bool ST>
void run(unsigned long long* d, const char* name) {
  for (int warps : {4, 8, 16}) {
    unsigned long long h = 0;
    for (int k = 0; k < 2; ++k) {
      cudaMemset(d, 0, 16);
      k_tm<X, ST><<<148, 32 * warps>>>(d);
    }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)warps * 32 * 128 * 4 * REP;
    printf("%-28s warps %2d: %6.1f B/clk/SM  (%.0f clk per 64 KB = one 128x128 fp32 S tile)\n", name, warps, bytes / h,
           65536.0 / (bytes / h));
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  run<32, false>(d, "tcgen05.ld 32x32b.x32");
  run<16, false>(d, "tcgen05.ld 32x32b.x8");
  run<32, true>(d, "tcgen05.st 32x32b.x32");
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
