// Probe (profiling aid, not part of the library): does tcgen05.mma kind::f16 accept A = f16 with
// B = bf16 (separate atype / btype fields of the instruction descriptor)?  D[128x128] = A[128x64]
// B[128x64]^T in four K=16 steps, A either from shared memory (SS) or from TMEM (TS, packed
// pairs per 32-bit column as the attention kernel stores P); checked against the host product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_mixed_test scripts/mma_mixed_test.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// byte offset of element (row r, k) of a 128-row x 64-col 16-bit tile, K-major SWIZZLE_128B
__host__ __device__ inline uint32_t swz(uint32_t r, uint32_t k) {
  const uint32_t chunk = (k * 2) / 16, within = (k * 2) % 16;
  return (r / 8) * 1024 + (r % 8) * 128 + ((chunk ^ (r % 8)) * 16) + within;
}

template <bool TS>
__global__ void k_probe(const uint16_t* a, const uint16_t* b, float* d, uint32_t atype, uint32_t btype) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t t = threadIdx.x, warp = t >> 5;
  uint8_t* sa = smem;            // 16 KB
  uint8_t* sb = smem + 16384;    // 16 KB
  for (uint32_t e = t; e < 128 * 64; e += blockDim.x) {
    const uint32_t r = e / 64, k = e % 64;
    *reinterpret_cast<uint16_t*>(sa + swz(r, k)) = a[e];
    *reinterpret_cast<uint16_t*>(sb + swz(r, k)) = b[e];
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  const uint32_t lane_base = (32 * warp) << 16;
  if (TS) {
    // A into TMEM columns [128, 160): lane = row, column c = elements (2c, 2c+1)
    const uint32_t r = t;
    for (uint32_t c = 0; c < 32; ++c) {
      const uint32_t v = (uint32_t)a[r * 64 + 2 * c] | ((uint32_t)a[r * 64 + 2 * c + 1] << 16);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tm + lane_base + 128 + c), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (atype << 7) | (btype << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  if (t == 0) {
    const uint64_t da = sdesc(smem_u32(sa), 16, 1024), db = sdesc(smem_u32(sb), 16, 1024);
    for (uint32_t k = 0; k < 4; ++k) {
      const uint32_t acc = k ? 1u : 0u;
      if (TS)
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
                     ::"r"(tm), "r"(tm + 128 + 8 * k), "l"(db + (uint64_t)((k * 32) >> 4)), "r"(idesc), "r"(acc));
      else
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                     ::"r"(tm), "l"(da + (uint64_t)((k * 32) >> 4)), "l"(db + (uint64_t)((k * 32) >> 4)), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (uint32_t c = 0; c < 128; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + lane_base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    d[t * 128 + c] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

static float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
static float bf2f(uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int n = 128 * 64;
  uint16_t *ha = (uint16_t*)malloc(2 * n), *hb = (uint16_t*)malloc(2 * n), *ha_bf = (uint16_t*)malloc(2 * n);
  srand(1);
  for (int i = 0; i < n; ++i) {
    const float x = (rand() % 2001 - 1000) / 500.f, y = (rand() % 2001 - 1000) / 500.f;
    ha[i] = __half_as_ushort(__float2half_rn(x));
    ha_bf[i] = __bfloat16_as_ushort(__float2bfloat16_rn(x));
    hb[i] = __bfloat16_as_ushort(__float2bfloat16_rn(y));
  }
  uint16_t *da, *db; float* dd;
  cudaMalloc(&da, 2 * n); cudaMalloc(&db, 2 * n); cudaMalloc(&dd, 4 * 128 * 128);
  cudaMemcpy(db, hb, 2 * n, cudaMemcpyHostToDevice);
  float* hd = (float*)malloc(4 * 128 * 128);
  cudaFuncSetAttribute(k_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  cudaFuncSetAttribute(k_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int ts = 0; ts < 2; ++ts)
    for (int mixed = 0; mixed < 2; ++mixed) {
      const uint16_t* A = mixed ? ha : ha_bf;
      cudaMemcpy(da, A, 2 * n, cudaMemcpyHostToDevice);
      cudaMemset(dd, 0, 4 * 128 * 128);
      if (ts) k_probe<true><<<1, 128, 40 * 1024>>>(da, db, dd, mixed ? 0u : 1u, 1u);
      else k_probe<false><<<1, 128, 40 * 1024>>>(da, db, dd, mixed ? 0u : 1u, 1u);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hd, dd, 4 * 128 * 128, cudaMemcpyDeviceToHost);
      double maxerr = 0, maxref = 0;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < 128; ++j) {
          double ref = 0;
          for (int k = 0; k < 64; ++k) ref += (double)(mixed ? h2f(A[i * 64 + k]) : bf2f(A[i * 64 + k])) * bf2f(hb[j * 64 + k]);
          maxerr = fmax(maxerr, fabs(ref - hd[i * 128 + j]));
          maxref = fmax(maxref, fabs(ref));
        }
      printf("%s A=%s B=bf16: max |err| %.3e (max |ref| %.2f)  %s\n", ts ? "TS" : "SS", mixed ? "f16 " : "bf16", maxerr,
             maxref, cudaGetErrorString(e));
    }
  return 0;
}
