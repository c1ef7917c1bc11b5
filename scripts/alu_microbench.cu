// Microbenchmark (profiling aid, not part of the library): per-SM throughput of the softmax
// instruction mix on sm_100a.  One CTA of W warps per SM; each thread runs ITER iterations of
// 8 independent chains of one instruction; clock64 around the loop; reports element-ops per
// clock per SM (one element = one fp32 lane result; packed x2 ops count 2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/alu_microbench scripts/alu_microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 512;

__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ffma1(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float fmax3(float a, float b, float c) { float d; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ uint32_t cvt_bf2(float a, float b) { uint32_t d; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ uint32_t cvt_h2(float a, float b) { uint32_t d; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) { uint32_t d; asm volatile("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ uint32_t shl_add(uint32_t a, uint32_t b) { uint32_t d; asm volatile("shl.b32 %0, %1, 23;\n\tadd.u32 %0, %0, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }

template <int OP>
__global__ void k_bench(unsigned long long* out, float seed) {
  float f[8]; uint32_t u[8]; uint64_t w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    f[j] = seed * (j + 1) * 1e-3f;
    u[j] = 0x3C003C00u + j;
    w[j] = ((uint64_t)__float_as_uint(f[j]) << 32) | __float_as_uint(f[j] + 1.f);
  }
  const uint64_t one2 = ((uint64_t)__float_as_uint(0.999f) << 32) | __float_as_uint(0.999f);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) f[j] = ex2f(f[j]);
      if (OP == 1) u[j] = ex2h2(u[j]);
      if (OP == 2) u[j] = ex2bf2(u[j]);
      if (OP == 3) w[j] = ffma2(w[j], one2, one2);
      if (OP == 4) w[j] = fadd2(w[j], one2);
      if (OP == 5) f[j] = ffma1(f[j], 0.999f, 0.5f);
      if (OP == 6) f[j] = fmax3(f[j], f[(j + 1) & 7], 0.5f);
      if (OP == 7) u[j] = cvt_bf2(f[j], __uint_as_float(u[j]));
      if (OP == 8) u[j] = cvt_h2(f[j], __uint_as_float(u[j]));
      if (OP == 9) u[j] = hfma2(u[j], 0x3C003C00u, 0x3C003C00u);
      if (OP == 10) u[j] = shl_add(u[j], 7u);
      if (OP == 11) { f[j] = ex2f(f[j]); w[j] = ffma2(w[j], one2, one2); }   // MUFU + FFMA2 co-issue
      if (OP == 12) { uint32_t d; asm volatile("add.u32 %0, %1, %2;" : "=r"(d) : "r"(u[j]), "r"(u[(j + 1) & 7])); u[j] = d; }
      if (OP == 13) { uint32_t d; asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(u[j]), "r"(u[(j + 3) & 7]), "r"(0x5A5A5A5Au)); u[j] = d; }
      if (OP == 14) { uint32_t d; asm volatile("{ .reg .pred p1; setp.eq.u32 p1, %1, %2; selp.u32 %0, 1, %1, p1; }" : "=r"(d) : "r"(u[j]), "r"(u[(j + 1) & 7])); u[j] = d; }
    }
  }
  const unsigned long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += f[j] + __uint_as_float(u[j]) + __uint_as_float((uint32_t)w[j]);
  if (acc == 1234.5f) out[1] = 1;
  if (threadIdx.x == 0) atomicMax(&out[0], t1 - t0);
}

template <int OP>
void run(unsigned long long* d, const char* name, double elems_per_op) {
  for (int warps : {4, 8, 16}) {
    unsigned long long h = 0;
    cudaMemset(d, 0, 16);
    k_bench<OP><<<148, 32 * warps>>>(d, 1.0f);
    cudaMemset(d, 0, 16);
    k_bench<OP><<<148, 32 * warps>>>(d, 1.0f);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double ops = 32.0 * warps * ITER * 8;
    printf("%-34s warps/SM %2d: %7.1f element-ops/clk/SM  (%.2f warp-instr/clk/SMSP)\n", name, warps,
           ops * elems_per_op / h, ops / 32.0 / 4 / h);
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  run<0>(d, "ex2.approx.ftz.f32 (MUFU.EX2)", 1);
  run<1>(d, "ex2.approx.f16x2", 2);
  run<2>(d, "ex2.approx.ftz.bf16x2", 2);
  run<3>(d, "fma.rn.f32x2 (FFMA2)", 2);
  run<4>(d, "add.rn.f32x2 (FADD2)", 2);
  run<5>(d, "fma.rn.f32 (FFMA)", 1);
  run<6>(d, "max.f32 3-input (FMNMX3)", 2);
  run<7>(d, "cvt.rn.bf16x2.f32 (F2FP)", 2);
  run<8>(d, "cvt.rn.f16x2.f32", 2);
  run<9>(d, "fma.rn.f16x2 (HFMA2)", 2);
  run<10>(d, "shl+add (2 int ops)", 1);
  run<11>(d, "MUFU.EX2 + FFMA2 pairs (per pair)", 1);
  run<12>(d, "add.u32 (IADD3, INT32 lane-op)", 1);
  run<13>(d, "lop3.b32 (LOP3, INT32 lane-op)", 1);
  run<14>(d, "setp.eq + selp (compare, 2 ops)", 1);
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
