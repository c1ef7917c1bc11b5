// Microbenchmark (profiling aid, not part of the library): throughput of candidate softmax
// inner loops (one thread = one 128-element row, as in the attention kernel), registers only.
// Reports SM clocks per 128x128 tile (16384 elements) for 2 warps per SMSP (the kernel's
// two softmax warpgroups).  V0 = the kernel's current f32 path; V1 = ex2.approx.ftz.bf16x2;
// V2 = ex2.approx.f16x2 with f32 sums; V3 = bf16x2 on [-1,0] fraction + exact exponent add.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/softmax_microbench scripts/softmax_microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TILES = 64;

__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) { uint32_t y; asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ void ffma2(float& o0, float& o1, float a0, float a1, float s, float m) {
  asm("{ .reg .b64 x, y, z, w; mov.b64 x, {%2, %3}; mov.b64 y, {%4, %4}; mov.b64 z, {%5, %5};\n\t"
      "fma.rn.f32x2 w, x, y, z; mov.b64 {%0, %1}, w; }" : "=f"(o0), "=f"(o1) : "f"(a0), "f"(a1), "f"(s), "f"(m));
}
__device__ __forceinline__ void fadd2(float& s0, float& s1, float a0, float a1) {
  asm("{ .reg .b64 x, y, w; mov.b64 x, {%0, %1}; mov.b64 y, {%2, %3};\n\t"
      "add.rn.f32x2 w, x, y; mov.b64 {%0, %1}, w; }" : "+f"(s0), "+f"(s1) : "f"(a0), "f"(a1));
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) { uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a)); return r; }
__device__ __forceinline__ uint32_t pack_f16(float a, float b) { uint32_t r; asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a)); return r; }
__device__ __forceinline__ float fmax3(float a, float b, float c) { float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f, j = t - 12582912.f, f = x - j;
  float p = fmaf(f, 0.05550411f, 0.24022651f);
  p = fmaf(p, f, 0.69314718f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}

__device__ __forceinline__ void ex2_poly2(float x0, float x1, float& y0, float& y1) {
  x0 = fmaxf(x0, -125.f);
  x1 = fmaxf(x1, -125.f);
  uint32_t t0, t1, p0, p1;
  asm("{ .reg .b64 x, t, j, f, p, c, m, nm, k3, k2, k1, one;\n\t"
      "mov.b64 x, {%4, %5};\n\t"
      "mov.b64 m, {0f4B400000, 0f4B400000};\n\t"
      "mov.b64 nm, {0fCB400000, 0fCB400000};\n\t"
      "add.rn.f32x2 t, x, m;\n\t"
      "add.rn.f32x2 j, t, nm;\n\t"
      "mov.b64 c, {0fBF800000, 0fBF800000};\n\t"
      "fma.rn.f32x2 f, j, c, x;\n\t"
      "mov.b64 k3, {0f3D61FBB0, 0f3D61FBB0};\n\t"
      "mov.b64 k2, {0f3E786F0F, 0f3E786F0F};\n\t"
      "mov.b64 k1, {0f3F31798D, 0f3F31798D};\n\t"
      "mov.b64 one, {0f3F7FFB49, 0f3F7FFB49};\n\t"
      "fma.rn.f32x2 p, f, k3, k2;\n\t"
      "fma.rn.f32x2 p, p, f, k1;\n\t"
      "fma.rn.f32x2 p, p, f, one;\n\t"
      "mov.b64 {%0, %1}, t;\n\t"
      "mov.b64 {%2, %3}, p; }"
      : "=r"(t0), "=r"(t1), "=r"(p0), "=r"(p1) : "f"(x0), "f"(x1));
  y0 = __uint_as_float(p0 + (t0 << 23));
  y1 = __uint_as_float(p1 + (t1 << 23));
}

// V4/V5: the attention kernel's current exp loop (64 elements per thread = half a row); EMU =
// bitmask over pair index mod 8 of pairs computed by ex2_poly2.  Reports clk per 128x128 tile
// when 256 threads (2 per row) process one tile per iteration.
template <int EMU, int DROP = 0>   // DROP bits: 1 = no row sum, 2 = no bf16 pack, 4 = no scale FFMA2
__global__ void __launch_bounds__(256) k_half(unsigned long long* out, float seed, uint32_t* sink) {
  float a[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) a[j] = seed * (float)((threadIdx.x * 131 + j * 17) & 255) * (1.f / 64.f) - 2.f;
  const float sl2 = 0.127f;
  float l = 0.f;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int t = 0; t < TILES; ++t) {
    const float negm = -(float)(t & 3) * 0.01f;
    float rsa[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t pk[32];
#pragma unroll
    for (int j = 0; j < 64; j += 2) {
      float x0 = a[j], x1 = a[j + 1];
      if (!(DROP & 4)) ffma2(x0, x1, a[j], a[j + 1], sl2, negm);
      float p0, p1;
      if ((EMU >> ((j >> 1) & 7)) & 1) ex2_poly2(x0, x1, p0, p1);
      else { p0 = ex2f(x0); p1 = ex2f(x1); }
      if (!(DROP & 1)) fadd2(rsa[(j >> 1) & 2], rsa[((j >> 1) & 2) + 1], p0, p1);
      pk[j >> 1] = (DROP & 2) ? (__float_as_uint(p0) ^ __float_as_uint(p1)) : pack_bf16(p0, p1);
    }
    l += (rsa[0] + rsa[1]) + (rsa[2] + rsa[3]);
#pragma unroll
    for (int j = 0; j < 32; ++j) acc ^= pk[j];
    a[t & 63] += __uint_as_float(acc & 0x3F800000u) * 1e-30f;   // loop-carried, cheap
  }
  const unsigned long long t1 = clock64();
  if (acc == 0x12345 && l == 1.f) sink[0] = acc;
  if (threadIdx.x == 0) atomicMax(&out[0], t1 - t0);
}

template <int V>
__global__ void __launch_bounds__(256) k_sm(unsigned long long* out, float seed, uint32_t* sink) {
  float a[128];
#pragma unroll
  for (int j = 0; j < 128; ++j) a[j] = seed * (float)((threadIdx.x * 131 + j * 17) & 255) * (1.f / 64.f) - 2.f;
  const float sl2 = 0.127f;
  float l = 0.f, mprev = 0.f;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int t = 0; t < TILES; ++t) {
    // max pass
    float mx[4] = {a[0], a[1], a[2], a[3]};
#pragma unroll
    for (int j = 4; j < 128; j += 8) {
      mx[0] = fmax3(mx[0], a[j], a[j + 1]); mx[1] = fmax3(mx[1], a[j + 2], a[j + 3]);
      mx[2] = fmax3(mx[2], a[j + 4], a[j + 5]); mx[3] = fmax3(mx[3], a[j + 6], a[j + 7]);
    }
    const float m = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2;
    const float negm = -fmaxf(m, mprev);
    mprev = m;
    float rs[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t pk[64];
    if (V == 0) {
#pragma unroll
      for (int j = 0; j < 128; j += 2) {
        float x0, x1;
        ffma2(x0, x1, a[j], a[j + 1], sl2, negm);
        const float p0 = ((j & 7) == 7) ? ex2_poly(x0) : ex2f(x0);
        const float p1 = (((j + 1) & 7) == 7) ? ex2_poly(x1) : ex2f(x1);
        fadd2(rs[(j >> 1) & 2], rs[((j >> 1) & 2) + 1], p0, p1);
        pk[j >> 1] = pack_bf16(p0, p1);
      }
    } else if (V == 1) {
#pragma unroll
      for (int j = 0; j < 128; j += 2) {
        float x0, x1;
        ffma2(x0, x1, a[j], a[j + 1], sl2, negm);
        const uint32_t p = ex2bf2(pack_bf16(x0, x1));
        fadd2(rs[(j >> 1) & 2], rs[((j >> 1) & 2) + 1], __uint_as_float(p << 16), __uint_as_float(p & 0xFFFF0000u));
        pk[j >> 1] = p;
      }
    } else if (V == 2) {
#pragma unroll
      for (int j = 0; j < 128; j += 2) {
        float x0, x1;
        ffma2(x0, x1, a[j], a[j + 1], sl2, negm);
        const uint32_t h = ex2h2(pack_f16(x0, x1));
        float p0, p1;
        asm("{ .reg .f16 lo, hi; mov.b32 {lo, hi}, %2; cvt.f32.f16 %0, lo; cvt.f32.f16 %1, hi; }" : "=f"(p0), "=f"(p1) : "r"(h));
        fadd2(rs[(j >> 1) & 2], rs[((j >> 1) & 2) + 1], p0, p1);
        pk[j >> 1] = pack_bf16(p0, p1);
      }
    } else {
      // V3: x = i + f, f in [-1, 0): bf16x2 exp of f (ulp <= 2^-8), 2^i added to the exponent
#pragma unroll
      for (int j = 0; j < 128; j += 2) {
        float x0, x1;
        ffma2(x0, x1, a[j], a[j + 1], sl2, negm);
        x0 = fmaxf(x0, -100.f); x1 = fmaxf(x1, -100.f);
        float i0, i1;
        asm("cvt.rmi.f32.f32 %0, %1;" : "=f"(i0) : "f"(x0));
        asm("cvt.rmi.f32.f32 %0, %1;" : "=f"(i1) : "f"(x1));
        float f0 = x0 - i0, f1 = x1 - i1;                 // [0, 1)
        uint32_t p = ex2bf2(pack_bf16(f0, f1));
        const uint32_t e = ((uint32_t)(int)i0 << 7 & 0xFFFFu) | ((uint32_t)(int)i1 << 23);
        p += e;
        fadd2(rs[(j >> 1) & 2], rs[((j >> 1) & 2) + 1], __uint_as_float(p << 16), __uint_as_float(p & 0xFFFF0000u));
        pk[j >> 1] = p;
      }
    }
    l = l * 0.5f + (rs[0] + rs[1]) + (rs[2] + rs[3]);
#pragma unroll
    for (int j = 0; j < 64; ++j) acc ^= pk[j];
#pragma unroll
    for (int j = 0; j < 128; ++j) a[j] = a[j] + __uint_as_float(acc & 1);   // loop-carried
  }
  const unsigned long long t1 = clock64();
  if (acc == 0x12345 && l == 1.f) sink[0] = acc;
  if (threadIdx.x == 0) atomicMax(&out[0], t1 - t0);
}

template <int V>
void run(unsigned long long* d, uint32_t* sink, const char* name) {
  for (int thr : {128, 256}) {
    unsigned long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d, 0, 8);
      k_sm<V><<<148, thr>>>(d, 1.0f, sink);
    }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double tiles = TILES * thr / 128.0;            // 128 threads = one 128x128 tile per iteration
    printf("%-44s threads/SM %3d: %7.0f clk per 128x128 tile\n", name, thr, h / tiles);
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned long long* d; uint32_t* sink;
  cudaMalloc(&d, 16); cudaMalloc(&sink, 16);
  run<0>(d, sink, "V0 f32 MUFU (1/8 poly) + F2FP");
  run<1>(d, sink, "V1 bf16x2 MUFU");
  run<2>(d, sink, "V2 f16x2 MUFU + cvt + F2FP");
  run<3>(d, sink, "V3 bf16x2 on fraction + exponent add");
  auto half = [&](auto kern, const char* name) {
    unsigned long long h = 0;
    for (int rep = 0; rep < 2; ++rep) { cudaMemset(d, 0, 8); kern<<<148, 256>>>(d, 1.0f, sink); }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-44s 256 threads (2 per row): %7.0f clk per 128x128 tile (ex-exchange, ex-max)\n", name, (double)h / TILES);
  };
  half(k_half<0x00>, "V4 kernel exp loop, no emulation");
  half(k_half<0x00, 1>, "  no emulation, no row sum");
  half(k_half<0x00, 2>, "  no emulation, no bf16 pack");
  half(k_half<0x00, 4>, "  no emulation, no scale FFMA2");
  half(k_half<0x00, 7>, "  MUFU only");
  half(k_half<0xFF, 7>, "  poly only");
  half(k_half<0x80>, "V4 kernel exp loop, 1/8 emulated");
  half(k_half<0x4A>, "V4 kernel exp loop, 3/8 emulated");
  half(k_half<0xAA>, "V4 kernel exp loop, 1/2 emulated");
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
