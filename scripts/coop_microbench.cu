// Microbenchmark (profiling aid, not part of the library): event-timed cost of a cooperative
// launch (grid.sync) vs a plain launch of the same tiny kernel, back to back on one stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/coop_microbench scripts/coop_microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_coop(int* x) { cg::this_grid().sync(); if (threadIdx.x == 0 && blockIdx.x == 0) x[0]++; }
__global__ void k_plain(int* x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0]++; }
int main() {
  int* d; cudaMalloc(&d, 4);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks : {148, 296}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a, s);
        for (int i = 0; i < 100; ++i) {
          if (mode == 0) k_plain<<<blocks, 512, 0, s>>>(d);
          else { void* args[] = {&d}; cudaLaunchCooperativeKernel((void*)k_coop, blocks, 512, args, 0, s); }
          if (mode == 2) k_plain<<<1, 32, 0, s>>>(d);
        }
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("blocks %d %-26s %7.2f us per launch\n", blocks,
                        mode == 0 ? "plain" : mode == 1 ? "cooperative" : "cooperative + plain", ms * 10);
      }
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
