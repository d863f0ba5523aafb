// gbar.cu -- cost of a grid-wide barrier in a cooperative kernel with one 512-thread CTA per SM
// (the s-GMRES block-iteration kernel's shape): cooperative_groups grid.sync() against a
// monotonic-counter barrier (one relaxed atomic per CTA, acquire polling).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gbar gbar.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_cg(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double a = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    a = a * 1.0000001 + 1.0;
    g.sync();
  }
  if (a == 12345.0) sink[0] = a;
}

__global__ void k_ctr(int iters, unsigned long long* bar, double* sink) {
  double a = threadIdx.x;
  const unsigned long long G = gridDim.x;
  unsigned long long gen = 0;
  for (int i = 0; i < iters; ++i) {
    a = a * 1.0000001 + 1.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      ++gen;
      __threadfence();
      atomicAdd(bar, 1ull);
      while (ld_acquire(bar) < gen * G) {
      }
    }
    __syncthreads();
  }
  if (a == 12345.0) sink[0] = a;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  unsigned long long* bar;
  cudaMalloc(&sink, 8);
  cudaMalloc(&bar, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int G : {sms - 1, sms}) {
    int iters = 2000;
    void* args1[] = {&iters, &sink};
    cudaLaunchCooperativeKernel((void*)k_cg, G, 512, args1);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_cg, G, 512, args1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("G=%d cg grid.sync      %.3f us per barrier\n", G, ms * 1e3 / iters);
    cudaMemset(bar, 0, 8);
    void* args2[] = {&iters, &bar, &sink};
    cudaLaunchCooperativeKernel((void*)k_ctr, G, 512, args2);
    cudaMemset(bar, 0, 8);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_ctr, G, 512, args2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("G=%d counter barrier   %.3f us per barrier\n", G, ms * 1e3 / iters);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
