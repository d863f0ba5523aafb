// tail_latency.cu -- latency of a single CTA's small global-memory work right after an
// all-SM streaming phase (the s-GMRES megakernel's least-squares tail): does it depend on
// the allocation the small buffers live in (TLB reach) or on L2 state?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tail_latency tail_latency.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// every CTA streams its slice of `big` (read), then CTA 0 does `rounds` dependent
// load->store round trips on `small` (stride words apart) and n stores
__global__ void k(double* big, size_t nbig, double* small, int stride, int rounds, int nstores,
                  unsigned long long* out, double* sink, int writes) {
  cg::grid_group grid = cg::this_grid();
  double acc = 0.0;
  const size_t per = nbig / gridDim.x;
  double* b = big + per * blockIdx.x;
  for (size_t i = threadIdx.x; i < per; i += blockDim.x) {
    const double v = __ldcg(b + i);
    acc += v;
    if (writes && (i & 3) == 0) b[i] = v + 1.0;
  }
  if (acc == 12345.0) sink[0] = acc;
  grid.sync();
  if (blockIdx.x != 0) return;
  __syncthreads();
  unsigned long long t0 = gt();
  double v = 0.0;
  if (threadIdx.x == 0)
    for (int r = 0; r < rounds; ++r) {
      v += __ldcg(small + (size_t)r * stride);
      small[(size_t)r * stride + 1] = v;
    }
  __syncthreads();
  unsigned long long t1 = gt();
  for (int e = threadIdx.x; e < nstores; e += blockDim.x) small[(size_t)e * 8 + 3] = (double)e;
  __syncthreads();
  unsigned long long t2 = gt();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    if (v == 12345.0) sink[1] = v;
  }
}

int main() {
  const size_t nbig = (size_t)400 << 20 >> 3;  // 400 MB
  double *big, *small_sep, *sink;
  unsigned long long* out;
  cudaMalloc(&big, nbig * 8 + (64 << 20));
  cudaMalloc(&small_sep, 64 << 20);
  cudaMalloc(&sink, 64);
  cudaMalloc(&out, 64);
  cudaMemset(big, 0, nbig * 8 + (64 << 20));
  cudaMemset(small_sep, 0, 64 << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* small_in = big + nbig;  // same allocation as the streamed data
  struct Case { const char* name; double* p; int stride; int writes; } cases[] = {
      {"separate alloc, stride 1 KB", small_sep, 128, 0},
      {"separate alloc, stride 2 MB", small_sep, 1 << 18, 0},
      {"same alloc, stride 1 KB", small_in, 128, 0},
      {"no streaming (nbig 0), separate", small_sep, 128, 0},
      {"streaming + 25% writes, separate", small_sep, 128, 1},
      {"streaming + 25% writes, 2 MB stride", small_sep, 1 << 18, 1},
  };
  for (int ci = 0; ci < 6; ++ci) {
    for (int rep = 0; rep < 3; ++rep) {
      size_t nb = ci == 3 ? 0 : nbig;
      int rounds = 16, nst = 200;
      void* args[] = {&big, &nb, &cases[ci].p, &cases[ci].stride, &rounds, &nst, &out, &sink, &cases[ci].writes};
      cudaLaunchCooperativeKernel((void*)k, sms, 512, args, 0, 0);
      unsigned long long h[2];
      cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      if (rep == 2) printf("%-36s 16 dependent ld/st rounds %.2f us, 200 stores %.2f us\n", cases[ci].name, h[0] * 1e-3, h[1] * 1e-3);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
}
