// Per-launch cost of empty (flag-skipped) kernels on the device: grid 296 x 288 threads, with
// dynamic shared memory sizes like the streaming kernels', with/without PDL.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_skip(const int* flag, double* out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ double sm[];
  if (__ldg(flag) == 0) return;
  sm[threadIdx.x] = 1.0;
  __syncthreads();
  out[blockIdx.x] = sm[(threadIdx.x + 1) % blockDim.x];
}

int main() {
  int* flag;
  double* out;
  cudaMalloc(&flag, 4);
  cudaMemset(flag, 0, 4);
  cudaMalloc(&out, 1 << 20);
  cudaFuncSetAttribute(k_skip, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int grid : {1, 148, 296})
      for (size_t smem : {(size_t)0, (size_t)48 * 1024, (size_t)100 * 1024, (size_t)200 * 1024}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = 288;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl;
        for (int i = 0; i < 50; ++i) cudaLaunchKernelEx(&cfg, k_skip, (const int*)flag, out);
        cudaEventRecord(a, st);
        const int N = 2000;
        for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, k_skip, (const int*)flag, out);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("pdl=%d grid=%d smem=%zuKB: %.2f us/launch\n", pdl, grid, smem / 1024, 1000.0 * ms / N);
      }
  // alternating smem sizes (carve-out changes)
  return 0;
}
