// Streaming-rate microbenchmark for the block-iteration megakernel's sweep shapes: one
// 512-thread CTA per SM with ~170 KB of shared memory (the candidate slice), each CTA owning a
// contiguous slice of n = 1024^2 points, sweeping NCOL basis columns of 8 MiB with U points per
// thread in flight.  Reports GB/s of basis bytes (and DRAM-only bytes when half of them were
// just read, i.e. L2-resident).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp stream_patterns.cu && /tmp/sp
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 512;
constexpr int64_t N = 1 << 20;
constexpr int NBLK = 12;  // 12 blocks of 4 columns = 402 MB > L2

template <int NCOL, int U, int PIPE>
__global__ void __launch_bounds__(NT, 1) k_sweep(const double* V, int64_t np, int b0, int b1, int P, double* out,
                                                 int warm, unsigned long long* tm) {
  extern __shared__ double sm[];
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * P;
  const int cnt = (int)(N - base < P ? N - base : P);
  if (warm) {  // block b1 into L2 first
    double w = 0.0;
    for (int c = 0; c < 4; ++c)
      for (int p = tid; p < cnt; p += NT) w += V[((int64_t)b1 * 4 + c) * np + base + p];
    if (w == 12345.678) out[blockIdx.x] = w;
  }
  grid.sync();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  // columns 0..3 from block b0, 4..7 from block b1
  const double* col[NCOL];
#pragma unroll
  for (int c = 0; c < NCOL; ++c) col[c] = V + ((int64_t)(c < 4 ? b0 : b1) * 4 + (c & 3)) * np + base;
  double acc[NCOL];
#pragma unroll
  for (int c = 0; c < NCOL; ++c) acc[c] = 0.0;
  if (!PIPE) {
    for (int p0 = tid; p0 < cnt; p0 += U * NT) {
      double v[U][NCOL];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < NCOL; ++c) v[u][c] = p0 + u * NT < cnt ? col[c][p0 + u * NT] : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double s = p0 + u * NT < cnt ? sm[p0 + u * NT] : 0.0;
#pragma unroll
        for (int c = 0; c < NCOL; ++c) acc[c] = fma(v[u][c], s, acc[c]);
      }
    }
  } else {
    double a[U][NCOL], b[U][NCOL];
    auto load = [&](double (&v)[U][NCOL], int p0) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < NCOL; ++c) v[u][c] = p0 + u * NT < cnt ? col[c][p0 + u * NT] : 0.0;
    };
    auto work = [&](const double (&v)[U][NCOL], int p0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double s = p0 + u * NT < cnt ? sm[p0 + u * NT] : 0.0;
#pragma unroll
        for (int c = 0; c < NCOL; ++c) acc[c] = fma(v[u][c], s, acc[c]);
      }
    };
    load(a, tid);
    for (int p0 = tid; p0 < cnt; p0 += 2 * U * NT) {
      load(b, p0 + U * NT);
      work(a, p0);
      load(a, p0 + 2 * U * NT);
      work(b, p0 + U * NT);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) s += acc[c];
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the loads alive
  grid.sync();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && tid == 0) tm[0] = t1 - t0;
}

template <int NCOL, int U, int PIPE>
void run(const char* name, const double* V, int64_t np, int P, double* out, bool warm_second) {
  auto k = k_sweep<NCOL, U, PIPE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const size_t smem = 180 * 1024;
  unsigned long long* tm;
  cudaMallocManaged(&tm, 8);
  float best = 1e9f;
  for (int rep = 0; rep < 6; ++rep) {
    float tot = 0.f;
    int cntl = 0;
    for (int b = 0; b + 1 < NBLK; ++b) {
      int b0 = (NCOL == 4 && warm_second) ? b + 1 : b, b1 = b + 1, w = warm_second ? 1 : 0;
      void* args[] = {(void*)&V, (void*)&np, (void*)&b0, (void*)&b1, (void*)&P, (void*)&out, (void*)&w, (void*)&tm};
      cudaLaunchCooperativeKernel((void*)k, 148, NT, args, smem, 0);
      cudaDeviceSynchronize();
      tot += tm[0] * 1e-6f;
      ++cntl;
    }
    if (rep > 0 && tot / cntl < best) best = tot / cntl;
  }
  const double bytes = (double)NCOL * N * 8;
  const double dram = warm_second ? (NCOL > 4 ? 4.0 * N * 8 : 0.0) : bytes;
  std::printf("%-34s %7.2f us  %7.0f GB/s (all)  %7.0f GB/s (DRAM part)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
              dram / (best * 1e-3) / 1e9);
}

int main() {
  const int64_t np = N;
  double *V, *out;
  cudaMalloc(&V, (size_t)NBLK * 4 * np * sizeof(double));
  cudaMemset(V, 0, (size_t)NBLK * 4 * np * sizeof(double));
  cudaMalloc(&out, 4096);
  const int P = (int)(((N + 147) / 148 + 1) & ~1);
  run<1, 1, 0>("1 col U=1 (sync + latency)", V, np, P, out, false);
  run<4, 4, 0>("4 cols U=4", V, np, P, out, false);
  run<4, 2, 0>("4 cols U=2", V, np, P, out, false);
  run<4, 8, 0>("4 cols U=8", V, np, P, out, false);
  run<4, 2, 1>("4 cols U=2 pipelined", V, np, P, out, false);
  run<4, 4, 1>("4 cols U=4 pipelined", V, np, P, out, false);
  run<8, 2, 0>("8 cols U=2", V, np, P, out, false);
  run<8, 3, 0>("8 cols U=3", V, np, P, out, false);
  run<8, 4, 0>("8 cols U=4", V, np, P, out, false);
  run<8, 2, 1>("8 cols U=2 pipelined", V, np, P, out, false);
  run<8, 2, 0>("8 cols U=2, 2nd block in L2", V, np, P, out, true);
  run<8, 3, 0>("8 cols U=3, 2nd block in L2", V, np, P, out, true);
  run<8, 4, 0>("8 cols U=4, 2nd block in L2", V, np, P, out, true);
  run<8, 2, 1>("8 cols U=2 pipe, 2nd block in L2", V, np, P, out, true);
  run<4, 4, 0>("4 cols U=4, block in L2", V, np, P, out, true);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
