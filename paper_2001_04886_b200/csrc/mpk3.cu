// mpk3.cu -- one-sweep 3D matrix powers for the 7-point stencil on one GPU (krylov_block,
// block.hpp:59-67; krylov_pair, sstep.hpp:71-81): out[j] = A^j (src * scale), j = 1..J
// (out[0] = src * scale when requested), J <= 4, reading the source once and writing each
// power once -- (J + 1) vectors of HBM traffic instead of the 2 J of J separate sweeps.
//
// 2.5D blocking: a CTA owns a 32 x 16 (x, y) tile and a run of z planes.  Source planes of the
// tile extended by J on every side stream into a shared-memory ring through asynchronous
// copies (zero-filled outside the grid) PF planes ahead; level j is computed on the tile
// extended by J - j, one plane behind level j - 1 (level j at plane t - j when source plane t
// has arrived), each level keeping its three newest planes in a shared-memory ring, so no level
// needs another CTA's results (the ghost columns are recomputed redundantly, and the z chunks
// start J planes early).  Every point is the reference's ascending-column sum (-z, -y, -x, C,
// +x, +y, +z; absent neighbours skipped; multiply and add rounded separately), so each power is
// bit-identical to J successive spmv calls.
#include <algorithm>
#include <cstring>

#include "device_util.cuh"
#include "skc_internal.hpp"

namespace skc {

namespace {

constexpr int M3_TX = 32, M3_TY = 16, M3_NT = 512, M3_PF = 3, M3_RS = M3_PF + 3;

struct Mpk3Desc {
  int nx, ny, nz;
  double c[7];
  const double* src;
  const double* scale;
  double* out[5];
  int Z;  // planes per CTA
  int tiles_x;
  const int* halt;
  const int* cond;
};

template <int J>
__host__ __device__ constexpr int m3_ex(int j) { return M3_TX + 2 * (J - j); }
template <int J>
__host__ __device__ constexpr int m3_ey(int j) { return M3_TY + 2 * (J - j); }
template <int J>
__host__ __device__ constexpr int m3_smem_doubles() {
  int s = M3_RS * m3_ex<J>(0) * m3_ey<J>(0);
  for (int j = 1; j < J; ++j) s += 3 * m3_ex<J>(j) * m3_ey<J>(j);
  return s;
}

__device__ __forceinline__ void cp_async8_zfill(void* smem, const void* gmem, bool valid) {
  const uint32_t s = smem_u32(smem);
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}

template <int J>
__global__ void __launch_bounds__(M3_NT, 2) k_mpk3t(const __grid_constant__ Mpk3Desc d) {
  SKC_PDL_ENTRY();
  if (skip_launch(d.halt, d.cond)) return;
  extern __shared__ __align__(16) double m3s[];
  constexpr int E0X = m3_ex<J>(0), E0Y = m3_ey<J>(0), E0 = E0X * E0Y;
  double* ring0 = m3s;  // source ring: plane q in slot q % RS
  double* lring[J > 1 ? J : 2];  // level j's three newest planes (j = 1..J-1)
  {
    double* p = m3s + M3_RS * E0;
#pragma unroll
    for (int j = 1; j < J; ++j) {
      lring[j] = p;
      p += 3 * m3_ex<J>(j) * m3_ey<J>(j);
    }
  }
  const int nx = d.nx, ny = d.ny, nz = d.nz;
  const int64_t plane = (int64_t)nx * ny;
  const int tx = blockIdx.x % d.tiles_x, ty = blockIdx.x / d.tiles_x;
  const int x0 = tx * M3_TX, y0 = ty * M3_TY;
  const int z0 = blockIdx.y * d.Z, z1 = min(nz, z0 + d.Z);
  if (z0 >= nz) return;
  const int tz0 = max(0, z0 - J), tsrc1 = min(nz, z1 + J);  // source planes [tz0, tsrc1)
  const int tid = threadIdx.x;
  const double sc = d.scale ? __ldg(d.scale) : 1.0;
  const bool scaled = d.scale != nullptr;

  auto load_plane = [&](int q) {  // source plane q of the extended tile into its ring slot
    double* dst = ring0 + (size_t)(q % M3_RS) * E0;
    const double* srcp = d.src + (int64_t)q * plane;
    for (int e = tid; e < E0; e += M3_NT) {
      const int ex = e % E0X, ey = e / E0X;
      const int gx = x0 - J + ex, gy = y0 - J + ey;
      const bool in = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
      cp_async8_zfill(dst + e, in ? srcp + (int64_t)gy * nx + gx : srcp, in);
    }
  };
  // prologue: planes tz0 .. tz0 + PF - 1 in flight (one commit group per plane slot, possibly empty)
#pragma unroll
  for (int i = 0; i < M3_PF; ++i) {
    if (tz0 + i < tsrc1) load_plane(tz0 + i);
    cp_async_commit();
  }
  // step t: level j at plane t - j (level J's last plane z1 - 1 at step z1 - 1 + J)
  for (int t = tz0; t <= z1 - 1 + J; ++t) {
    // plane t + PF in flight, plane t landed (its group is PF groups back)
    if (t + M3_PF < tsrc1) load_plane(t + M3_PF);
    cp_async_commit();
    cp_async_wait<M3_PF>();
    __syncthreads();
#pragma unroll
    for (int j = 1; j <= J; ++j) {
      const int p = t - j;  // this step's plane of level j
      const int lo = max(0, z0 - (J - j)), hi = min(nz, z1 + (J - j));
      if (p >= lo && p < hi) {
        const int EX = M3_TX + 2 * (J - j), EY = M3_TY + 2 * (J - j);
        const int PX = EX + 2;  // previous level's extent width
        const int off = J - j;  // this level's extent starts off points before the tile
        // previous level's planes p-1, p, p+1
        const double* pm;
        const double* pc;
        const double* pp;
        if (j == 1) {
          pm = ring0 + (size_t)(((p - 1) % M3_RS + M3_RS) % M3_RS) * E0;
          pc = ring0 + (size_t)(p % M3_RS) * E0;
          pp = ring0 + (size_t)((p + 1) % M3_RS) * E0;
        } else {
          const int PE = PX * (EY + 2);
          pm = lring[j - 1] + (size_t)(((p - 1) % 3 + 3) % 3) * PE;
          pc = lring[j - 1] + (size_t)(p % 3) * PE;
          pp = lring[j - 1] + (size_t)((p + 1) % 3) * PE;
        }
        double* cur = j < J ? lring[j] + (size_t)(p % 3) * EX * EY : nullptr;
        const bool hz0 = p > 0, hz1 = p + 1 < nz;
        const bool store = p >= z0 && p < z1;
        for (int e = tid; e < EX * EY; e += M3_NT) {
          const int ex = e % EX, ey = e / EX;
          const int gx = x0 - off + ex, gy = y0 - off + ey;
          if (gx < 0 || gx >= nx || gy < 0 || gy >= ny) continue;
          const int q = (ey + 1) * PX + (ex + 1);  // this point in the previous level's extent
          auto val = [&](const double* pl, int o) {
            const double v = pl[q + o];
            return j == 1 && scaled ? __dmul_rn(v, sc) : v;
          };
          double a = 0.0;
          if (hz0) a = __dadd_rn(a, __dmul_rn(d.c[0], val(pm, 0)));
          if (gy > 0) a = __dadd_rn(a, __dmul_rn(d.c[1], val(pc, -PX)));
          if (gx > 0) a = __dadd_rn(a, __dmul_rn(d.c[2], val(pc, -1)));
          const double vc = val(pc, 0);
          a = __dadd_rn(a, __dmul_rn(d.c[3], vc));
          if (gx + 1 < nx) a = __dadd_rn(a, __dmul_rn(d.c[4], val(pc, 1)));
          if (gy + 1 < ny) a = __dadd_rn(a, __dmul_rn(d.c[5], val(pc, PX)));
          if (hz1) a = __dadd_rn(a, __dmul_rn(d.c[6], val(pp, 0)));
          if (cur) cur[e] = a;
          const bool interior = ex >= off && ex < off + M3_TX && ey >= off && ey < off + M3_TY;
          if (store && interior) {
            const int64_t gp = (int64_t)p * plane + (int64_t)gy * nx + gx;
            if (d.out[j]) d.out[j][gp] = a;
            if (j == 1 && d.out[0]) d.out[0][gp] = vc;  // level 0 = src * scale as stored
          }
        }
      }
      __syncthreads();
    }
  }
  cp_async_wait<0>();
}

template <int J>
void run_mpk3t(Ctx& c, Mpk3Desc& dd) {
  const int tiles_x = (dd.nx + M3_TX - 1) / M3_TX, tiles_y = (dd.ny + M3_TY - 1) / M3_TY;
  const int tiles = tiles_x * tiles_y;
  // about two resident CTAs per SM: z chunks of at least 8 J planes
  int zc = std::max(1, (2 * c.sm_count + tiles - 1) / tiles);
  int Z = (dd.nz + zc - 1) / zc;
  Z = std::max(Z, std::min(dd.nz, 8 * J));
  dd.Z = Z;
  dd.tiles_x = tiles_x;
  const size_t smem = sizeof(double) * (size_t)m3_smem_doubles<J>();
  ensure_smem(k_mpk3t<J>, smem);
  launch_k(c, k_mpk3t<J>, dim3(tiles, (dd.nz + Z - 1) / Z), M3_NT, smem, dd);
}

}  // namespace

bool launch_mpk3(Ctx& c, const DevOp& op, const double* src, const double* scale, double* const* out, int J,
                 const int* halt, const int* cond, const char* name) {
  if (op.dim != 3 || op.kind != kStencilConst || op.halo_rows != 0 || J < 1 || J > 4) return false;
  Mpk3Desc d;
  std::memset(&d, 0, sizeof d);
  d.nx = (int)op.nx;
  d.ny = (int)op.ny;
  d.nz = (int)op.nz;
  for (int t = 0; t < 7; ++t) d.c[t] = op.coef[t];
  d.src = src;
  d.scale = scale;
  int nout = 0;
  for (int j = 0; j <= J; ++j) {
    d.out[j] = out[j];
    nout += out[j] != nullptr;
  }
  d.halt = halt;
  d.cond = cond;
  Launch lh(c, name, 8.0 * (double)op.n * (1 + nout));
  switch (J) {
    case 1: run_mpk3t<1>(c, d); break;
    case 2: run_mpk3t<2>(c, d); break;
    case 3: run_mpk3t<3>(c, d); break;
    default: run_mpk3t<4>(c, d); break;
  }
  CK(cudaGetLastError());
  return true;
}

}  // namespace skc
