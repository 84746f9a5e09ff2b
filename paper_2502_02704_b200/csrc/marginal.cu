// Marginal recursion: the relax tables of every fine step without sweeping f.
//
// Let M_xy[i][jx][jy] = sum_z w_z f[i][jx][jy][jz] and M_xz = sum_y w_y f
// (w = 1, or the trapezoidal end weights).  Both parts of one fine step act on
// a v_x row with coefficients that do not depend on (v_y, v_z):
//   * the upwind x transport (ref/kinetic.py:110-112) is linear with
//     coefficient c_x[jx];
//   * the BGK relaxation (ref/kinetic.py:130-134) is f = r f* + r ls M with a
//     separable Maxwellian M = (g_x amp) g_y g_z (ref/lifting.py:47-57).
// Summing over v_z (resp. v_y) therefore commutes with both, and
//   M(f*_s)(i) = T_x[ r M(f*_{s-1}) + r ls (g_x amp) g_y S_z ](i)
// with S_z = sum_z w_z g_z (resp. g_z S_y for M_xz), evaluated on the cell and
// its upwind neighbour.  The 1-D marginals of f*_s are row / column sums of
// M(f*_s), so the moments and the relax table R_s of every step follow
// (finalize_impl.cuh, ref/moments.py:91-113) from data 2/N_v the size of f.
// The multi-step sweep (fsweep.cu) then applies the precomputed tables.
//
// Rounding: the sums are taken in a different order than a direct reduction of
// f*_s (transport-then-sum vs sum-then-transport), a few ulps per step, far
// inside the 1e-10 parity bound.  Each marginal entry is a fixed tree, the
// same for every index and its mirror, so even data keeps an exactly zero
// folded first moment (ref/moments.py:80-88).
#include <cuda_runtime.h>

#include "common.cuh"
#include "finalize_impl.cuh"
#include "ptx.cuh"

namespace pbgk {

constexpr int kMargThreads = 256;

__device__ __forceinline__ double wq(int trap, int j, int n) {
  return (trap && (j == 0 || j == n - 1)) ? 0.5 : 1.0;
}

// One CTA per x cell i.  Shared memory: the three table rows (cells i-1, i,
// i+1), the per-warp column partials, then the finalize scratch.
__global__ void __launch_bounds__(kMargThreads) marg_kernel(const MargArgs m, const FinalArgs f) {
  extern __shared__ double sm[];
  __shared__ double sh[16];
  __shared__ double ssum[6];  // S_y, S_z of cells l, c, r
  const int i = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = m.nx, nvx = m.nvx, nvy = m.nvy, nvz = m.nvz;
  const int TL = f.TL;
  const int MS = nvx * (nvy + nvz);
  double* rows = sm;                  // [3][TL]
  double* Mn = rows + 3 * TL;         // [NW][nvy + nvz] column partials
  double* fs = Mn + (kMargThreads / 32) * (nvy + nvz);  // finalize scratch: mx | my | mz | ...
  // neighbour cells: ghost -1 = absorbing zero; periodic wrap; outflow edge
  auto nb = [&](int j) {
    if (j >= 0 && j < nx) return j;
    if (m.bc == 1) return (j + nx) % nx;
    if (m.bc == 2) return j < 0 ? 0 : nx - 1;
    return -1;
  };
  const int cl = nb(i - 1), cr = nb(i + 1);
  pdl_wait();  // tables and M(f*_{s-1}) come from the preceding kernels
  pdl_trigger();
  for (int q = 0; q < 3; ++q) {
    const int cc = q == 0 ? cl : (q == 1 ? i : cr);
    for (int j = tid; j < TL; j += kMargThreads)
      rows[q * TL + j] = (cc >= 0) ? m.tab_in[(size_t)cc * TL + j] : 0.0;
  }
  __syncthreads();
  if (warp < 6) {
    const int q = warp >> 1, ax = warp & 1;  // ax 0: S_y, 1: S_z
    const int n = ax == 0 ? nvy : nvz;
    const double* g = rows + q * TL + (ax == 0 ? f.gyo : f.gzo);
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s += (f.trap && (j == 0 || j == n - 1)) ? 0.5 * g[j] : g[j];
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) s += __shfl_xor_sync(0xffffffffu, s, w);
    if (lane == 0) ssum[warp] = s;
  }
  __syncthreads();
  const bool synth = (m.min == nullptr);
  const int nneg = nvx / 2;
  constexpr int NW = kMargThreads / 32;
  // warp w owns the v_x rows jx = w, w + NW, ...; lane owns columns
  // j2 = lane, lane + 32, ... of both parts.  m_x[jx] is the row's lane
  // partials (ascending j2) folded by an xor tree; the column marginals are
  // per-warp partials over the warp's rows (ascending jx) added in warp order.
  // Fixed trees, the same for every index and its mirror.
  double* mx = fs;
  double* my = mx + nvx;
  double* mz = my + nvy;
  double* colp = Mn;  // [NW][nvy + nvz] column partials
  const int ncol = nvy + nvz;
  constexpr int CPL = 4;  // columns per lane per part (nvy, nvz <= 128)
  double cs[2][CPL];
#pragma unroll
  for (int pz = 0; pz < 2; ++pz)
#pragma unroll
    for (int u = 0; u < CPL; ++u) cs[pz][u] = 0.0;
  for (int jx = warp; jx < nvx; jx += NW) {
    const double c = m.cx[jx];
    const bool down = jx < nneg;  // c_x < 0 exactly for jx < nvx/2 (ref/grid.py:100-103)
    const int qn = down ? 2 : 0;  // upwind neighbour: i+1 or i-1
    const int cn = down ? cr : cl;
    const double wx = wq(f.trap, jx, nvx);
    // per row: relax coefficients (cell, neighbour)
    const double* rc = rows + TL;
    const double* rn = rows + qn * TL;
    const double ac = (synth ? rc[1] : rc[0] * rc[1]) * rc[f.gxo + jx];
    const double an = (synth ? rn[1] : rn[0] * rn[1]) * rn[f.gxo + jx];
#pragma unroll
    for (int pz = 0; pz < 2; ++pz) {
      const int n2 = pz == 0 ? nvy : nvz;
      const int base = pz == 0 ? jx * nvy : nvx * nvy + jx * nvz;
      const int g2o = pz == 0 ? f.gyo : f.gzo;
      const double Sc = ssum[2 + (pz == 0 ? 1 : 0)], Sn = ssum[2 * qn + (pz == 0 ? 1 : 0)];
      double mc[CPL], mv[CPL];
#pragma unroll
      for (int u = 0; u < CPL; ++u) {
        const int j2 = lane + 32 * u;
        mc[u] = mv[u] = 0.0;
        if (!synth && j2 < n2) {
          mc[u] = __ldcg(m.min + (size_t)i * MS + base + j2);
          if (cn >= 0) mv[u] = __ldcg(m.min + (size_t)cn * MS + base + j2);
        }
      }
      double rs = 0.0;
#pragma unroll
      for (int u = 0; u < CPL; ++u) {
        const int j2 = lane + 32 * u;
        if (j2 < n2) {
          const double gmc = ac * rc[g2o + j2];
          const double x = synth ? gmc * Sc : fma(gmc, Sc, rc[0] * mc[u]);
          double xn = 0.0;
          if (cn >= 0) {
            const double gmn = an * rn[g2o + j2];
            xn = synth ? gmn * Sn : fma(gmn, Sn, rn[0] * mv[u]);
          }
          const double fl = __dmul_rn(c, x), pv = __dmul_rn(c, xn);
          const double d = down ? __dsub_rn(pv, fl) : __dsub_rn(fl, pv);
          const double o = __dsub_rn(x, __dmul_rn(m.dtdx, d));
          m.mout[(size_t)i * MS + base + j2] = o;
          if (pz == 0) rs += f.trap ? o * wq(1, j2, n2) : o;
          cs[pz][u] += f.trap ? o * wx : o;
        }
      }
      if (pz == 0) {
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, w);
        if (lane == 0) mx[jx] = rs;
      }
    }
  }
#pragma unroll
  for (int pz = 0; pz < 2; ++pz)
#pragma unroll
    for (int u = 0; u < CPL; ++u) {
      const int j2 = lane + 32 * u;
      if (j2 < (pz == 0 ? nvy : nvz)) colp[warp * ncol + (pz == 0 ? 0 : nvy) + j2] = cs[pz][u];
    }
  __syncthreads();
  for (int t = tid; t < ncol; t += kMargThreads) {
    double s2 = 0.0;
    for (int w = 0; w < NW; ++w) s2 += colp[w * ncol + t];
    (t < nvy ? my[t] : mz[t - nvy]) = s2;
  }
  __syncthreads();
  finalize_cell<true>(f, i, fs, sh);
}

size_t marg_smem_bytes(int nvx, int nvy, int nvz, int TL) {
  if (nvy > 128 || nvz > 128) return ~(size_t)0;  // columns per lane (CPL) bound
  return (size_t)(3 * TL + (kMargThreads / 32) * (nvy + nvz) + 2 * (nvx + nvy + nvz)) * sizeof(double);
}

cudaError_t launch_marg(const MargArgs& m, const FinalArgs& f, cudaStream_t st) {
  const size_t smem = marg_smem_bytes(m.nvx, m.nvy, m.nvz, f.TL);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(marg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return launch_pdl(marg_kernel, m.nx, kMargThreads, smem, st, m, f);
}

}  // namespace pbgk
