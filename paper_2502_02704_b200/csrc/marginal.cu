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
// Two kernels per step: marg_rows_kernel (one CTA per cell and chunk of v_x
// rows: the recursion itself, streaming, every load of a row in flight at
// once) writes M(f*_s), the row sums m_x and per-chunk column partials;
// marg_final_kernel (one CTA per cell) adds the chunk partials in chunk order
// into m_y, m_z and runs the finalize (moments -> R_s).
//
// Rounding: the sums are taken in a different order than a direct reduction of
// f*_s (transport-then-sum vs sum-then-transport), a few ulps per step, far
// inside the 1e-10 parity bound.  Each marginal entry is a fixed tree, the
// same for every index and its mirror, so even data keeps an exactly zero
// folded first moment (ref/moments.py:80-88).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "finalize_impl.cuh"
#include "ptx.cuh"

namespace pbgk {

constexpr int kRowThreads = 256;  // 8 warps, rpc / 8 rows each
constexpr int kFinThr = 128;

__device__ __forceinline__ double wq(int trap, int j, int n) {
  return (trap && (j == 0 || j == n - 1)) ? 0.5 : 1.0;
}

__device__ __forceinline__ int nb_cell(int j, int nx, int bc) {
  if (j >= 0 && j < nx) return j;
  if (bc == 1) return (j + nx) % nx;
  if (bc == 2) return j < 0 ? 0 : nx - 1;
  return -1;  // absorbing ghost: zero
}

// Cell blockIdx.x, v_x rows [blockIdx.y * rpc, +rpc).  Warp w takes rows
// w, w + 8, ... of the chunk; lane takes columns lane + 32 u of both parts.
// m_x[jx] = the row's lane partials (ascending u) folded by an xor tree;
// column partials over the chunk's rows in ascending jx.
template <int RPW, int kCPL, bool TRAP>
__global__ void __launch_bounds__(kRowThreads) marg_rows_kernel(const MargArgs m) {
  extern __shared__ double sm[];
  __shared__ double ssum[6];  // S_y, S_z of cells l, c, r
  const int i = blockIdx.x, chunk = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = m.nx, nvx = m.nvx, nvy = m.nvy, nvz = m.nvz;
  const int ncol = nvy + nvz, MS = nvx * ncol;
  const int cl = nb_cell(i - 1, nx, m.bc), cr = nb_cell(i + 1, nx, m.bc);
  // shared: per cell q (l, c, r): r, ls, then g_y | g_z; then per-row column values
  double* g = sm;                      // [3][2 + ncol]
  double* cp = g + 3 * (2 + ncol);     // [rpc][ncol]
  pdl_wait();  // tables and M(f*_{s-1}) come from the preceding kernels
  pdl_trigger();
  for (int q = 0; q < 3; ++q) {
    const int cc = q == 0 ? cl : (q == 1 ? i : cr);
    for (int k = tid; k < 2 + ncol; k += kRowThreads) {
      const int col = k < 2 ? k : (k - 2 < nvy ? m.gyo + k - 2 : m.gzo + k - 2 - nvy);
      g[q * (2 + ncol) + k] = cc >= 0 ? __ldg(m.tab_in + (size_t)cc * m.TL + col) : 0.0;
    }
  }
  __syncthreads();
  if (warp < 6) {
    const int q = warp >> 1, ax = warp & 1;  // ax 0: S_y, 1: S_z
    const int n = ax == 0 ? nvy : nvz;
    const double* gv = g + q * (2 + ncol) + 2 + (ax == 0 ? 0 : nvy);
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s += (TRAP && (j == 0 || j == n - 1)) ? 0.5 * gv[j] : gv[j];
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) s += __shfl_xor_sync(0xffffffffu, s, w);
    if (lane == 0) ssum[warp] = s;
  }
  __syncthreads();
  const bool synth = (m.min == nullptr);
  const int nneg = nvx / 2;
  const int r0 = chunk * m.rpc;
  // all loads of the warp's rows first
  double mc[RPW][2][kCPL], mv[RPW][2][kCPL];
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int jx = r0 + warp + 8 * k;
    const int cn = jx < nneg ? cr : cl;
#pragma unroll
    for (int pz = 0; pz < 2; ++pz) {
      const int n2 = pz == 0 ? nvy : nvz;
      const size_t base = pz == 0 ? (size_t)jx * nvy : (size_t)nvx * nvy + (size_t)jx * nvz;
#pragma unroll
      for (int u = 0; u < kCPL; ++u) {
        const int j2 = lane + 32 * u;
        mc[k][pz][u] = mv[k][pz][u] = 0.0;
        if (!synth && jx < nvx && j2 < n2) {
          mc[k][pz][u] = __ldcg(m.min + (size_t)i * MS + base + j2);
          if (cn >= 0) mv[k][pz][u] = __ldcg(m.min + (size_t)cn * MS + base + j2);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int jx = r0 + warp + 8 * k;
    const int rl = warp + 8 * k;  // row within the chunk
    if (jx >= nvx || rl >= m.rpc) continue;
    const double c = m.cx[jx];
    const bool down = jx < nneg;  // c_x < 0 exactly for jx < nvx/2 (ref/grid.py:100-103)
    const int qn = down ? 2 : 0;  // upwind neighbour: i+1 or i-1
    const bool ghost = (down ? cr : cl) < 0;
    const double* gc = g + (2 + ncol);
    const double* gn = g + qn * (2 + ncol);
    // relax coefficient of the row: (r ls g_x amp), or (ls g_x amp) for the lift
    const double gxc = __ldg(m.tab_in + (size_t)i * m.TL + m.gxo + jx);
    const double gxn = ghost ? 0.0 : __ldg(m.tab_in + (size_t)(down ? cr : cl) * m.TL + m.gxo + jx);
    const double ac = (synth ? gc[1] : gc[0] * gc[1]) * gxc;
    const double an = (synth ? gn[1] : gn[0] * gn[1]) * gxn;
    const double wx = wq(TRAP, jx, nvx);
    double rs = 0.0;
#pragma unroll
    for (int pz = 0; pz < 2; ++pz) {
      const int n2 = pz == 0 ? nvy : nvz;
      const size_t base = pz == 0 ? (size_t)jx * nvy : (size_t)nvx * nvy + (size_t)jx * nvz;
      const double Sc = ssum[2 + (pz == 0 ? 1 : 0)], Sn = ssum[2 * qn + (pz == 0 ? 1 : 0)];
      const int go = 2 + (pz == 0 ? 0 : nvy);
#pragma unroll
      for (int u = 0; u < kCPL; ++u) {
        const int j2 = lane + 32 * u;
        if (j2 < n2) {
          const double gmc = ac * gc[go + j2];
          const double x = synth ? gmc * Sc : fma(gmc, Sc, gc[0] * mc[k][pz][u]);
          double xn = 0.0;
          if (!ghost) {
            const double gmn = an * gn[go + j2];
            xn = synth ? gmn * Sn : fma(gmn, Sn, gn[0] * mv[k][pz][u]);
          }
          const double fl = __dmul_rn(c, x), pv = __dmul_rn(c, xn);
          const double d = down ? __dsub_rn(pv, fl) : __dsub_rn(fl, pv);
          const double o = __dsub_rn(x, __dmul_rn(m.dtdx, d));
          m.mout[(size_t)i * MS + base + j2] = o;
          if (pz == 0) rs += TRAP ? o * wq(1, j2, n2) : o;
          cp[rl * ncol + (pz == 0 ? 0 : nvy) + j2] = TRAP ? o * wx : o;
        }
      }
    }
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, w);
    if (lane == 0) m.mx[(size_t)i * nvx + jx] = rs;
  }
  __syncthreads();
  const int nrow = min(m.rpc, nvx - r0);
  for (int t = tid; t < ncol; t += kRowThreads) {
    double s2 = 0.0;
    for (int rl = 0; rl < nrow; ++rl) s2 += cp[rl * ncol + t];
    m.colp[((size_t)i * m.nrc + chunk) * ncol + t] = s2;
  }
}

// One CTA per cell: m_y, m_z = chunk partials in chunk order, then the
// moments and R_s (finalize_impl.cuh).
__global__ void __launch_bounds__(kFinThr) marg_final_kernel(const MargArgs m, const FinalArgs f) {
  extern __shared__ double sm[];
  __shared__ double sh[16];
  const int i = blockIdx.x, tid = threadIdx.x;
  const int nvx = m.nvx, ncol = m.nvy + m.nvz;
  pdl_wait();
  pdl_trigger();
  for (int t = tid; t < nvx; t += kFinThr) sm[t] = __ldcg(m.mx + (size_t)i * nvx + t);
  for (int t = tid; t < ncol; t += kFinThr) {
    double s2 = 0.0;
    for (int c = 0; c < m.nrc; ++c) s2 += __ldcg(m.colp + ((size_t)i * m.nrc + c) * ncol + t);
    sm[nvx + t] = s2;  // m_y | m_z follow m_x
  }
  __syncthreads();
  finalize_cell<true>(f, i, sm, sh);
}

// rows per CTA (8 warps x RPW): 8 for tiny grids, else PBGK_MARG_RPC (16 or
// 32; 32 only for <= 64 columns)
static int marg_rpc(int nvx, int ncolmax) {
  static const int env = getenv("PBGK_MARG_RPC") ? atoi(getenv("PBGK_MARG_RPC")) : 16;
  if (nvx <= 8) return 8;
  if (env >= 32 && nvx >= 32 && ncolmax <= 64) return 32;
  return 16;
}

size_t marg_smem_bytes(int nvx, int nvy, int nvz, int TL) {
  (void)TL;
  if (nvy > 128 || nvz > 128) return ~(size_t)0;  // columns per lane bound (4)
  const int ncol = nvy + nvz;
  return (size_t)(3 * (2 + ncol) + marg_rpc(nvx, std::max(nvy, nvz)) * ncol) * sizeof(double);
}

size_t marg_scratch_doubles(int nx, int nvx, int nvy, int nvz) {
  const int rpc = marg_rpc(nvx, std::max(nvy, nvz)), nrc = (nvx + rpc - 1) / rpc;
  return (size_t)nx * nvx + (size_t)nx * nrc * (nvy + nvz);
}

cudaError_t launch_marg(const MargArgs& m0, const FinalArgs& f, double* scratch, cudaStream_t st) {
  MargArgs m = m0;
  m.rpc = marg_rpc(m.nvx, std::max(m.nvy, m.nvz));
  m.nrc = (m.nvx + m.rpc - 1) / m.rpc;
  m.mx = scratch;
  m.colp = scratch + (size_t)m.nx * m.nvx;
  m.TL = f.TL;
  m.gxo = f.gxo;
  m.gyo = f.gyo;
  m.gzo = f.gzo;
  m.trap = f.trap;
  const size_t smem = marg_smem_bytes(m.nvx, m.nvy, m.nvz, f.TL);
  // columns per lane: the longer of the two column axes over 32 lanes
  const int cpl = (std::max(m.nvy, m.nvz) + 31) / 32;
  void (*rk)(const MargArgs) = nullptr;
#define PBGK_RK(R, C) (m.trap ? marg_rows_kernel<R, C, true> : marg_rows_kernel<R, C, false>)
  if (m.rpc == 8) rk = cpl <= 1 ? PBGK_RK(1, 1) : (cpl == 2 ? PBGK_RK(1, 2) : PBGK_RK(1, 4));
  else if (m.rpc == 16) rk = cpl <= 1 ? PBGK_RK(2, 1) : (cpl == 2 ? PBGK_RK(2, 2) : PBGK_RK(2, 4));
  else rk = cpl <= 1 ? PBGK_RK(4, 1) : (cpl == 2 ? PBGK_RK(4, 2) : PBGK_RK(2, 4));
#undef PBGK_RK
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(m.nx, m.nrc);
  cfg.blockDim = dim3(kRowThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = getenv("PBGK_NO_PDL") ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, rk, m);
  if (e != cudaSuccess) return e;
  const size_t fsm = (size_t)2 * (m.nvx + m.nvy + m.nvz) * sizeof(double);
  return launch_pdl(marg_final_kernel, m.nx, kFinThr, fsm, st, m, f);
}

}  // namespace pbgk
