// Moment recursion: the relax tables of every fine step without sweeping f.
//
// Both parts of one fine step act on a v_x row with coefficients that do not
// depend on (v_y, v_z):
//   * the upwind x transport (ref/kinetic.py:110-112) is linear with
//     coefficient c_x[jx];
//   * the BGK relaxation (ref/kinetic.py:130-134) is f = r f* + r ls M with a
//     separable Maxwellian M = (g_x amp) g_y g_z (ref/lifting.py:47-57).
// So any weighted sum of f over (v_y, v_z) commutes with both.  Per x cell
// and v_x row the recursion carries five of them (w = 1, or the trapezoidal
// end weights):
//   Q0 = sum_yz f                          (= the marginal m_x[jx])
//   Q1 = sum_z sum_{y<h} c_y (f_y - f_{n-1-y})   (folded first moment in v_y)
//   Q2 = sum_yz c_y^2 f,   Q3, Q4 = the same in v_z
// and one step is  Q_k(f*_s)(i) = T_x[ r Q_k(f*_{s-1}) + r ls (g_x amp) G_k ](i)
// on the cell and its upwind neighbour, G_k the matching sums of g_y g_z of
// the table row (G_0 = S_y0 S_z0, G_1 = S_y1 S_z0, ...).  From Q(f*_s) the
// moments follow (ref/moments.py:91-113): rho and u_x, the x part of theta
// exactly as the reference (marginal m_x, folded first moment, two-pass
// second moment); u_y = sum Q1 dvol / rho; the y part of theta
// sum (c_y - u_y)^2 m_y = Q2 - 2 u_y Q1 + u_y^2 Q0 (one-pass; a few ulps for
// the low-Mach states here, relative error ~ eps (1 + u^2/theta) in general),
// likewise z.  Then R_s = the table row of finalize_impl.cuh, same formulas.
//
// The recursion moves 5 N_vx doubles per cell and step -- about 5/N_v^2 of
// f -- and one warp per cell does the whole step (no CTA barrier).  The
// multi-step sweep (fsweep.cu) applies the tables to f; the window's final
// projection is taken from f itself (the reference-order marginal sweep).
//
// Folded sums keep an exactly zero velocity for even data (ref/moments.py:
// 80-88): Q1, Q3 and G_1, G_3 vanish identically and the transport keeps
// them at zero.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace pbgk {

constexpr int kWarpsPerCta = 8;

__device__ __forceinline__ double wsum(double x) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) x += __shfl_xor_sync(0xffffffffu, x, w);
  return x;
}

__device__ __forceinline__ double wq(bool trap, int j, int n) {
  return (trap && (j == 0 || j == n - 1)) ? 0.5 : 1.0;
}

__device__ __forceinline__ int nb_cell(int j, int nx, int bc) {
  if (j >= 0 && j < nx) return j;
  if (bc == 1) return (j + nx) % nx;
  if (bc == 2) return j < 0 ? 0 : nx - 1;
  return -1;  // absorbing ghost: zero
}

// Sums of one axis' g over the lanes of a warp (lane-strided, xor tree):
// s0 = sum w g, s1 = sum_{j<h} w c (g_j - g_{n-1-j}), s2 = sum w c^2 g.
__device__ __forceinline__ void axis_sums(const double* g, const double* c, int n, bool trap, int lane,
                                          double& s0, double& s1, double& s2) {
  s0 = s1 = s2 = 0.0;
  const int h = n / 2;
  for (int j = lane; j < n; j += 32) {
    const double w = wq(trap, j, n);
    s0 += w == 0.5 ? 0.5 * g[j] : g[j];
    s2 += (w * c[j]) * (c[j] * g[j]);
    if (j < h) s1 += (w * c[j]) * (g[j] - g[n - 1 - j]);
  }
  s0 = wsum(s0);
  s1 = wsum(s1);
  s2 = wsum(s2);
}

// G sums of the table rows of a lift (the window's first step): one warp per
// cell.  gsum[i] = {S_y0, S_y1, S_y2, S_z0, S_z1, S_z2}.
__global__ void __launch_bounds__(32 * kWarpsPerCta) mrec_init_kernel(const MargArgs m) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  const int w = blockIdx.y;
  pdl_wait();
  pdl_trigger();
  if (i >= m.nx) return;
  const double* row = m.tab_in + w * m.t_ws + (size_t)i * m.TL;
  double a0, a1, a2, b0, b1, b2;
  axis_sums(row + m.gyo, m.cy, m.nvy, m.trap, lane, a0, a1, a2);
  axis_sums(row + m.gzo, m.cz, m.nvz, m.trap, lane, b0, b1, b2);
  if (lane == 0) {
    double* g = m.gsum_out + w * m.g_ws + (size_t)i * 6;
    g[0] = a0; g[1] = a1; g[2] = a2; g[3] = b0; g[4] = b1; g[5] = b2;
  }
}

// One recursion step of cell i of window w by the calling warp (step `step`;
// JPL = v_x rows per lane; mxs: nvx doubles of warp-private shared memory).
// Every global read of data written by earlier steps goes through L2
// (ld.global.cg): the persistent kernel below runs several steps per launch.
template <int JPL, bool TRAP>
__device__ __forceinline__ void mrec_cell(const MargArgs& m, const FinalArgs& f, int step, int i, int w,
                                          double* mxs) {
  const int lane = threadIdx.x & 31;
  const int nx = m.nx, nvx = m.nvx, nvy = m.nvy, nvz = m.nvz;
  if (m.nst != nullptr && step > m.nst[w]) return;  // this window has fewer steps
  const double* qmin = m.min ? m.min + w * m.q_ws : nullptr;
  double* qout = m.mout + w * m.q_ws;
  const double* tab_in = m.tab_in + w * m.t_ws;
  double* tab_out = f.tab + w * m.t_ws;
  const double* gsum_in = m.gsum_in + w * m.g_ws;
  double* gsum_out = m.gsum_out + w * m.g_ws;
  const double dt = m.dts ? m.dts[w] : f.dt;
  const double dtdx = m.dts ? dt / m.dx : m.dtdx;  // the host's dt / dx
  ErrKey* err = m.errw ? m.errw + w : f.err;
  const int cl = nb_cell(i - 1, nx, m.bc), cr = nb_cell(i + 1, nx, m.bc);
  const bool synth = (qmin == nullptr);
  const int nneg = nvx / 2;
  const int QS = 5 * nvx;
  // per cell q (l, c, r): r, ls and G_0..G_4 (uniform over the warp)
  double rq[3], lq[3], G[3][5];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int cc = q == 0 ? cl : (q == 1 ? i : cr);
    rq[q] = lq[q] = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) G[q][k] = 0.0;
    if (cc >= 0) {
      const double* row = tab_in + (size_t)cc * m.TL;
      const double* gs = gsum_in + (size_t)cc * 6;
      rq[q] = __ldcg(row);
      lq[q] = __ldcg(row + 1);
      const double sy0 = __ldcg(gs), sy1 = __ldcg(gs + 1), sy2 = __ldcg(gs + 2);
      const double sz0 = __ldcg(gs + 3), sz1 = __ldcg(gs + 4), sz2 = __ldcg(gs + 5);
      G[q][0] = sy0 * sz0;
      G[q][1] = sy1 * sz0;
      G[q][2] = sy2 * sz0;
      G[q][3] = sz1 * sy0;
      G[q][4] = sz2 * sy0;
    }
  }
  // loads first: Q of the cell and of the row's upwind neighbour
  double qc[5][JPL], qn[5][JPL], gxc[JPL], gxn[JPL];
#pragma unroll
  for (int u = 0; u < JPL; ++u) {
    const int jx = lane + 32 * u;
    const int cn = jx < nneg ? cr : cl;
    gxc[u] = gxn[u] = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) qc[k][u] = qn[k][u] = 0.0;
    if (jx < nvx) {
      gxc[u] = __ldcg(tab_in + (size_t)i * m.TL + m.gxo + jx);
      if (cn >= 0) gxn[u] = __ldcg(tab_in + (size_t)cn * m.TL + m.gxo + jx);
      if (!synth) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          qc[k][u] = __ldcg(qmin + (size_t)i * QS + k * nvx + jx);
          if (cn >= 0) qn[k][u] = __ldcg(qmin + (size_t)cn * QS + k * nvx + jx);
        }
      }
    }
  }
  // v_x field term (ref/kinetic.py:114-123, linear in the v_x rows): the
  // cell's relaxed rows go through warp-private shared memory first
  const bool field = m.E != nullptr;
  double cpf = 0.0, cmf = 0.0;
  double* xs = mxs + nvx;  // [5][nvx]
  if (field) {
    const double hE = __dmul_rn(0.5, m.E[i]);
    cpf = hE + m.half_emax;
    cmf = hE - m.half_emax;
#pragma unroll
    for (int u = 0; u < JPL; ++u) {
      const int jx = lane + 32 * u;
      if (jx >= nvx) continue;
      const double ac = (synth ? lq[1] : rq[1] * lq[1]) * gxc[u];
#pragma unroll
      for (int k = 0; k < 5; ++k)
        xs[k * nvx + jx] = synth ? ac * G[1][k] : fma(ac, G[1][k], rq[1] * qc[k][u]);
    }
    __syncwarp();
  }
  // the step: relax (cell and upwind neighbour), upwind transport, in the
  // one-step sweep's order; then the jx sums of the moments
  double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0, q4 = 0.0;  // sum_jx w_x Q_k
  int bad = 0;
#pragma unroll
  for (int u = 0; u < JPL; ++u) {
    const int jx = lane + 32 * u;
    if (jx >= nvx) continue;
    const bool down = jx < nneg;  // c_x < 0 exactly for jx < nvx/2 (ref/grid.py:100-103)
    const bool ghost = (down ? cr : cl) < 0;
    const double c = m.cx[jx];
    // neighbour constants by selects (a runtime index would spill to local memory)
    const double rn = down ? rq[2] : rq[0], ln = down ? lq[2] : lq[0];
    const double ac = (synth ? lq[1] : rq[1] * lq[1]) * gxc[u];
    const double an = (synth ? ln : rn * ln) * gxn[u];
    const double wx = wq(TRAP, jx, nvx);
    double o[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const double Gn = down ? G[2][k] : G[0][k];
      const double x = synth ? ac * G[1][k] : fma(ac, G[1][k], rq[1] * qc[k][u]);
      const double xn = ghost ? 0.0 : (synth ? an * Gn : fma(an, Gn, rn * qn[k][u]));
      const double fl = __dmul_rn(c, x), pv = __dmul_rn(c, xn);
      const double d = down ? __dsub_rn(pv, fl) : __dsub_rn(fl, pv);
      o[k] = __dsub_rn(x, __dmul_rn(dtdx, d));
      if (field) {
        // Rusanov flux on interior v_x faces of the relaxed rows, zero at the
        // cube faces: G(lo, hi) = cp lo + cm hi (the sweep's reassociation)
        const double ghi = jx + 1 < nvx ? fma(cpf, x, cmf * xs[k * nvx + jx + 1]) : 0.0;
        const double glo = jx > 0 ? fma(cpf, xs[k * nvx + jx - 1], cmf * x) : 0.0;
        o[k] = fma(-(dt / m.dvx), ghi - glo, o[k]);  // the host's dt / dv_x
      }
      qout[(size_t)i * QS + k * nvx + jx] = o[k];
      bad |= !isfinite(o[k]);
    }
    mxs[jx] = o[0];
    q0 += TRAP ? o[0] * wx : o[0];
    q1 += TRAP ? o[1] * wx : o[1];
    q2 += TRAP ? o[2] * wx : o[2];
    q3 += TRAP ? o[3] * wx : o[3];
    q4 += TRAP ? o[4] * wx : o[4];
  }
  __syncwarp();
  q0 = wsum(q0);
  q1 = wsum(q1);
  q2 = wsum(q2);
  q3 = wsum(q3);
  q4 = wsum(q4);
  const int nonfinite = __any_sync(0xffffffffu, bad);
  // moments (ref/moments.py:100-112): rho and u_x from m_x as the reference
  // (q0 is sum_jx w_x m_x in the finalize's lane order), folded first moment
  const double* cx = m.cx;
  double s1 = 0.0;
  const int h = nvx / 2;
  for (int j = lane; j < h; j += 32)
    s1 += (mxs[j] - mxs[nvx - 1 - j]) * (TRAP ? cx[j] * wq(true, j, nvx) : cx[j]);
  s1 = wsum(s1);
  const double dvol = f.dvol;
  const double rho = q0 * dvol;
  const double u0 = (s1 * dvol) / rho;
  const double u1 = (q1 * dvol) / rho;
  const double u2 = (q3 * dvol) / rho;
  double ex = 0.0;
  for (int j = lane; j < nvx; j += 32) {
    const double d = cx[j] - u0;
    ex += (d * d) * (TRAP ? mxs[j] * wq(true, j, nvx) : mxs[j]);
  }
  ex = wsum(ex);
  const double ey = (q2 - 2.0 * u1 * q1) + (u1 * u1) * q0;
  const double ez = (q4 - 2.0 * u2 * q3) + (u2 * u2) * q0;
  const double e2 = ((0.0 + ex) + ey) + ez;
  const double th = (e2 * dvol) / (3.0 * rho);
  if (lane == 0) {
    if (rho <= 0.0) atomicMin(err, err_key(0, step, kErrProjectRho));
    if (rho <= 0.0 || th <= 0.0) atomicMin(err, err_key(0, step, kErrLiftState));
  }
  // the table row of R_s (finalize_impl.cuh, same expressions and sum order)
  const double inv2t = 1.0 / (2.0 * th);
  const double tt = 6.283185307179586 * th;
  const double amp = rho / (tt * sqrt(tt));  // (2 pi theta)^1.5, ref/lifting.py:50
  double* row = tab_out + (size_t)i * f.TL;
  double sxa = 0.0;
  for (int j = lane; j < nvx; j += 32) {
    const double d = cx[j] - u0;
    const double g = exp(-(d * d) * inv2t) * amp;
    sxa += (TRAP && (j == 0 || j == nvx - 1)) ? 0.5 * g : g;
    row[f.gxo + j] = g;
  }
  sxa = wsum(sxa);
  double a[2][3];
#pragma unroll
  for (int ax = 0; ax < 2; ++ax) {
    const int n = ax == 0 ? nvy : nvz;
    const double* c = ax == 0 ? m.cy : m.cz;
    const double ua = ax == 0 ? u1 : u2;
    const int off = ax == 0 ? f.gyo : f.gzo;
    const int hh = n / 2;
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int j = lane; j < n; j += 32) {
      const double d = c[j] - ua;
      const double g = exp(-(d * d) * inv2t);
      const double w = wq(TRAP, j, n);
      t0 += w == 0.5 ? 0.5 * g : g;
      t2 += (w * c[j]) * (c[j] * g);
      if (j < hh) {
        const double dm = c[n - 1 - j] - ua;
        t1 += (w * c[j]) * (g - exp(-(dm * dm) * inv2t));
      }
      row[off + j] = g;
    }
    a[ax][0] = wsum(t0);
    a[ax][1] = wsum(t1);
    a[ax][2] = wsum(t2);
  }
  for (int j = f.gyo + nvy + lane; j < f.gzo; j += 32) row[j] = 0.0;
  for (int j = f.gzo + nvz + lane; j < f.TL; j += 32) row[j] = 0.0;
  const double mass = ((sxa * a[0][0]) * a[1][0]) * dvol;
  const double scale = rho / mass;
  const double tau = f.tau_arr != nullptr ? f.tau_arr[i] : f.tau;
  const double lam = (dt * tau) / f.eps;
  const double r = 1.0 / (1.0 + lam);
  const double ls = lam * scale;
  if (lane == 0) {
    row[0] = r;
    row[1] = ls;
    double* gs = gsum_out + (size_t)i * 6;
    gs[0] = a[0][0]; gs[1] = a[0][1]; gs[2] = a[0][2];
    gs[3] = a[1][0]; gs[4] = a[1][1]; gs[5] = a[1][2];
    // f_s = R_s(f*_s) is finite iff f*_s and the table row are (BlowUpError(step))
    if (nonfinite || !isfinite(r) || !isfinite(ls) || !isfinite(amp) || !isfinite(u0) ||
        !isfinite(u1) || !isfinite(u2) || !isfinite(th))
      atomicMin(err, err_key(0, step, kErrNonFinite));
  }
}

#ifndef PBGK_MREC_MINB
#define PBGK_MREC_MINB 2  // 128 registers, 16 warps per SM: the step is latency-bound (config 2 +3.5 %, config 4 +1 %)
#endif
template <int JPL, bool TRAP>
__global__ void __launch_bounds__(32 * kWarpsPerCta, PBGK_MREC_MINB)
    mrec_step_kernel(const MargArgs m, const FinalArgs f) {
  extern __shared__ double sm[];
  const int wid = threadIdx.x >> 5;
  const int i = blockIdx.x * kWarpsPerCta + wid;
  pdl_wait();  // tables, G sums and Q(f*_{s-1}) come from the preceding kernels
  pdl_trigger();
  if (i >= m.nx) return;
  mrec_cell<JPL, TRAP>(m, f, f.step, i, blockIdx.y, sm + (size_t)wid * 6 * m.nvx);
}

// Device-wide barrier of a co-resident (cooperatively launched) grid:
// generation counter, the last arriver resets the count and bumps it.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// All steps 1..S of the recursion in one launch (small grids: the per-step
// launches are latency-bound).  Per-step tables at tab_in + s * t_step (tab_in
// = the step-0 tables), state ping-pong q[2] (q0: Q of a given f0, or null:
// a lift), G sums ping-pong in gsum; one grid barrier per step.  Windows of a
// batch: grid.y as in mrec_step_kernel.
template <int JPL, bool TRAP>
__global__ void __launch_bounds__(32 * kWarpsPerCta) mrec_multi_kernel(MargArgs m, FinalArgs f,
                                                                        const double* q0, double* qa,
                                                                        double* qb, double* gsum,
                                                                        long long t_step, int S,
                                                                        unsigned* bar, unsigned* prog,
                                                                        unsigned prog_base) {
  extern __shared__ double sm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kWarpsPerCta + wid;
  const int w = blockIdx.y;
  const unsigned nblocks = gridDim.x * gridDim.y;
  pdl_wait();
  pdl_trigger();
  const size_t g6 = (size_t)6 * m.nx;
  const double* tab0 = m.tab_in;
  // G sums of the step-0 tables
  if (i < m.nx) {
    const double* row = tab0 + w * m.t_ws + (size_t)i * m.TL;
    double a0, a1, a2, b0, b1, b2;
    axis_sums(row + m.gyo, m.cy, m.nvy, m.trap, lane, a0, a1, a2);
    axis_sums(row + m.gzo, m.cz, m.nvz, m.trap, lane, b0, b1, b2);
    if (lane == 0) {
      double* g = gsum + w * m.g_ws + (size_t)i * 6;
      g[0] = a0; g[1] = a1; g[2] = a2; g[3] = b0; g[4] = b1; g[5] = b2;
    }
  }
  for (int s = 1; s <= S; ++s) {
    grid_barrier(bar, nblocks);
    // steps < s are complete everywhere: publish for concurrent passes
    if (prog != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
      __threadfence();
      st_release_gpu(prog, prog_base + (unsigned)(s - 1));
    }
    MargArgs ms = m;
    ms.min = s == 1 ? q0 : ((s - 1) & 1 ? qa : qb);
    ms.mout = (s & 1) ? qa : qb;
    ms.tab_in = tab0 + (size_t)(s - 1) * t_step;
    ms.gsum_in = gsum + ((s - 1) & 1) * g6;
    ms.gsum_out = gsum + (s & 1) * g6;
    ms.dts = m.dts + (size_t)(s - 1) * gridDim.y;
    FinalArgs fs = f;
    fs.tab = const_cast<double*>(tab0) + (size_t)s * t_step;
    if (i < m.nx) mrec_cell<JPL, TRAP>(ms, fs, s, i, w, sm + (size_t)wid * 6 * m.nvx);
  }
  if (prog != nullptr) {
    grid_barrier(bar, nblocks);
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
      __threadfence();
      st_release_gpu(prog, prog_base + (unsigned)S);
    }
  }
}

// Q of a given distribution (the recursion's start for a window that begins
// from f0): one warp per (cell, v_x row); lanes over v_z, sequential over v_y;
// fixed trees, mirror-symmetric (folded sums are exactly 0 for even data).
template <bool TRAP>
__global__ void __launch_bounds__(32 * kWarpsPerCta) mrec_from_f_kernel(const MargArgs m, const double* f) {
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  const int nvx = m.nvx, nvy = m.nvy, nvz = m.nvz;
  pdl_wait();
  pdl_trigger();
  if (w >= (long long)m.nx * nvx) return;
  const int i = (int)(w / nvx), jx = (int)(w - (long long)i * nvx);
  const double* row = f + ((size_t)i * nvx + jx) * nvy * nvz;
  const int hy = nvy / 2, hz = nvz / 2;
  double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0, q4 = 0.0;
  for (int jy = 0; jy < nvy; ++jy) {
    const double wy = wq(TRAP, jy, nvy), cy = m.cy[jy];
    const double* fy = row + (size_t)jy * nvz;
    const double* fm = row + (size_t)(nvy - 1 - jy) * nvz;
    for (int jz = lane; jz < nvz; jz += 32) {
      const double wz = wq(TRAP, jz, nvz), cz = m.cz[jz];
      const double v = fy[jz];
      const double ww = wy * wz;
      q0 += ww * v;
      q2 += (ww * cy) * (cy * v);
      q4 += (ww * cz) * (cz * v);
      if (jy < hy) q1 += (ww * cy) * (v - fm[jz]);
      if (jz < hz) q3 += (ww * cz) * (v - fy[nvz - 1 - jz]);
    }
  }
  q0 = wsum(q0);
  q1 = wsum(q1);
  q2 = wsum(q2);
  q3 = wsum(q3);
  q4 = wsum(q4);
  if (lane == 0) {
    double* o = m.mout + (size_t)i * 5 * nvx;
    o[jx] = q0;
    o[nvx + jx] = q1;
    o[2 * nvx + jx] = q2;
    o[3 * nvx + jx] = q3;
    o[4 * nvx + jx] = q4;
  }
}

cudaError_t launch_q_from_f(const MargArgs& m, const double* f, cudaStream_t st) {
  const long long warps = (long long)m.nx * m.nvx;
  const int grid = (int)((warps + kWarpsPerCta - 1) / kWarpsPerCta);
  auto k = m.trap ? mrec_from_f_kernel<true> : mrec_from_f_kernel<false>;
  return launch_pdl(k, grid, 32 * kWarpsPerCta, 0, st, m, f);
}

size_t marg_smem_bytes(int nvx, int nvy, int nvz, int TL) {
  (void)nvy; (void)nvz; (void)TL;
  if (nvx > 128) return ~(size_t)0;  // rows per lane bound (4)
  return (size_t)kWarpsPerCta * 6 * nvx * sizeof(double);  // m_x + the field's relaxed rows
}

// Q (5 nvx per cell) lives in the caller's ping-pong buffers
size_t marg_state_doubles(int nvx) { return (size_t)5 * nvx; }

// Step s >= 1 for `nwin` windows (grid.y; the caller sets the per-window
// strides, 0 for one window).  s == 1: the input tables are a lift or
// identity rows, their G sums come first.  The G sums ping-pong between the
// two halves (6 nx doubles each) of each window's `gsum` block (stride g_ws).
cudaError_t launch_marg(const MargArgs& m0, const FinalArgs& f, double* gsum, int s, int nwin,
                        cudaStream_t st) {
  MargArgs m = m0;
  m.TL = f.TL;
  m.gxo = f.gxo;
  m.gyo = f.gyo;
  m.gzo = f.gzo;
  m.trap = f.trap;
  m.cy = f.cy;
  m.cz = f.cz;
  const size_t g6 = (size_t)6 * m.nx;
  m.gsum_in = gsum + ((s - 1) & 1) * g6;
  m.gsum_out = gsum + (s & 1) * g6;
  const dim3 grid((m.nx + kWarpsPerCta - 1) / kWarpsPerCta, nwin);
  if (s == 1) {
    MargArgs mi = m;
    mi.gsum_out = const_cast<double*>(m.gsum_in);
    cudaError_t e = launch_pdl_grid(mrec_init_kernel, grid, 32 * kWarpsPerCta, 0, st, mi);
    if (e != cudaSuccess) return e;
  }
  const int jpl = (m.nvx + 31) / 32;
  void (*k)(const MargArgs, const FinalArgs) = nullptr;
#define PBGK_MK(J) (m.trap ? mrec_step_kernel<J, true> : mrec_step_kernel<J, false>)
  k = jpl <= 1 ? PBGK_MK(1) : (jpl == 2 ? PBGK_MK(2) : (jpl == 3 ? PBGK_MK(3) : PBGK_MK(4)));
#undef PBGK_MK
  return launch_pdl_grid(k, grid, 32 * kWarpsPerCta, marg_smem_bytes(m.nvx, m.nvy, m.nvz, f.TL), st, m, f);
}

// CTAs of the one-launch recursion for nx cells and nwin windows, and how
// many fit one SM (registers / shared memory).
void marg_all_shape(int nx, int nvx, int nvy, int nvz, int TL, bool trap, int nwin, int* ctas,
                    int* per_sm) {
  const int jpl = (nvx + 31) / 32;
  void (*k)(MargArgs, FinalArgs, const double*, double*, double*, double*, long long, int, unsigned*,
            unsigned*, unsigned) = nullptr;
#define PBGK_MK(J) (trap ? mrec_multi_kernel<J, true> : mrec_multi_kernel<J, false>)
  k = jpl <= 1 ? PBGK_MK(1) : (jpl == 2 ? PBGK_MK(2) : (jpl == 3 ? PBGK_MK(3) : PBGK_MK(4)));
#undef PBGK_MK
  *ctas = ((nx + kWarpsPerCta - 1) / kWarpsPerCta) * nwin;
  *per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k, 32 * kWarpsPerCta,
                                                marg_smem_bytes(nvx, nvy, nvz, TL));
}

// All S steps in one cooperative launch when the grid is co-resident (see
// mrec_multi_kernel); returns cudaErrorCooperativeLaunchTooLarge otherwise.
cudaError_t launch_marg_all(const MargArgs& m0, const FinalArgs& f, const double* q0, double* qa,
                            double* qb, double* gsum, long long t_step, int S, int nwin,
                            unsigned* bar, cudaStream_t st, unsigned* prog, unsigned prog_base,
                            int max_ctas) {
  MargArgs m = m0;
  m.TL = f.TL;
  m.gxo = f.gxo;
  m.gyo = f.gyo;
  m.gzo = f.gzo;
  m.trap = f.trap;
  m.cy = f.cy;
  m.cz = f.cz;
  const int jpl = (m.nvx + 31) / 32;
  void (*k)(MargArgs, FinalArgs, const double*, double*, double*, double*, long long, int, unsigned*,
            unsigned*, unsigned) = nullptr;
#define PBGK_MK(J) (m.trap ? mrec_multi_kernel<J, true> : mrec_multi_kernel<J, false>)
  k = jpl <= 1 ? PBGK_MK(1) : (jpl == 2 ? PBGK_MK(2) : (jpl == 3 ? PBGK_MK(3) : PBGK_MK(4)));
#undef PBGK_MK
  const size_t smem = marg_smem_bytes(m.nvx, m.nvy, m.nvz, f.TL);
  const dim3 grid((m.nx + kWarpsPerCta - 1) / kWarpsPerCta, nwin);
  int dev = 0, nsm = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 32 * kWarpsPerCta, smem);
  if (e != cudaSuccess) return e;
  if ((long long)grid.x * grid.y > (long long)per * nsm) return cudaErrorCooperativeLaunchTooLarge;
  if (max_ctas > 0 && (long long)grid.x * grid.y > max_ctas) return cudaErrorCooperativeLaunchTooLarge;
  e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(32 * kWarpsPerCta);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, m, f, q0, qa, qb, gsum, t_step, S, bar, prog, prog_base);
}

}  // namespace pbgk
