// Per-cell finalisation, shared by finalize.cu (one CTA per cell) and the
// sweep kernel (fused: the CTA that writes a cell's last tile partials).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace pbgk {

// Sum of one marginal entry over its tiles, outer-major / inner-minor (the
// fixed order for every entry); loads are batched 8 ahead so the L2
// latencies overlap while the additions stay in order.
static __device__ __forceinline__ double tile_sum(const double* P, int PS, int base, int n_out,
                                                  int s_out, int n_in, int s_in, int off) {
  const int n = n_out * n_in;
  double s = 0.0;
  int q = 0;
  for (; q + 8 <= n; q += 8) {
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int o = (q + r) / n_in, in = q + r - o * n_in;
      v[r] = __ldcg(P + (size_t)(base + o * s_out + in * s_in) * PS + off);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) s += v[r];
  }
  for (; q < n; ++q) {
    const int o = q / n_in, in = q - o * n_in;
    s += __ldcg(P + (size_t)(base + o * s_out + in * s_in) * PS + off);
  }
  return s;
}

static __device__ __forceinline__ double warp_allsum(double x) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) x += __shfl_xor_sync(0xffffffffu, x, w);
  return x;
}

// One x cell, by the whole calling CTA (blockDim >= 128; warps 0-3 reduce).
// sm: 2*(nvx+nvy+nvz) doubles of scratch, sh: 16 doubles.  Block-uniform call.
static __device__ __forceinline__ void finalize_cell(const FinalArgs& a, int i, double* sm, double* sh) {
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nvx = a.nvx, nvy = a.nvy, nvz = a.nvz;
  double* mx = sm;
  double* my = mx + nvx;
  double* mz = my + nvy;
  double* gx = mz + nvz;
  double* gy = gx + nvx;
  double* gz = gy + nvy;
  const double* cs[3] = {a.cx, a.cy, a.cz};
  const int nv[3] = {nvx, nvy, nvz};
  double* ms[3] = {mx, my, mz};
  double* gs[3] = {gx, gy, gz};

  if (a.mode == kFinIdentity) {
    double* row = a.tab + (size_t)i * a.TL;
    for (int j = tid; j < a.TL; j += blockDim.x) row[j] = (j == 0) ? 1.0 : 0.0;
    return;
  }

  double rho, u0, u1, u2, th;
  int nonfinite = 0;
  if (a.mom_in != nullptr) {
    rho = a.mom_in[i];
    u0 = a.mom_in[a.nx + i];
    u1 = a.mom_in[2 * a.nx + i];
    u2 = a.mom_in[3 * a.nx + i];
    th = a.mom_in[4 * a.nx + i];
  } else {
    const Tiling& T = a.t;
    const int per = T.nty * T.ntz;
    const double* P = a.part + (size_t)i * T.NT * T.PS;
    for (int j = tid; j < nvx + nvy + nvz; j += blockDim.x) {
      double s = 0.0;
      if (j < nvx) {
        const int jx = j;
        int tx, r0;
        if (jx < T.nneg) {
          tx = jx / T.A;
          r0 = tx * T.A;
        } else {
          tx = T.ntn + (jx - T.nneg) / T.A;
          r0 = T.nneg + (tx - T.ntn) * T.A;
        }
        const int off = jx - r0;
        s = tile_sum(P, T.PS, tx * per, T.nty, T.ntz, T.ntz, 1, off);
        mx[jx] = s;
      } else if (j < nvx + nvy) {
        const int jy = j - nvx;
        const int ty = jy / T.By, off = T.A + jy - ty * T.By;
        const int ntx = T.ntn + T.ntp;
        s = tile_sum(P, T.PS, ty * T.ntz, ntx, per, T.ntz, 1, off);
        my[jy] = s;
      } else {
        const int jz = j - nvx - nvy;
        const int tz = jz / T.Bz, off = T.A + T.By + jz - tz * T.Bz;
        const int ntx = T.ntn + T.ntp;
        s = tile_sum(P, T.PS, tz, ntx, per, T.nty, T.ntz, off);
        mz[jz] = s;
      }
    }
    // finiteness of f* (all its values feed these sums; a NaN/Inf anywhere
    // leaves a non-finite marginal) -- the guard of ref/kinetic.py:157-159
    int bad = 0;
    for (int j = tid; j < nvx + nvy + nvz; j += blockDim.x) bad |= !isfinite(sm[j]);
    nonfinite = __syncthreads_or(bad);
    if (warp == 0) {
      double s = 0.0;
      for (int j = lane; j < nvx; j += 32) s += mx[j];
      s = warp_allsum(s);
      if (lane == 0) sh[0] = s;
    } else if (warp < 4) {
      const int ax = warp - 1;  // warps 1..3 -> axes 0..2
      const int n = nv[ax], h = n / 2;
      const double* m = ms[ax];
      const double* c = cs[ax];
      double s = 0.0;
      for (int j = lane; j < h; j += 32) s += (m[j] - m[n - 1 - j]) * c[j];
      s = warp_allsum(s);
      if (lane == 0) sh[1 + ax] = s;
    }
    __syncthreads();
    rho = sh[0] * a.dvol;
    u0 = (sh[1] * a.dvol) / rho;
    u1 = (sh[2] * a.dvol) / rho;
    u2 = (sh[3] * a.dvol) / rho;
    if (warp < 3) {
      const int n = nv[warp];
      const double* m = ms[warp];
      const double* c = cs[warp];
      const double ua = (warp == 0) ? u0 : (warp == 1 ? u1 : u2);
      double s = 0.0;
      for (int j = lane; j < n; j += 32) {
        const double d = c[j] - ua;
        s += (d * d) * m[j];
      }
      s = warp_allsum(s);
      if (lane == 0) sh[4 + warp] = s;
    }
    __syncthreads();
    const double e2 = ((0.0 + sh[4]) + sh[5]) + sh[6];
    th = (e2 * a.dvol) / (3.0 * rho);
    if (tid == 0 && rho <= 0.0) atomicMin(a.err, err_key(0, a.step, kErrProjectRho));
  }
  if (a.mom_out != nullptr && tid == 0) {
    a.mom_out[i] = rho;
    a.mom_out[a.nx + i] = u0;
    a.mom_out[2 * a.nx + i] = u1;
    a.mom_out[3 * a.nx + i] = u2;
    a.mom_out[4 * a.nx + i] = th;
  }
  if (a.mode == kFinProject) {
    if (a.check_finite && nonfinite && tid == 0) atomicMin(a.err, err_key(0, a.step, kErrNonFinite));
    return;
  }

  if (tid == 0 && (rho <= 0.0 || th <= 0.0)) atomicMin(a.err, err_key(0, a.step, kErrLiftState));
  const double inv2t = 1.0 / (2.0 * th);
  const double amp = rho / pow(6.283185307179586 * th, 1.5);
  const double us[3] = {u0, u1, u2};
  for (int ax = 0; ax < 3; ++ax) {
    for (int j = tid; j < nv[ax]; j += blockDim.x) {
      const double d = cs[ax][j] - us[ax];
      double g = exp(-(d * d) * inv2t);
      if (ax == 0) g = g * amp;
      gs[ax][j] = g;
    }
  }
  __syncthreads();
  if (warp < 3) {
    double s = 0.0;
    for (int j = lane; j < nv[warp]; j += 32) s += gs[warp][j];
    s = warp_allsum(s);
    if (lane == 0) sh[8 + warp] = s;
  }
  __syncthreads();
  double r = 0.0, ls = 1.0;
  if (a.mode == kFinRelax || a.mode == kFinSynthNorm) {
    const double mass = ((sh[8] * sh[9]) * sh[10]) * a.dvol;
    const double scale = rho / mass;
    if (a.mode == kFinRelax) {
      const double tau = a.tau_arr != nullptr ? a.tau_arr[i] : a.tau;
      const double lam = (a.dt * tau) / a.eps;
      r = 1.0 / (1.0 + lam);
      ls = lam * scale;
    } else {
      ls = scale;
    }
  }
  // f_s = R_s(f*_s) is finite iff f*_s and the table row are (BlowUpError(step))
  if (a.mode == kFinRelax && tid == 0 &&
      (nonfinite || !isfinite(r) || !isfinite(ls) || !isfinite(amp) || !isfinite(u0) ||
       !isfinite(u1) || !isfinite(u2) || !isfinite(th)))
    atomicMin(a.err, err_key(0, a.step, kErrNonFinite));
  double* row = a.tab + (size_t)i * a.TL;
  for (int j = tid; j < a.TL; j += blockDim.x) {
    double v = 0.0;
    if (j == 0) v = r;
    else if (j == 1) v = ls;
    else if (j >= a.gxo && j < a.gxo + nvx) v = gx[j - a.gxo];
    else if (j >= a.gyo && j < a.gyo + nvy) v = gy[j - a.gyo];
    else if (j >= a.gzo && j < a.gzo + nvz) v = gz[j - a.gzo];
    row[j] = v;
  }
}


}  // namespace pbgk
