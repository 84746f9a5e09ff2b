// Per-cell finalisation, shared by finalize.cu (one CTA per cell) and the
// sweep kernel (fused: the CTA that writes a cell's last tile partials).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace pbgk {

// Gather of the tile partials.  The tiles contributing to one marginal entry
// are enumerated outer-major / inner-minor (the same order for every entry and
// its mirror); that list is cut into chunks of kChunk tiles, each chunk summed
// in order by one thread (all its loads issued before the first add), and the
// chunk sums of an entry are then added in chunk order.  Adjacent threads take
// adjacent entries of the same chunk, so each load instruction is coalesced.
#ifndef PBGK_FIN_CHUNK
#define PBGK_FIN_CHUNK 16
#endif
constexpr int kChunk = PBGK_FIN_CHUNK;

struct EntryList {
  int base, n_out, s_out, n_in, s_in, off;
};

// Tile list of entry j of axis ax (0: c_x, 1: c_y, 2: c_z).
static __device__ __forceinline__ EntryList entry_list(const Tiling& T, int ax, int j) {
  const int per = T.nty * T.ntz, ntx = T.ntn + T.ntp;
  EntryList e;
  if (ax == 0) {
    int tx, r0;
    if (j < T.nneg) {
      tx = j / T.A;
      r0 = tx * T.A;
    } else {
      tx = T.ntn + (j - T.nneg) / T.A;
      r0 = T.nneg + (tx - T.ntn) * T.A;
    }
    e = {tx * per, T.nty, T.ntz, T.ntz, 1, j - r0};
  } else if (ax == 1) {
    const int ty = j / T.By;
    e = {ty * T.ntz, ntx, per, T.ntz, 1, T.A + j - ty * T.By};
  } else {
    const int tz = j / T.Bz;
    e = {tz, ntx, per, T.nty, T.ntz, T.A + T.By + j - tz * T.Bz};
  }
  return e;
}

static __device__ __forceinline__ int list_len(const Tiling& T, int ax) {
  return ax == 0 ? T.nty * T.ntz : (ax == 1 ? (T.ntn + T.ntp) * T.ntz : (T.ntn + T.ntp) * T.nty);
}

// Sum of tiles [q0, q1) of list e (q1 - q0 <= kChunk), in list order.
static __device__ __forceinline__ double chunk_sum(const double* P, int PS, const EntryList& e,
                                                   int q0, int q1) {
  // branch-free walk: pointer advanced by s_in records, or by the wrap
  // stride at the end of an inner run; positions past q1 re-load the first
  // address and add +0.0 (exact: s starts at +0.0 and can never become -0.0)
  int o = q0 / e.n_in, in = q0 - o * e.n_in;
  const double* p0 = P + (size_t)(e.base + o * e.s_out + in * e.s_in) * PS + e.off;
  const long long d_in = (long long)e.s_in * PS;
  const long long d_wrap = (long long)(e.s_out - (e.n_in - 1) * e.s_in) * PS;
  const int cnt = q1 - q0;
  const double* p = p0;
  double v[kChunk];
#pragma unroll
  for (int r = 0; r < kChunk; ++r) {
    const double* q = r < cnt ? p : p0;
    v[r] = __ldcg(q);
    ++in;
    const bool wrap = in == e.n_in;
    p += wrap ? d_wrap : d_in;
    in = wrap ? 0 : in;
  }
  double s = 0.0;
#pragma unroll
  for (int r = 0; r < kChunk; ++r) s += r < cnt ? v[r] : 0.0;
  return s;
}

// Doubles of chunk-sum scratch finalize_cell needs beyond its 2*(nvx+nvy+nvz).
static __host__ __device__ __forceinline__ int chunk_scratch(const Tiling& T, int nvx, int nvy,
                                                             int nvz) {
  const int ntx = T.ntn + T.ntp;
  const int lx = T.nty * T.ntz, ly = ntx * T.ntz, lz = ntx * T.nty;
  return nvx * ((lx + kChunk - 1) / kChunk) + nvy * ((ly + kChunk - 1) / kChunk) +
         nvz * ((lz + kChunk - 1) / kChunk);
}

static __device__ __forceinline__ double warp_allsum(double x) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) x += __shfl_xor_sync(0xffffffffu, x, w);
  return x;
}

// Tile partials of cell i -> marginals m_x | m_y | m_z in sm (contiguous),
// by the whole calling CTA; ends with a CTA barrier.
static __device__ __forceinline__ void gather_marginals(const FinalArgs& a, int i, double* sm) {
  const int tid = threadIdx.x;
  const int nvx = a.nvx, nvy = a.nvy, nvz = a.nvz;
  const Tiling& T = a.t;
  const double* P = a.part + (size_t)i * T.NT * T.PS;
  double* csum = sm + 2 * (nvx + nvy + nvz);
  const int k0 = (list_len(T, 0) + kChunk - 1) / kChunk;
  const int k1 = (list_len(T, 1) + kChunk - 1) / kChunk;
  const int k2 = (list_len(T, 2) + kChunk - 1) / kChunk;
  const int t1 = k0 * nvx, t2 = t1 + k1 * nvy, t3 = t2 + k2 * nvz;
  // one chunk per entry (small tilings): the chunk sum IS the marginal
  const bool single = (t3 == nvx + nvy + nvz);
  double* dst = single ? sm : csum;
  for (int t = tid; t < t3; t += blockDim.x) {
    const int ax = t < t1 ? 0 : (t < t2 ? 1 : 2);
    const int q = t - (ax == 0 ? 0 : (ax == 1 ? t1 : t2));
    const int n = ax == 0 ? nvx : (ax == 1 ? nvy : nvz);
    const int c = q / n, j = q - c * n;
    const int len = list_len(T, ax);
    const EntryList e = entry_list(T, ax, j);
    const int q1 = min(len, (c + 1) * kChunk);
    dst[t] = chunk_sum(P, T.PS, e, c * kChunk, q1);
  }
  __syncthreads();
  if (!single) {
    for (int j = tid; j < nvx + nvy + nvz; j += blockDim.x) {
      const int ax = j < nvx ? 0 : (j < nvx + nvy ? 1 : 2);
      const int jj = j - (ax == 0 ? 0 : (ax == 1 ? nvx : nvx + nvy));
      const int n = ax == 0 ? nvx : (ax == 1 ? nvy : nvz);
      const int kk = ax == 0 ? k0 : (ax == 1 ? k1 : k2);
      const double* cs0 = csum + (ax == 0 ? 0 : (ax == 1 ? t1 : t2)) + jj;
      double s = 0.0;
      for (int c = 0; c < kk; ++c) s += cs0[c * n];
      sm[j] = s;  // mx | my | mz are contiguous
    }
    __syncthreads();
  }
}

// One x cell, by the whole calling CTA (blockDim >= 128; warps 0-3 reduce).
// sm: 2*(nvx+nvy+nvz) doubles of scratch, sh: 16 doubles.  Block-uniform call.
// HAVE_MARG: the marginals are already in sm (marginal recursion, marginal.cu).
template <bool HAVE_MARG = false>
static __device__ __forceinline__ void finalize_cell(const FinalArgs& a, int i, double* sm, double* sh) {
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nvx = a.nvx, nvy = a.nvy, nvz = a.nvz;
  double* mx = sm;
  double* my = mx + nvx;
  double* mz = my + nvy;
  // per-axis selectors (ternaries, not arrays: a runtime index would put
  // an array on the stack)
  auto nv = [&](int ax) { return ax == 0 ? nvx : (ax == 1 ? nvy : nvz); };
  auto cs = [&](int ax) { return ax == 0 ? a.cx : (ax == 1 ? a.cy : a.cz); };
  auto ms = [&](int ax) { return ax == 0 ? mx : (ax == 1 ? my : mz); };

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
    if (!HAVE_MARG) gather_marginals(a, i, sm);
    if (a.relax_tab != nullptr) {
      // the marginals of R(f*) from those of f*: warp ax sums the factors of
      // axis ax (lane-strided, then the butterfly: a fixed tree), then every
      // entry adds its axis factor times the other two sums
      const double* row = a.relax_tab + (size_t)i * a.TL;
      if (warp < 3) {
        const int n = nv(warp);
        const int off = warp == 0 ? a.gxo : (warp == 1 ? a.gyo : a.gzo);
        double s = 0.0;
        for (int j = lane; j < n; j += 32) s += row[off + j];
        s = warp_allsum(s);
        if (lane == 0) sh[8 + warp] = s;
      }
      __syncthreads();
      const double r = row[0], ls = row[1];
      for (int j = tid; j < nvx + nvy + nvz; j += blockDim.x) {
        const int ax = j < nvx ? 0 : (j < nvx + nvy ? 1 : 2);
        const int jj = j - (ax == 0 ? 0 : (ax == 1 ? nvx : nvx + nvy));
        const int off = ax == 0 ? a.gxo : (ax == 1 ? a.gyo : a.gzo);
        const double other = ax == 0 ? sh[9] * sh[10] : (ax == 1 ? sh[8] * sh[10] : sh[8] * sh[9]);
        sm[j] = r * fma(ls * row[off + jj], other, sm[j]);  // mx | my | mz are contiguous
      }
      __syncthreads();
    }
    // finiteness of f* (all its values feed these sums; a NaN/Inf anywhere
    // leaves a non-finite marginal) -- the guard of ref/kinetic.py:157-159;
    // warps 1..3 test their axis while reducing the folded first moment
    // trapezoid: the marginals carry the weights of the two summed axes; the
    // remaining axis is weighted here (end nodes 1/2, exact)
    auto wq = [&](int j, int n) { return (a.trap && (j == 0 || j == n - 1)) ? 0.5 : 1.0; };
    if (warp == 0) {
      double s = 0.0;
      for (int j = lane; j < nvx; j += 32) s += a.trap ? mx[j] * wq(j, nvx) : mx[j];
      s = warp_allsum(s);
      if (lane == 0) sh[0] = s;
    } else if (warp < 4) {
      const int ax = warp - 1;  // warps 1..3 -> axes 0..2
      const int n = nv(ax), h = n / 2;
      const double* m = ms(ax);
      const double* c = cs(ax);
      double s = 0.0;
      for (int j = lane; j < h; j += 32) s += (m[j] - m[n - 1 - j]) * (a.trap ? c[j] * wq(j, n) : c[j]);
      s = warp_allsum(s);
      int bad = 0;
      for (int j = lane; j < n; j += 32) bad |= !isfinite(m[j]);
      bad = __any_sync(0xffffffffu, bad);
      if (lane == 0) {
        sh[1 + ax] = s;
        sh[12 + ax] = bad ? 1.0 : 0.0;
      }
    }
    __syncthreads();
    nonfinite = (sh[12] != 0.0) || (sh[13] != 0.0) || (sh[14] != 0.0);
    rho = sh[0] * a.dvol;
    u0 = (sh[1] * a.dvol) / rho;
    u1 = (sh[2] * a.dvol) / rho;
    u2 = (sh[3] * a.dvol) / rho;
    if (warp < 3) {
      const int n = nv(warp);
      const double* m = ms(warp);
      const double* c = cs(warp);
      const double ua = (warp == 0) ? u0 : (warp == 1 ? u1 : u2);
      double s = 0.0;
      for (int j = lane; j < n; j += 32) {
        const double d = c[j] - ua;
        s += (d * d) * (a.trap ? m[j] * wq(j, n) : m[j]);
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
  const double tt = 6.283185307179586 * th;
  const double amp = rho / (tt * sqrt(tt));  // (2 pi theta)^1.5, ref/lifting.py:50
  double* row = a.tab + (size_t)i * a.TL;
  // warp a < 3: the Maxwellian factors of axis a, their sum (lane-strided
  // sequential + xor butterfly, the fixed tree of every reduction here) and
  // the row segment; warp 3: the row's zero padding
  if (warp < 3) {
    const int ax = warp;
    const int n = nv(ax);
    const double* c = cs(ax);
    const double ua = ax == 0 ? u0 : (ax == 1 ? u1 : u2);
    const int off = ax == 0 ? a.gxo : (ax == 1 ? a.gyo : a.gzo);
    double s = 0.0;
    for (int j = lane; j < n; j += 32) {
      const double d = c[j] - ua;
      double g = exp(-(d * d) * inv2t);
      if (ax == 0) g = g * amp;
      s += (a.trap && (j == 0 || j == n - 1)) ? 0.5 * g : g;
      row[off + j] = g;
    }
    s = warp_allsum(s);
    if (lane == 0) sh[8 + ax] = s;
  } else if (warp == 3) {
    for (int j = a.gyo + nvy + lane; j < a.gzo; j += 32) row[j] = 0.0;
    for (int j = a.gzo + nvz + lane; j < a.TL; j += 32) row[j] = 0.0;
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
  if (tid == 0) {
    row[0] = r;
    row[1] = ls;
    // f_s = R_s(f*_s) is finite iff f*_s and the table row are (BlowUpError(step))
    if (a.mode == kFinRelax &&
        (nonfinite || !isfinite(r) || !isfinite(ls) || !isfinite(amp) || !isfinite(u0) ||
         !isfinite(u1) || !isfinite(u2) || !isfinite(th)))
      atomicMin(a.err, err_key(0, a.step, kErrNonFinite));
  }
}


}  // namespace pbgk
