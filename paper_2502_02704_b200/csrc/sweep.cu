// Fused fine-step sweep: one HBM read and one HBM write of f per fine step.
//
// Step s of the fine propagator (ref/kinetic.py:152-160) is
//     f*_s = T_dt(f_{s-1}),   f_s = R_s(f*_s) = (f*_s + lam M[f*_s]) / (1 + lam).
// R_s needs per-x-cell velocity reductions of f*_s, a grid-wide dependency.
// The sweep therefore runs skewed: pass s reads f*_{s-1} (already in HBM),
// applies R_{s-1} pointwise from a small per-cell table row (lambda and the
// separable Maxwellian factors, written by finalize.cu), applies T_dt for step
// s, writes f*_s and accumulates fixed-order marginal partials of f*_s.  The
// first pass of a window synthesises f_0 = L(U) from the lift tables instead
// of reading it (SYNTH); the last pass applies R_S only (dtdx == 0) and may
// skip the write (the window only needs P(f_S)).
//
// Work decomposition (persistent, 1 CTA per SM):
//   velocity box "tile" (A rows of v_x, By of v_y, Bz of v_z) x all x cells.
//   Every tile has one sign of c_x, so its upwind neighbour plane is on one
//   side: c_x >= 0 tiles march upward in x, c_x < 0 tiles march downward and
//   a register sliding window holds f_pre of the previous plane.  The
//   (tile, plane) sequence is cut into gridDim.x contiguous segments; a
//   segment pays one halo plane per tile it touches.
//   Each plane's box arrives by one 4-D TMA copy (plus a 1-D bulk copy of the
//   cell's table row) into a ring of `ns` shared-memory stages.
//
// Reductions are deterministic and mirror-symmetric (same tree for every
// marginal index), so even data keeps an exactly-zero folded first moment
// (ref/moments.py:80-88).
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "ptx.cuh"

namespace pbgk {

constexpr unsigned FULL = 0xffffffffu;

// Reduce-scatter of C per-lane line values over the W..1 lane bits of an
// aligned lane group.  After the split levels each lane holds C' = max(C/LZ,1)
// line totals; `base` is the index of the first one.  Every line total is the
// same binary tree over lanes (fp add is commutative), for every line.
template <int C, int W>
struct LineRS {
  static __device__ __forceinline__ void run(double* v, int lz, int& base) {
    if constexpr (W == 0) {
      return;
    } else if constexpr (C >= 2) {
      const bool upper = (lz & W) != 0;
#pragma unroll
      for (int q = 0; q < C / 2; ++q) {
        const double lo = v[q], hi = v[q + C / 2];
        const double send = upper ? lo : hi;
        const double keep = upper ? hi : lo;
        v[q] = keep + __shfl_xor_sync(FULL, send, W);
      }
      if (upper) base += C / 2;
      LineRS<C / 2, W / 2>::run(v, lz, base);
    } else {
      v[0] += __shfl_xor_sync(FULL, v[0], W);
      LineRS<1, W / 2>::run(v, lz, base);
    }
  }
};

struct TileGeom {
  int r0, r1, y0, z0;
  bool down;
};

__device__ __forceinline__ TileGeom tile_geom(const Tiling& t, int nvx, int tile) {
  const int per = t.nty * t.ntz;
  const int tx = tile / per;
  const int rem = tile - tx * per;
  const int ty = rem / t.ntz;
  const int tz = rem - ty * t.ntz;
  TileGeom g;
  if (tx < t.ntn) {
    g.r0 = tx * t.A;
    g.r1 = min(g.r0 + t.A, t.nneg);
    g.down = true;
  } else {
    g.r0 = t.nneg + (tx - t.ntn) * t.A;
    g.r1 = min(g.r0 + t.A, nvx);
    g.down = false;
  }
  g.y0 = ty * t.By;
  g.z0 = tz * t.Bz;
  return g;
}

// Item j of the segment [g0, g1): each run of consecutive planes of one tile
// is preceded by its halo (upwind neighbour) plane.
struct Item {
  int tile;
  int plane;  // x cell to load
  bool halo;
  bool ghost;  // absorbing ghost: f_pre == 0, nothing to load
  bool down;
};

__device__ __forceinline__ long long seg_items(long long g0, long long g1, int nx) {
  if (g1 <= g0) return 0;
  const long long len0 = min((long long)nx - g0 % nx, g1 - g0);
  const long long rest = g1 - g0 - len0;
  const long long runs = 1 + (rest + nx - 1) / nx;
  return (g1 - g0) + runs;
}

__device__ __forceinline__ Item seg_item(const SweepArgs& a, long long g0, long long g1,
                                         long long j) {
  const int nx = a.nx;
  const long long len0 = min((long long)nx - g0 % nx, g1 - g0);
  long long g;
  bool halo;
  if (j < 1 + len0) {
    halo = (j == 0);
    g = halo ? g0 : g0 + j - 1;
  } else {
    const long long jj = j - 1 - len0;
    const long long r = jj / (1 + nx);
    const long long q = jj - r * (1 + nx);
    const long long gs = g0 + len0 + r * nx;
    halo = (q == 0);
    g = halo ? gs : gs + q - 1;
  }
  Item it;
  it.tile = (int)(g / nx);
  const int p = (int)(g - (long long)it.tile * nx);
  const TileGeom tg = tile_geom(a.t, a.nvx, it.tile);
  it.down = tg.down;
  int i = tg.down ? nx - 1 - p : p;
  it.halo = halo;
  it.ghost = false;
  if (halo) {
    i += tg.down ? 1 : -1;
    if (i < 0 || i >= nx) {
      if (a.periodic) {
        i = (i + nx) % nx;
      } else {
        it.ghost = true;
        i = 0;
      }
    }
  }
  it.plane = i;
  return it;
}

template <int V, int LZ, int K, int NTHR, bool SYNTH, bool FIELD, bool TMA>
__global__ void __launch_bounds__(NTHR, 1)
    sweep_kernel(const __grid_constant__ CUtensorMap fmap, const SweepArgs a, int ns) {
  constexpr int NL = NTHR / LZ;  // line groups
  constexpr int NW = NTHR / 32;
  constexpr int BZ = LZ * V;
  static_assert(32 % LZ == 0, "LZ must divide the warp");
  extern __shared__ __align__(128) unsigned char smem[];

  const Tiling& T = a.t;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int lz = tid % LZ;
  const int lg = tid / LZ;
  const int hoff = (T.rows_load - T.A) >> 1;  // neighbour rows loaded for the field term
  const int lines = T.A * T.By;

  const uint32_t box_bytes = SYNTH ? 0u : (uint32_t)(T.rows_load * T.By * BZ * 8);
  const uint32_t tab_bytes = (uint32_t)(a.TL * 8);
  const uint32_t stage_bytes = TMA ? ((box_bytes + tab_bytes + 127u) & ~127u) : 0u;
  double* LT = reinterpret_cast<double*>(smem + (size_t)ns * stage_bytes);  // [2][lines]
  double* PZ = LT + 2 * lines;                                              // [2][NW][BZ]
  uint64_t* bars = reinterpret_cast<uint64_t*>(PZ + 2 * NW * BZ);           // [ns]

  const long long g0 = (a.total * blockIdx.x) / gridDim.x;
  const long long g1 = (a.total * (blockIdx.x + 1)) / gridDim.x;
  const long long n_items = seg_items(g0, g1, a.nx);

  if (TMA) {
    if (tid == 0) {
      for (int s = 0; s < ns; ++s) mbar_init(&bars[s], 1);
      fence_mbar_init();
    }
    __syncthreads();
  }

  auto issue = [&](long long j) {
    const Item it = seg_item(a, g0, g1, j);
    const int s = (int)(j % ns);
    uint64_t* bar = &bars[s];
    unsigned char* st = smem + (size_t)s * stage_bytes;
    if (it.ghost) {
      mbar_arrive_expect_tx(bar, 0);
      return;
    }
    const TileGeom tg = tile_geom(T, a.nvx, it.tile);
    mbar_arrive_expect_tx(bar, box_bytes + tab_bytes);
    if (!SYNTH) tma_load_4d(st, &fmap, tg.z0, tg.y0, tg.r0 - hoff, it.plane, bar);
    tma_load_1d(st + box_bytes, a.tab + (size_t)it.plane * a.TL, tab_bytes, bar);
  };

  if (TMA && tid == 0) {
    prefetch_tensormap(&fmap);
    const long long pre = n_items < ns ? n_items : ns;
    for (long long j = 0; j < pre; ++j) issue(j);
  }

  double prev[K][V];
  double cur[K][V];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int v = 0; v < V; ++v) prev[k][v] = 0.0;
  bool bad = false;

  for (long long j = 0; j < n_items; ++j) {
    const Item it = seg_item(a, g0, g1, j);
    const TileGeom tg = tile_geom(T, a.nvx, it.tile);
    const int s = (int)(j % ns);
    const double* SF = reinterpret_cast<const double*>(smem + (size_t)s * stage_bytes);
    const double* ST = reinterpret_cast<const double*>(smem + (size_t)s * stage_bytes + box_bytes);
    const double* GT = a.tab + (size_t)it.plane * a.TL;
    if (TMA) mbar_wait(&bars[s], (uint32_t)((j / ns) & 1));

    auto tab = [&](int idx) -> double { return TMA ? ST[idx] : __ldg(GT + idx); };
    // raw f*_{s-1} value at box row `brow` (halo-offset row index), line b, box z `zz`
    auto raw = [&](int brow, int b, int zz) -> double {
      if (SYNTH) return 0.0;
      if (TMA) return SF[(brow * T.By + b) * BZ + zz];
      const int jx = tg.r0 - hoff + brow, jy = tg.y0 + b, jz = tg.z0 + zz;
      if (jx < 0 || jx >= a.nvx || jy >= a.nvy || jz >= a.nvz) return 0.0;
      return __ldg(a.fin + (size_t)it.plane * a.plane + ((size_t)jx * a.nvy + jy) * a.nvz + jz);
    };

    if (it.ghost) {
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int v = 0; v < V; ++v) cur[k][v] = 0.0;
    } else {
      const double r = tab(0), ls = tab(1);
      double gz[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int jz = tg.z0 + lz * V + v;
        gz[v] = (jz < a.nvz) ? tab(a.gzo + jz) : 0.0;
      }
      double out[K][V];
      double lp[K];
      double pz[V];
#pragma unroll
      for (int v = 0; v < V; ++v) pz[v] = 0.0;
      const double hE = (FIELD && !it.halo) ? __dmul_rn(0.5, a.E[it.plane]) : 0.0;

#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int l = lg + k * NL;
        const int ls_ = (l < lines) ? l : 0;  // keep smem reads inside the box
        const int aa = ls_ / T.By;
        const int b = ls_ - aa * T.By;
        const int jx = tg.r0 + aa;
        const int jy = tg.y0 + b;
        const bool okl = (l < lines) && (jx < tg.r1) && (jy < a.nvy);
        const int jxs = okl ? jx : tg.r0;
        const int jys = okl ? jy : 0;
        const double gxy = okl ? tab(a.gxo + jxs) * tab(a.gyo + jys) : 0.0;
        // f_pre at the neighbour rows (field term only)
        double gxm = 0.0, gxp = 0.0;
        if (FIELD && !it.halo && okl) {
          if (jx > 0) gxm = tab(a.gxo + jx - 1) * tab(a.gyo + jy);
          if (jx + 1 < a.nvx) gxp = tab(a.gxo + jx + 1) * tab(a.gyo + jy);
        }
        const double c = okl ? __ldg(a.cx + jxs) : 0.0;
        lp[k] = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int zz = lz * V + v;
          const bool ok = okl && (tg.z0 + zz < a.nvz);
          double x;
          if (SYNTH) {
            x = (gxy * gz[v]) * ls;
          } else {
            x = fma(ls, gxy * gz[v], raw(aa + hoff, b, zz)) * r;
          }
          if (a.check_step > 0 && ok && !isfinite(x)) bad = true;
          cur[k][v] = x;
          if (it.halo) continue;
          double o = x;
          if (a.dtdx != 0.0) {
            const double y = prev[k][v];
            const double fhi = it.down ? __dmul_rn(c, y) : __dmul_rn(c, x);
            const double flo = it.down ? __dmul_rn(c, x) : __dmul_rn(c, y);
            o = __dsub_rn(x, __dmul_rn(a.dtdx, __dsub_rn(fhi, flo)));
          }
          if (FIELD) {
            // ref/kinetic.py:114-123, Rusanov flux on interior v_x faces of f_pre
            double fm = 0.0, fp = 0.0;
            if (okl && jx > 0) {
              fm = SYNTH ? (gxm * gz[v]) * ls : fma(ls, gxm * gz[v], raw(aa + hoff - 1, b, zz)) * r;
            }
            if (okl && jx + 1 < a.nvx) {
              fp = SYNTH ? (gxp * gz[v]) * ls : fma(ls, gxp * gz[v], raw(aa + hoff + 1, b, zz)) * r;
            }
            const double ghi = (jx + 1 < a.nvx)
                                   ? __dsub_rn(__dmul_rn(hE, __dadd_rn(x, fp)),
                                               __dmul_rn(a.half_emax, __dsub_rn(fp, x)))
                                   : 0.0;
            const double glo = (jx > 0) ? __dsub_rn(__dmul_rn(hE, __dadd_rn(fm, x)),
                                                    __dmul_rn(a.half_emax, __dsub_rn(x, fm)))
                                        : 0.0;
            o = __dsub_rn(o, __dmul_rn(a.dtdv, __dsub_rn(ghi, glo)));
          }
          const double m = ok ? o : 0.0;
          out[k][v] = m;
          pz[v] += m;
          lp[k] += m;
        }
        if (!it.halo && a.fout != nullptr && okl) {
          double* dst = a.fout + (size_t)it.plane * a.plane + ((size_t)jx * a.nvy + jy) * a.nvz +
                        tg.z0 + lz * V;
          if constexpr (V == 2) {
            if (tg.z0 + lz * V + 1 < a.nvz) {
              st_global_v2(dst, out[k][0], out[k][1]);
            } else if (tg.z0 + lz * V < a.nvz) {
              dst[0] = out[k][0];
            }
          } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
              if (tg.z0 + lz * V + v < a.nvz) dst[v] = out[k][v];
          }
        }
      }
      if (!it.halo) {
        // line totals -> LT, z partials -> PZ (double-buffered by item parity)
        double* LTb = LT + (j & 1) * lines;
        double* PZb = PZ + (j & 1) * NW * BZ;
        int base = 0;
        LineRS<K, LZ / 2>::run(lp, lz, base);
        constexpr int CF = (K / LZ) > 1 ? (K / LZ) : 1;
        constexpr int WMASK = (LZ / K) > 1 ? (LZ / K - 1) : 0;
        if ((lz & WMASK) == 0) {
#pragma unroll
          for (int c2 = 0; c2 < CF; ++c2) {
            const int l = lg + (base + c2) * NL;
            if (l < lines) LTb[l] = lp[c2];
          }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
#pragma unroll
          for (int w = LZ; w < 32; w <<= 1) pz[v] += __shfl_xor_sync(FULL, pz[v], w);
        }
        if (lane < LZ) {
#pragma unroll
          for (int v = 0; v < V; ++v) PZb[warp * BZ + lane * V + v] = pz[v];
        }
      }
    }

    __syncthreads();
    if (TMA && tid == 0 && j + ns < n_items) {
      fence_proxy_async();
      issue(j + ns);
    }
    if (!it.halo && !it.ghost) {
      const double* LTb = LT + (j & 1) * lines;
      const double* PZb = PZ + (j & 1) * NW * BZ;
      double* dst = a.part + ((size_t)it.plane * T.NT + it.tile) * T.PS;
      if (tid < T.A) {
        if (tg.r0 + tid < tg.r1) {
          double s2 = 0.0;
          for (int b = 0; b < T.By; ++b) s2 += LTb[tid * T.By + b];
          dst[tid] = s2;
        }
      } else if (tid < T.A + T.By) {
        const int b = tid - T.A;
        if (tg.y0 + b < a.nvy) {
          double s2 = 0.0;
          for (int aa = 0; aa < T.A; ++aa) s2 += LTb[aa * T.By + b];
          dst[T.A + b] = s2;
        }
      } else if (tid < T.A + T.By + BZ) {
        const int zz = tid - T.A - T.By;
        if (tg.z0 + zz < a.nvz) {
          double s2 = 0.0;
          for (int w = 0; w < NW; ++w) s2 += PZb[w * BZ + zz];
          dst[T.A + T.By + zz] = s2;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int v = 0; v < V; ++v) prev[k][v] = cur[k][v];
  }
  if (bad) atomicMin(a.err, err_key(0, a.check_step, kErrNonFinite));
}

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------

struct SweepCfg {
  int V, LZ, K, NTHR;
  bool tma;
};

template <int V, int LZ, int K, int NTHR, bool TMA>
static cudaError_t launch_cfg(const CUtensorMap& map, const SweepArgs& a, bool synth, bool field,
                              int grid, int ns, size_t smem, cudaStream_t st) {
  void (*fn)(const CUtensorMap, const SweepArgs, int);
  if (synth)
    fn = field ? sweep_kernel<V, LZ, K, NTHR, true, true, TMA>
               : sweep_kernel<V, LZ, K, NTHR, true, false, TMA>;
  else
    fn = field ? sweep_kernel<V, LZ, K, NTHR, false, true, TMA>
               : sweep_kernel<V, LZ, K, NTHR, false, false, TMA>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, NTHR, smem, st>>>(map, a, ns);
  return cudaGetLastError();
}

// Shared memory the kernel needs for `ns` stages.
size_t sweep_smem_bytes(const SweepArgs& a, int V, int LZ, int NTHR, bool synth, bool tma, int ns) {
  const int BZ = LZ * V;
  const size_t box = synth ? 0 : (size_t)a.t.rows_load * a.t.By * BZ * 8;
  const size_t stage = tma ? ((box + (size_t)a.TL * 8 + 127) & ~(size_t)127) : 0;
  const size_t lines = (size_t)a.t.A * a.t.By;
  return (size_t)ns * stage + 2 * lines * 8 + 2 * (size_t)(NTHR / 32) * BZ * 8 + (size_t)ns * 8 + 16;
}

cudaError_t launch_sweep(int cfg_id, const CUtensorMap& map, const SweepArgs& a, bool synth,
                         bool field, int grid, int ns, size_t smem, cudaStream_t st) {
  switch (cfg_id) {
    case 0: return launch_cfg<2, 32, 8, 512, true>(map, a, synth, field, grid, ns, smem, st);
    case 1: return launch_cfg<2, 16, 8, 512, true>(map, a, synth, field, grid, ns, smem, st);
    case 2: return launch_cfg<2, 16, 4, 512, true>(map, a, synth, field, grid, ns, smem, st);
    case 3: return launch_cfg<3, 16, 4, 512, true>(map, a, synth, field, grid, ns, smem, st);
    case 4: return launch_cfg<2, 8, 4, 256, true>(map, a, synth, field, grid, ns, smem, st);
    case 5: return launch_cfg<2, 4, 4, 256, true>(map, a, synth, field, grid, ns, smem, st);
    default: return launch_cfg<1, 32, 4, 256, false>(map, a, synth, field, grid, ns, smem, st);
  }
}

}  // namespace pbgk
