// Multi-step sweep with the v_x field term (configs 3a / 3b): up to 4 fine
// steps of f per pass over HBM.
//
// The field term of ref/kinetic.py:114-123 couples the v_x rows of one x cell
// (the Rusanov flux on the interior v_x faces), so the tiles of msweep.cu --
// a few v_x rows marching in x in the upwind direction of their sign -- do
// not close under it.  Here a warp owns WHOLE v_x columns instead:
//
//   * a warp column = all nvx rows x one v_y x 8 v_z; lane (s, c) = (lane/4,
//     lane%4) holds rows s V .. s V + V - 1 (V = nvx / 8) of v_z pair c, so
//     the v_x neighbours of a thread's rows are its own registers or (the
//     segment's end rows) one shuffle from lane s -+ 1.
//   * a warp marches a segment [x0, x1) of x planes in +x for both signs of
//     c_x: level l (relax with the table of step s0 + l, then transport)
//     works one plane behind level l - 1, so at input position p level l
//     holds the relaxed plane p - l - 1 of its input and the one before it
//     (two carries per element and level), receives plane p - l from level
//     l - 1, and emits plane p - l - 1 of its output.  The last level's
//     output (plane p - n) is stored: 16 / n bytes of HBM per cell-update
//     (ref: 16).  Segments overlap by n planes on either side (their halo).
//   * relax + transport of level l on plane q, per element
//     (ref/kinetic.py:110-123,130-134):
//         y = r x + (r ls g_y g_x[j]) g_z                  (relaxed f)
//         x' = kappa_j y_j + a_j y_nb + DCP y_{j-1} - DCM y_{j+1}
//     with a_j = (dt/dx)|c_x|, y_nb = y at plane q-1 (c_x > 0) or q+1
//     (c_x < 0), DCP / DCM = (dt/dv)(E_q/2 +- e_max/2) and kappa_j = 1 - a_j
//     - (dt/dv) e_max on interior rows, 1 - a_j - DCP on row 0 and
//     1 - a_j + DCM on row nvx - 1 (no flux through the cube faces): the
//     reference's f - (dt/dx)(F+ - F-) - (dt/dv)(G+ - G-) re-associated (a
//     few ulps per step; held to the oracle at 1e-12).
//   * loads: every lane cp.asyncs its own V 16-byte chunks of an input plane
//     into its own slots of a per-warp ring (no cross-lane f traffic), lanes
//     0..4V+6 the level table slices [r, ls, g_x | g_y | E_q | g_z of the
//     warp's 8 v_z]; no CTA barrier anywhere -- every warp is an independent
//     pipeline of D positions.
//   * SYNTH (the window's first pass from moments): level 0 input is the lift
//     f_0 = ls g_x g_y g_z of tab[0] (ref/lifting.py:47-57), no f read.
//
// Ghost planes (bc 0 absorbing: 0; bc 2 outflow: the edge plane of the same
// level) are substituted where level l's neighbour plane falls outside the
// domain; periodic segments wrap (ref/kinetic.py:101-108).  Finiteness
// (ref/kinetic.py:157-159): the stored values are summed per thread;
// non-finite -> status kind 6 at the pass's first step (the host re-runs the
// propagation on the one-step path for the exact BlowUpError(step)).
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace pbgk {

namespace es {
constexpr int NW = 4;             // warps per CTA (independent pipelines)
constexpr int NTHR = 32 * NW;
constexpr int ZW = 8;             // v_z per warp column (4 lanes x 2)
__host__ __device__ constexpr int slice(int V) { return 8 * V + 12; }  // doubles per level slice
// per-warp stage: V double2 per lane + L level slices
__host__ __device__ constexpr int stage_bytes(int V, int L) { return 32 * V * 16 + L * slice(V) * 8; }
}  // namespace es

__device__ __forceinline__ void cp_async_8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The position stream of one warp: items (column, x segment) gw, gw + W, ...;
// an item's input positions p = ps .. pe (inclusive), see the header.
struct EsIt {
  int item, p, pe, x0, x1, y, z0;
  bool done;
  __device__ __forceinline__ void setup(const ESweepArgs& a, int n) {
    const int nitems = a.ncol * a.nseg;
    if (item >= nitems) {
      done = true;
      return;
    }
    const int col = item / a.nseg;
    const int seg = item - col * a.nseg;
    const int nzb = a.nvz / es::ZW;
    y = col / nzb;
    z0 = (col - y * nzb) * es::ZW;
    x0 = seg * a.seglen;
    x1 = min(a.nx, x0 + a.seglen);
    if (a.bc == 1) {
      p = x0 - n;
      pe = x1 + n - 1;
    } else {
      p = max(x0 - n, 0);
      pe = min(x1 + n - 1, a.nx - 1 + n);
    }
    done = false;
  }
  __device__ __forceinline__ void init(const ESweepArgs& a, int n, int first) {
    item = first;
    setup(a, n);
  }
  __device__ __forceinline__ void next(const ESweepArgs& a, int n, int stride) {
    if (done) return;
    if (++p > pe) {
      item += stride;
      setup(a, n);
    }
  }
};

__device__ __forceinline__ int es_wrap(int q, int nx) { return ((q % nx) + nx) % nx; }

template <int V, int L, bool SYNTH, int D>
__global__ void __launch_bounds__(es::NTHR, 2)
    esweep_kernel(const __grid_constant__ ESweepArgs a) {
  using namespace es;
  constexpr int SL = slice(V);
  constexpr int NX8 = 8 * V;  // nvx
  constexpr uint32_t STB = (uint32_t)stage_bytes(V, L);
  constexpr uint32_t FB = 32u * V * 16u;  // f area of a stage
  extern __shared__ __align__(128) unsigned char smem[];
  double2* AK = reinterpret_cast<double2*>(smem);  // [L][nvx] (kappa_interior, a)
  unsigned char* ring0 = smem + (size_t)L * NX8 * sizeof(double2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int s = lane >> 2, c = lane & 3;
  const int n = a.nlev;
  const int nx = a.nx;
  const bool periodic = a.bc == 1;
  const bool outflow = a.bc == 2;

  for (int j = tid; j < L * NX8; j += NTHR) {
    const int l = j / NX8, jx = j - l * NX8;
    const double cv = a.cx[jx];
    const double av = a.dtdx[l] * (cv < 0.0 ? -cv : cv);
    AK[j] = make_double2(1.0 - av - a.dtdv[l] * (2.0 * a.half_emax), av);
  }
  pdl_wait();
  pdl_trigger();
  __syncthreads();

  unsigned char* ring = ring0 + (size_t)warp * D * STB;
  const int gw = blockIdx.x * NW + warp;
  const int nwarps = gridDim.x * NW;
  const bool up = a.cx[s * V] > 0.0;  // the segment's rows share the sign of c_x
  const bool row_lo = s == 0, row_hi = s == 7;

  // issue the loads of one position into stage `st`
  auto issue = [&](const EsIt& it, int st) {
    unsigned char* S = ring + (size_t)st * STB;
    if (!it.done) {
      if (!SYNTH) {
        const int q = periodic ? es_wrap(it.p, nx) : it.p;
        if (q >= 0 && q < nx) {
          const double* src = a.fin + (((size_t)q * NX8 + s * V) * a.nvy + it.y) * a.nvz + it.z0 + 2 * c;
#pragma unroll
          for (int v = 0; v < V; ++v)
            cp_async_16(S + (v * 32 + lane) * 16, src + (size_t)v * a.nvy * a.nvz);
        }
      }
      // level slices: lanes [0, 4V+1) r, ls, g_x (16-byte chunks), 4V+1..4V+4
      // g_z chunks, 4V+5 g_y, 4V+6 E_q
      constexpr int NC = 4 * V + 7;
#pragma unroll
      for (int l = 0; l < L; ++l) {
        if (l >= n) break;
        int q = it.p - l;
        if (periodic) q = es_wrap(q, nx);
        if (q < 0 || q >= nx) continue;
        const double* row = a.tab[l] + (size_t)q * a.TL;
        double* dst = reinterpret_cast<double*>(S + FB) + l * SL;
#pragma unroll
        for (int k0 = 0; k0 < NC; k0 += 32) {
          const int k = k0 + lane;
          if (k <= 4 * V) {
            cp_async_16(dst + 2 * k, row + 2 * k);
          } else if (k < 4 * V + 5) {
            const int m = k - (4 * V + 1);
            cp_async_16(dst + NX8 + 4 + 2 * m, row + a.gzo + it.z0 + 2 * m);
          } else if (k == 4 * V + 5) {
            cp_async_8(dst + NX8 + 2, row + a.gyo + it.y);
          } else if (k == 4 * V + 6) {
            cp_async_8(dst + NX8 + 3, a.E + q);
          }
        }
      }
    }
    cp_async_commit();
  };

  // level carries: relaxed input planes p-l-1 (yh) and p-l-2 (yp), E of p-l-1
  double yh[L][V][2], yp[L][V][2], eh[L];
#pragma unroll
  for (int l = 0; l < L; ++l) {
    eh[l] = 0.0;
#pragma unroll
    for (int v = 0; v < V; ++v) yh[l][v][0] = yh[l][v][1] = yp[l][v][0] = yp[l][v][1] = 0.0;
  }
  double acc = 0.0;

  EsIt pf, cu;
  pf.init(a, n, gw);
  cu.init(a, n, gw);
#pragma unroll
  for (int i = 0; i < D - 1; ++i) {
    issue(pf, i);
    pf.next(a, n, nwarps);
  }
  int stg = 0;
  int ist = D - 1;
  int item = -1;

  // one level on the stage's slice: relax the incoming plane (x, plane p-l)
  // into ynew, transport + field of the held plane (p-l-1) into x.  FAST: all
  // planes interior (no ghosts, no skipped levels)
  auto level = [&](auto lc, auto fastc, double (&x)[V][2], const double* S, int p) {
    constexpr int l = decltype(lc)::value;
    constexpr bool FAST = decltype(fastc)::value;
    const double* T = S + l * SL;
    const int qn = p - l;  // plane of the incoming input (non-periodic: may be a ghost)
    bool ghost = false;
    if (!FAST && !periodic) {
      if (qn < 0 || qn > nx) return false;  // nothing of this level (or later) at this position
      ghost = qn == nx;
    }
    double yn[V][2];
    double en = 0.0;
    if (!ghost) {
      const double2 rl = *reinterpret_cast<const double2*>(T);           // r, ls
      const double2 ge = *reinterpret_cast<const double2*>(T + NX8 + 2);  // g_y, E
      const double2 gz = *reinterpret_cast<const double2*>(T + NX8 + 4 + 2 * c);
      en = ge.y;
      constexpr bool LIFT = SYNTH && l == 0;
      const double rlg = LIFT ? rl.y * ge.x : (rl.x * rl.y) * ge.x;
      double gx[V];
#pragma unroll
      for (int v = 0; v < V; v += 2) {
        const double2 g2 = *reinterpret_cast<const double2*>(T + 2 + s * V + v);
        gx[v] = g2.x;
        gx[v + 1] = g2.y;
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const double w = rlg * gx[v];
        if (LIFT) {
          yn[v][0] = w * gz.x;
          yn[v][1] = w * gz.y;
        } else {
          yn[v][0] = fma(w, gz.x, rl.x * x[v][0]);
          yn[v][1] = fma(w, gz.y, rl.x * x[v][1]);
        }
      }
    } else {
      // right ghost plane nx of this level: 0 (absorbing) or plane nx-1 (outflow)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        yn[v][0] = outflow ? yh[l][v][0] : 0.0;
        yn[v][1] = outflow ? yh[l][v][1] : 0.0;
      }
    }
    const int qh = qn - 1;
    const bool work = FAST || periodic || qh >= 0;
    if (work) {
      // left ghost plane -1 of this level when the held plane is 0
      if (!FAST && !periodic && qh == 0) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          yp[l][v][0] = outflow ? yh[l][v][0] : 0.0;
          yp[l][v][1] = outflow ? yh[l][v][1] : 0.0;
        }
      }
      const double hE = 0.5 * eh[l];
      const double DCP = a.dtdv[l] * (hE + a.half_emax);
      const double DCM = a.dtdv[l] * (hE - a.half_emax);
      double lo[2], hi[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        lo[k] = __shfl_up_sync(0xffffffffu, yh[l][V - 1][k], 4);
        hi[k] = __shfl_down_sync(0xffffffffu, yh[l][0][k], 4);
        if (row_lo) lo[k] = 0.0;
        if (row_hi) hi[k] = 0.0;
      }
      const double2* AKl = AK + l * NX8 + s * V;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const double2 ka = AKl[v];
        double kap = ka.x;
        if (v == 0 && row_lo) kap = ka.x + 2.0 * a.dtdv[l] * a.half_emax - DCP;
        if (v == V - 1 && row_hi) kap = ka.x + 2.0 * a.dtdv[l] * a.half_emax + DCM;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double ym = v > 0 ? yh[l][v - 1][k] : lo[k];
          const double yq = v < V - 1 ? yh[l][v + 1][k] : hi[k];
          const double nb = up ? yp[l][v][k] : yn[v][k];
          x[v][k] = fma(kap, yh[l][v][k], fma(ka.y, nb, fma(DCP, ym, -(DCM * yq))));
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      yp[l][v][0] = yh[l][v][0];
      yp[l][v][1] = yh[l][v][1];
      yh[l][v][0] = yn[v][0];
      yh[l][v][1] = yn[v][1];
    }
    eh[l] = en;
    return work;
  };

#pragma unroll 1
  while (!cu.done) {
    __syncwarp();
    issue(pf, ist);
    pf.next(a, n, nwarps);
    if (++ist == D) ist = 0;
    cp_async_wait<D - 1>();
    __syncwarp();
    if (cu.item != item) {
      // a new item: its carries restart (the halo positions refill them)
      item = cu.item;
#pragma unroll
      for (int l = 0; l < L; ++l) {
        eh[l] = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) yh[l][v][0] = yh[l][v][1] = yp[l][v][0] = yp[l][v][1] = 0.0;
      }
    }
    const unsigned char* S = ring + (size_t)stg * STB;
    const double* ST = reinterpret_cast<const double*>(S + FB);
    const int p = cu.p;
    double x[V][2];
    if (!SYNTH) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const double2 u = *reinterpret_cast<const double2*>(S + (v * 32 + lane) * 16);
        x[v][0] = u.x;
        x[v][1] = u.y;
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) x[v][0] = x[v][1] = 0.0;
    }
    const bool fast = periodic || (p >= n + 1 && p <= nx - 1);
    // (each level decides from its own planes whether it runs: a skipped
    // level's successors either skip too or only see a ghost input)
    if (fast && n == L) {
      level(std::integral_constant<int, 0>{}, std::true_type{}, x, ST, p);
      if constexpr (L > 1) level(std::integral_constant<int, 1>{}, std::true_type{}, x, ST, p);
      if constexpr (L > 2) level(std::integral_constant<int, 2>{}, std::true_type{}, x, ST, p);
      if constexpr (L > 3) level(std::integral_constant<int, 3>{}, std::true_type{}, x, ST, p);
    } else {
      level(std::integral_constant<int, 0>{}, std::false_type{}, x, ST, p);
      if constexpr (L > 1) if (n > 1) level(std::integral_constant<int, 1>{}, std::false_type{}, x, ST, p);
      if constexpr (L > 2) if (n > 2) level(std::integral_constant<int, 2>{}, std::false_type{}, x, ST, p);
      if constexpr (L > 3) if (n > 3) level(std::integral_constant<int, 3>{}, std::false_type{}, x, ST, p);
    }
    // output plane p - n of the last level (inside the segment, the last
    // level's held plane is a real plane, so it ran)
    const int qo = p - n;
    if (qo >= cu.x0 && qo < cu.x1) {
      double* dst = a.fout + (((size_t)qo * NX8 + s * V) * a.nvy + cu.y) * a.nvz + cu.z0 + 2 * c;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        st_global_v2(dst + (size_t)v * a.nvy * a.nvz, x[v][0], x[v][1]);
        acc += x[v][0] + x[v][1];
      }
    }
    if (++stg == D) stg = 0;
    cu.next(a, n, nwarps);
  }
  cp_async_wait<0>();
  if (!isfinite(acc)) atomicMin(a.err, err_key(0, a.step0, kErrNonFiniteMulti));
}

// shapes the kernel runs: nvx = 8 V (V = 2, 4, 6, 8), nvz % 8 == 0, the
// table layout of capi.cu (g_x at 2, g_z 16-byte aligned)
#ifndef PBGK_ES_L4
#define PBGK_ES_L4 3  // levels of the nvx = 32 build (dev A/B knob: 2, 3 or 4)
#endif
int esweep_levels(int nvx, int nvz) {
  if (nvx % 8 != 0 || nvz % es::ZW != 0) return 0;
  switch (nvx / 8) {
    case 2: return 4;
    case 4: return PBGK_ES_L4;
    case 6: return 2;
  }
  return 0;  // (nvx = 64: two levels need 768 B of spills; one-step passes)
}

constexpr int kEsD = 4;  // ring stages per warp

size_t esweep_smem_bytes(int nvx) {
  const int V = nvx / 8;
  const int L = esweep_levels(nvx, 8);
  return (size_t)L * nvx * 16 + (size_t)es::NW * kEsD * es::stage_bytes(V, L);
}

int esweep_ctas_per_sm(int nvx);

template <int V, int L, bool SYNTH>
static cudaError_t launch_es(const ESweepArgs& a, int grid, size_t smem, cudaStream_t st) {
  auto fn = esweep_kernel<V, L, SYNTH, kEsD>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(fn, grid, es::NTHR, smem, st, a);
}

template <int V, int L>
static int occ(size_t smem) {
  int n = 0;
  auto fn = esweep_kernel<V, L, false, kEsD>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, es::NTHR, smem) != cudaSuccess) return 0;
  return n;
}

int esweep_ctas_per_sm(int nvx) {
  const size_t smem = esweep_smem_bytes(nvx);
  switch (nvx / 8) {
    case 2: return occ<2, 4>(smem);
    case 4: return occ<4, PBGK_ES_L4>(smem);
    case 6: return occ<6, 2>(smem);
  }
  return 0;
}

cudaError_t launch_esweep(const ESweepArgs& a, bool synth, int grid, size_t smem, cudaStream_t st) {
  switch (a.nvx / 8) {
    case 2: return synth ? launch_es<2, 4, true>(a, grid, smem, st) : launch_es<2, 4, false>(a, grid, smem, st);
    case 4:
      return synth ? launch_es<4, PBGK_ES_L4, true>(a, grid, smem, st)
                   : launch_es<4, PBGK_ES_L4, false>(a, grid, smem, st);
    case 6: return synth ? launch_es<6, 2, true>(a, grid, smem, st) : launch_es<6, 2, false>(a, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace pbgk
