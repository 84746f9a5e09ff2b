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
//   * FINAL (the window's last pass): the column's marginal partial record
//     [m_x rows | m_y | m_z] of the last level's output f*_S written per
//     plane for finalize.cu (kFinProject, the projection P(f_S) of
//     ref/moments.py:60-112; it applies the linear, separable R_S of
//     ref/kinetic.py:130-134 to the marginals) instead of f_S: no store and
//     no read-back of f_S.  Fixed trees, the same for every entry and its
//     mirror (even data keeps an exactly zero folded first moment).
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
// predicated copies: every lane runs the same instructions (no divergent
// branches on the loader roles)
__device__ __forceinline__ void cp_async_16_if(uint32_t dst, const void* src, bool on) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %2, 0; @p cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(dst),
      "l"(src), "r"((int)on)
      : "memory");
}
__device__ __forceinline__ void cp_async_8_if(uint32_t dst, const void* src, bool on) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %2, 0; @p cp.async.ca.shared.global [%0], [%1], 8; }" ::"r"(dst),
      "l"(src), "r"((int)on)
      : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The position stream of one warp: items (column, x segment) gw, gw + W, ...;
// an item's input positions p = ps .. pe (inclusive), see the header.
struct EsIt {
  int item, p, pe, x0, x1, y, z0, col;
  long long foff;  // (y nvz + z0): the column's offset inside a v_x row of a plane (doubles)
  bool done;
  __device__ __forceinline__ void setup(const ESweepArgs& a, int n) {
    const int nitems = a.ncol * a.nseg;
    if (item >= nitems) {
      done = true;
      return;
    }
    col = item / a.nseg;
    const int seg = item - col * a.nseg;
    const int nzb = a.nvz / es::ZW;
    y = col / nzb;
    z0 = (col - y * nzb) * es::ZW;
    foff = (long long)y * a.nvz + z0;
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

template <int V, int L, bool SYNTH, int D, bool FINAL>
__global__ void __launch_bounds__(es::NTHR, 2)
    esweep_kernel(const __grid_constant__ ESweepArgs a) {
  using namespace es;
  constexpr int H = V / 2;    // rows of each c_x sign per lane
  constexpr int SL = slice(V);
  constexpr int NX8 = 8 * V;  // nvx
  constexpr int NS = L;  // table slices per stage
  constexpr uint32_t STB = (uint32_t)stage_bytes(V, NS);
  constexpr uint32_t FB = 32u * V * 16u;  // f area of a stage
  extern __shared__ __align__(128) unsigned char smem[];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int s = lane >> 2, c = lane & 3;
  const int n = a.nlev;
  const int nx = a.nx;
  const bool periodic = a.bc == 1;
  const bool outflow = a.bc == 2;

  pdl_wait();
  pdl_trigger();

  unsigned char* ring = smem + (size_t)warp * D * STB;
  const int gw = blockIdx.x * NW + warp;
  const int nwarps = gridDim.x * NW;
  // this lane's rows: v < H the c_x < 0 rows s H + v (their upwind plane is
  // q + 1), v >= H the c_x > 0 rows nvx/2 + s H + (v - H) (upwind plane q - 1)
  const int rd0 = s * H, ru0 = NX8 / 2 + s * H;
  double ac[V];  // |c_x| of the rows
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const double cv = a.cx[v < H ? rd0 + v : ru0 + (v - H)];
    ac[v] = cv < 0.0 ? -cv : cv;
  }
  const bool row_lo = s == 0, row_hi = s == 7;  // the lane holds row 0 / row nvx - 1
  const int lane_up = (lane + 4) & 31, lane_dn = (lane + 28) & 31;  // lanes s + 1 / s - 1 (mod 8)

  // the loader role of this lane for a level slice [r, ls, g_x | g_y, E | g_z
  // of the warp's 8 v_z]: lanes 0 .. 4V the 16-byte chunks of r, ls, g_x, the
  // next four those of g_z, then one 8-byte copy each of g_y and E; per-lane
  // source offset (from the table row, or from E) and destination offset,
  // the column's part of the source added per item
  constexpr int NC = 4 * V + 7;
  static_assert(NC <= 32, "one loader round per level");
  const bool r16 = lane <= 4 * V + 4, r8 = lane == 4 * V + 5 || lane == 4 * V + 6;
  const bool rz = lane > 4 * V && lane <= 4 * V + 4, ry = lane == 4 * V + 5, rE = lane == 4 * V + 6;
  const int soff0 = lane <= 4 * V ? 2 * lane : (rz ? a.gzo + 2 * (lane - (4 * V + 1)) : (ry ? a.gyo : 0));
  const int doff = lane <= 4 * V ? 2 * lane : (rz ? NX8 + 4 + 2 * (lane - (4 * V + 1)) : (ry ? NX8 + 2 : NX8 + 3));
  const long long rs = (long long)a.nvy * a.nvz;      // one v_x row of a plane
  const long long plane = (long long)NX8 * rs;
  const long long lane_f = (long long)rd0 * rs + 2 * c;  // this lane's first row + v_z pair
  const uint32_t ring_u = smem_u32(ring);

  // issue the loads of one position into stage `st`
  auto issue = [&](const EsIt& it, int st) {
    const uint32_t S = ring_u + (uint32_t)st * STB;
    if (!it.done) {
      int q0 = it.p;
      if (periodic) q0 = q0 < 0 ? q0 + nx : (q0 >= nx ? q0 - nx : q0);
      if (!SYNTH) {
        const bool on = q0 >= 0 && q0 < nx;
        const double* src = a.fin + ((long long)q0 * plane + lane_f + it.foff);
#pragma unroll
        for (int v = 0; v < V; ++v)
          cp_async_16_if(S + (v * 32 + lane) * 16, src + (long long)(v < H ? v : NX8 / 2 - H + v) * rs, on);
      }
      const int so = soff0 + (rz ? it.z0 : (ry ? it.y : 0));
#pragma unroll
      for (int l = 0; l < NS; ++l) {
        if (l >= n) break;
        int q = q0 - l;
        if (periodic && q < 0) q += nx;
        const bool on = q >= 0 && q < nx;
        const double* src = rE ? a.E + q : a.tab[l] + ((long long)q * a.TL + so);
        const uint32_t dst = S + FB + (uint32_t)(l * SL + doff) * 8u;
        cp_async_16_if(dst, src, on && r16);
        cp_async_8_if(dst, src, on && r8);
      }
    }
    cp_async_commit();
  };

  // Level carries, double-buffered by the parity of the position (no register
  // moves: slot ph holds the plane relaxed at the previous position, slot
  // ph ^ 1 receives this position's):
  //   yh: the relaxed input plane, all rows
  //   xd: the c_x > 0 rows' output, which a level computes one position
  //       earlier than its c_x < 0 rows' (see `level`) and hands on with them
  //   eh: E of the held plane
  double yh[L][2][V][2], xd[L][2][H][2], eh[L][2];
  auto zero_carries = [&]() {
#pragma unroll
    for (int l = 0; l < L; ++l)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        eh[l][b] = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) yh[l][b][v][0] = yh[l][b][v][1] = 0.0;
#pragma unroll
        for (int v = 0; v < H; ++v) xd[l][b][v][0] = xd[l][b][v][1] = 0.0;
      }
  };
  zero_carries();
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

  // One level at one position.  In: x = plane m = p - l of the level's input
  // (all rows).  The level relaxes it (y_m), then transports
  //   * its c_x < 0 rows on plane m - 1 (held y_{m-1}, upwind neighbour y_m,
  //     v_x neighbours from y_{m-1}, E_{m-1}), and
  //   * its c_x > 0 rows on plane m itself (y_m, upwind neighbour y_{m-1},
  //     v_x neighbours from y_m, E_m), kept for one position,
  // and hands plane m - 1 on: the c_x < 0 rows just computed with the c_x > 0
  // rows computed at the previous position.  One carry per element either
  // way.  Out: x = plane m - 1 of the level's output.  FAST: every plane
  // interior (no ghosts, no skipped levels).
  auto level = [&](auto lc, auto phc, auto fastc, double (&x)[V][2], const double* S, int p) {
    constexpr int l = decltype(lc)::value;
    constexpr int PH = decltype(phc)::value;
    constexpr bool FAST = decltype(fastc)::value;
    const double* T = S + l * SL;
    const int m = p - l;
    bool ghost = false;
    double(&yn)[V][2] = yh[l][PH ^ 1];
    double(&yo)[V][2] = yh[l][PH];
    if (!FAST && !periodic) {
      if (m < 0 || m > nx) {
        // nothing of this level (or a later one) at this position; its (unused)
        // carries change slots, so that only one slot is live between positions
#pragma unroll
        for (int v = 0; v < V; ++v) yn[v][0] = yo[v][0], yn[v][1] = yo[v][1];
#pragma unroll
        for (int v = 0; v < H; ++v) xd[l][PH ^ 1][v][0] = xd[l][PH][v][0], xd[l][PH ^ 1][v][1] = xd[l][PH][v][1];
        eh[l][PH ^ 1] = eh[l][PH];
        return;
      }
      ghost = m == nx;
    }
    double en = 0.0;
    if (!ghost) {
      const double2 rl = *reinterpret_cast<const double2*>(T);            // r, ls
      const double2 ge = *reinterpret_cast<const double2*>(T + NX8 + 2);  // g_y, E
      const double2 gz = *reinterpret_cast<const double2*>(T + NX8 + 4 + 2 * c);
      en = ge.y;
      constexpr bool LIFT = SYNTH && l == 0;
      const double rlg = LIFT ? rl.y * ge.x : (rl.x * rl.y) * ge.x;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const double w = rlg * T[2 + (v < H ? rd0 + v : ru0 + (v - H))];
        if (LIFT) {
          yn[v][0] = w * gz.x;
          yn[v][1] = w * gz.y;
        } else {
          yn[v][0] = fma(w, gz.x, rl.x * x[v][0]);
          yn[v][1] = fma(w, gz.y, rl.x * x[v][1]);
        }
      }
    } else {
      // right ghost plane nx of this level: 0 (absorbing) or plane nx - 1 (outflow)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        yn[v][0] = outflow ? yo[v][0] : 0.0;
        yn[v][1] = outflow ? yo[v][1] : 0.0;
      }
    }
    eh[l][PH ^ 1] = en;
    // left ghost plane -1 when the incoming plane is 0
    if (!FAST && !periodic && m == 0) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        yo[v][0] = outflow ? yn[v][0] : 0.0;
        yo[v][1] = outflow ? yn[v][1] : 0.0;
      }
    }
    const double dv = a.dtdv[l], dxl = a.dtdx[l];
    const double k0 = 1.0 - dv * (2.0 * a.half_emax);  // interior rows: 1 - a_j - (dt/dv) e_max
    // c_x < 0 rows, plane m - 1: v_x neighbours from the held plane
    {
      const double hE = 0.5 * eh[l][PH];
      const double DCP = dv * (hE + a.half_emax), DCM = dv * (hE - a.half_emax);
      double lo[2], hi[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        // below: row s H - 1 (lane s - 1's last c_x < 0 row; none for row 0);
        // above: row (s + 1) H (lane s + 1's first c_x < 0 row; for s = 7 row
        // nvx / 2, lane s = 0's first c_x > 0 row)
        lo[k] = __shfl_sync(0xffffffffu, yo[H - 1][k], lane_dn);
        hi[k] = __shfl_sync(0xffffffffu, row_lo ? yo[H][k] : yo[0][k], lane_up);
        if (row_lo) lo[k] = 0.0;
      }
#pragma unroll
      for (int v = 0; v < H; ++v) {
        const double av = dxl * ac[v];
        double kap = k0 - av;
        if (v == 0 && row_lo) kap = (1.0 - av) - DCP;  // row 0: no flux through the cube face
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double ym = v > 0 ? yo[v - 1][k] : lo[k];
          const double yq = v < H - 1 ? yo[v + 1][k] : hi[k];
          x[v][k] = fma(kap, yo[v][k], fma(av, yn[v][k], fma(DCP, ym, -(DCM * yq))));
        }
      }
    }
    // c_x > 0 rows, plane m: v_x neighbours from the incoming plane; handed
    // on at the next position
    {
      const double hE = 0.5 * en;
      const double DCP = dv * (hE + a.half_emax), DCM = dv * (hE - a.half_emax);
      double lo[2], hi[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        // below: row nvx/2 + s H - 1 (lane s - 1's last c_x > 0 row; for s = 0
        // row nvx/2 - 1, lane s = 7's last c_x < 0 row); above: lane s + 1's
        // first c_x > 0 row (none for row nvx - 1)
        lo[k] = __shfl_sync(0xffffffffu, row_hi ? yn[H - 1][k] : yn[V - 1][k], lane_dn);
        hi[k] = __shfl_sync(0xffffffffu, yn[H][k], lane_up);
        if (row_hi) hi[k] = 0.0;
      }
#pragma unroll
      for (int v = H; v < V; ++v) {
        const double av = dxl * ac[v];
        double kap = k0 - av;
        if (v == V - 1 && row_hi) kap = (1.0 - av) + DCM;  // row nvx - 1
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double ym = v > H ? yn[v - 1][k] : lo[k];
          const double yq = v < V - 1 ? yn[v + 1][k] : hi[k];
          x[v][k] = xd[l][PH][v - H][k];
          xd[l][PH ^ 1][v - H][k] = fma(kap, yn[v][k], fma(av, yo[v][k], fma(DCP, ym, -(DCM * yq))));
        }
      }
    }
  };

  auto position = [&](auto phc, auto fastc, const unsigned char* S, int p, const EsIt& it) {
    constexpr bool FAST = decltype(fastc)::value;
    constexpr int PHV = decltype(phc)::value;
    const double* ST = reinterpret_cast<const double*>(S + FB);
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
    level(std::integral_constant<int, 0>{}, phc, fastc, x, ST, p);
    if constexpr (L > 1) if (FAST || n > 1) level(std::integral_constant<int, 1>{}, phc, fastc, x, ST, p);
    if constexpr (L > 2) if (FAST || n > 2) level(std::integral_constant<int, 2>{}, phc, fastc, x, ST, p);
    if constexpr (L > 3) if (FAST || n > 3) level(std::integral_constant<int, 3>{}, phc, fastc, x, ST, p);
    (void)PHV;
    // output plane p - n of the last level
    const int qo = p - n;
    if (qo >= it.x0 && qo < it.x1) {
      if constexpr (FINAL) {
        // the column's partial record of plane qo of f*_S (finalize applies R_S
        // to the marginals: FinalArgs relax_tab).  Two or four values are
        // reduced per shuffle round -- a lane keeps some and sends the others,
        // the partner keeps those -- so every total is the tree of a plain
        // butterfly: a row total = the lane's two v_z, then the 4 v_z pairs;
        // an m_z entry = the lane's rows in order, then the 8 row groups;
        // m_y = the kept row totals over all lanes.
        static_assert(V == 2 || V == 4 || V == 6, "row totals per lane");
        double t[V], zs[2] = {0.0, 0.0};
#pragma unroll
        for (int v = 0; v < V; ++v) {
          t[v] = x[v][0] + x[v][1];
          zs[0] = v == 0 ? x[v][0] : zs[0] + x[v][0];
          zs[1] = v == 0 ? x[v][1] : zs[1] + x[v][1];
        }
        // row totals over c (lanes xor 1, xor 2): V values -> V / 2 -> ...
        const bool c0 = c & 1, c1 = (c >> 1) & 1;
        constexpr int V2 = V / 2;
        double u[V2];
#pragma unroll
        for (int v = 0; v < V2; ++v) {
          const double keep = c0 ? t[V2 + v] : t[v];
          const double send = c0 ? t[v] : t[V2 + v];
          u[v] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        }
        // u[v] = rows (c0 ? V2 + v : v) summed over the pair (c, c ^ 1)
        double rowt;       // one finished row total per lane (V == 6: two on c1 == 0 lanes, one on the others)
        double rowt2 = 0.0;
        int rv, rv2 = -1;  // its row slot v
        if constexpr (V2 == 1) {
          rowt = u[0] + __shfl_xor_sync(0xffffffffu, u[0], 2);
          rv = c0 ? 1 : 0;
        } else if constexpr (V2 == 2) {
          const double keep = c1 ? u[1] : u[0];
          const double send = c1 ? u[0] : u[1];
          rowt = keep + __shfl_xor_sync(0xffffffffu, send, 2);
          rv = (c0 ? V2 : 0) + (c1 ? 1 : 0);
        } else {
          // three values over two lanes: slot 0 / 1 exchanged, slot 2 a butterfly
          const double keep = c1 ? u[1] : u[0];
          const double send = c1 ? u[0] : u[1];
          rowt = keep + __shfl_xor_sync(0xffffffffu, send, 2);
          rv = (c0 ? V2 : 0) + (c1 ? 1 : 0);
          rowt2 = u[2] + __shfl_xor_sync(0xffffffffu, u[2], 2);
          rv2 = c1 ? -1 : (c0 ? V2 : 0) + 2;
        }
        // m_z over the row groups s (lanes xor 4, 8, 16)
        const bool s0b = s & 1;
        double zt = (s0b ? zs[1] : zs[0]) + __shfl_xor_sync(0xffffffffu, s0b ? zs[0] : zs[1], 4);
        zt += __shfl_xor_sync(0xffffffffu, zt, 8);
        zt += __shfl_xor_sync(0xffffffffu, zt, 16);
        // m_y: every finished row total once (rowt2 only where it is kept)
        // (V == 2: both c1 lanes hold the same row total, one of them counts)
        double tot = ((V2 == 1 && c1) ? 0.0 : rowt) + ((V2 == 3 && !c1) ? rowt2 : 0.0);
#pragma unroll
        for (int m = 1; m <= 16; m <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, m);
        acc += tot;
        double* R = a.part + ((long long)qo * a.ncol + it.col) * a.PS;
        R[rv < H ? rd0 + rv : ru0 + (rv - H)] = rowt;
        if (V2 == 3 && rv2 >= 0) R[rv2 < H ? rd0 + rv2 : ru0 + (rv2 - H)] = rowt2;
        if (s < 2) R[NX8 + 1 + 2 * c + s] = zt;
        if (lane == 0) R[NX8] = tot;
      } else {
        double* dst = a.fout + ((long long)qo * plane + lane_f + it.foff);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          st_global_v2(dst + (long long)(v < H ? v : NX8 / 2 - H + v) * rs, x[v][0], x[v][1]);
          acc += x[v][0] + x[v][1];
        }
      }
    }
  };

  // one position (parity PH of the carries' slots); false at the end
  auto step = [&](auto phc) {
    constexpr int PH = decltype(phc)::value;
    if (cu.done) return false;
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
        eh[l][PH] = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v) yh[l][PH][v][0] = yh[l][PH][v][1] = 0.0;
#pragma unroll
        for (int v = 0; v < H; ++v) xd[l][PH][v][0] = xd[l][PH][v][1] = 0.0;
      }
    }
    const unsigned char* S = ring + (size_t)stg * STB;
    const int p = cu.p;
    // FAST: every level's planes p - l and p - l - 1 are interior, all levels run
    const bool fast = n == L && (periodic || (p >= n + 1 && p <= nx - 1));
    if (fast) position(phc, std::true_type{}, S, p, cu);
    else position(phc, std::false_type{}, S, p, cu);
    if (++stg == D) stg = 0;
    cu.next(a, n, nwarps);
    return true;
  };
#pragma unroll 1
  while (true) {
    if (!step(std::integral_constant<int, 0>{})) break;
    if (!step(std::integral_constant<int, 1>{})) break;
  }
  cp_async_wait<0>();
  if (!isfinite(acc)) atomicMin(a.err, err_key(0, a.step0, kErrNonFiniteMulti));
}

// shapes the kernel runs: nvx = 8 V (V = 2, 4, 6, 8: a lane holds V / 2 rows
// of each c_x sign), nvz % 8 == 0, the table layout of capi.cu (g_x at 2, g_z
// 16-byte aligned)
#ifndef PBGK_ES_L2
#define PBGK_ES_L2 4  // levels of the nvx = 16 build (dev A/B knobs)
#endif
#ifndef PBGK_ES_L4
#define PBGK_ES_L4 3  // nvx = 32 (4: 150 B of spills, 13 % slower)
#endif
#ifndef PBGK_ES_L6
#define PBGK_ES_L6 2  // nvx = 48 (3 spills)
#endif
#ifndef PBGK_ES_L8
#define PBGK_ES_L8 0  // nvx = 64: off (2 levels spill; one-step field passes)
#endif
int esweep_levels(int nvx, int nvz) {
  if (nvx % 16 != 0 || nvz % es::ZW != 0) return 0;
  switch (nvx / 8) {
    case 2: return PBGK_ES_L2;
    case 4: return PBGK_ES_L4;
    case 6: return PBGK_ES_L6;
    case 8: return PBGK_ES_L8;
  }
  return 0;
}

#ifndef PBGK_ES_D
#define PBGK_ES_D 4
#endif
constexpr int kEsD = PBGK_ES_D;  // ring stages per warp

size_t esweep_smem_bytes(int nvx, bool fin) {
  (void)fin;  // (the FINAL pass loads the same slices)
  const int V = nvx / 8;
  const int L = esweep_levels(nvx, 8);
  return (size_t)es::NW * kEsD * es::stage_bytes(V, L);
}

// the tiling of the FINAL pass's partial records for finalize.cu: one tile per
// warp column (all v_x rows x 1 v_y x 8 v_z)
void esweep_tiling(int nvx, int nvy, int nvz, Tiling* t) {
  t->A = nvx;
  t->By = 1;
  t->Bz = es::ZW;
  t->rows_load = nvx;
  t->nneg = 0;
  t->ntn = 0;
  t->ntp = 1;
  t->nty = nvy;
  t->ntz = nvz / es::ZW;
  t->NT = t->nty * t->ntz;
  t->PS = nvx + 10;
}

int esweep_ctas_per_sm(int nvx);

template <int V, int L, bool SYNTH, bool FINAL>
static cudaError_t launch_es(const ESweepArgs& a, int grid, size_t smem, cudaStream_t st) {
  auto fn = esweep_kernel<V, L, SYNTH, kEsD, FINAL>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(fn, grid, es::NTHR, smem, st, a);
}

template <int V, int L>
static int occ(size_t smem) {
  int n = 0;
  auto fn = esweep_kernel<V, L, false, kEsD, true>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, es::NTHR, smem) != cudaSuccess) return 0;
  return n;
}

// resident CTAs per SM (of the FINAL build: the larger stage)
int esweep_ctas_per_sm(int nvx) {
  const size_t smem = esweep_smem_bytes(nvx, true);
  switch (nvx / 8) {
    case 2: return occ<2, PBGK_ES_L2>(smem);
    case 4: return occ<4, PBGK_ES_L4>(smem);
    case 6: return occ<6, PBGK_ES_L6>(smem);
  }
  return 0;
}

template <int V, int L>
static cudaError_t launch_es_v(const ESweepArgs& a, bool synth, int grid, size_t smem, cudaStream_t st) {
  const bool fin = a.tabR != nullptr;
  if (synth) return fin ? launch_es<V, L, true, true>(a, grid, smem, st) : launch_es<V, L, true, false>(a, grid, smem, st);
  return fin ? launch_es<V, L, false, true>(a, grid, smem, st) : launch_es<V, L, false, false>(a, grid, smem, st);
}

cudaError_t launch_esweep(const ESweepArgs& a, bool synth, int grid, size_t smem, cudaStream_t st) {
  switch (a.nvx / 8) {
    case 2: return launch_es_v<2, PBGK_ES_L2>(a, synth, grid, smem, st);
    case 4: return launch_es_v<4, PBGK_ES_L4>(a, synth, grid, smem, st);
    case 6: return launch_es_v<6, PBGK_ES_L6>(a, synth, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace pbgk
