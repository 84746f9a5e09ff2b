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
// Work decomposition (persistent CTAs, 2 per SM):
//   velocity box "tile" (A rows of v_x, By of v_y, Bz of v_z) x all x cells.
//   Every tile has one sign of c_x, so its upwind neighbour plane is on one
//   side: c_x >= 0 tiles march upward in x, c_x < 0 tiles march downward, and
//   each thread keeps f_pre of the previous plane for its elements in
//   registers.  The (tile, plane) sequence is cut into gridDim.x contiguous
//   segments; a segment pays one halo plane per tile run it touches.
//   Each plane's box arrives by one 4-D TMA copy (plus a 1-D bulk copy of the
//   cell's table row) into a ring of `ns` shared-memory stages.
//   Thread layout: LZ lanes x V consecutive v_z per box line (a line is one
//   (v_x, v_y) pair of the box), K lines per thread.
//
// Reductions are deterministic and mirror-symmetric (the same tree for every
// marginal index), so even data keeps an exactly-zero folded first moment
// (ref/moments.py:80-88).  Non-finite values are not tested per element here:
// they propagate into the marginals and the finalize kernel flags the step.
//
// Template variants: SYNTH (first pass from lift tables), FIELD (the v_x
// Rusanov term of ref/kinetic.py:114-123), TMA (vs a cooperative-load
// fallback for odd shapes), and three extensions: MUSCL (minmod x transport,
// output one plane behind the loads, 2 lead / 1 trail halo items per run),
// TRAP (trapezoidal velocity quadrature: end nodes weigh 1/2 in the
// reductions), NORED (the multi-step path's field passes: no marginal
// partials, a finiteness sum instead; field variants only).  bc 3 (runtime) is a slab of an x-sharded domain whose halo
// planes sit in the padded buffers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

#ifndef PBGK_HINT_LOAD
#define PBGK_HINT_LOAD 0
#endif
#ifndef PBGK_HINT_STORE
#define PBGK_HINT_STORE 0
#endif
#ifndef PBGK_HINT_PART
#define PBGK_HINT_PART 1
#endif
#ifndef PBGK_OUT_ROT
#define PBGK_OUT_ROT 1
#endif

namespace pbgk {

constexpr unsigned FULL = 0xffffffffu;

// Reduce-scatter of C per-lane line values over the W..1 lane bits of an
// aligned lane group.  After the split levels each lane holds max(C/LZ, 1)
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

// Walks the items of a segment [g0, g1) of the (tile, position) sequence:
// every run of consecutive positions of one tile is preceded by LEAD halo
// items (its upwind neighbour planes: 1 for upwind, 2 for MUSCL) and, with
// TRAIL, followed by one look-ahead item (MUSCL's downwind neighbour of the
// run's last plane).  Item kinds: lead halo, first / later plane of the run,
// trail.  Positions of halo / trail items may fall outside [0, nx).
enum ItemKind : int { kLead = 0, kFirst = 1, kNormal = 2, kTrail = 3 };

template <int LEAD, int TRAIL>
struct ItemIter {
  int g, g1;    // next plane-item index (global linear) and segment end
  int tile, p;  // tile and position of g
  int lead_left;
  bool first;
  bool trail_next;
  int trail_tile, trail_p;

  __device__ __forceinline__ void init(int g0, int end, int nx) {
    g = g0;
    g1 = end;
    tile = g0 / nx;
    p = g0 - tile * nx;
    lead_left = g0 < end ? LEAD : 0;
    first = true;
    trail_next = false;
  }
  __device__ __forceinline__ bool done() const { return g >= g1 && lead_left == 0 && !trail_next; }
  // current item: (tile, position, kind); then advance
  __device__ __forceinline__ void next(int nx, int& t_out, int& p_out, int& kind) {
    if (TRAIL && trail_next) {
      t_out = trail_tile;
      p_out = trail_p;
      kind = kTrail;
      trail_next = false;
      return;
    }
    t_out = tile;
    if (lead_left > 0) {
      p_out = p - lead_left;
      kind = kLead;
      --lead_left;
      return;
    }
    p_out = p;
    kind = first ? kFirst : kNormal;
    first = false;
    ++g;
    if (++p == nx || g >= g1) {  // end of this run
      if (TRAIL) {
        trail_next = true;
        trail_tile = tile;
        trail_p = p;
      }
      if (p == nx) {
        p = 0;
        ++tile;
      }
      if (g < g1) {
        lead_left = LEAD;
        first = true;
      }
    }
  }
};

// x cell of march position p of a tile (p may be outside [0, nx) for halo /
// trail items); -1 = absorbing ghost (f == 0).  Ghost planes: periodic wrap,
// zero-gradient copy of the edge plane (outflow) or zero (absorbing).  bc 3
// (a slab of an x-sharded domain): -1 and nx are the halo planes, kept as
// such; the slab's buffers are padded by one plane / table row per side.
__device__ __forceinline__ int item_plane(int nx, int bc, const TileGeom& tg, int p) {
  int i = tg.down ? nx - 1 - p : p;
  if ((i < 0 || i >= nx) && bc != 3)
    i = (bc == 1) ? ((i % nx) + nx) % nx : (bc == 2 ? (i < 0 ? 0 : nx - 1) : -1);
  return i;
}

// Lane z layout: V consecutive v_z per lane (16/32-byte vectors) for even V;
// interleaved (element v of lane lz at v*LZ + lz) for odd V, so that every
// store instruction of a warp covers whole 32-byte sectors.
template <int V, int LZ>
__device__ __forceinline__ constexpr int zpos(int lz, int v) {
  return (V % 2 == 0 || V == 1) ? lz * V + v : v * LZ + lz;
}

template <int V, int LZ>
__device__ __forceinline__ void lds_lane(const double* p, double (&x)[V]) {
  if constexpr (V % 2 == 0) {
#pragma unroll
    for (int v = 0; v < V; v += 2) {
      const double2 t = *reinterpret_cast<const double2*>(p + v);
      x[v] = t.x;
      x[v + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) x[v] = p[v * LZ];
  }
}

template <int V>
__device__ __forceinline__ void lds_vec(const double* p, double (&x)[V]) {
  if constexpr (V % 2 == 0) {
#pragma unroll
    for (int v = 0; v < V; v += 2) {
      const double2 t = *reinterpret_cast<const double2*>(p + v);
      x[v] = t.x;
      x[v + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) x[v] = p[v];
  }
}

// Store of one lane's V outputs of a line: one 32-byte vector (V = 4), 16-byte
// pairs (other even V) or masked scalars (odd V / partial rows).
template <int V, int LZ, bool FAST>
__device__ __forceinline__ void store_line(double* d, const double (&o)[V], unsigned zmask,
                                           bool keep = false, uint64_t pol = 0) {
  if constexpr (V == 4) {
    if (FAST || zmask == 0xfu) {
      st_global_v4(d, o[0], o[1], o[2], o[3]);
      return;
    }
  } else if constexpr (V % 2 == 0) {
    if (FAST || zmask == (1u << V) - 1) {
#pragma unroll
      for (int v = 0; v < V; v += 2) {
        if (keep) st_global_v2_hint(d + v, o[v], o[v + 1], pol);
        else st_global_v2(d + v, o[v], o[v + 1]);
      }
      return;
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v)
    if (FAST || ((zmask >> v) & 1u)) d[zpos<V, LZ>(0, v)] = o[v];
}

template <int V, int LZ, int K, int NTHR, int MINB, bool SYNTH, bool FIELD, bool TMA, bool MUSCL,
          bool TRAP, bool NORED = false>
__global__ void __launch_bounds__(NTHR, MINB)
    sweep_kernel(const __grid_constant__ CUtensorMap fmap, const SweepArgs a, int ns) {
  static_assert(!(TRAP && FIELD), "the field term is defined on midpoint velocity cells only");
  static_assert(!(MUSCL && FIELD), "MUSCL x transport has no v_x field term");
  constexpr int LEAD = MUSCL ? 2 : 1, TRAIL = MUSCL ? 1 : 0;
  // field term formulation: expanded per-cell coefficients (even V) or
  // relaxed neighbour rows (odd V); see the body
  constexpr bool FEXP = (V % 2 == 0);
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
  const int lgBy = __ffs(T.By) - 1;  // By is a power of two
  const int nx = a.nx;

  const uint32_t box_elems = (uint32_t)(T.rows_load * T.By * BZ);
  const uint32_t box_bytes = SYNTH ? 0u : box_elems * 8u;
  const uint32_t tab_bytes = (uint32_t)(a.TL * 8);
  const uint32_t stage_bytes = (box_bytes + tab_bytes + 127u) & ~127u;
  double* LT = reinterpret_cast<double*>(smem + (size_t)ns * stage_bytes);  // [2][lines]
  double* PZ = LT + 2 * lines;                                              // [2][NW][BZ]
  double* SCX = PZ + 2 * NW * BZ;                                           // [nvx] x-velocity centres
  uint64_t* bars = reinterpret_cast<uint64_t*>(SCX + ((a.nvx + 1) & ~1));   // [ns]

  const int g0 = (int)((a.total * blockIdx.x) / gridDim.x);
  const int g1 = (int)((a.total * (blockIdx.x + 1)) / gridDim.x);

  for (int j = tid; j < a.nvx; j += NTHR) SCX[j] = a.cx[j];
  if (TMA && tid == 0) {
    for (int s = 0; s < ns; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  // the prologue above reads only constant inputs; f, the tables and the
  // partial buffer belong to the preceding kernels of the step chain
  pdl_wait();
  pdl_trigger();
  __syncthreads();

  // producer state (thread 0 only): loads run ns items ahead
  // L2 policies: f is streamed once per sweep (evict first); the partial
  // records are re-read by finalize right after the sweep (evict last)
  const uint64_t pol_stream = make_policy_evict_first();
  const uint64_t pol_keep = make_policy_evict_last();

  // producer: lane 0 of the LAST warp (the first warps carry the per-plane
  // partial sums), with the tile geometry cached across its run
  const int ptid = NTHR - 32;
  ItemIter<LEAD, TRAIL> prod;
  prod.init(g0, g1, nx);
  int pstg = 0;  // ring stage of the next issue
  int ptile = -1;
  TileGeom ptg{};
  auto issue_next = [&]() {
    int t, p, h;
    prod.next(nx, t, p, h);
    if (t != ptile) {
      ptile = t;
      ptg = tile_geom(T, a.nvx, t);
    }
    const TileGeom& tg = ptg;
    const int i = item_plane(nx, a.bc, tg, p);
    const int s = pstg;
    if (++pstg == ns) pstg = 0;
    uint64_t* bar = &bars[s];
    unsigned char* st = smem + (size_t)s * stage_bytes;
    if (i < 0 && a.bc != 3) {
      mbar_arrive_expect_tx(bar, 0);
      return;
    }
    const int im = i + (a.bc == 3 ? 1 : 0);  // plane / row in memory (slab buffers are padded)
    mbar_arrive_expect_tx(bar, box_bytes + tab_bytes);
    if (!SYNTH) {
      // L2-resident ping-pong (f fits in L2): the loaded f*_{s-1} is dead
      // after this read, the stored f*_s is re-read by the next step
      if (PBGK_HINT_LOAD || a.l2_keep)
        tma_load_4d_hint(st, &fmap, tg.z0, tg.y0, tg.r0 - hoff, im, bar, pol_stream);
      else
        tma_load_4d(st, &fmap, tg.z0, tg.y0, tg.r0 - hoff, im, bar);
    }
    tma_load_1d(st + box_bytes, a.tab + (size_t)im * a.TL, tab_bytes, bar);
  };
  if (TMA && tid == ptid) {
    prefetch_tensormap(&fmap);
    for (int s = 0; s < ns && !prod.done(); ++s) issue_next();
  }

  // Line k of this thread: l = lg + k NL (strided over the box's lines)
  auto line_of = [&](int k) {  // natural line index aa*By + b, or -1 outside the box
    const int l = lg + k * NL;
    return l < lines ? l : -1;
  };
  // per-thread line geometry inside the box (fixed for the kernel): smem
  // offset of the lane's first element of line k, and the line's (row,
  // column) inside the box packed as a<<16|b
  int soff[K], lab[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    int l = line_of(k);
    if (l < 0) l = 0;
    const int aa = l >> lgBy, b = l & (T.By - 1);
    soff[k] = ((aa + hoff) * T.By + b) * BZ + zpos<V, LZ>(lz, 0);
    lab[k] = (aa << 16) | b;
  }
  // per-tile line constants (recomputed when the tile changes)
  int gxi[K], gyi[K], goff[K];
  double cvx[K];
  unsigned vmask = 0;  // bit k: line k is inside the tile and the grid
  // trapezoidal quadrature (a.trap): lines / lanes on the end nodes of an axis
  // take weight 1/2 (exact) in the marginal partials
  unsigned xedge = 0, yedge = 0, zedge = 0;
  unsigned xlo = 0, xhi = 0;  // field term: lines on the first / last v_x row
  unsigned zmask = 0;  // bit v: element v of this lane is inside the grid
  bool full = false;   // every line and element of this thread is valid
  int cur_tile = -1;
  TileGeom tg{};

  // prev[k][v]: the upwind flux c_x f_pre of the previous plane in march
  // order (the F of ref/kinetic.py:110-112 on the face shared with this plane)
  double prev[K][V];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int v = 0; v < V; ++v) prev[k][v] = 0.0;
  // MUSCL: the relaxed values of the two previous planes in march order
  double xm1[MUSCL ? K : 1][V], xm2[MUSCL ? K : 1][V];

  double facc = 0.0;  // noreduce: sum of this thread's outputs (finiteness)
  ItemIter<LEAD, TRAIL> it;
  it.init(g0, g1, nx);
  int j = 0;        // item counter (LT/PZ parity)
  int stg = 0;      // ring stage of item j
  uint32_t ph = 0;  // mbarrier phase of that stage
  while (!it.done()) {
    int t, p, kind;
    it.next(nx, t, p, kind);
    const bool halo = kind == kLead;
    if (t != cur_tile) {
      cur_tile = t;
      tg = tile_geom(T, a.nvx, t);
      vmask = 0;
      xedge = yedge = zedge = 0;
      xlo = xhi = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int l = line_of(k);
        int jx = tg.r0 + (lab[k] >> 16), jy = tg.y0 + (lab[k] & 0xffff);
        if (l >= 0 && jx < tg.r1 && jy < a.nvy) vmask |= 1u << k;
        jx = min(jx, a.nvx - 1);
        jy = min(jy, a.nvy - 1);
        gxi[k] = a.gxo + jx;
        gyi[k] = a.gyo + jy;
        goff[k] = (jx * a.nvy + jy) * a.nvz + tg.z0 + zpos<V, LZ>(lz, 0);
        cvx[k] = SCX[jx];
        if (jx == 0 || jx == a.nvx - 1) xedge |= 1u << k;
        if (jx == 0) xlo |= 1u << k;
        if (jx == a.nvx - 1) xhi |= 1u << k;
        if (jy == 0 || jy == a.nvy - 1) yedge |= 1u << k;
      }
      zmask = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int jz = tg.z0 + zpos<V, LZ>(lz, v);
        if (jz < a.nvz) zmask |= 1u << v;
        if (jz == 0 || jz == a.nvz - 1) zedge |= 1u << v;
      }
      full = (vmask == (1u << K) - 1) && (zmask == (1u << V) - 1);
    }
    const int i = item_plane(nx, a.bc, tg, p);
    // output: upwind -> this plane (not for halos); MUSCL -> the previous
    // plane of the run (lags one item), emitted by every item after the first
    const bool out_plane = MUSCL ? (kind == kNormal || kind == kTrail) : !halo;
    const int i_out = MUSCL ? item_plane(nx, a.bc, tg, p - 1) : i;
    const int sh = a.bc == 3 ? 1 : 0;  // slab buffers: one padding plane / row
    const double* SF = reinterpret_cast<const double*>(smem + (size_t)stg * stage_bytes);
    const double* ST = reinterpret_cast<const double*>(smem + (size_t)stg * stage_bytes + box_bytes);
    // the cell's field value is read before the stage wait so its global-load
    // latency overlaps the wait (the wait's memory clobber keeps the order)
    // (not for odd V: those kernels run at the register limit)
    double e_cell = 0.0;
    if (FIELD && FEXP && out_plane) e_cell = __ldg(a.E + i);
    if (TMA) {
      mbar_wait(&bars[stg], ph);
    } else if (i >= 0 || a.bc == 3) {
      // generic path: cooperative synchronous load of the box and the table row
      double* sf = reinterpret_cast<double*>(smem);
      for (uint32_t e = tid; e < box_elems && !SYNTH; e += NTHR) {
        const int zz = e % BZ, rest = e / BZ;
        const int b = rest % T.By, br = rest / T.By;
        const int jx = tg.r0 - hoff + br, jy = tg.y0 + b, jz = tg.z0 + zz;
        double v = 0.0;
        if (jx >= 0 && jx < a.nvx && jy < a.nvy && jz < a.nvz)
          v = a.fin[(size_t)(i + sh) * a.plane + ((size_t)jx * a.nvy + jy) * a.nvz + jz];
        sf[e] = v;
      }
      for (int e = tid; e < a.TL; e += NTHR) sf[box_bytes / 8 + e] = a.tab[(size_t)(i + sh) * a.TL + e];
      __syncthreads();
    }

    if (!MUSCL && i < 0 && a.bc != 3) {
      // absorbing ghost plane: f_pre == 0
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int v = 0; v < V; ++v) prev[k][v] = 0.0;
    } else {
      const double r = ST[0], ls = ST[1];
      double gz[V];
      if (zmask == (1u << V) - 1) {
        lds_lane<V, LZ>(ST + a.gzo + tg.z0 + zpos<V, LZ>(lz, 0), gz);
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
          gz[v] = ((zmask >> v) & 1u) ? ST[a.gzo + tg.z0 + zpos<V, LZ>(lz, v)] : 0.0;
      }
      const bool transport = a.dtdx != 0.0;
      const double dtdx = a.dtdx;
      double hE = 0.0;
      if (FIELD && out_plane) hE = __dmul_rn(0.5, FEXP ? e_cell : __ldg(a.E + i));
      // v_x Rusanov flux of ref/kinetic.py:114-123 reassociated per cell:
      // G(lo, hi) = E/2 (lo + hi) - e_max/2 (hi - lo) = cp lo + cm hi.  The
      // update -dt/dv (G_{j+1/2} - G_{j-1/2}) of row j is linear in the
      // relaxed rows x (j), fp (j+1), fm (j-1):
      //   interior  -dt/dv ((cp - cm) x + cm fp - cp fm)
      //   j = 0     -dt/dv (cp x + cm fp)          (no lower face)
      //   j = n-1   -dt/dv (-cm x - cp fm)         (no upper face)
      // and fp = r raw_p + s g_x[j+1] g_y g_z with s = r ls (s = ls, no raw,
      // for the synthesised first pass), likewise fm.  So per cell: kx_* on x,
      // kp / km on the raw neighbours, and per line kg on g_z -- 4 FMAs per
      // element instead of relaxing both neighbours (within a few ulps of the
      // reference's order, far inside the 1e-10 parity bound)
      const double cp = hE + a.half_emax, cm = hE - a.half_emax;
      double kx_in = 0.0, kx_lo = 0.0, kx_hi = 0.0, kp = 0.0, km = 0.0, fCm = 0.0, fCp = 0.0;
      if (FIELD && FEXP) {
        const double D = -a.dtdv;
        kx_in = D * (cp - cm);
        kx_lo = D * cp;
        kx_hi = -(D * cm);
        const double s = SYNTH ? ls : r * ls;
        fCm = (D * s) * cm;
        fCp = -((D * s) * cp);
        kp = (D * r) * cm;
        km = -((D * r) * cp);
      }
      double* gdst = (a.fout != nullptr && out_plane) ? a.fout + (size_t)(i_out + sh) * a.plane : nullptr;
      double lp[K];
      double pz[V];
#pragma unroll
      for (int v = 0; v < V; ++v) pz[v] = 0.0;
      // z partial += m (weight of the line's x, y nodes), line total += m
      // (weight of the z node); the weights are 1 except for trapezoidal
      // quadrature, where end nodes count 1/2 (exact scalings)
      auto accum = [&](double m, int k, int v, double& sl) {
        if constexpr (TRAP) {
          const double wl = (((xedge >> k) & 1u) ? 0.5 : 1.0) * (((yedge >> k) & 1u) ? 0.5 : 1.0);
          pz[v] += m * wl;
          sl += m * (((zedge >> v) & 1u) ? 0.5 : 1.0);
        } else {
          pz[v] += m;
          sl += m;
        }
      };

      // One plane: relax R_{s-1} of the loaded f*_{s-1}, transport, store,
      // marginal partials.  FAST: full tile, transport on, output plane
      // written (every step but the first/last of a window) -- no masks and no
      // per-line tests; otherwise the general masked path.  DOWNT: c_x < 0
      // (the upwind neighbour is plane i+1, already in `prev`).  RO: full
      // tile, no transport and no store (a window's final relax + projection
      // of f*_S, read-only): FAST's unmasked partials without the update.
      auto body = [&](auto fast_c, auto down_c, auto ro_c) {
        constexpr bool RO = decltype(ro_c)::value;
        constexpr bool FAST = decltype(fast_c)::value && !RO;
        constexpr bool FULL = FAST || RO;
        constexpr bool DOWNT = decltype(down_c)::value;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const bool ok = FULL || ((vmask >> k) & 1u);
          const double gxy = ST[gxi[k]] * ST[gyi[k]];
          const double c = cvx[k];
          double x[V];
          if (SYNTH) {
#pragma unroll
            for (int v = 0; v < V; ++v) x[v] = (gxy * gz[v]) * ls;
          } else {
            // (f* + ls M) r with M = gxy gz, as (r f*) + (r ls gxy) gz
            const double w = r * (ls * gxy);
            double raw[V];
            lds_lane<V, LZ>(SF + soff[k], raw);
#pragma unroll
            for (int v = 0; v < V; ++v) x[v] = fma(w, gz[v], r * raw[v]);
          }
          double fl[V];  // this plane's upwind flux c f_pre
          if constexpr (!RO) {
#pragma unroll
            for (int v = 0; v < V; ++v) fl[v] = __dmul_rn(c, x[v]);
          }
          if (FULL || out_plane) {
            double o[V];
            if (!RO && (FAST || transport)) {
#pragma unroll
              for (int v = 0; v < V; ++v) {
                // f* = f - (dt/dx)(F_{i+1/2} - F_{i-1/2}); upward: F_{i+1/2} = c f_i,
                // F_{i-1/2} = c f_{i-1}; downward: F_{i+1/2} = c f_{i+1}, F_{i-1/2} = c f_i
                const double d = DOWNT ? __dsub_rn(prev[k][v], fl[v]) : __dsub_rn(fl[v], prev[k][v]);
                o[v] = __dsub_rn(x[v], __dmul_rn(dtdx, d));
              }
            } else {
#pragma unroll
              for (int v = 0; v < V; ++v) o[v] = x[v];
            }
            if (FIELD && FEXP && (FAST || transport)) {
              // ref/kinetic.py:114-123: Rusanov flux on interior v_x faces of
              // f_pre, expanded over the relaxed neighbours (see kx_* above):
              // -dt/dv (G_hi - G_lo) = kx x + kp rp + km rm + kg gz
              const bool has_lo = !((xlo >> k) & 1u), has_hi = !((xhi >> k) & 1u);
              const double gpl = has_hi ? ST[gxi[k] + 1] : 0.0;
              const double gmi = has_lo ? ST[gxi[k] - 1] : 0.0;
              const double kg = ST[gyi[k]] * fma(fCm, gpl, fCp * gmi);
              const double kx = has_lo ? (has_hi ? kx_in : kx_hi) : (has_hi ? kx_lo : 0.0);
              if (SYNTH) {
#pragma unroll
                for (int v = 0; v < V; ++v) o[v] = fma(kg, gz[v], fma(kx, x[v], o[v]));
              } else {
                // neighbour rows outside the cube are zero-filled by the load
                double rm[V], rp[V];
                lds_lane<V, LZ>(SF + soff[k] - T.By * BZ, rm);
                lds_lane<V, LZ>(SF + soff[k] + T.By * BZ, rp);
#pragma unroll
                for (int v = 0; v < V; ++v)
                  o[v] = fma(kg, gz[v], fma(km, rm[v], fma(kp, rp[v], fma(kx, x[v], o[v]))));
              }
            } else if (FIELD && (FAST || transport)) {
              // the same flux with both neighbour rows relaxed first (fewer
              // live per-cell coefficients: measured faster for odd V, whose
              // kernels run at the register limit)
              const int jx = gxi[k] - a.gxo;
              const bool has_lo = jx > 0, has_hi = jx + 1 < a.nvx;
              double fm[V], fp[V];
              const double gym = ST[gyi[k]];
              const double gxm = has_lo ? ST[gxi[k] - 1] * gym : 0.0;
              const double gxp = has_hi ? ST[gxi[k] + 1] * gym : 0.0;
              if (SYNTH) {
#pragma unroll
                for (int v = 0; v < V; ++v) {
                  fm[v] = (gxm * gz[v]) * ls;
                  fp[v] = (gxp * gz[v]) * ls;
                }
              } else {
                const double wm = r * (ls * gxm), wp = r * (ls * gxp);
                double rm[V], rp[V];
                lds_lane<V, LZ>(SF + soff[k] - T.By * BZ, rm);
                lds_lane<V, LZ>(SF + soff[k] + T.By * BZ, rp);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                  fm[v] = fma(wm, gz[v], r * rm[v]);
                  fp[v] = fma(wp, gz[v], r * rp[v]);
                }
              }
#pragma unroll
              for (int v = 0; v < V; ++v) {
                const double ghi = has_hi ? fma(cp, x[v], cm * fp[v]) : 0.0;
                const double glo = has_lo ? fma(cp, fm[v], cm * x[v]) : 0.0;
                o[v] = fma(-a.dtdv, ghi - glo, o[v]);
              }
            }
            double sl = 0.0;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const double m = FULL ? o[v] : ((ok && ((zmask >> v) & 1u)) ? o[v] : 0.0);
              accum(m, k, v, sl);
            }
            lp[k] = sl;
            if (!RO && (FAST || (gdst != nullptr && ok))) {
              store_line<V, LZ, FAST>(gdst + goff[k], o, zmask, a.l2_keep != 0, pol_keep);
            }
          }
          if constexpr (!RO) {
#pragma unroll
            for (int v = 0; v < V; ++v) prev[k][v] = fl[v];
          }
        }
      };
      // MUSCL (minmod) x transport, one plane behind the loads: item q
      // relaxes plane q, forms the slope of plane q-1 from planes q-2..q and
      // the face flux between q-1 and q (march order), and outputs plane q-1
      // (oracle/bgk.py transport_muscl, same operation order).
      auto body_m = [&](auto fast_c, auto down_c) {
        constexpr bool FAST = decltype(fast_c)::value;
        constexpr bool DOWNT = decltype(down_c)::value;
        if constexpr (MUSCL) {
          const bool ghost = i < 0;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const bool ok = FAST || ((vmask >> k) & 1u);
            double x[V];
            if (ghost) {
#pragma unroll
              for (int v = 0; v < V; ++v) x[v] = 0.0;
            } else {
              const double gxy = ST[gxi[k]] * ST[gyi[k]];
              if (SYNTH) {
#pragma unroll
                for (int v = 0; v < V; ++v) x[v] = (gxy * gz[v]) * ls;
              } else {
                const double w = r * (ls * gxy);
                double raw[V];
                lds_lane<V, LZ>(SF + soff[k], raw);
#pragma unroll
                for (int v = 0; v < V; ++v) x[v] = fma(w, gz[v], r * raw[v]);
              }
            }
            const double c = cvx[k];
            double F[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
              // physical order: a = f_i - f_{i-1}, b = f_{i+1} - f_i for plane i = q-1
              const double am = DOWNT ? __dsub_rn(xm1[k][v], x[v]) : __dsub_rn(xm1[k][v], xm2[k][v]);
              const double bm = DOWNT ? __dsub_rn(xm2[k][v], xm1[k][v]) : __dsub_rn(x[v], xm1[k][v]);
              const double sg = (__dmul_rn(am, bm) > 0.0) ? copysign(fmin(fabs(am), fabs(bm)), am) : 0.0;
              const double hs = __dmul_rn(0.5, sg);
              F[v] = __dmul_rn(c, DOWNT ? __dsub_rn(xm1[k][v], hs) : __dadd_rn(xm1[k][v], hs));
            }
            if (FAST || out_plane) {
              double o[V];
#pragma unroll
              for (int v = 0; v < V; ++v) {
                const double d = DOWNT ? __dsub_rn(prev[k][v], F[v]) : __dsub_rn(F[v], prev[k][v]);
                o[v] = __dsub_rn(xm1[k][v], __dmul_rn(dtdx, d));
              }
              double sl = 0.0;
#pragma unroll
              for (int v = 0; v < V; ++v) {
                const double m = FAST ? o[v] : ((ok && ((zmask >> v) & 1u)) ? o[v] : 0.0);
                accum(m, k, v, sl);
              }
              lp[k] = sl;
              if (FAST || (gdst != nullptr && ok)) {
                store_line<V, LZ, FAST>(gdst + goff[k], o, zmask, a.l2_keep != 0, pol_keep);
              }
            }
#pragma unroll
            for (int v = 0; v < V; ++v) {
              xm2[k][v] = xm1[k][v];
              xm1[k][v] = x[v];
              prev[k][v] = F[v];
            }
          }
        }
      };
      using T1 = std::integral_constant<bool, true>;
      using F1 = std::integral_constant<bool, false>;
      if constexpr (MUSCL) {
        if (full && out_plane && gdst != nullptr) {
          if (tg.down) body_m(T1{}, T1{}); else body_m(T1{}, F1{});
        } else {
          if (tg.down) body_m(F1{}, T1{}); else body_m(F1{}, F1{});
        }
      } else if (!SYNTH && (a.debug & 4)) {
        // ablation: copy-through skeleton (TMA in, STG out, no arithmetic)
        if (gdst != nullptr && out_plane) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            double raw[V];
            lds_lane<V, LZ>(SF + soff[k], raw);
            if constexpr (V == 2) st_global_v2(gdst + goff[k], raw[0], raw[1]);
          }
        }
      } else if (full && out_plane && transport && gdst != nullptr) {
        if (tg.down) body(T1{}, T1{}, F1{}); else body(T1{}, F1{}, F1{});
      } else {
        bool ro = false;
        if constexpr (!FIELD && !SYNTH && !MUSCL) {
          if (full && out_plane && !transport && gdst == nullptr) {
            body(F1{}, F1{}, T1{});
            ro = true;
          }
        }
        if (!ro) {
          if (tg.down) body(F1{}, T1{}, F1{}); else body(F1{}, F1{}, F1{});
        }
      }

      if (NORED && out_plane) {
        // no partials: sum the plane's outputs for the finiteness flag
#pragma unroll
        for (int k = 0; k < K; ++k) facc += lp[k];
      } else if (out_plane && !(a.debug & 1)) {
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
            const int l = line_of(base + c2);
            if (l >= 0) LTb[l] = lp[c2];
          }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
#pragma unroll
          for (int w = LZ; w < 32; w <<= 1) pz[v] += __shfl_xor_sync(FULL, pz[v], w);
        }
        if (lane < LZ) {
#pragma unroll
          for (int v = 0; v < V; ++v) PZb[warp * BZ + zpos<V, LZ>(lane, v)] = pz[v];
        }
      }
    }

    __syncthreads();
    if (TMA && tid == ptid && !prod.done()) {
      fence_proxy_async();
      issue_next();
    }
    if (!NORED && out_plane && i_out >= 0 && !(a.debug & 1)) {
      // one output per thread, in equal contiguous chunks per warp so no warp
      // carries the serial sums alone (contiguous lanes keep smem reads
      // conflict-free)
      const double* LTb = LT + (j & 1) * lines;
      const double* PZb = PZ + (j & 1) * NW * BZ;
      double* dst = a.part + ((size_t)i_out * T.NT + t) * T.PS;
#if PBGK_OUT_ROT
      // z outputs first, then x, then y, on consecutive threads starting at a
      // warp that rotates with the item (the serial sums move round the CTA)
      int q = tid - (j & (NW - 1)) * 32;
      if (q < 0) q += NTHR;
      const int o = q < BZ ? T.A + T.By + q : (q < BZ + T.A + T.By ? q - BZ : 1 << 20);
#else
      const int chunk = (T.A + T.By + BZ + NW - 1) / NW;
      const int o = lane < chunk ? warp * chunk + lane : 1 << 20;
#endif
      if (o < T.A) {
        if (tg.r0 + o < tg.r1) {
          double s2 = 0.0;
          for (int b = 0; b < T.By; ++b) {
            const int y = tg.y0 + b;
            s2 += (TRAP && (y == 0 || y == a.nvy - 1)) ? 0.5 * LTb[o * T.By + b] : LTb[o * T.By + b];
          }
          
#if PBGK_HINT_PART
          st_global_f64_hint(dst + o, s2, pol_keep);
#else
          *(dst + o) = s2;
#endif

        }
      } else if (o < T.A + T.By) {
        const int b = o - T.A;
        if (tg.y0 + b < a.nvy) {
          double s2 = 0.0;
          for (int aa = 0; aa < T.A; ++aa) {
            const int x = tg.r0 + aa;
            s2 += (TRAP && (x == 0 || x == a.nvx - 1)) ? 0.5 * LTb[aa * T.By + b] : LTb[aa * T.By + b];
          }
          
#if PBGK_HINT_PART
          st_global_f64_hint(dst + T.A + b, s2, pol_keep);
#else
          *(dst + T.A + b) = s2;
#endif

        }
      } else if (o < T.A + T.By + BZ) {
        const int zz = o - T.A - T.By;
        if (tg.z0 + zz < a.nvz) {
          double s2 = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) s2 += PZb[w * BZ + zz];
          
#if PBGK_HINT_PART
          st_global_f64_hint(dst + T.A + T.By + zz, s2, pol_keep);
#else
          *(dst + T.A + T.By + zz) = s2;
#endif

        }
      }
    }
    if (!TMA) __syncthreads();  // the single stage is refilled next item
    ++j;
    if (++stg == ns) {
      stg = 0;
      ph ^= 1u;
    }
  }
  if (NORED && !isfinite(facc)) atomicMin(a.err, err_key(0, a.out_step, kErrNonFinite));
}

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------

// MODES: bit 0 = first-order upwind kernels, bit 1 = MUSCL kernels, bit 2 =
// upwind with the v_x field term, bit 3 = trapezoidal-quadrature variants of
// the bit 0 / bit 1 kernels; a shape only instantiates what it serves.
template <int V, int LZ, int K, int NTHR, int MINB, bool TMA, int MODES>
static cudaError_t launch_cfg(const CUtensorMap& map, const SweepArgs& a, bool synth, bool field,
                              int grid, int ns, size_t smem, cudaStream_t st) {
  void (*fn)(const CUtensorMap, const SweepArgs, int) = nullptr;
  constexpr bool TR = (MODES & 8) != 0;
  if (a.trap) {
    if constexpr (TR) {
      if (a.muscl) {
        if constexpr ((MODES & 2) != 0)
          fn = synth ? sweep_kernel<V, LZ, K, NTHR, MINB, true, false, TMA, true, true>
                     : sweep_kernel<V, LZ, K, NTHR, MINB, false, false, TMA, true, true>;
      } else if (!field) {
        if constexpr ((MODES & 1) != 0)
          fn = synth ? sweep_kernel<V, LZ, K, NTHR, MINB, true, false, TMA, false, true>
                     : sweep_kernel<V, LZ, K, NTHR, MINB, false, false, TMA, false, true>;
      }
    }
  } else if (a.muscl) {
    if constexpr ((MODES & 2) != 0)
      fn = synth ? sweep_kernel<V, LZ, K, NTHR, MINB, true, false, TMA, true, false>
                 : sweep_kernel<V, LZ, K, NTHR, MINB, false, false, TMA, true, false>;
  } else {
    if (field) {
      if constexpr ((MODES & 4) != 0) {
        if (a.noreduce)
          fn = synth ? sweep_kernel<V, LZ, K, NTHR, MINB, true, true, TMA, false, false, true>
                     : sweep_kernel<V, LZ, K, NTHR, MINB, false, true, TMA, false, false, true>;
        else
          fn = synth ? sweep_kernel<V, LZ, K, NTHR, MINB, true, true, TMA, false, false>
                     : sweep_kernel<V, LZ, K, NTHR, MINB, false, true, TMA, false, false>;
      }
    } else {
      if constexpr ((MODES & 1) != 0)
        fn = synth ? sweep_kernel<V, LZ, K, NTHR, MINB, true, false, TMA, false, false>
                   : sweep_kernel<V, LZ, K, NTHR, MINB, false, false, TMA, false, false>;
    }
  }
  if (fn == nullptr) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(fn, grid, NTHR, smem, st, map, a, ns);
}

// Shared memory the kernel needs for `ns` stages.

}  // namespace pbgk
