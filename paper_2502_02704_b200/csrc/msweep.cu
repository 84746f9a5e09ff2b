// Multi-step sweep, round 2: up to 8 fine steps of f per pass.
//
// Same algorithm as fsweep.cu (the relax tables R_s of every step come from
// the moment recursion, marginal.cu; a velocity tile marches in x and every
// level keeps the upwind flux of the previous plane in registers; only the
// last level is stored: 16/L bytes of HBM per cell-update), re-laid out for
// latency hiding and a lean per-element instruction stream:
//
//   * box A = 8 v_x rows x BY = 8 v_y x BZ = 16 v_z (8 KB); a warp owns one
//     box row, so the per-row scalars (relax factor, transport coefficients)
//     are warp-uniform; a thread owns a 2 x 2 patch (two adjacent v_y lines x
//     two adjacent v_z): its table factors are two g_y and two g_z, each one
//     8-byte shared load whose warp-wide footprint is <= 128 B (one data-pipe
//     cycle; measured with tools/ubench/lds_bench.cu: a 16-byte load whose
//     lanes differ inside a quarter warp costs four).
//   * two warp groups split the levels: group 0 runs levels [0, LA) of plane
//     p and hands its output to group 1 through a hand-off area of the stage,
//     group 1 runs levels [LA, L) of plane p, the output and the reductions
//     while group 0 moves on to plane p+1 (LA = 5 of 8).  A third warpgroup
//     only issues the loads and hands its registers to the other two
//     (setmaxnreg: 32 / 120 / 104 registers from a 96-register start).
//   * relax + transport of level l, per element (ref/kinetic.py:110-112,
//     130-134):  z = x + (ls gxa gy) gz,  out = (keep r) z + q_prev,
//     q = (a r) z,  with a = (dt/dx)|c_x| and keep = 1 - a: the reference's
//     f* = f - (dt/dx)(F_i+1 - F_i) after f = r (f* + ls M), re-associated (a
//     few ulps; the multi-step path is held to the oracle at 1e-12).  a per
//     (v_x row, level) sits in a shared table computed once per launch;
//     a r and keep r = r - a r per warp and level.
//   * loads: loader thread 0 issues the TMA box of a plane, the loader
//     threads the 16-byte cp.async chunks of the table-row slices the tile needs
//     (r, ls | gxa of its rows | gy | gz per level: 0.3 KB instead of whole
//     rows); full / mid / empty mbarriers per ring stage, no CTA barrier on
//     the steady path.
//   * FINAL (the window's last pass): R_S applied to the last level's output
//     and the per-(plane, tile) marginal partial records [m_x rows | m_y |
//     m_z] written for finalize.cu (kFinProject) -- the projection P(f_S)
//     without storing f_S and reading it back.  Fixed trees, the same for
//     every marginal index and its mirror (even data keeps an exactly zero
//     folded first moment, ref/moments.py:80-88).
//   * SYNTH (the window's first pass from moments): level 0 input is the lift
//     f_0 = ls gxa gy gz of tab[0] (ref/lifting.py:47-57), no f read.
//
// Finiteness (ref/kinetic.py:157-159): the stored level's values (or, FINAL,
// the m_x partials) are summed per thread; non-finite -> status kind 6 at the
// pass's first step, on which the host re-runs the propagation on the
// one-step path for the exact BlowUpError(step).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"
#include "sweep_impl.cuh"

// development A/B knobs (tools/ab_ms.sh)
#ifndef PBGK_MS_ZSPLIT
#define PBGK_MS_ZSPLIT 0
#endif
#ifndef PBGK_MS_STHINT
#define PBGK_MS_STHINT 1
#endif
#ifndef PBGK_MS_HINT
#define PBGK_MS_HINT 2
#endif
#ifndef PBGK_MS_GYASM
#define PBGK_MS_GYASM 1
#endif
#ifndef PBGK_MS_AONLY
#define PBGK_MS_AONLY 1
#endif

namespace pbgk {

namespace ms {
constexpr int A = 8;      // v_x rows per box = warps per group
constexpr int BZ = 16;    // v_z per box line (128 B)
constexpr int NW = A;     // warps per group
constexpr int NTG = 32 * NW;
constexpr int NTHR = 2 * NTG;
constexpr int BY = 8;     // v_y lines per box row
constexpr int TS = 2 + A + BY + BZ;  // table slice (doubles): r, ls | gxa rows | g_y | g_z
// PRE: (ls gxa, keep r, a r, -) per box row | g_y | g_z -- the per-row factors
// of every (cell, step) precomputed once per window (ms_prep_kernel)
constexpr int TSP = 4 * A + BY + BZ;
__host__ __device__ constexpr int slice_doubles(bool pre) { return pre ? TSP : TS; }
}  // namespace ms

enum MsMode : int { kMsSynth = 1, kMsFinal = 2 };


// The item sequence of a CTA's segment [g0, g1) of (tile, plane) positions:
// every run of consecutive planes of one tile is preceded by `nlev` lead
// positions (its upwind halo planes; lead position k completes k levels);
// the run's positions (lead + planes) are grouped P per item, the last item
// of a run possibly short.
struct MsRuns {
  long long g, g1;
  int nx, nlev;
  __device__ __forceinline__ void init(long long g0_, long long g1_, int nx_, int nlev_) {
    g = g0_;
    g1 = g1_;
    nx = nx_;
    nlev = nlev_;
  }
  // next run: tile, first plane position p0, end p1; false at the end
  __device__ __forceinline__ bool next(int& t, int& p0, int& p1) {
    if (g >= g1) return false;
    t = (int)(g / nx);
    p0 = (int)(g - (long long)t * nx);
    p1 = (int)min((long long)nx, p0 + (g1 - g));
    g += p1 - p0;
    return true;
  }
};

template <int NT_>
__device__ __forceinline__ void named_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NT_) : "memory");
}

#ifndef PBGK_MS_NG
#define PBGK_MS_NG 2
#endif

// NG = 2: two warp groups split the levels (16 warps, one CTA per SM);
// NG = 1: one group runs every level (8 warps, two CTAs per SM)
#ifndef PBGK_MS_LW
#define PBGK_MS_LW 1
#endif
// LW (two groups only): a loader warpgroup (warps 16-19) issues every load
// (the TMA boxes and the table chunks), so group 0 runs nothing but its
// levels, and hands most of its registers to the compute groups (setmaxnreg)
constexpr bool kMsLW = PBGK_MS_LW && PBGK_MS_NG == 2;
constexpr int kMsLoaders = 128;  // a whole warpgroup, so that it can hand its registers to the others
constexpr int kMsThreads = PBGK_MS_NG * ms::NTG + (kMsLW ? kMsLoaders : 0);
// Registers after the role split.  The kernel starts at 96 per thread (640
// threads); what the compute groups gain must come out of what the loader
// warpgroup releases (the CTA's pool holds only released registers -- asking
// for more never returns): 128 x (96 - 32) = 8192 >= 256 x (R0 - 96) + 256 x
// (R1 - 96).
#ifndef PBGK_MS_R0
#define PBGK_MS_R0 120
#endif
#ifndef PBGK_MS_R1
#define PBGK_MS_R1 104
#endif
#ifndef PBGK_MS_RL
#define PBGK_MS_RL 32
#endif
static_assert(128 * (96 - PBGK_MS_RL) >= 256 * (PBGK_MS_R0 - 96) + 256 * (PBGK_MS_R1 - 96), "register pool");
// the FINAL pass (group 1 also reduces the partial records) may split differently
#ifndef PBGK_MS_R0F
#define PBGK_MS_R0F PBGK_MS_R0
#endif
#ifndef PBGK_MS_R1F
#define PBGK_MS_R1F PBGK_MS_R1
#endif
static_assert(128 * (96 - PBGK_MS_RL) >= 256 * (PBGK_MS_R0F - 96) + 256 * (PBGK_MS_R1F - 96), "register pool");
template <int N>
__device__ __forceinline__ void reg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

template <int L, int MODE, int P, int NG, bool PRE>
__global__ void __launch_bounds__(kMsThreads, NG == 1 ? 2 : 1)
    msweep_kernel(const __grid_constant__ CUtensorMap fmap, const MSweepArgs a, int ns) {
  using namespace ms;
  constexpr int TS = slice_doubles(PRE);  // (shadows ms::TS) doubles per level slice of a stage
  constexpr bool SYNTH = (MODE & kMsSynth) != 0;
  constexpr bool FINAL = (MODE & kMsFinal) != 0;
  constexpr bool LW = kMsLW && NG == 2;
  constexpr int NLD = LW ? kMsLoaders : NTG;  // loader threads
#ifndef PBGK_MS_LA
#define PBGK_MS_LA 0
#endif
  // levels [0, LA) run in group 0 (which also issues the loads), [LA, L) in
  // group 1; LH = the larger share (carry registers)
  // (measured on config 4, 8 levels: with the loads in group 0, 3 + 5 is 6 %
  // faster than 4 + 4 -- group 0 also walks the loader; 2 + 6 spills.  With
  // the loader warpgroup group 1 -- the output, the finiteness sums, FINAL's
  // reductions -- is the heavier one: a config 4 window's passes take 8.79 ms
  // at 3 + 5, 8.67 at 4 + 4, 8.30 at 5 + 3, 8.84 at 6 + 2)
#ifndef PBGK_MS_LAF
#define PBGK_MS_LAF 4
#endif
#ifndef PBGK_MS_LAFW
#define PBGK_MS_LAFW 6  // FINAL with the loader warpgroup: group 1 also reduces (window passes 7.70 ms at 5 + 3, 7.61 at 6 + 2, 7.57 at 7 + 1 with spills)
#endif
  // FINAL: group 1 also applies R_S and reduces the partial records, so it
  // takes one level fewer (4 + 4)
  constexpr int LA = NG == 1 ? L
                             : (PBGK_MS_LA > 0 && PBGK_MS_LA < L ? PBGK_MS_LA
                                                                 : (L == 8 ? (LW ? (FINAL ? PBGK_MS_LAFW : 5) : (FINAL ? PBGK_MS_LAF : 3)) : L / 2));
  constexpr int LH = LA > L - LA ? LA : L - LA;
  constexpr int NTHR_K = NG * NTG + (LW ? kMsLoaders : 0);
  constexpr int NTAB = L + (FINAL ? 1 : 0);
  constexpr uint32_t BOXB = (uint32_t)(A * BY * BZ * 8);
  // the group hand-off area of a plane: after its box and tables, not in the
  // TMA destination (shared stores into the box the async proxy fills cost
  // ~35 % of the pass, measured)
  constexpr uint32_t HOFF = (BOXB + NTAB * TS * 8 + 127u) & ~127u;
  constexpr uint32_t PLB = NG == 2 ? HOFF + BOXB : HOFF;  // one plane of a stage
  constexpr uint32_t STAGEB = P * PLB;
  constexpr int REC = A + BY + BZ;
  constexpr int RS = 1 + BY + BZ;             // per-warp partial block (FINAL)
  constexpr int FR = 8;                       // FINAL records reduced per barrier
  constexpr int NCH = (2 + A + BY + BZ) / 2;  // 16-byte chunks of one plain table slice (R_S; every level without PRE)
  constexpr int NCHP = PRE ? TSP / 2 : NCH;   // chunks of one level slice
  constexpr int NCHT = L * NCHP + (FINAL ? NCH : 0);  // chunks of one plane
  constexpr int CPT = (P * NCHT + NLD - 1) / NLD;  // chunks per loader thread
  extern __shared__ __align__(128) unsigned char smem[];

  const Tiling& T = a.t;
  const int tid = threadIdx.x;
  const int nx = a.nx, nvx = a.nvx;
  // window of a batched launch (grid.y; 0 otherwise) and its buffers
  const int win = blockIdx.y;
  double* const fout = a.fout != nullptr ? a.fout + (size_t)win * a.f_ws : nullptr;
  double* const part = a.part != nullptr ? a.part + (size_t)win * a.p_ws : nullptr;
  ErrKey* const errp = a.errw != nullptr ? a.errw + win : a.err;
  const int nlev = a.nlev;
  double* AK = reinterpret_cast<double*>(smem + (size_t)ns * STAGEB);     // [nvx][L] a = (dt/dx)|c_x| (not PRE)
  double* RB = reinterpret_cast<double*>(AK + (PRE ? 0 : L * nvx * (PBGK_MS_AONLY ? 1 : 2)));  // FINAL: [2][FR][NW][RS]
  long long* RI = reinterpret_cast<long long*>(RB + (FINAL ? 2 * FR * NW * RS : 0));  // [2][FR]
  uint64_t* full = reinterpret_cast<uint64_t*>(RI + (FINAL ? 2 * FR : 0));
  uint64_t* mid = full + ns;
  uint64_t* empty = mid + ns;

  const long long g0 = (a.total * blockIdx.x) / gridDim.x;
  const long long g1 = (a.total * (blockIdx.x + 1)) / gridDim.x;

  // transport coefficients per (row, level): a = (dt/dx) |c_x|, keep = 1 - a
  // (up rows: f* = (1-a) f + a f_{i-1}; down rows: (1-a) f + a f_{i+1})
  for (int j = tid; j < (PRE ? 0 : L * nvx); j += NTHR_K) {
    const int jx = j / L, l = j - jx * L;
    const double c = a.cx[jx];
    const double dtl = a.dts == nullptr ? a.dtdx[l] : (l < nlev ? a.dts[(size_t)(a.s0 + l) * a.dts_g + win] / a.dx : 0.0);
    const double av = dtl * (c < 0.0 ? -c : c);
#if PBGK_MS_AONLY
    AK[j] = av;
#else
    reinterpret_cast<double2*>(AK)[j] = make_double2(1.0 - av, av);
#endif
  }
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1 + NLD);  // the boxes' expect-tx arrive + one cp.async arrive per loader
      mbar_init(&mid[s], NW);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  pdl_wait();
  pdl_trigger();
  __syncthreads();

  const int grp = tid / NTG;        // 0: (loads +) levels [0, LA); 1: levels [LA, L) + output; 2: the loader warp (LW)
  const int gt = tid - grp * NTG;
  const bool loader = LW ? grp == 2 : grp == 0;
  const int lid = gt;               // loader thread index (LW: within the loader warpgroup)

  const int w = gt >> 5;            // box row
  const int lane = tid & 31;
  const int yp = lane >> 3;         // lines y = 2 yp, 2 yp + 1
  const int zp = lane & 7;          // v_z zp and zp + 8: not adjacent, so the two g_z loads of a
                                    // level stay 8 bytes wide (ptxas fuses adjacent ones)
  const int yl = 2 * yp;
  // box offset of the patch (doubles); a quarter warp (one yp) reads half a
  // 128-byte box line per 8-byte access: no bank conflicts
  constexpr int ZM = PBGK_MS_ZSPLIT ? 1 : 2, ZS = PBGK_MS_ZSPLIT ? 8 : 1;  // v_z of element v: ZM zp + ZS v
  const int zo = ZM * zp;
  const int boff = (w * BY + yl) * BZ + zo;

  double prev[LH][2][2];
#pragma unroll
  for (int l = 0; l < LH; ++l)
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int v = 0; v < 2; ++v) prev[l][k][v] = 0.0;
  double acc = 0.0;
  int stg = 0;
  uint32_t ph = 0;

  // levels [BASE, BASE + LH) of one plane: relax with the level's table, then
  // (levels < depth) transport; level == depth (a lead position) only
  // relaxes and passes its flux on.  FULLC: a run plane of a full pass (no
  // runtime conditions -- the steady path)
  auto levels = [&](double (&x)[2][2], const double* tabs, int depth, const double* AKr, auto fullc,
                    auto basec) {
    constexpr bool FULLC = decltype(fullc)::value;
    constexpr int BASE = decltype(basec)::value;
    constexpr int CNT = BASE == 0 ? LA : L - LA;
#pragma unroll
    for (int ll = 0; ll < CNT; ++ll) {
      const int l = BASE + ll;
      if (!FULLC && (l >= nlev || l > depth)) break;
      const double* S = tabs + l * TS;
      const bool lift0 = SYNTH && l == 0;
      double W, kr, ar;
      double gy[2], gz[2];
      if constexpr (PRE) {
        // (ls gxa, keep r, a r) of this row, cell and level from the window's table
        const double2 wk2 = *reinterpret_cast<const double2*>(S + 4 * w);
        W = wk2.x;
        kr = wk2.y;
        ar = S[4 * w + 2];
        gy[0] = lds_f64(S + 4 * A + yl);
        gy[1] = lds_f64(S + 4 * A + yl + 1);
        gz[0] = lds_f64(S + 4 * A + BY + zo);
        gz[1] = lds_f64(S + 4 * A + BY + zo + ZS);
      } else {
        const double2 rl = *reinterpret_cast<const double2*>(S);  // r, ls
        const double gxa = S[2 + w];
        gy[0] = lds_f64(S + 2 + A + yl);
        gy[1] = lds_f64(S + 2 + A + yl + 1);
        gz[0] = lds_f64(S + 2 + A + BY + zo);
        gz[1] = lds_f64(S + 2 + A + BY + zo + ZS);
#if PBGK_MS_AONLY
        const double av = AKr[l];
        // (a r, (1 - a) r) as a r and r - a r
        ar = lift0 ? av : av * rl.x;
        kr = (lift0 ? 1.0 : rl.x) - ar;
#else
        const double2 ak = reinterpret_cast<const double2*>(AKr)[l];
        kr = lift0 ? ak.x : ak.x * rl.x;
        ar = lift0 ? ak.y : ak.y * rl.x;
#endif
        W = rl.y * gxa;  // ls gxa
      }
      if (FULLC || l < depth) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double wk = W * gy[k];
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const double z = lift0 ? wk * gz[v] : fma(wk, gz[v], x[k][v]);
            x[k][v] = fma(kr, z, prev[ll][k][v]);
            prev[ll][k][v] = ar * z;
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double wk = W * gy[k];
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const double z = lift0 ? wk * gz[v] : fma(wk, gz[v], x[k][v]);
            prev[ll][k][v] = ar * z;
          }
        }
      }
    }
  };
  auto load_x = [&](double (&x)[2][2], const double* box) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      x[k][0] = box[boff + k * BZ];
      x[k][1] = box[boff + k * BZ + ZS];
    }
  };
  auto zero_prev = [&]() {
#pragma unroll
    for (int l = 0; l < LH; ++l)
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int v = 0; v < 2; ++v) prev[l][k][v] = 0.0;
  };
  using TRUE_ = std::integral_constant<bool, true>;
  using FALSE_ = std::integral_constant<bool, false>;
  // the walk over the segment's runs and their items, the same for both
  // groups; item(tg, p0, u0, n, fullc): positions p0 - nlev + u0 .. + n - 1
  auto walk = [&](auto&& item) {
    MsRuns runs;
    runs.init(g0, g1, nx, nlev);
    int t, p0, p1;
    while (runs.next(t, p0, p1)) {
      const TileGeom tg = tile_geom(T, nvx, t);
      const int nitems = (p1 - p0) + nlev;
      // FULLC items: every position a run plane (u >= nlev), P of them, all levels
      int f0 = (nlev + P - 1) / P, f1 = nitems / P;
      if (nlev != L || f1 < f0) f0 = f1 = (nitems + P - 1) / P;
#pragma unroll 1
      for (int j = 0; j < f0; ++j) item(tg, t, p0, j * P, min(P, nitems - j * P), FALSE_{});
#pragma unroll 1
      for (int j = f0; j < f1; ++j) item(tg, t, p0, j * P, P, TRUE_{});
#pragma unroll 1
      for (int j = f1; j * P < nitems; ++j) item(tg, t, p0, j * P, min(P, nitems - j * P), FALSE_{});
    }
  };
  // plane of position p0 - nlev + u of a run
  auto plane_of = [&](const TileGeom& tg, int p0, int u, bool interior) {
    const int p = p0 - nlev + u;
    if (interior) return tg.down ? nx - 1 - p : p;
    return item_plane(nx, a.bc, tg, p);
  };

  // FINAL: the records [m_x rows | m_y | m_z] of a batch of (plane, tile)
  // items from the per-warp partials -- rows from the warps, m_y / m_z summed
  // over the warps in order (the same tree for every entry and its mirror)
  int nfin = 0;
  auto flush = [&](int set, int cnt) {
    named_sync<NTG>(1);
    for (int e = gt; e < cnt * REC; e += NTG) {
      const int q = e / REC, ent = e - q * REC;
      const double* R0 = RB + (size_t)(set * FR + q) * NW * RS;
      double s;
      if (ent < A) {
        // the row total of warp `ent` from its line totals (a fixed tree)
        const double* Lt = R0 + (size_t)ent * RS + 1;
        static_assert(BY == 8, "row total tree");
        s = ((Lt[0] + Lt[1]) + (Lt[2] + Lt[3])) + ((Lt[4] + Lt[5]) + (Lt[6] + Lt[7]));
        acc += s;
      } else {
        const int off = ent < A + BY ? 1 + (ent - A) : 1 + BY + (ent - A - BY);
        s = R0[off];
#pragma unroll
        for (int qq = 1; qq < NW; ++qq) s += R0[(size_t)qq * RS + off];
      }
      part[(size_t)RI[set * FR + q] * T.PS + ent] = s;
    }
  };
  // the pass's last level of a run plane: R_S (FINAL), the store, the
  // partial records (FINAL) or the finiteness sum
  const uint64_t pol_out = (PBGK_MS_STHINT && (NG == 1 || grp == 1)) ? make_policy_evict_first() : 0;
  auto emit = [&](double (&x)[2][2], const double* tabs, int i, int t, long long goff) {
    if (FINAL && fout != nullptr) {
      // R_S (ref/kinetic.py:130-134) of the last level's output, when f_S is
      // stored; otherwise the records are those of f*_S and finalize forms
      // the marginals of R_S(f*_S) from them (FinalArgs relax_tab)
      const double* S = tabs + L * TS;
      const double2 rl = *reinterpret_cast<const double2*>(S);
      const double W = rl.y * S[2 + w];
      const double gz[2] = {S[2 + A + BY + zo], S[2 + A + BY + zo + ZS]};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double wk = W * S[2 + A + yl + k];
#pragma unroll
        for (int v = 0; v < 2; ++v) x[k][v] = rl.x * fma(wk, gz[v], x[k][v]);
      }
    }
    if (fout != nullptr) {
      double* d = fout + (size_t)i * a.plane + goff;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (PBGK_MS_STHINT) {
          // f streams out: its lines leave L2 first (the table rows stay)
          st_global_v2_hint(d + (size_t)k * a.nvz, x[k][0], x[k][1], pol_out);
        } else {
          d[(size_t)k * a.nvz] = x[k][0];
          d[(size_t)k * a.nvz + ZS] = x[k][1];
        }
      }
    }
    if constexpr (FINAL) {
      // per-warp partials: line totals (the 8 lanes of a line pair), the row
      // total, the v_z partials over the warp's lines; fixed butterfly trees
      // (symmetric under index reversal)
      // Two values reduced over 2^k lanes in k shuffles: in the first round a
      // lane keeps one value and sends the other (the partner keeps that one),
      // the later rounds are a butterfly of the kept value.  Every total is
      // the tree ((a0 + a1) + (a2 + a3)) + ... of a plain butterfly.
      double lt[2], zs[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) lt[k] = x[k][0] + x[k][1];
#pragma unroll
      for (int v = 0; v < 2; ++v) zs[v] = x[0][v] + x[1][v];
      const bool zodd = zp & 1, yodd = yp & 1;
      // line totals over the 8 lanes of a line pair: even zp ends with line
      // yl, odd zp with line yl + 1
      double ltot = (zodd ? lt[1] : lt[0]) + __shfl_xor_sync(0xffffffffu, zodd ? lt[0] : lt[1], 1);
      ltot += __shfl_xor_sync(0xffffffffu, ltot, 2);
      ltot += __shfl_xor_sync(0xffffffffu, ltot, 4);
      // v_z partials over the warp's lines: even yp ends with element 0, odd
      // yp with element 1
      double ztot = (yodd ? zs[1] : zs[0]) + __shfl_xor_sync(0xffffffffu, yodd ? zs[0] : zs[1], 8);
      ztot += __shfl_xor_sync(0xffffffffu, ztot, 16);
      // into the batch slot of this record; the records of a batch are
      // reduced after one barrier (FR records per barrier); the row total is
      // summed from the line totals there
      const int slot = nfin % FR, set = (nfin / FR) & 1;
      double* R = RB + ((size_t)(set * FR + slot) * NW + w) * RS;
      if (zp < 2) R[1 + yl + zp] = ltot;
      if (yp < 2) R[1 + BY + zo + ZS * yp] = ztot;
      if (gt == 0) RI[set * FR + slot] = (long long)i * T.NT + t;
      if (++nfin % FR == 0) flush(set, FR);
    } else {
      acc += (x[0][0] + x[0][1]) + (x[1][0] + x[1][1]);
    }
  };

  if (grp == 0 || (LW && grp == 2)) {
    // ---------------- group 0: loads (or the loader warp's), levels [0, LA) ----------------
    // this thread's table chunks of an item: (plane, level, slice) fixed for
    // the launch; source pointer with the run's tile offset set per run, the
    // plane row added per item
    const double* cptr[CPT];
    int cdst[CPT], cpl[CPT];
    bool crow[CPT];  // a row chunk of the window's per-row table (cell stride 4 nvx, else TL)
    auto decode = [&](const TileGeom& tg) {
#pragma unroll
      for (int r = 0; r < CPT; ++r) {
        const int j = lid + r * NLD;
        const bool inr = j < P * NCHT;
        const int pl = inr ? j / NCHT : 0;
        const int jj = inr ? j - pl * NCHT : 0;
        const bool rslot = FINAL && jj >= L * NCHP;  // the R_S slice (plain layout)
        // (the R_S slice is loaded only when f_S is stored)
        const bool ok = inr && !(rslot && fout == nullptr);
        const int l = rslot ? L : jj / NCHP;
        const int c = rslot ? jj - L * NCHP : jj - l * NCHP;
        const double* base = rslot ? a.tabR : a.tab[l < L ? l : 0];
        size_t wso = (size_t)win * a.t_ws;  // the window's tables
        int so, dof;
        bool rowc = false;
        if (PRE && !rslot) {
          if (c < 2 * A) {
            // a box row's (ls gxa, keep r | a r, -) from the window's row table;
            // levels the pass does not run read the last one's rows (unused)
            const int lc = l < nlev ? l : nlev - 1;
            base = a.trip + (size_t)lc * a.trip_ls;
            wso = (size_t)win * a.trip_ws;
            so = (tg.r0 + (c >> 1)) * 4 + 2 * (c & 1); dof = 2 * c;
            rowc = true;
          } else if (c < 2 * A + BY / 2) {
            const int q = c - 2 * A;
            so = a.gyo + tg.y0 + 2 * q; dof = 4 * A + 2 * q;
          } else {
            const int q = c - 2 * A - BY / 2;
            so = a.gzo + tg.z0 + 2 * q; dof = 4 * A + BY + 2 * q;
          }
        } else if (c == 0) {
          so = 0; dof = 0;
        } else if (c <= A / 2) {
          so = a.gxo + tg.r0 + 2 * (c - 1); dof = 2 + 2 * (c - 1);
        } else if (c <= A / 2 + BY / 2) {
          const int q = c - 1 - A / 2;
          so = a.gyo + tg.y0 + 2 * q; dof = 2 + A + 2 * q;
        } else {
          const int q = c - 1 - A / 2 - BY / 2;
          so = a.gzo + tg.z0 + 2 * q; dof = 2 + A + BY + 2 * q;
        }
        cpl[r] = ok ? pl : -1;
        cptr[r] = base + wso + so;
        crow[r] = rowc;
        cdst[r] = (int)(pl * (PLB / 8) + BOXB / 8) + l * TS + dof;
      }
    };
    // loader state: its own walk over the runs (one item per issue)
    MsRuns lruns;
    lruns.init(g0, g1, nx, nlev);
    int lt = 0, lp0 = 0, lnit = 0, lu = 0;
    bool lmore = true;
    TileGeom ltg{};
    int pstg = 0;
    uint32_t pph = 0;
    const int dist = ns - 2;  // items loaded ahead (group 1 trails by about one item)
    // L2 policies: the table slices of a plane are re-read by every tile
    // (keep), f streams through once per pass
    const uint64_t pol_keep = PBGK_MS_HINT >= 1 ? make_policy_evict_last() : 0;
    const uint64_t pol_stream = PBGK_MS_HINT >= 2 ? make_policy_evict_first() : 0;
    auto issue_next = [&]() {
      if (!lmore) return;
      if (lu >= lnit) {
        int lp1;
        if (!lruns.next(lt, lp0, lp1)) {
          lmore = false;
          return;
        }
        lnit = (lp1 - lp0) + nlev;
        lu = 0;
        ltg = tile_geom(T, nvx, lt);
        decode(ltg);
      }
      const int n = min(P, lnit - lu);
      int ip[P];
#pragma unroll
      for (int pl = 0; pl < P; ++pl) {
        const int u = lu + pl;
        int i = -1;
        if (pl < n) {
          const int pp = lp0 - nlev + u;
          i = ltg.down ? nx - 1 - pp : pp;
          if ((unsigned)i >= (unsigned)nx) i = item_plane(nx, a.bc, ltg, pp);  // halo positions
        }
        ip[pl] = i;
      }
      lu += n;
      const int s = pstg;
      // the stage's previous item must be released by group 1
      mbar_wait(&empty[s], pph ^ 1u);
      unsigned char* st = smem + (size_t)s * STAGEB;
      if (lid == 0) {
        uint32_t bytes = 0;
#pragma unroll
        for (int pl = 0; pl < P; ++pl)
          if (ip[pl] >= 0 && !SYNTH) bytes += BOXB;
        mbar_arrive_expect_tx(&full[s], bytes);
#pragma unroll
        for (int pl = 0; pl < P; ++pl)
          if (ip[pl] >= 0 && !SYNTH)
          {
            if (PBGK_MS_HINT >= 2)
              tma_load_4d_hint(st + pl * PLB, &fmap, ltg.z0, ltg.y0, ltg.r0, ip[pl] + win * nx, &full[s],
                               pol_stream);
            else
              tma_load_4d(st + pl * PLB, &fmap, ltg.z0, ltg.y0, ltg.r0, ip[pl] + win * nx, &full[s]);
          }
      }
      {
        // the table-row slices of every level of the item's planes: 16-byte
        // cp.async chunks (L2 hits)
#pragma unroll
        for (int r = 0; r < CPT; ++r) {
          const int pl = cpl[r];
          int i = -1;
#pragma unroll
          for (int q = 0; q < P; ++q)
            if (pl == q) i = ip[q];
          if (i >= 0) {
            const double* src = cptr[r] + ((PRE && crow[r]) ? (size_t)i * (4 * nvx) : (size_t)i * a.TL);
            if (PBGK_MS_HINT >= 1)
              cp_async_16_hint(reinterpret_cast<double*>(st) + cdst[r], src, pol_keep);
            else
              cp_async_16(reinterpret_cast<double*>(st) + cdst[r], src);
          }
        }
      }
      cp_async_mbar_arrive(&full[s]);
      if (++pstg == ns) {
        pstg = 0;
        pph ^= 1u;
      }
    };
    if (lid == 0 && loader) prefetch_tensormap(&fmap);
    if (a.prog != nullptr && loader) {
      // the recursion runs concurrently on other SMs: wait for this pass's
      // tables (bounded: a stalled recursion becomes status kind 5)
      if (lid == 0) {
        long long spins = 0;
        while (ld_acquire_gpu(a.prog) < a.need) {
          __nanosleep(256);
          if (++spins > 20000000LL) {
            atomicMin(errp, err_key(0, a.step0, kErrSync));
            break;
          }
        }
        fence_proxy_async();
      }
      if (LW) named_sync<kMsLoaders>(2);
      else named_sync<NTG>(2);
    }
    if (LW && grp == 2) {
      // the loader warpgroup: every item's loads, as far ahead as the ring
      // allows; its registers go to the compute groups
      reg_dec<PBGK_MS_RL>();
      while (lmore) issue_next();
      asm volatile("cp.async.wait_all;" ::: "memory");
      return;
    }
    if constexpr (LW && (FINAL ? PBGK_MS_R0F : PBGK_MS_R0) > 96) reg_inc<(FINAL ? PBGK_MS_R0F : PBGK_MS_R0)>();
    if (!LW)
      for (int q = 0; q < dist; ++q) issue_next();
    walk([&](const TileGeom& tg, int t, int p0, int u0, int n, auto fullc) {
      constexpr bool FULLC = decltype(fullc)::value;
      mbar_wait(&full[stg], ph);
      const double* AKr = AK + (tg.r0 + w) * L * (PBGK_MS_AONLY ? 1 : 2);
#pragma unroll 1
      for (int pl = 0; pl < (FULLC ? P : n); ++pl) {
        const int u = u0 + pl;
        const int depth = u < nlev ? u : nlev;
        const int i = plane_of(tg, p0, u, FULLC);
        double* box = reinterpret_cast<double*>(smem + (size_t)stg * STAGEB + pl * PLB);
        if (!FULLC && i < 0) {
          zero_prev();  // absorbing ghost plane (lead positions only): zero flux at every level
          continue;
        }
        const double* tabs = box + BOXB / 8;
        double x[2][2];
        if (!SYNTH) load_x(x, box);
        levels(x, tabs, depth, AKr, fullc, std::integral_constant<int, 0>{});
        if constexpr (NG == 1) {
          if (FULLC || depth == nlev) {
            const long long goff =
                ((long long)(tg.r0 + w) * a.nvy + tg.y0 + yl) * a.nvz + tg.z0 + zo;
            emit(x, tabs, i, t, goff);
          }
          continue;
        }
        // hand-off to group 1: every plane it continues (a run plane, or a
        // lead position deep enough to reach its levels)
        if (FULLC || depth == nlev || depth >= LA) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            double* ho = box + HOFF / 8;
            ho[boff + k * BZ] = x[k][0];
            ho[boff + k * BZ + ZS] = x[k][1];
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(NG == 1 ? &empty[stg] : &mid[stg]);
      if (++stg == ns) {
        stg = 0;
        ph ^= 1u;
      }
      if (!LW) issue_next();
    });
    if (NG == 1 && FINAL && nfin % FR) flush((nfin / FR) & 1, nfin % FR);
    if (NG == 1 && !isfinite(acc)) atomicMin(errp, err_key(0, a.step0, kErrNonFiniteMulti));
    return;
  }

  // ---------------- group 1: levels [LH, L), output ----------------
  if constexpr (LW && (FINAL ? PBGK_MS_R1F : PBGK_MS_R1) > 96) reg_inc<(FINAL ? PBGK_MS_R1F : PBGK_MS_R1)>();
  walk([&](const TileGeom& tg, int t, int p0, int u0, int n, auto fullc) {
    constexpr bool FULLC = decltype(fullc)::value;
    mbar_wait(&mid[stg], ph);
    const double* AKr = AK + (tg.r0 + w) * L * (PBGK_MS_AONLY ? 1 : 2);
    const long long goff = ((long long)(tg.r0 + w) * a.nvy + tg.y0 + yl) * a.nvz + tg.z0 + zo;
#pragma unroll 1
    for (int pl = 0; pl < (FULLC ? P : n); ++pl) {
      const int u = u0 + pl;
      const int depth = u < nlev ? u : nlev;
      const int i = plane_of(tg, p0, u, FULLC);
      const double* box = reinterpret_cast<const double*>(smem + (size_t)stg * STAGEB + pl * PLB);
      if (!FULLC && i < 0) {
        zero_prev();
        continue;
      }
      if (!(FULLC || depth == nlev || depth >= LA)) continue;
      const double* tabs = box + BOXB / 8;
      double x[2][2];
      load_x(x, box + HOFF / 8);
      levels(x, tabs, depth, AKr, fullc, std::integral_constant<int, LA>{});
      if (!(FULLC || depth == nlev)) continue;
      emit(x, tabs, i, t, goff);
    }
    __syncwarp();
    // the stage's shared-memory reads are in registers: a relaxed arrive, so
    // the warp does not wait for its global stores to complete
    if (lane == 0) mbar_arrive_relaxed(&empty[stg]);
    if (++stg == ns) {
      stg = 0;
      ph ^= 1u;
    }
  });
  if (FINAL && nfin % FR) flush((nfin / FR) & 1, nfin % FR);
  if (!isfinite(acc)) atomicMin(errp, err_key(0, a.step0, kErrNonFiniteMulti));
}

#ifndef PBGK_MS_P
#define PBGK_MS_P 1
#endif

size_t msweep_smem_bytes(int L, int mode, int nvx, int ns, bool pre) {
  const bool fin = mode & kMsFinal;
  const size_t box = (size_t)ms::A * ms::BY * ms::BZ * 8;
  const size_t stage =
      PBGK_MS_P * (((box + (size_t)(L + (fin ? 1 : 0)) * ms::slice_doubles(pre) * 8 + 127) & ~(size_t)127) +
                   (PBGK_MS_NG == 2 ? box : 0));
  return (size_t)ns * stage + (pre ? 0 : (size_t)L * nvx * 16) +
         (fin ? 2 * 8 * ms::NW * (1 + ms::BY + ms::BZ) * 8 + 2 * 8 * 8 : 0) + (size_t)3 * ns * 8;
}

// The per-row factors of every (window, step, cell): W = ls gxa, keep r =
// r - a r, a r with a = (dt_s / dx) |c_x| (ref/kinetic.py:110-112,130-134, the
// pass kernel's re-association, the same rounded operations); step 0 of a
// window from moments is the lift (keep = 1 - a, a; no r).  One thread per
// (step, cell, row); grid.z = window.
__global__ void __launch_bounds__(256)
    ms_prep_kernel(const double* T, long long t_ws, long long tstep, int TL, int gxo, const double* cx,
                   const double* dts, int dts_g, double dx, int S, int nx, int nvx, int lift0, double* trip,
                   long long trip_ws) {
  pdl_wait();
  pdl_trigger();
  const int win = blockIdx.z;
  const long long n = (long long)S * nx * nvx;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(j % nvx);
    const long long sc = j / nvx;
    const int cell = (int)(sc % nx), s = (int)(sc / nx);
    const double* t = T + (size_t)win * t_ws + (size_t)s * tstep + (size_t)cell * TL;
    const double r = __ldg(t), ls = __ldg(t + 1), gxa = __ldg(t + gxo + row);
    const double c = cx[row];
    const double av = __dmul_rn(__ddiv_rn(dts[(size_t)s * dts_g + win], dx), c < 0.0 ? -c : c);
    const bool lift = lift0 && s == 0;
    const double ar = lift ? av : __dmul_rn(av, r);
    const double kr = __dsub_rn(lift ? 1.0 : r, ar);
    double* o = trip + (size_t)win * trip_ws + (size_t)j * 4;
    reinterpret_cast<double2*>(o)[0] = make_double2(__dmul_rn(ls, gxa), kr);
    reinterpret_cast<double2*>(o)[1] = make_double2(ar, 0.0);
  }
}

cudaError_t launch_ms_prep(const double* T, long long t_ws, long long tstep, int TL, int gxo, const double* cx,
                           const double* dts, int dts_g, double dx, int S, int nx, int nvx, int lift0,
                           double* trip, long long trip_ws, int nwin, cudaStream_t st) {
  const long long n = (long long)S * nx * nvx;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  return launch_pdl_grid(ms_prep_kernel, dim3(blocks, 1, nwin), 256, 0, st, T, t_ws, tstep, TL, gxo, cx, dts,
                         dts_g, dx, S, nx, nvx, lift0, trip, trip_ws);
}

int msweep_threads() { return kMsThreads; }

// CTAs per SM the pass kernel is built for
int msweep_ctas_per_sm() { return PBGK_MS_NG == 1 ? 2 : 1; }

// Box shape of the kernel for a velocity grid (0 if it does not tile):
// 8 rows of each c_x sign, 8 v_y, 16 v_z, no partial boxes.
int msweep_tiling(int nvx, int nvy, int nvz, Tiling* t) {
  if (nvx % (2 * ms::A) != 0 || nvy % ms::BY != 0 || nvz % ms::BZ != 0) return 0;
  t->A = ms::A;
  t->By = ms::BY;
  t->Bz = ms::BZ;
  t->rows_load = ms::A;
  t->nneg = nvx / 2;
  t->ntn = t->nneg / ms::A;
  t->ntp = (nvx - t->nneg) / ms::A;
  t->nty = nvy / ms::BY;
  t->ntz = nvz / ms::BZ;
  t->NT = (t->ntn + t->ntp) * t->nty * t->ntz;
  t->PS = (ms::A + ms::BY + ms::BZ + 1) & ~1;
  return 1;
}

template <int L, int MODE, bool PRE>
static cudaError_t launch_ms(const CUtensorMap& map, const MSweepArgs& a, dim3 grid, int ns, size_t smem,
                             cudaStream_t st) {
  auto fn = msweep_kernel<L, MODE, PBGK_MS_P, PBGK_MS_NG, PRE>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.prog != nullptr) {
    fn<<<grid, kMsThreads, smem, st>>>(map, a, ns);
    return cudaGetLastError();
  }
  return launch_pdl_grid(fn, grid, kMsThreads, smem, st, map, a, ns);
}

template <int L, bool PRE>
static cudaError_t launch_ms_mode(int mode, const CUtensorMap& map, const MSweepArgs& a, dim3 grid, int ns,
                                  size_t smem, cudaStream_t st) {
  switch (mode) {
    case 0: return launch_ms<L, 0, PRE>(map, a, grid, ns, smem, st);
    case kMsSynth: return launch_ms<L, kMsSynth, PRE>(map, a, grid, ns, smem, st);
    case kMsFinal: return launch_ms<L, kMsFinal, PRE>(map, a, grid, ns, smem, st);
    case kMsSynth | kMsFinal: return launch_ms<L, kMsSynth | kMsFinal, PRE>(map, a, grid, ns, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

// L: compiled level counts (a pass may run fewer, a.nlev <= L); nwin > 1: a
// batch of windows (grid.y)
cudaError_t launch_msweep(int L, int mode, const CUtensorMap& map, const MSweepArgs& a, int grid_x, int nwin,
                          int ns, size_t smem, cudaStream_t st) {
  const dim3 grid(grid_x, nwin);
  // a.trip: the per-row factors precomputed (ms_prep_kernel), else from the
  // tables in the kernel (passes that wait on a concurrent recursion)
  const bool pre = a.trip != nullptr;
  switch (L) {
    case 4: return pre ? launch_ms_mode<4, true>(mode, map, a, grid, ns, smem, st)
                       : launch_ms_mode<4, false>(mode, map, a, grid, ns, smem, st);
    case 8: return pre ? launch_ms_mode<8, true>(mode, map, a, grid, ns, smem, st)
                       : launch_ms_mode<8, false>(mode, map, a, grid, ns, smem, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace pbgk
