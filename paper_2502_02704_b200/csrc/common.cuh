// Shared definitions of the fine-propagator kernels.
//
// Data layout in HBM (fp64, C order, identical to the reference's numpy array,
// ref/lifting.py:16-23):  f[i][jx][jy][jz],  i = x cell, jz fastest.
// Per-cell side tables (one row of TL doubles per x cell):
//   [0] r    relax: 1/(1+lambda)             synth: unused
//   [1] ls   relax: lambda*rho/mass           synth: 1 (raw lift) or rho/mass
//   [gxo .. gxo+nvx)  gx*amp      (ref/lifting.py:47-50)
//   [gyo .. gyo+nvy)  gy
//   [gzo .. gzo+nvz)  gz
// Moments (SoA, 5*nx): rho, u_x, u_y, u_z, theta.
// Partial marginals: part[(i*NT + tile)*PS + {0..A) m_x rows, A..A+By) m_y, A+By..) m_z].
#pragma once
#include <cuda_runtime.h>
#include <utility>
#include <cstdlib>
#include <cstdint>

namespace pbgk {

// Error codes are 64-bit keys (unit << 40) | (step << 8) | kind, reduced with
// atomicMin: the lowest unit (window / slice) wins, then the earliest step,
// then the lowest kind, which is the reference's raise order inside one step
// (SURVEY 8(b) Errors).  All ones = clean.
typedef unsigned long long ErrKey;
enum ErrKind : int {
  kErrProjectRho = 0,   // DegenerateStateError in project (ref/moments.py:102-104)
  kErrLiftState = 1,    // DegenerateStateError in lift / conserved->primitive
  kErrNonFinite = 2,    // BlowUpError(step)
  kErrUnphysical = 3,   // BlowUpError(step) from G's positivity guard
  kErrOvershoot = 4,    // CorrectionOvershootError(slice_index)
  kErrSync = 5,         // internal: a pass gave up waiting for the concurrent recursion
  kErrNonFiniteMulti = 6,  // internal: non-finite f somewhere in a multi-step pass that starts at
                           // `step`; the host re-runs that propagation on the one-step path
};
constexpr ErrKey kNoError = ~0ull;
__host__ __device__ constexpr ErrKey err_key(unsigned long long unit, unsigned long long step,
                                             int kind) {
  return (unit << 40) | (step << 8) | (unsigned long long)kind;
}

struct Tiling {
  int A, By, Bz;     // velocity box of one tile (rows, jy, jz)
  int rows_load;     // A, or A+2 when the v_x field term needs neighbour rows
  int nneg;          // rows [0,nneg) have c_x < 0 and march downward in x
  int ntn, ntp;      // row tiles in the negative / non-negative group
  int nty, ntz, NT;  // y / z tiles, total tiles
  int PS;            // stride of one tile's partial record (doubles)
};

struct SweepArgs {
  int nx, nvx, nvy, nvz;
  long long plane;   // nvx*nvy*nvz
  Tiling t;
  long long total;   // NT*nx plane items (halos excluded)
  const double* fin;
  double* fout;      // nullptr: marginals only
  const double* tab;
  int TL, gxo, gyo, gzo;
  const double* cx;  // x-velocity centres
  double dtdx;       // 0: no transport (pure relax/copy pass)
  int bc;            // 0 absorbing, 1 periodic, 2 outflow (zero gradient)
  const double* E;   // per-cell field or nullptr
  double half_emax;  // 0.5*max|E|
  double dtdv;       // dt / dv_x
  double* part;
  ErrKey* err;
  int check_step;    // >0: flag non-finite f_pre as step `check_step`
  int muscl;         // 1: MUSCL (minmod) x transport instead of first-order upwind
  int l2_keep;       // 1: f stores evict_last / loads evict_first (f ping-pong fits in L2)
  int trap;          // 1: trapezoidal velocity quadrature (end nodes weigh 1/2)
  int debug;         // development ablations (PBGK_DEBUG): 1 no reductions, 4 copy-through
  int noreduce;      // multi-step path with the field term: no marginal partials (the
                     // recursion gives the tables); f*'s finiteness flagged as step out_step
  int out_step;
};

// Multi-step sweep (fsweep.cu): L consecutive fine steps per pass over f,
// the relax tables of every step known beforehand (marginal recursion,
// marginal.cu), no reductions.  Level l reads the tables tab[l] and moves by
// dtdx[l]; the pass reads f*_s (or synthesises f_0) and writes f*_{s+L}.
constexpr int kMaxLevels = 4;
struct FSweepArgs {
  int nx, nvx, nvy, nvz;
  long long plane;
  Tiling t;
  long long total;
  const double* fin;   // null: level 0 synthesises f_0 from tab[0]
  double* fout;
  const double* tab[kMaxLevels];
  int TL, gxo, gyo, gzo;
  const double* cx;
  double dtdx[kMaxLevels];
  int bc;
  ErrKey* err;
  int step0;           // step number of level 0's output (BlowUpError keys)
  // concurrent recursion (single propagations): wait until *prog >= need
  // before the first table load (null: the tables are already complete)
  const unsigned* prog;
  unsigned need;
};

// Multi-step sweep, round 2 (msweep.cu): up to kMaxL levels per pass,
// warp-specialised; tab[l] the relax table applied before level l's
// transport, tabR (FINAL mode) R_S of the window's last step, part the
// partial records of P(f_S) on the kernel's own tiling.
constexpr int kMaxL = 8;
struct MSweepArgs {
  int nx, nvx, nvy, nvz;
  long long plane;
  Tiling t;
  long long total;       // NT * nx plane items (halos excluded)
  double* fout;          // null: nothing stored (FINAL: partials only)
  const double* tab[kMaxL];
  const double* tabR;
  int nlev;              // levels of this pass (<= the compiled L)
  int TL, gxo, gyo, gzo;
  const double* cx;
  double dtdx[kMaxL];
  int bc;
  ErrKey* err;
  int step0;
  double* part;
  const unsigned* prog;
  unsigned need;
  // a batch of windows in one launch (grid.y = window; small grids, where one
  // window cannot fill the GPU): per-window strides (doubles) of f in / out
  // (the tensor map spans nx * windows planes), of the tables and of the
  // partial records; per-window failure keys; per-window dt of step s on the
  // device at dts[(s0 + l) * dts_g + window] (null: dtdx[l] for every window)
  long long f_ws, t_ws, p_ws;
  ErrKey* errw;
  const double* dts;
  int dts_g, s0;
  double dx;
  // per-row factors (ls gxa, keep r, a r, -) of level l and cell i at
  // trip + l trip_ls + i 4 nvx (+ window trip_ws), precomputed once per window
  // (ms_prep_kernel); null: the kernel forms them from the tables and dtdx
  const double* trip;
  long long trip_ls, trip_ws;
};

// Multi-step sweep with the v_x field term (esweep.cu): up to kMaxLevels
// levels per pass, a warp per (whole v_x column, x segment) item; tab[l] the
// relax table applied before level l's transport (SYNTH: fin null, tab[0]
// the lift tables), dtdx / dtdv per level, E per x cell.
struct ESweepArgs {
  int nx, nvx, nvy, nvz;
  const double* fin;   // null: level 0 synthesises f_0 from tab[0]
  double* fout;
  const double* tab[kMaxLevels];
  int TL, gyo, gzo;
  const double* cx;
  const double* E;
  double half_emax;
  double dtdx[kMaxLevels], dtdv[kMaxLevels];
  int nlev;
  int bc;              // 0 absorbing, 1 periodic, 2 outflow
  int ncol;            // warp columns: nvy * nvz / 8
  int nseg, seglen;    // x segments per column and their length (planes)
  ErrKey* err;
  int step0;
  // FINAL (the window's last pass, tabR non-null): instead of the store, the
  // partial records [m_x rows | m_y | m_z of the column's 8 v_z] of the last
  // level's output f*_S for every (plane, warp column), written to part
  // (stride PS doubles, NT = ncol records per plane) for finalize.cu
  // (kFinProject with relax_tab = tabR: R_S applied to the marginals)
  const double* tabR;
  double* part;
  int PS;
};

// Moment recursion (marginal.cu): five weighted sums of f over (v_y, v_z)
// per x cell and v_x row obey a closed recursion under the upwind x transport
// and the separable BGK relaxation (both act on a v_x row with coefficients
// independent of v_y, v_z).  One step maps Q(f*_{s-1}) and the tables of
// R_{s-1} to Q(f*_s), the moments and the tables of R_s.
struct MargArgs {
  int nx, nvx, nvy, nvz, bc;
  const double* min;   // Q(f*_{s-1}): nx * 5 nvx doubles; null: f_{s-1} = lift (tab_in r = 0)
  double* mout;        // Q(f*_s)
  const double* tab_in;
  const double* cx;
  const double* cy;
  const double* cz;
  double dtdx;
  int TL, gxo, gyo, gzo, trap;
  const double* gsum_in;  // per cell: sums of g_y, g_z of tab_in (6 doubles)
  double* gsum_out;       // the same for the output tables
  // batch of windows (grid.y = window): per-window strides (doubles) of the
  // state, the tables and the G sums; per-window dt of this step, step counts
  // and failure keys (null: a single window, dtdx / FinalArgs dt and err)
  long long q_ws, t_ws, g_ws;
  const double* dts;
  const int* nst;
  ErrKey* errw;
  double dx;
  const double* E;     // v_x field per cell (null: none); half_emax = max|E| / 2
  double half_emax, dvx;
};

enum FinalMode : int {
  kFinRelax = 0,      // tables of the normalised Maxwellian + lambda (bgk_relax)
  kFinSynthRaw = 1,   // tables of the un-normalised lift (window start)
  kFinSynthNorm = 2,  // tables of the mass-normalised lift
  kFinIdentity = 3,   // r=1, ls=0: f_pre = f (a loaded distribution as is)
  kFinProject = 4,    // moments only
};

struct FinalArgs {
  int nx, nvx, nvy, nvz;
  Tiling t;
  const double* part;
  const double* mom_in;  // non-null: moments given (lift), partials ignored
  const double* cx;
  const double* cy;
  const double* cz;
  double dvol;
  double* mom_out;       // may be null
  double* tab;           // may be null
  int TL, gxo, gyo, gzo;
  int mode;
  double dt, eps, tau;   // lambda = dt*tau/eps (ref/kinetic.py:131)
  const double* tau_arr; // optional per-cell tau values
  ErrKey* err;
  int step;
  int check_finite;      // kFinProject: flag non-finite marginals as BlowUpError(step)
  int trap;              // trapezoidal velocity quadrature (end nodes weigh 1/2)
  // non-null (midpoint quadrature): the partials are those of f*; the
  // marginals of f = R(f*) = r (f* + ls g_x g_y g_z) (ref/kinetic.py:130-134,
  // linear and separable) are formed from them with this table before the
  // projection: m_x[j] = r (m*_x[j] + ls g_x[j] (sum g_y) (sum g_z)), ...
  const double* relax_tab;
};

// finalize over a batch of windows (grid.y = window): per-window strides
// (doubles) of the partial records, the moments in / out and the tables, and
// per-window failure keys (null: FinalArgs err)
struct FinalBatch {
  long long part_ws, mom_in_ws, mom_out_ws, tab_ws;
  ErrKey* errw;
};

// Coarse propagator arguments (fluid.cu).  model 0: the reference's Rusanov
// Euler G; model 1: the drift-diffusion G of the diffusive scaling (extension).
struct FluidArgs {
  int nx;
  double dx;
  int periodic;
  double dt_max;  // <= 0: none
  double cfl;
  const double* force;  // nx or null
  ErrKey* err;
  int model;
  double diff;          // model 1: diffusivity D = m2 / tau
  int fastg;            // set by the launcher: per-cell wave / flux arrays fit in smem
};

// Launch with programmatic dependent launch enabled: the kernel may begin
// launching while the preceding kernel of the stream finishes; it must call
// pdl_wait() (ptx.cuh) before consuming that kernel's results.
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl_grid(void (*kernel)(KArgs...), dim3 grid, int block, size_t smem,
                                          cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  static const bool off = getenv("PBGK_NO_PDL") != nullptr;  // development A/B knob
  attr[0].val.programmaticStreamSerializationAllowed = off ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem,
                                     cudaStream_t st, Args&&... args) {
  return launch_pdl_grid(kernel, dim3(grid), block, smem, st, std::forward<Args>(args)...);
}

}  // namespace pbgk
