/*
 * pbgk.h — C ABI of the B200 fine kinetic propagator (libpbgk.so).
 *
 * Drop-in boundary for the hot path of arXiv 2502.02704's reference package
 * `parabgk` (Python/numpy; /root/reference/pkg/src/parabgk, "ref/" below).
 * The reference has no FFI of its own: its boundary is the Python API
 * re-exported at ref/__init__.py:8-31.  Each entry point here replaces the
 * numpy body of one reference function; the Python host package
 * `paper_2502_02704_b200` keeps the reference signatures and calls these
 * through ctypes (see INTEGRATION.md for the binding a parabgk maintainer
 * would add).
 *
 * Conventions
 *  - All array arguments are DEVICE pointers (cudaMalloc / torch CUDA
 *    storage) unless named h_*; fp64 only; C order.
 *  - Distribution f: double[nx][nvx][nvy][nvz] (ref/lifting.py:16-23).
 *  - Moments: double[5][nx] = rho, u_x, u_y, u_z, theta (ref/moments.py:29-34).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Return value: 0 on success, negative on an API/CUDA failure (message in
 *    pbgk_last_error()).  Numerical failures are NOT return codes: when
 *    `h_code` is non-NULL the call synchronises `stream` and stores the
 *    solver status there: -1 = clean, otherwise the key
 *        (unit << 40) | (step << 8) | kind
 *    (unit = window / slice index where it applies, else 0) with
 *      kind 0  rho <= 0 in a projection        -> DegenerateStateError
 *      kind 1  degenerate state in lift or in
 *              conserved->primitive            -> DegenerateStateError
 *      kind 2  non-finite state after `step`    -> BlowUpError(step)
 *      kind 3  rho or p <= 0 in G after `step`  -> BlowUpError(step)
 *      kind 4  correction overshoot             -> CorrectionOvershootError(unit)
 *      kind 5  internal: a multi-step pass timed out waiting for the
 *              concurrent relax-table recursion  -> RuntimeError
 *      (kind 6 is internal to the library: "non-finite within a multi-step
 *      pass"; pbgk_propagate / pbgk_propagate_windows re-run that
 *      propagation on the one-step path and return its exact key)
 *    Keys are min-reduced: lowest unit, then earliest step, then the
 *    reference's raise order within a step (ref/moments.py:102-104,
 *    ref/lifting.py:44-45, ref/kinetic.py:157-159, ref/fluid.py:117-122).
 *  - Threads: pbgk_last_error() is per thread; a context holds mutable
 *    workspaces (tables, partial records, failure word, tensor-map cache), so
 *    calls on one context must not run concurrently from several threads, and
 *    its own workspaces are used on one stream at a time (the *_async / *_range
 *    entry points take caller-owned buffers and may run on a second stream).
 */
#ifndef PBGK_H
#define PBGK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pbgk_ctx pbgk_ctx;

/* Phase grid + boundary (ref/grid.py:39-87, :89-116). */
typedef struct pbgk_grid_desc {
  int32_t nx, nvx, nvy, nvz;
  double x_min, x_max, v_max;
  int32_t bc;       /* x boundary: 0 ABSORBING (zero inflow ghost, ref/kinetic.py:106-108),
                       1 PERIODIC, 2 OUTFLOW (zero-gradient ghost; extension asked by
                       BASELINE.json, not in the reference), 3 SLAB (one x-slab of a
                       sharded domain, halos supplied by the caller; see pbgk_slab_*) */
  int32_t device;   /* CUDA device ordinal the context (and every call on it) uses */
} pbgk_grid_desc;

/* Library identification. */
int pbgk_version(void);
const char* pbgk_last_error(void);

/* Context: grid constants, tiling, device workspace (tables, partials). */
int pbgk_ctx_create(const pbgk_grid_desc* grid, pbgk_ctx** out);
void pbgk_ctx_destroy(pbgk_ctx* ctx);
/* Workspace bytes held by a context (diagnostics). */
size_t pbgk_ctx_workspace_bytes(const pbgk_ctx* ctx);

/* lift(U, grid, normalize_mass) — replaces ref/lifting.py:36-58. */
int pbgk_lift(pbgk_ctx* ctx, const double* mom, int normalize_mass, double* f_out, void* stream,
              long long* h_code);

/* project(f, grid) — replaces ref/moments.py:91-113. */
int pbgk_project(pbgk_ctx* ctx, const double* f, double* mom_out, void* stream, long long* h_code);

/* transport_update(f, dt, grid, params, bc) — replaces ref/kinetic.py:86-124.
 * E: per-cell field (nx) or NULL; e_max = max|E| (field term only if > 0). */
int pbgk_transport(pbgk_ctx* ctx, const double* f, double* f_out, double dt, const double* E,
                   double e_max, void* stream);

/* bgk_relax(f, dt, grid, params) — replaces ref/kinetic.py:127-134.
 * lambda = dt*tau/eps with tau = tau_cells[i] when tau_cells != NULL. */
int pbgk_relax(pbgk_ctx* ctx, const double* f, double* f_out, double dt, double eps, double tau,
               const double* tau_cells, void* stream, long long* h_code);

/* Finiteness guard of ref/kinetic.py:157-159 on a distribution: status key
 * (0 << 40) | (step << 8) | 2 if any value of f is NaN/Inf. */
int pbgk_check_finite(pbgk_ctx* ctx, const double* f, int step, void* stream, long long* h_code);

/* The fine propagator loop of propagate_kinetic (ref/kinetic.py:137-161) for a
 * given step schedule h_dts[0..nsteps) (computed by the caller exactly as the
 * reference does, ref/kinetic.py:146-156).
 * Start: f0 (distribution) or, when f0 == NULL, mom0 (the window lift
 *   L(U) of ref/parareal.py:129, never materialised).
 * End:   f_out receives f_S when write_final != 0; mom_out (may be NULL)
 *   receives P(f_S) (ref/parareal.py:136).  f_tmp is a second f-sized buffer
 *   (ping-pong); f0 must not alias f_out or f_tmp. */
int pbgk_propagate(pbgk_ctx* ctx, const double* f0, const double* mom0, double* f_out,
                   double* f_tmp, int write_final, double* mom_out, int nsteps,
                   const double* h_dts, double eps, double tau, const double* E, double e_max,
                   void* stream, long long* h_code);

/* The fine stage of one parareal iteration on this GPU: P(F(L(U_w))) for
 * nwin windows back to back (ref/parareal.py:123-142 without the G part),
 * mom_in / mom_out double[nwin][5][nx] on the device, window w taking
 * h_nsteps[w] steps of h_dts (concatenated), f_a / f_b two f-sized device
 * scratch buffers.  One host synchronisation for the whole batch; h_codes[w]
 * receives window w's failure key (-1 clean).  Same kernels and order as
 * pbgk_propagate per window, so results are bitwise those of nwin calls. */
int pbgk_propagate_windows(pbgk_ctx* ctx, int nwin, const double* mom_in, double* mom_out,
                           double* f_a, double* f_b, const int* h_nsteps, const double* h_dts,
                           double eps, double tau, const double* E, double e_max, void* stream,
                           long long* h_codes);

/* Coarse Euler propagator G (ref/fluid.py:91-125) on one GPU: advance
 * `nwin` independent primitive states mom_in[w] (double[nwin][5][nx]) over
 * [h_t0[w], h_t1[w]] into mom_out[w]; when `minuend` is non-NULL the output
 * is minuend[w] - G(mom_in[w]) (the parareal jump, ref/parareal.py:142);
 * `minuend` may alias `mom_out` (each entry is read, then written, by one thread).
 * dt_max <= 0 means no cap.  force: per-cell E or NULL.  Failure keys carry
 * the window index (0-based) as unit. */
int pbgk_fluid_propagate(pbgk_ctx* ctx, int nwin, const double* mom_in, double* mom_out,
                         const double* minuend, const double* h_t0, const double* h_t1,
                         double dt_max, double cfl, const double* force, void* stream,
                         long long* h_code);

/* Sequential parareal correction (ref/parareal.py:217-248) on one GPU:
 *   U_n = G(U_{n-1}) + jump_n   for n = start..n_g  (primitive variables),
 * snaps: double[n_g+1][5][nx] (updated in place from index start),
 * old:   double[n_g+1][5][nx] (iterate before the correction),
 * jumps: double[n_g][5][nx];  h_times: coarse times (n_g+1).
 * h_err receives the successive-iterate sup error; failure keys carry the
 * 1-based slice index as unit (kind 4: CorrectionOvershootError). */
int pbgk_parareal_correct(pbgk_ctx* ctx, int n_g, int start, double* snaps, const double* old,
                          const double* jumps, const double* h_times, double dt_max, double cfl,
                          const double* force, void* stream, double* h_err, long long* h_code);

/* Selects the coarse propagator used by pbgk_fluid_propagate and
 * pbgk_parareal_correct on this context: model 0 = the reference's Rusanov
 * Euler G (default); model 1 = the drift-diffusion G of the diffusive scaling
 * (EXTENSION, no reference counterpart -- SPEC:8; PAPER eq. (DDbis) with the
 * central scheme of PAPER:351): d_t rho = D d_x(d_x rho - E rho), output
 * (rho, u = 0, theta = 1), D = `diffusivity` (> 0). */
int pbgk_fluid_model(pbgk_ctx* ctx, int model, double diffusivity);

/* Velocity quadrature of the context: 0 = the reference's midpoint cells
 * (default), 1 = trapezoidal (EXTENSION: BASELINE config 0's wording; n
 * nodes on [-v_max, v_max] including the ends, dv = 2 v_max/(n-1), end
 * nodes weigh 1/2 in every velocity sum).  Call before any use. */
int pbgk_ctx_set_quadrature(pbgk_ctx* ctx, int quadrature);

/* x transport of every sweep on this context: 0 = the reference's first-order
 * upwind flux (default); 1 = MUSCL reconstruction with the minmod limiter
 * (EXTENSION: BASELINE north_star "upwind/MUSCL", PAPER flux limiters;
 * no reference counterpart; two ghost planes per side by the x boundary).
 * MUSCL has no v_x field term: sweeps with E != 0 fail on a MUSCL context. */
int pbgk_set_x_scheme(pbgk_ctx* ctx, int scheme);

/* Multi-step path of pbgk_propagate / pbgk_propagate_windows (upwind
 * scheme, bc 0..2): the relax tables R_s of every step come first from the
 * moment recursion -- per x cell and v_x row five weighted sums of f over
 * (v_y, v_z) (the marginal m_x, the folded first moments and the second
 * moments in v_y and v_z) evolve in closed form under the upwind x transport,
 * the v_x field flux and the separable BGK relaxation -- then f is read and
 * written once per `levels` fine steps.  With the v_x field term the passes
 * are the field-term kernel's (pbgk_set_esweep), else one step each (the
 * one-step field sweep on the recursion's tables).  Same
 * results as the one-step path to rounding (sums and transport associated
 * differently); 0 = always the one-step path; -1 (default) = the measured
 * best.  `levels` (1..4) applies to the round-1 pass kernel (fsweep.cu);
 * pbgk_set_msweep selects the round-2 kernel and its level count. */
int pbgk_set_fusion(pbgk_ctx* ctx, int levels);

/* Round-2 pass kernel of the multi-step path (msweep.cu, default on): up to
 * 8 fine steps per pass over f, warp-specialised (a loader warpgroup issues
 * the TMA boxes and the table-row slices and hands its registers to the two
 * compute groups), 3 fp64 instructions per element and level, and
 * the window's final relax + projection folded into its last pass (partial
 * records of P(f_S), no store of f_S unless the caller wants it).  Needs
 * v_x / v_y / v_z counts divisible by 16 / 8 / 16 (else the round-1 kernel
 * runs).  on = 0 selects the round-1 kernel; levels = 0 (auto: 8), 4 or 8.
 * Replaces the numpy loop of ref/kinetic.py:152-160 like pbgk_propagate. */
int pbgk_set_msweep(pbgk_ctx* ctx, int on, int levels);
/* Levels per pass the round-2 kernel runs on this context (0: not used). */
int pbgk_msweep_levels(pbgk_ctx* ctx);
/* Multi-step passes WITH the v_x field term (esweep.cu, default on): a warp
 * owns whole v_x columns and marches an x segment, up to 4 fine steps per
 * pass (3 at nvx = 32) with the field flux's v_x neighbours in registers /
 * shuffles; the window's last pass applies R_S and writes the partial
 * records of P(f_S) instead of f_S when only the moments are wanted (midpoint
 * quadrature).  Needs nvx = 16, 32 or 48 and nvz % 8 == 0 (else, and with
 * on = 0, the field runs one step per pass).  An explicit pbgk_set_fusion
 * level count caps its levels.  Replaces ref/kinetic.py:152-160 with a force
 * (ref/kinetic.py:114-123) like pbgk_propagate. */
int pbgk_set_esweep(pbgk_ctx* ctx, int on);
/* Levels per pass of the field-term kernel on this context (0: not used). */
int pbgk_esweep_levels(pbgk_ctx* ctx);
/* Device bytes the multi-step path may spend on per-step relax tables: the
 * batched windows of pbgk_propagate_windows run in groups that fit (a single
 * propagation whose tables do not fit runs one-step).  0 = the default
 * (PBGK_BATCH_BYTES, else a quarter of the free device memory within 2..16
 * GiB).  Results do not depend on the grouping. */
int pbgk_set_batch_bytes(pbgk_ctx* ctx, double bytes);

/* ---- x-sharded fine propagation (slabs) --------------------------------- */
/* A context created with bc = 3 is one x-slab of a larger domain (one rank
 * of an x-sharded F, EXTENSION: SURVEY 8(f) rank 2).  Its f buffers are
 * PADDED, double[nx+2][nvx][nvy][nvz], and so are its table buffers,
 * double[nx+2][TL]: index 0 and nx+1 are halo planes / rows that the caller
 * fills between steps (neighbours' boundary planes f*_s and table rows R_s;
 * zeros for an absorbing global edge, the edge itself for outflow).  Every
 * sweep / finalize is the unsharded one restricted to the slab, so the
 * sharded F is bitwise the single-GPU F. */
int pbgk_table_len(const pbgk_ctx* ctx);
/* Exact cell width (a slab inherits the global dx; (x_max-x_min)/nx of the
 * slab's bounds may round differently). */
int pbgk_ctx_set_dx(pbgk_ctx* ctx, double dx);
/* Table rows 1..nx: kind 0 identity (relax = id, for an f given directly),
 * kind 1 lift tables of the moments mom (double[5][nx]).  Starts a
 * propagation: resets the context's failure key. */
int pbgk_slab_tables(pbgk_ctx* ctx, int kind, const double* mom, double* tab_pad, void* stream,
                     long long* h_code);
/* One sweep: relax the padded input by tab_pad, transport by dt (0: relax
 * only), write the interior planes of fout_pad (NULL: partials only);
 * fin_pad NULL synthesises the input from the lift tables. */
int pbgk_slab_sweep(pbgk_ctx* ctx, const double* fin_pad, const double* tab_pad, double* fout_pad,
                    double dt, const double* E, double e_max, void* stream);
/* After a sweep: mode 0 = relax tables R(dt, eps, tau) into rows 1..nx of
 * tab_pad (BlowUpError(step) on non-finite marginals); mode 1 = the moments
 * of the swept planes into mom_out (double[5][nx]).  `field`: the sweep had
 * the v_x field term (its partial layout).  Asynchronous unless h_code is
 * non-NULL, which synchronises and returns the earliest failure key since
 * pbgk_slab_tables (-1 clean). */
int pbgk_slab_finalize(pbgk_ctx* ctx, int mode, int field, double* tab_pad, double* mom_out,
                       double dt, double eps, double tau, int step, void* stream, long long* h_code);

/* ---- pipelined parareal (side stream) ---------------------------------- */
/* Leave `slots` CTA slots out of the persistent sweep grid (sized for every
 * slot of every SM), so a side-stream G / correction CTA (launched "lean":
 * the fewest threads covering nx) is resident beside the sweeps instead of
 * stalling one of their CTAs.  0 = whole GPU (default). */
int pbgk_set_grid_reserve(pbgk_ctx* ctx, int slots);

/* pbgk_fluid_propagate without host synchronisation: window times are
 * device arrays, failure keys are atomicMin-ed into the device word
 * *d_status (caller initialises it to -1 = clean). */
int pbgk_fluid_propagate_async(pbgk_ctx* ctx, int nwin, const double* mom_in, double* mom_out,
                               const double* minuend, const double* d_t0, const double* d_t1,
                               double dt_max, double cfl, const double* force, void* stream,
                               long long* d_status);

/* The correction sweep of pbgk_parareal_correct restricted to windows
 * first..last (1-based, inclusive), asynchronous: d_times are the coarse
 * times on the device, the sup error is max-accumulated into *d_errmax
 * (caller zeroes it) and failure keys into *d_status.  Consecutive ranges
 * give bitwise the result of one full sweep. */
int pbgk_parareal_correct_range(pbgk_ctx* ctx, int first, int last, double* snaps,
                                const double* old, const double* jumps, const double* d_times,
                                double dt_max, double cfl, const double* force, void* stream,
                                double* d_errmax, long long* d_status);

/* ---- measurement (bench.py) ------------------------------------------- */
/* Human-readable tiling / launch plan of a context (diagnostics). */
int pbgk_ctx_describe(const pbgk_ctx* ctx, char* buf, size_t n);

/* Total kernel launches issued by this library in the process. */
long long pbgk_launch_count(void);

typedef struct pbgk_profile {
  double sweep_ms;        /* summed device time of profiled sweep launches     */
  double sweep_bytes;     /* their algorithmic HBM bytes (f read + f written)  */
  long long sweeps;       /* number of profiled sweep launches                 */
  double finalize_ms;     /* summed device time of finalize launches           */
  long long finalizes;
  double msweep_ms;       /* multi-step sweeps (fsweep.cu): device time        */
  double msweep_bytes;    /* their algorithmic HBM bytes (f read + f written)  */
  long long msweeps;      /* number of profiled multi-step sweeps              */
  long long msweep_steps; /* fine steps they advanced                          */
  double marg_ms;         /* marginal recursion steps (marginal.cu)            */
  long long margs;
} pbgk_profile;

/* When enabled, every sweep / finalize launch on this context is bracketed
 * by CUDA events recorded on its own stream. */
int pbgk_profile_enable(pbgk_ctx* ctx, int on);
/* Synchronises the recorded events, returns the sums and resets them. */
int pbgk_profile_read(pbgk_ctx* ctx, pbgk_profile* out);

#ifdef __cplusplus
}
#endif
#endif /* PBGK_H */
