// Coarse propagator G: first-order Rusanov Euler solver (ref/fluid.py:39-125)
// and the sequential parareal correction (ref/parareal.py:217-248), on one GPU.
//
// One CTA owns one window's state (conserved variables of all nx cells in
// shared memory).  Every expression is evaluated in the reference's operation
// order with explicitly rounded fp64 intrinsics (no FMA contraction), so the
// result is bitwise that of numpy for the same input; the CFL max is
// order-independent.  Each thread recomputes both faces of its cells (no face
// buffer), which keeps the smem footprint at 40*nx bytes.
#include <cuda_runtime.h>

#include "common.cuh"

namespace pbgk {

#define DM __dmul_rn
#define DA __dadd_rn
#define DS __dsub_rn
#define DD __ddiv_rn

// ref/fluid.py:39-42
__device__ __forceinline__ double press(double v0, double v1, double v2, double v3, double v4) {
  const double ke = DD(DM(0.5, DA(DA(DM(v1, v1), DM(v2, v2)), DM(v3, v3))), v0);
  return DD(DS(v4, ke), 1.5);
}

struct St {
  double v[5];
};

// ref/fluid.py:45-56
__device__ __forceinline__ void eflux(const St& s, double h[5]) {
  const double ux = DD(s.v[1], s.v[0]);
  const double p = press(s.v[0], s.v[1], s.v[2], s.v[3], s.v[4]);
  h[0] = s.v[1];
  h[1] = DA(DM(s.v[1], ux), p);
  h[2] = DM(s.v[2], ux);
  h[3] = DM(s.v[3], ux);
  h[4] = DM(ux, DA(s.v[4], p));
}

__device__ __forceinline__ double wave(const St& s) {
  const double p = press(s.v[0], s.v[1], s.v[2], s.v[3], s.v[4]);
  return DA(fabs(DD(s.v[1], s.v[0])), sqrt(DD(p, s.v[0])));
}

// ref/fluid.py:59-66
__device__ __forceinline__ void rusanov(const St& l, const St& r, double H[5]) {
  const double s = fmax(wave(l), wave(r));
  double hl[5], hr[5];
  eflux(l, hl);
  eflux(r, hr);
  const double hs = DM(0.5, s);
#pragma unroll
  for (int c = 0; c < 5; ++c) H[c] = DS(DM(0.5, DA(hl[c], hr[c])), DM(hs, DS(r.v[c], l.v[c])));
}

__device__ __forceinline__ St load_state(const double* V, int nx, int i) {
  St s;
#pragma unroll
  for (int c = 0; c < 5; ++c) s.v[c] = V[c * nx + i];
  return s;
}

__device__ __forceinline__ St ghost_state(const double* V, int nx, int i, int periodic) {
  // ref/fluid.py:78-88: periodic wrap or transmissive copy
  if (i < 0) return load_state(V, nx, periodic ? nx - 1 : 0);
  if (i >= nx) return load_state(V, nx, periodic ? 0 : nx - 1);
  return load_state(V, nx, i);
}

__device__ double block_max(double x, double* red) {
  for (int w = 16; w >= 1; w >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, w));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = x;
  __syncthreads();
  double m = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
  return m;
}

// prim -> conserved (ref/moments.py:116-119; einsum('ij,ij->i') over 3
// components evaluates as (a0 b0 + a2 b2) + a1 b1 in numpy 2.x)
__device__ __forceinline__ void to_cons(double rho, double u0, double u1, double u2, double th,
                                        double v[5]) {
  v[0] = rho;
  v[1] = DM(rho, u0);
  v[2] = DM(rho, u1);
  v[3] = DM(rho, u2);
  const double uu = DA(DA(DM(u0, u0), DM(u2, u2)), DM(u1, u1));
  v[4] = DA(DM(DM(0.5, rho), uu), DM(DM(1.5, rho), th));
}

// Advances the state held in smem V (5 x nx, conserved) over `span`.
// Returns 0 or (step << 8) | kind (kErrNonFinite / kErrUnphysical).
constexpr int kMaxCellsPerThread = 4;

__device__ ErrKey g_advance(double* V, double* red, int* flag, const FluidArgs& a, double span) {
  const int nx = a.nx;
  const double guard = 1e-12;  // ref/fluid.py:30
  double done = 0.0;
  unsigned long long step = 0;
  while (DS(span, done) > DM(guard, span)) {
    double rate = 0.0;
    for (int i = threadIdx.x; i < nx; i += blockDim.x) rate = fmax(rate, wave(load_state(V, nx, i)));
    rate = block_max(rate, red);
    // ref/fluid.py:75, :106-109
    double dt = DD(DM(a.cfl, a.dx), rate);
    if (a.dt_max > 0.0) dt = fmin(dt, a.dt_max);
    dt = fmin(dt, DS(span, done));
    int dx_exp;
    const double dtdx = frexp(a.dx, &dx_exp) == 0.5 ? DM(dt, DD(1.0, a.dx)) : DD(dt, a.dx);  // exact either way
    ++step;
    double nv[kMaxCellsPerThread][5];
    int bad = 0;
#pragma unroll
    for (int k = 0; k < kMaxCellsPerThread; ++k) {
      const int i = threadIdx.x + k * blockDim.x;
      if (i >= nx) break;
      const St c = load_state(V, nx, i);
      const St l = ghost_state(V, nx, i - 1, a.periodic);
      const St r = ghost_state(V, nx, i + 1, a.periodic);
      double HL[5], HR[5];
      rusanov(l, c, HL);
      rusanov(c, r, HR);
      double* w = nv[k];
#pragma unroll
      for (int q = 0; q < 5; ++q) w[q] = DS(c.v[q], DM(dtdx, DS(HR[q], HL[q])));
      if (a.force != nullptr) {  // ref/fluid.py:113-115 (old state)
        const double E = a.force[i];
        w[1] = DA(w[1], DM(DM(dt, c.v[0]), E));
        w[4] = DA(w[4], DM(DM(dt, c.v[1]), E));
      }
      bool fin = true;
#pragma unroll
      for (int q = 0; q < 5; ++q) fin = fin && isfinite(w[q]);
      if (!fin) bad |= 1;
      else if (w[0] <= 0.0 || press(w[0], w[1], w[2], w[3], w[4]) <= 0.0) bad |= 2;
    }
    if (bad) atomicOr(flag, bad);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kMaxCellsPerThread; ++k) {
      const int i = threadIdx.x + k * blockDim.x;
      if (i >= nx) break;
#pragma unroll
      for (int q = 0; q < 5; ++q) V[q * nx + i] = nv[k][q];
    }
    __syncthreads();
    const int f = *flag;
    // ref/fluid.py:117-122: the finiteness guard is tested first
    if (f) return (step << 8) | (unsigned long long)((f & 1) ? kErrNonFinite : kErrUnphysical);
    done = DA(done, dt);
  }
  return 0;
}

// g_advance with each cell's wave speed and Euler flux evaluated once per step
// into shared memory (S[nx], Hf[5][nx] after V): the faces then need no
// division.  Every value is the same function of the same cell state as in
// g_advance (rusanov() recomputes them per face), so the result is bitwise
// identical; needs 11 nx doubles of shared memory (a.fastg).
__device__ ErrKey g_advance_fast(double* V, double* red, int* flag, const FluidArgs& a,
                                 double span) {
  const int nx = a.nx;
  double* S = V + 5 * nx;
  double* Hf = S + nx;
  const double guard = 1e-12;  // ref/fluid.py:30
  int dx_exp;
  const bool pow2 = frexp(a.dx, &dx_exp) == 0.5;
  double done = 0.0;
  unsigned long long step = 0;
  while (DS(span, done) > DM(guard, span)) {
    double rate = 0.0;
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
      const St c = load_state(V, nx, i);
      const double w = wave(c);
      double h[5];
      eflux(c, h);
      S[i] = w;
#pragma unroll
      for (int q = 0; q < 5; ++q) Hf[q * nx + i] = h[q];
      rate = fmax(rate, w);
    }
    rate = block_max(rate, red);  // its barriers also publish S and Hf
    double dt = DD(DM(a.cfl, a.dx), rate);
    if (a.dt_max > 0.0) dt = fmin(dt, a.dt_max);
    dt = fmin(dt, DS(span, done));
    const double dtdx = pow2 ? DM(dt, DD(1.0, a.dx)) : DD(dt, a.dx);  // exact either way
    ++step;
    double nv[kMaxCellsPerThread][5];
    int bad = 0;
#pragma unroll
    for (int k = 0; k < kMaxCellsPerThread; ++k) {
      const int i = threadIdx.x + k * blockDim.x;
      if (i >= nx) break;
      const int il = i > 0 ? i - 1 : (a.periodic ? nx - 1 : 0);
      const int ir = i < nx - 1 ? i + 1 : (a.periodic ? 0 : nx - 1);
      const St c = load_state(V, nx, i);
      const St l = load_state(V, nx, il);
      const St r = load_state(V, nx, ir);
      const double hsl = DM(0.5, fmax(S[il], S[i])), hsr = DM(0.5, fmax(S[i], S[ir]));
      double* w = nv[k];
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const double hc = Hf[q * nx + i];
        const double HL = DS(DM(0.5, DA(Hf[q * nx + il], hc)), DM(hsl, DS(c.v[q], l.v[q])));
        const double HR = DS(DM(0.5, DA(hc, Hf[q * nx + ir])), DM(hsr, DS(r.v[q], c.v[q])));
        w[q] = DS(c.v[q], DM(dtdx, DS(HR, HL)));
      }
      if (a.force != nullptr) {  // ref/fluid.py:113-115 (old state)
        const double E = a.force[i];
        w[1] = DA(w[1], DM(DM(dt, c.v[0]), E));
        w[4] = DA(w[4], DM(DM(dt, c.v[1]), E));
      }
      bool fin = true;
#pragma unroll
      for (int q = 0; q < 5; ++q) fin = fin && isfinite(w[q]);
      if (!fin) bad |= 1;
      else if (w[0] <= 0.0 || press(w[0], w[1], w[2], w[3], w[4]) <= 0.0) bad |= 2;
    }
    if (bad) atomicOr(flag, bad);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kMaxCellsPerThread; ++k) {
      const int i = threadIdx.x + k * blockDim.x;
      if (i >= nx) break;
#pragma unroll
      for (int q = 0; q < 5; ++q) V[q * nx + i] = nv[k][q];
    }
    __syncthreads();
    const int f = *flag;
    if (f) return (step << 8) | (unsigned long long)((f & 1) ? kErrNonFinite : kErrUnphysical);
    done = DA(done, dt);
  }
  return 0;
}

// Drift-diffusion G (extension; oracle/bgk.py dd_propagate, same operation
// order): rho only, held in V[0..nx).  Conservative central fluxes
//   J_{i+1/2} = (rho_{i+1} - rho_i)/dx - 0.5 (E_i rho_i + E_{i+1} rho_{i+1}),
//   rho_i += (dt D / dx) (J_{i+1/2} - J_{i-1/2}),
// dt = min(cfl dx^2 / (D (2 + dx e_max)), dt_max, remaining).  Ghosts: periodic
// wrap, else zero-gradient copies of rho and E.
__device__ ErrKey g_advance_dd(double* V, double* red, int* flag, const FluidArgs& a, double span) {
  const int nx = a.nx;
  const double guard = 1e-12;
  double em = 0.0;
  if (a.force != nullptr) {
    for (int i = threadIdx.x; i < nx; i += blockDim.x) em = fmax(em, fabs(a.force[i]));
    em = block_max(em, red);
  }
  double cap = DD(DM(DM(a.cfl, a.dx), a.dx), DM(a.diff, DA(2.0, DM(a.dx, em))));
  if (a.dt_max > 0.0) cap = fmin(cap, a.dt_max);
  auto E = [&](int i) { return a.force != nullptr ? a.force[i] : 0.0; };
  // x / dx is exactly x * (1 / dx) when dx is a power of two (every config
  // here: x in [0, 1] on 2^k cells): the fp64 divisions leave the critical path
  int dx_exp;
  const bool pow2 = frexp(a.dx, &dx_exp) == 0.5;
  const double rdx = pow2 ? DD(1.0, a.dx) : 0.0;
  auto over_dx = [&](double x) { return pow2 ? DM(x, rdx) : DD(x, a.dx); };
  // the field at each cell and its neighbours is constant over the window
  double eC[kMaxCellsPerThread], eL[kMaxCellsPerThread], eR[kMaxCellsPerThread];
#pragma unroll
  for (int k = 0; k < kMaxCellsPerThread; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    const int ii = i < nx ? i : nx - 1;
    const int il = ii > 0 ? ii - 1 : (a.periodic ? nx - 1 : 0);
    const int ir = ii < nx - 1 ? ii + 1 : (a.periodic ? 0 : nx - 1);
    eC[k] = E(ii);
    eL[k] = E(il);
    eR[k] = E(ir);
  }
  double done = 0.0;
  unsigned long long step = 0;
  while (DS(span, done) > DM(guard, span)) {
    const double dt = fmin(cap, DS(span, done));
    const double coef = over_dx(DM(dt, a.diff));
    ++step;
    // ping-pong between V[0..nx) and V[nx..2nx): one barrier per step
    const double* Vin = V + ((step - 1) & 1) * nx;
    double* Vout = V + (step & 1) * nx;
    int bad = 0;
#pragma unroll
    for (int k = 0; k < kMaxCellsPerThread; ++k) {
      const int i = threadIdx.x + k * blockDim.x;
      if (i >= nx) break;
      const int il = i > 0 ? i - 1 : (a.periodic ? nx - 1 : 0);
      const int ir = i < nx - 1 ? i + 1 : (a.periodic ? 0 : nx - 1);
      const double gi = Vin[i], gl = Vin[il], gr = Vin[ir];
      const double ei = eC[k], el = eL[k], er = eR[k];
      const double JR = DS(over_dx(DS(gr, gi)), DM(0.5, DA(DM(ei, gi), DM(er, gr))));
      const double JL = DS(over_dx(DS(gi, gl)), DM(0.5, DA(DM(el, gl), DM(ei, gi))));
      const double v = DA(gi, DM(coef, DS(JR, JL)));
      Vout[i] = v;
      if (!isfinite(v)) bad |= 1;
      else if (v <= 0.0) bad |= 2;
    }
    if (bad) atomicOr(flag, bad);
    __syncthreads();
    const int f = *flag;
    if (f) return (step << 8) | (unsigned long long)((f & 1) ? kErrNonFinite : kErrUnphysical);
    done = DA(done, dt);
  }
  if (step & 1) {  // the state ended in V[nx..2nx)
    for (int i = threadIdx.x; i < nx; i += blockDim.x) V[i] = V[nx + i];
    __syncthreads();
  }
  return 0;
}

// Loads window state into smem V: conserved variables (Euler) or rho (DD).
__device__ __forceinline__ void load_window(const FluidArgs& a, const double* src, double* V) {
  const int nx = a.nx;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) {
    if (a.model == 1) {
      V[i] = src[i];
      continue;
    }
    double v[5];
    to_cons(src[i], src[nx + i], src[2 * nx + i], src[3 * nx + i], src[4 * nx + i], v);
#pragma unroll
    for (int q = 0; q < 5; ++q) V[q * nx + i] = v[q];
  }
}

__device__ __forceinline__ ErrKey advance(double* V, double* red, int* flag, const FluidArgs& a,
                                          double span) {
  if (a.model == 1) return g_advance_dd(V, red, flag, a, span);
  return a.fastg ? g_advance_fast(V, red, flag, a, span) : g_advance(V, red, flag, a, span);
}

// conserved -> primitive (ref/moments.py:122-129); returns false if degenerate.
// Drift-diffusion: (rho, 0, 0, 0, 1), never degenerate (rho > 0 is checked per step).
__device__ bool to_prim(const FluidArgs& a, const double* V, int nx, int i, double out[5]) {
  if (a.model == 1) {
    out[0] = V[i];
    out[1] = 0.0;
    out[2] = 0.0;
    out[3] = 0.0;
    out[4] = 1.0;
    return true;
  }
  const double rho = V[i], m0 = V[nx + i], m1 = V[2 * nx + i], m2 = V[3 * nx + i],
               en = V[4 * nx + i];
  const double u0 = DD(m0, rho), u1 = DD(m1, rho), u2 = DD(m2, rho);
  const double mu = DA(DA(DM(m0, u0), DM(m2, u2)), DM(m1, u1));
  const double eint = DS(en, DM(0.5, mu));
  out[0] = rho;
  out[1] = u0;
  out[2] = u1;
  out[3] = u2;
  out[4] = DD(eint, DM(1.5, rho));
  return !(rho <= 0.0) && !(eint <= 0.0);
}

// Batched independent G solves: blockIdx.x = window.  out = minuend - G(in)
// when minuend != null (the parareal jump, ref/parareal.py:142).
template <int M>
__global__ void __launch_bounds__(1024) fluid_batch_kernel(FluidArgs a0, const double* in, double* out,
                                                           const double* minuend, const double* t0,
                                                           const double* t1) {
  FluidArgs a = a0;
  a.model = M;  // compile-time model: each variant carries only its own G

  extern __shared__ double V[];
  __shared__ double red[32];
  __shared__ int flag;
  const int w = blockIdx.x, nx = a.nx;
  const double* src = in + (size_t)w * 5 * nx;
  if (threadIdx.x == 0) flag = 0;
  load_window(a, src, V);
  __syncthreads();
  const double span = DS(t1[w], t0[w]);
  double* dst = out + (size_t)w * 5 * nx;
  const double* mn = minuend ? minuend + (size_t)w * 5 * nx : nullptr;
  if (span == 0.0) {  // ref/fluid.py:98-99: the input itself (DD: rho, 0, 1)
    for (int i = threadIdx.x; i < 5 * nx; i += blockDim.x) {
      double v = src[i];
      if (a.model == 1 && i >= nx) v = (i >= 4 * nx) ? 1.0 : 0.0;
      dst[i] = mn ? DS(mn[i], v) : v;
    }
    return;
  }
  const ErrKey code = advance(V, red, &flag, a, span);
  if (code) {
    if (threadIdx.x == 0) atomicMin(a.err, ((ErrKey)w << 40) | code);
    return;
  }
  bool ok = true;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) {
    double p[5];
    ok = to_prim(a, V, nx, i, p) && ok;
#pragma unroll
    for (int q = 0; q < 5; ++q) dst[q * nx + i] = mn ? DS(mn[q * nx + i], p[q]) : p[q];
  }
  if (!ok) atomicMin(a.err, err_key(w, 0, kErrLiftState));
}

// Sequential correction sweep (one CTA): U_n = G(U_{n-1}) + jump_n for
// n = start..last, overshoot guard, sup error (ref/parareal.py:226-248).
// The error is max-accumulated into *err_out (non-negative doubles order as
// their bit patterns), so a sweep split into consecutive ranges gives the
// same value as one launch.
template <int M>
__global__ void __launch_bounds__(1024) correct_kernel(FluidArgs a0, int last, int start, double* snaps,
                                                       const double* old, const double* jumps,
                                                       const double* times, double* err_out) {
  FluidArgs a = a0;
  a.model = M;

  extern __shared__ double V[];
  __shared__ double red[32];
  __shared__ int flag;
  __shared__ int over;
  const int nx = a.nx;
  double emax = 0.0;
  if (threadIdx.x == 0) {
    flag = 0;
    over = 0;
  }
  __syncthreads();
  for (int n = start; n <= last; ++n) {
    const double* src = snaps + (size_t)(n - 1) * 5 * nx;
    load_window(a, src, V);
    __syncthreads();
    const double span = DS(times[n], times[n - 1]);
    double* dst = snaps + (size_t)n * 5 * nx;
    const double* jp = jumps + (size_t)(n - 1) * 5 * nx;
    const double* od = old + (size_t)n * 5 * nx;
    ErrKey code = 0;
    if (span != 0.0) code = advance(V, red, &flag, a, span);
    if (code) {
      if (threadIdx.x == 0) atomicMin(a.err, ((ErrKey)n << 40) | code);
      return;
    }
    bool bad = false;
    bool degen = false;
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
      double p[5];
      if (span != 0.0) {
        if (!to_prim(a, V, nx, i, p)) degen = true;
      } else {
#pragma unroll
        for (int q = 0; q < 5; ++q) p[q] = src[q * nx + i];
        if (a.model == 1) {
          p[1] = p[2] = p[3] = 0.0;
          p[4] = 1.0;
        }
      }
      double c[5];
#pragma unroll
      for (int q = 0; q < 5; ++q) c[q] = DA(p[q], jp[q * nx + i]);
      bool fin = true;
#pragma unroll
      for (int q = 0; q < 5; ++q) fin = fin && isfinite(c[q]);
      if (!fin || c[0] <= 0.0 || c[4] <= 0.0) bad = true;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        emax = fmax(emax, fabs(DS(c[q], od[q * nx + i])));
        dst[q * nx + i] = c[q];
      }
    }
    if (bad) atomicOr(&over, 1);
    if (degen) atomicOr(&over, 2);
    __syncthreads();
    if (over) {
      // a degenerate G result raises inside propagate_fluid, before the guard
      if (threadIdx.x == 0)
        atomicMin(a.err, err_key(n, 0, (over & 2) ? kErrLiftState : kErrOvershoot));
      return;
    }
  }
  emax = block_max(emax, red);
  if (threadIdx.x == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(err_out),
              (unsigned long long)__double_as_longlong(emax));
}

// Threads of a G CTA: one per cell up to 1024; `lean` (side-stream launches
// that must fit next to a sweep CTA): the fewest covering nx at
// kMaxCellsPerThread cells each.
static int fluid_threads(int nx, bool lean = false) {
  int t = 32;
  const int need = lean ? (nx + kMaxCellsPerThread - 1) / kMaxCellsPerThread : nx;
  while (t < need && t < 1024) t <<= 1;
  return t;
}

cudaError_t launch_fluid_batch(const FluidArgs& a, int nwin, const double* in, double* out,
                               const double* minuend, const double* t0, const double* t1,
                               cudaStream_t st, bool lean) {
  const int thr = fluid_threads(a.nx, lean);
  if ((size_t)thr * kMaxCellsPerThread < (size_t)a.nx) return cudaErrorInvalidValue;
  FluidArgs b = a;
  // Euler G: per-cell wave speeds / fluxes in shared memory when they fit
  b.fastg = (a.model == 0 && (size_t)11 * a.nx * sizeof(double) <= 220 * 1024) ? 1 : 0;
  const size_t smem = (size_t)(b.fastg ? 11 : 5) * a.nx * sizeof(double);
  auto k = a.model == 1 ? fluid_batch_kernel<1> : fluid_batch_kernel<0>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<nwin, thr, smem, st>>>(b, in, out, minuend, t0, t1);
  return cudaGetLastError();
}

cudaError_t launch_correct(const FluidArgs& a, int last, int start, double* snaps, const double* old,
                           const double* jumps, const double* times, double* err_out,
                           cudaStream_t st, bool lean) {
  const int thr = fluid_threads(a.nx, lean);
  if ((size_t)thr * kMaxCellsPerThread < (size_t)a.nx) return cudaErrorInvalidValue;
  FluidArgs b = a;
  // Euler G: per-cell wave speeds / fluxes in shared memory when they fit
  b.fastg = (a.model == 0 && (size_t)11 * a.nx * sizeof(double) <= 220 * 1024) ? 1 : 0;
  const size_t smem = (size_t)(b.fastg ? 11 : 5) * a.nx * sizeof(double);
  cudaError_t e =
      cudaFuncSetAttribute(a.model == 1 ? correct_kernel<1> : correct_kernel<0>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.model == 1)
    correct_kernel<1><<<1, thr, smem, st>>>(b, last, start, snaps, old, jumps, times, err_out);
  else
    correct_kernel<0><<<1, thr, smem, st>>>(b, last, start, snaps, old, jumps, times, err_out);
  return cudaGetLastError();
}

}  // namespace pbgk
