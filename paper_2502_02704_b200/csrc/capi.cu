// extern "C" boundary of libpbgk.so (declared in include/pbgk.h).
//
// Host orchestration of the fine propagator: context (grid constants, tiling,
// device workspace, TMA descriptors), the skewed sweep/finalize sequence of
// propagate_kinetic, and the single-GPU coarse solver / correction launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pbgk.h"
#include "common.cuh"

namespace pbgk {
cudaError_t launch_sweep(int cfg_id, const CUtensorMap& map, const SweepArgs& a, bool synth,
                         bool field, int grid, int ns, size_t smem, cudaStream_t st);
size_t sweep_smem_bytes(const SweepArgs& a, int V, int LZ, int NTHR, bool synth, bool tma, int ns);
cudaError_t launch_finalize(const FinalArgs& a, cudaStream_t st);
cudaError_t launch_fsweep(int cfg_id, const CUtensorMap& map, const FSweepArgs& a, bool synth, int L,
                          int grid, int ns, size_t smem, cudaStream_t st);
size_t fsweep_smem_bytes(const FSweepArgs& a, int V, int LZ, bool synth, int L, int ns);
bool fsweep_has_cfg(int cfg_id);
int fsweep_ctas_per_sm(int L);
cudaError_t launch_msweep(int L, int mode, const CUtensorMap& map, const MSweepArgs& a, int grid_x, int nwin,
                          int ns, size_t smem, cudaStream_t st);
cudaError_t launch_finalize_batch(const FinalArgs& a, const FinalBatch& b, int nwin, cudaStream_t st);
size_t msweep_smem_bytes(int L, int mode, int nvx, int ns, bool pre);
cudaError_t launch_ms_prep(const double* T, long long t_ws, long long tstep, int TL, int gxo, const double* cx,
                           const double* dts, int dts_g, double dx, int S, int nx, int nvx, int lift0,
                           double* trip, long long trip_ws, int nwin, cudaStream_t st);
int msweep_ctas_per_sm();
int msweep_tiling(int nvx, int nvy, int nvz, Tiling* t);
int esweep_levels(int nvx, int nvz);
size_t esweep_smem_bytes(int nvx, bool fin);
void esweep_tiling(int nvx, int nvy, int nvz, Tiling* t);
int esweep_ctas_per_sm(int nvx);
cudaError_t launch_esweep(const ESweepArgs& a, bool synth, int grid, size_t smem, cudaStream_t st);
cudaError_t launch_marg(const MargArgs& m, const FinalArgs& f, double* gsum, int s, int nwin,
                        cudaStream_t st);
size_t marg_state_doubles(int nvx);
cudaError_t launch_q_from_f(const MargArgs& m, const double* f, cudaStream_t st);
cudaError_t launch_marg_all(const MargArgs& m0, const FinalArgs& f, const double* q0, double* qa,
                            double* qb, double* gsum, long long t_step, int S, int nwin,
                            unsigned* bar, cudaStream_t st, unsigned* prog, unsigned prog_base,
                            int max_ctas);
void marg_all_shape(int nx, int nvx, int nvy, int nvz, int TL, bool trap, int nwin, int* ctas,
                    int* per_sm);
size_t marg_smem_bytes(int nvx, int nvy, int nvz, int TL);
cudaError_t launch_set_key(ErrKey* p, ErrKey v, cudaStream_t st);
cudaError_t launch_fluid_batch(const FluidArgs& a, int nwin, const double* in, double* out,
                               const double* minuend, const double* t0, const double* t1,
                               cudaStream_t st, bool lean = false);
cudaError_t launch_correct(const FluidArgs& a, int last, int start, double* snaps, const double* old,
                           const double* jumps, const double* times, double* err_out,
                           cudaStream_t st, bool lean = false);
}  // namespace pbgk

using namespace pbgk;

namespace {

thread_local std::string g_last_error;

int fail(const std::string& msg) {
  g_last_error = msg;
  return -1;
}

#define CK(expr)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(std::string(#expr) + ": " + cudaGetErrorString(e_));            \
  } while (0)

// device buffer of at least n elements (grown, never shrunk)
template <typename T>
int ensure_dev(T*& p, size_t& cap, size_t n, cudaStream_t st) {
  if (n <= cap) return 0;
  if (p) {
    CK(cudaStreamSynchronize(st));
    CK(cudaFree(p));
    p = nullptr;
    cap = 0;
  }
  CK(cudaMalloc(&p, n * sizeof(T)));
  cap = n;
  return 0;
}

// bytes of per-step relax tables the multi-step path may hold (a group of
// batched windows, or one long propagation)
// Default: a quarter of the device memory free at first use, between 2 and
// 16 GiB (config 3b's windows carry 2 GB of tables each: at 2 GiB their
// recursions ran one window at a time, 16 % of an iteration; at 16 GiB 8 %).
double default_batch_budget() {
  static const double b = [] {
    if (getenv("PBGK_BATCH_BYTES")) return atof(getenv("PBGK_BATCH_BYTES"));
    size_t free_b = 0, total_b = 0;
    const double gib = 1073741824.0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return 2.0 * gib;
    return std::min(16.0 * gib, std::max(2.0 * gib, 0.25 * (double)free_b));
  }();
  return b;
}

// compile-time tile shapes of sweep.cu (index = cfg id)
struct CfgShape {
  int V, LZ, K, NTHR;
  bool tma;
  int minb;  // CTAs per SM the launch bounds target
};
const CfgShape kCfg[] = {
    // first-order upwind (and the v_x field term), 4 lines per thread
    {2, 32, 4, 256, true, 2},   // 0: nvz % 64 == 0, full 512-byte v_z rows per box line
    {3, 16, 4, 256, true, 2},   // 1: nvz % 48 == 0
    {2, 16, 4, 256, true, 2},   // 2: nvz % 32 == 0
    {2, 8, 4, 256, true, 2},    // 3: nvz % 16 == 0
    {2, 4, 4, 256, true, 2},    // 4: nvz % 8 == 0
    {1, 32, 4, 256, false, 2},  // 5: anything (no TMA; also MUSCL)
    // MUSCL: three planes of per-line state; one CTA per SM, 255 registers
    {2, 32, 4, 256, true, 1},   // 6: nvz % 64 == 0 (measured slower than cfg 0; unused)
    {3, 16, 4, 256, true, 1},   // 7: nvz % 48 == 0
    {2, 16, 4, 256, true, 1},   // 8: nvz % 32 == 0
    {2, 8, 4, 256, true, 1},    // 9: nvz % 16 == 0
    {2, 4, 4, 256, true, 1},    // 10: nvz % 8 == 0
    {6, 8, 2, 256, true, 2},    // 11: nvz % 48 == 0, 48 contiguous bytes per lane (plain sweep)
};


struct Plan {
  int cfg;
  Tiling t;
  int grid;
  int ns;
  int per_sm;  // resident CTAs per SM the grid was sized for
};

struct MapEntry {
  const void* ptr;
  int rows_load, By, Bz, planes;
  CUtensorMap map;
};

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace

struct EvPair {
  cudaEvent_t a, b;
  int kind;  // 0 sweep, 1 finalize, 2 multi-step sweep, 3 marginal recursion step
  double bytes;
  int steps;
};

struct pbgk_ctx {
  int g_model = 0;       // coarse G: 0 Euler (reference), 1 drift-diffusion (extension)
  int x_scheme = 0;      // 0 first-order upwind (reference), 1 MUSCL-minmod (extension)
  int l2_keep = 0;       // f ping-pong small enough to live in L2 (sweep cache policies)
  int quad = 0;          // velocity quadrature: 0 midpoint (reference), 1 trapezoidal (extension)
  int slot_reserve = 0;  // CTA slots the sweep grid leaves free (pipelined parareal side stream)
  double g_diff = 1.0;   // drift-diffusion D
  pbgk_grid_desc g;
  bool prof = false;
  std::vector<EvPair> ev_pool, ev_used;
  double dx, dv[3], dvol;
  int dev, nsm;
  size_t smem_optin, smem_per_sm;
  double* d_c[3] = {nullptr, nullptr, nullptr};
  Plan plan[4];  // [0] upwind, [1] upwind + v_x field term, [2] MUSCL, [3] multi-step sweep
  int TL, gxo, gyo, gzo;
  double* d_part = nullptr;
  size_t part_elems = 0;
  double* d_tab[2] = {nullptr, nullptr};
  double* d_scratch = nullptr;  // 5*nx moments / small host-visible staging
  ErrKey* d_err = nullptr;
  ErrKey* err_slot = nullptr;   // where sweeps / finalizes record failures (d_err, or a window's slot)
  ErrKey* d_keys = nullptr;     // pbgk_propagate_windows: one failure key per window
  ErrKey* h_keys = nullptr;
  int keys_cap = 0;
  ErrKey* h_err = nullptr;  // pinned
  double* h_dbl = nullptr;  // pinned small
  double* d_times = nullptr;
  double* d_times2 = nullptr;             // coarse times of the correction sweep
  size_t times2_cap = 0;
  // host copies of what the small per-call upload buffers hold: an unchanged
  // upload (the same schedule / time grid in every parareal iteration) is skipped
  std::vector<double> sh_times, sh_times2, sh_bdts;
  std::vector<int> sh_bnst;
  size_t times_cap = 0;
  std::vector<MapEntry> maps;
  size_t ws_bytes = 0;
  // multi-step path (fsweep.cu + marginal.cu): levels per pass (0 = off,
  // -1 = the per-shape default of fuse_levels); Q of a given f0
  int fuse = -1;
  int one_step = 0;  // force the one-step path (exact re-run after a kind-6 status)
  double* d_q0 = nullptr;
  // the recursion's per-(window, step) tables, per-window state ping-pong,
  // G sums, per-step dt and step counts (multi-step path)
  double* d_bt = nullptr;
  double* d_bq = nullptr;
  double* d_bg = nullptr;
  double* d_bdts = nullptr;
  int* d_bnst = nullptr;
  size_t bt_cap = 0, bq_cap = 0, bg_cap = 0, bdts_cap = 0, bnst_cap = 0;
  unsigned* d_gbar = nullptr;  // grid barrier of the one-launch recursion
  // concurrent recursion of single propagations: side stream, events, the
  // device progress word (monotonic: each propagation takes a fresh base)
  cudaStream_t st_side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
  unsigned* d_prog = nullptr;
  unsigned prog_next = 1;
  int rec_reserve = 0;  // SMs the passes leave to a concurrent recursion (0: serial)
  int no_concurrent = 0;  // serial recursion (re-run after a pass gave up waiting, status kind 5)
  // round-2 multi-step sweep (msweep.cu): on/off (pbgk_set_msweep), levels
  // per pass (0 = auto: 8), its tilings for K = 1 / 2 lines per thread (NT =
  // 0: the velocity grid does not tile) and its partial records (the
  // window's final projection)
  int ms = 1;
  int ms_levels = 0;
  double batch_bytes = 0.0;  // table budget of the multi-step path (0: the default)
  Tiling ms_t = {};
  double* d_fb[2] = {nullptr, nullptr};  // f of a batch of windows (ms_windows_batched)
  size_t fb_cap[2] = {0, 0};
  double* d_mpart = nullptr;
  size_t mpart_cap = 0;
  double* d_trip = nullptr;  // per-row factors of a window's steps (ms_prep_kernel)
  size_t trip_cap = 0;
  // multi-step passes with the v_x field term (esweep.cu): on/off
  // (pbgk_set_esweep), CTAs per SM of its build for this nvx (0: unknown yet)
  int es = 1;
  int es_per_sm = 0;
};

namespace {

std::atomic<long long> g_launches{0};

// bytes of per-step relax tables the multi-step path may hold (a group of
// batched windows, or one long propagation): the context's setting, else
// PBGK_BATCH_BYTES, else a quarter of the free device memory within 2..16 GiB
double batch_budget(const pbgk_ctx* c) { return c->batch_bytes > 0.0 ? c->batch_bytes : default_batch_budget(); }

// CUDA-event bracket around one launch when profiling is on.
struct ProfScope {
  pbgk_ctx* c;
  cudaStream_t st;
  EvPair* ev = nullptr;
  ProfScope(pbgk_ctx* c_, cudaStream_t st_, int kind, double bytes, int steps = 1) : c(c_), st(st_) {
    ++g_launches;
    if (!c->prof) return;
    if (c->ev_pool.empty()) {
      EvPair p;
      cudaEventCreate(&p.a);
      cudaEventCreate(&p.b);
      c->ev_pool.push_back(p);
    }
    c->ev_used.push_back(c->ev_pool.back());
    c->ev_pool.pop_back();
    ev = &c->ev_used.back();
    ev->kind = kind;
    ev->bytes = bytes;
    ev->steps = steps;
    cudaEventRecord(ev->a, st);
  }
  ~ProfScope() {
    if (ev) cudaEventRecord(ev->b, st);
  }
};

// Tile choice for one configuration of the sweep.
bool make_plan(pbgk_ctx* c, bool field, bool muscl, Plan& out, int only = -1) {
  const int nvx = c->g.nvx, nvy = c->g.nvy, nvz = c->g.nvz;
  const int nneg = nvx / 2;  // centres (j - (n-1)/2) dv are < 0 exactly for j < n/2
  const int npos = nvx - nneg;
  // tile shapes in measured order of preference (cfg ids of sweep.cu)
  std::vector<int> cands;
  const bool even = (nvz % 2 == 0);
  // MUSCL (measured, round 1): 64-wide rows keep 2 CTAs/SM (cfg 0, K=4 with a
  // few spilled registers); the other shapes prefer 1 CTA/SM with 255 registers
  const int* ids = nullptr;
  // 48-wide rows: V = 6 lanes (48 contiguous bytes, 16-byte stores) for the
  // plain sweep (+14% over V = 3 interleaved); the field term keeps V = 3
  static const int upw[5] = {0, 11, 2, 3, 4}, fld[5] = {0, 1, 2, 3, 4}, mus[5] = {0, 7, 8, 9, 10};
  ids = muscl ? mus : (field ? fld : upw);
  if (even && nvz % 64 == 0) cands.push_back(ids[0]);
  else if (even && nvz % 48 == 0) cands.push_back(ids[1]);
  else if (even && nvz % 32 == 0) cands.push_back(ids[2]);
  else if (even && nvz % 16 == 0) cands.push_back(ids[3]);
  else if (even && nvz % 8 == 0) cands.push_back(ids[4]);
  cands.push_back(5);
  if (const char* force = getenv("PBGK_FORCE_CFG")) {  // development knob
    cands.assign(1, atoi(force));
  }
  if (only >= 0) cands.assign(1, only);
  if (const char* force = getenv("PBGK_FORCE_FIELD_CFG"))  // development knob
    if (field) cands.assign(1, atoi(force));
  double best = 1e300;
  bool found = false;
  for (int id : cands) {
    const CfgShape& s = kCfg[id];
    const int Bz = s.V * s.LZ;
    const int lines = s.K * (s.NTHR / s.LZ);
    for (int A = 1; A <= lines; A *= 2) {
      if (A > std::max(nneg, npos) && A > 1) break;
      int By = lines / A;
      while (By > nvy && By > 1) By >>= 1;  // power of two (the kernel shifts by log2 By)
      if (By < 1 || By > 256 || A + (field ? 2 : 0) > 256) continue;
      if (A + By + Bz > s.NTHR) continue;
      if (const char* fa = getenv("PBGK_FORCE_A")) {  // development knob
        if (A != atoi(fa)) continue;
      } else if (field && A > 8) {
        continue;  // field term: <= 8 rows per box (measured: 64^3 A=8 +7 % over A=32)
      } else if (!field && s.V == 6 && A > 4) {
        continue;  // 48-wide V = 6 boxes: 4 x 16 lines (measured +3.5 % over 8 x 8)
      }
      Tiling t;
      t.A = A;
      t.By = By;
      t.Bz = Bz;
      t.rows_load = A + (field ? 2 : 0);
      t.nneg = nneg;
      t.ntn = (nneg + A - 1) / A;
      t.ntp = (npos + A - 1) / A;
      t.nty = (nvy + By - 1) / By;
      t.ntz = (nvz + Bz - 1) / Bz;
      t.NT = (t.ntn + t.ntp) * t.nty * t.ntz;
      t.PS = (A + By + Bz + 1) & ~1;  // even: 16-B aligned records (bulk copies)
      // loaded elements per useful element, plus marginal-partial traffic
      const double loaded = (double)t.NT * t.rows_load * By * Bz;
      const double useful = (double)nvx * nvy * nvz;
      const double part = 2.0 * t.NT * t.PS;
      // shared memory for 2 stages at least
      SweepArgs dummy{};
      dummy.nvx = nvx;
      dummy.t = t;
      dummy.TL = c->TL;
      const size_t sm2 = sweep_smem_bytes(dummy, s.V, s.LZ, s.NTHR, false, s.tma, 2);
      if (sm2 > c->smem_optin) continue;
      // halo overhead: one extra plane per tile run per CTA segment
      const double items = (double)t.NT * c->g.nx;
      const double runs = std::min<double>(c->nsm, items) + t.NT;
      const double halo = runs / items;
      const double penalty = (s.tma ? 1.0 : 4.0);
      const double util = (double)(A * By) / lines;  // busy fraction of the thread lines
      const double score = penalty * ((loaded + part) / useful) * (1.0 + halo) * (1.5 - 0.5 * util) +
                           (id == 5 ? 100.0 : 0.0);
      if (score < best) {
        best = score;
        out.cfg = id;
        out.t = t;
        found = true;
      }
    }
  }
  if (!found) return false;
  const CfgShape& s = kCfg[out.cfg];
  SweepArgs dummy{};
  dummy.nvx = nvx;
  dummy.t = out.t;
  dummy.TL = c->TL;
  // two CTAs per SM when the ring fits in half the shared memory, else one
  const size_t half = (c->smem_per_sm / 2) - 2048;
  // ring depth (same-box A/B, round 1): 64-wide boxes 3 stages; 32-wide 4 for
  // the plain sweep, 3 with the field term; 48-wide (V = 6) and the narrow /
  // odd shapes 2
  int ns_max = (s.V == 2 && s.LZ == 32) ? 3 : ((s.V == 2 && s.LZ == 16) ? (field ? 3 : 4) : 2);
  if (const char* e = getenv("PBGK_NS")) ns_max = atoi(e);  // development knob
  int ns = ns_max;
  while (ns > 2 && sweep_smem_bytes(dummy, s.V, s.LZ, s.NTHR, false, s.tma, ns) > half) --ns;
  int per_sm = 2;
  if (s.minb == 1 || sweep_smem_bytes(dummy, s.V, s.LZ, s.NTHR, false, s.tma, ns) > half) {
    per_sm = 1;
    ns = ns_max;
    while (ns > 2 && sweep_smem_bytes(dummy, s.V, s.LZ, s.NTHR, false, s.tma, ns) > c->smem_optin) --ns;
  }
  out.ns = s.tma ? ns : 1;
  const long long items = (long long)out.t.NT * c->g.nx;
  long long grid = (long long)c->nsm * per_sm;
  if (grid > items) grid = items;
  out.grid = (int)std::max<long long>(grid, 1);
  out.per_sm = per_sm;
  return true;
}

// nplanes > 0: a batch of windows stacked along x (nx * windows planes)
const CUtensorMap* tensor_map(pbgk_ctx* c, const double* ptr, const Tiling& t, int cfg, int nplanes = 0) {
  static CUtensorMap dummy;
  if (!kCfg[cfg].tma || ptr == nullptr) return &dummy;
  const int planes = nplanes > 0 ? nplanes : c->g.nx + (c->g.bc == 3 ? 2 : 0);
  for (auto& m : c->maps)
    if (m.ptr == ptr && m.rows_load == t.rows_load && m.By == t.By && m.Bz == t.Bz && m.planes == planes)
      return &m.map;
  auto enc = get_encode();
  if (!enc) return nullptr;
  MapEntry e;
  e.ptr = ptr;
  e.rows_load = t.rows_load;
  e.By = t.By;
  e.Bz = t.Bz;
  e.planes = planes;
  // slab contexts (bc 3) address padded buffers: one halo plane per side
  const cuuint64_t dims[4] = {(cuuint64_t)c->g.nvz, (cuuint64_t)c->g.nvy, (cuuint64_t)c->g.nvx,
                              (cuuint64_t)planes};
  const cuuint64_t strides[3] = {(cuuint64_t)c->g.nvz * 8, (cuuint64_t)c->g.nvy * c->g.nvz * 8,
                                 (cuuint64_t)c->g.nvx * c->g.nvy * c->g.nvz * 8};
  const cuuint32_t box[4] = {(cuuint32_t)t.Bz, (cuuint32_t)t.By, (cuuint32_t)t.rows_load, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  // 128B: box rows can be as short as 128 bytes; 256B promotion would fetch the
  // neighbouring row of another tile (measured +50% DRAM reads)
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  if (const char* p = getenv("PBGK_L2PROMO")) {  // development knob
    const int v = atoi(p);
    promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                   : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                             : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                        : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
  CUresult r = enc(&e.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(ptr), dims,
                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    g_last_error = buf;
    return nullptr;
  }
  if (c->maps.size() > 64) c->maps.erase(c->maps.begin());
  c->maps.push_back(e);
  return &c->maps.back().map;
}

SweepArgs base_args(pbgk_ctx* c, const Plan& p) {
  SweepArgs a{};
  a.nx = c->g.nx;
  a.nvx = c->g.nvx;
  a.nvy = c->g.nvy;
  a.nvz = c->g.nvz;
  a.plane = (long long)c->g.nvx * c->g.nvy * c->g.nvz;
  a.t = p.t;
  a.total = (long long)p.t.NT * c->g.nx;
  a.tab = c->d_tab[0];
  a.TL = c->TL;
  a.gxo = c->gxo;
  a.gyo = c->gyo;
  a.gzo = c->gzo;
  a.cx = c->d_c[0];
  a.bc = c->g.bc;
  a.part = c->d_part;
  a.err = c->err_slot ? c->err_slot : c->d_err;
  static const int debug = getenv("PBGK_DEBUG") ? atoi(getenv("PBGK_DEBUG")) : 0;  // dev ablations
  a.debug = debug & ~2;  // bit 2 (no CTA barrier) was removed: it races the TMA ring
  return a;
}

FinalArgs fin_args(pbgk_ctx* c, const Plan& p) {
  FinalArgs f{};
  f.nx = c->g.nx;
  f.nvx = c->g.nvx;
  f.nvy = c->g.nvy;
  f.nvz = c->g.nvz;
  f.t = p.t;
  f.part = c->d_part;
  f.cx = c->d_c[0];
  f.cy = c->d_c[1];
  f.cz = c->d_c[2];
  f.dvol = c->dvol;
  f.TL = c->TL;
  f.gxo = c->gxo;
  f.gyo = c->gyo;
  f.gzo = c->gzo;
  f.err = c->err_slot ? c->err_slot : c->d_err;
  f.trap = c->quad;
  f.tau = 1.0;
  f.eps = 1.0;
  return f;
}

// One sweep over f (see sweep.cu).  `in` null => SYNTH from `tab`.
int run_sweep(pbgk_ctx* c, int pid, bool field, const double* in, const double* tab, double* out,
              double dtdx, const double* E, double half_emax, double dtdv, int check_step,
              cudaStream_t st, int noreduce = 0) {
  const Plan& p = c->plan[pid];
  const CfgShape& s = kCfg[p.cfg];
  SweepArgs a = base_args(c, p);
  a.fin = in;
  a.fout = out;
  a.tab = tab;
  a.dtdx = dtdx;
  a.E = field ? E : nullptr;
  a.half_emax = half_emax;
  a.dtdv = dtdv;
  a.check_step = check_step;
  a.muscl = (c->x_scheme == 1 && dtdx != 0.0) ? 1 : 0;
  a.l2_keep = c->l2_keep;
  a.trap = c->quad;
  a.noreduce = noreduce;
  a.out_step = check_step;
  if (a.muscl && field) return fail("MUSCL x transport has no v_x field term (use the upwind scheme)");
  const bool synth = (in == nullptr);
  const CUtensorMap* map = tensor_map(c, synth ? nullptr : in, p.t, p.cfg);
  if (!map) return fail("tensor map: " + g_last_error);
  const size_t smem = sweep_smem_bytes(a, s.V, s.LZ, s.NTHR, synth, s.tma, p.ns);
  const double fbytes = 8.0 * (double)a.plane * a.nx;
  ProfScope ps(c, st, 0, (synth ? 0.0 : fbytes) + (out ? fbytes : 0.0));
  // persistent grid, minus the CTA slots left to side-stream work
  int grid = p.grid;
  if (c->slot_reserve > 0) grid = std::max(1, std::min(grid, c->nsm * p.per_sm - c->slot_reserve));
  CK(launch_sweep(p.cfg, *map, a, synth, field, grid, p.ns, smem, st));
  return 0;
}

int run_final(pbgk_ctx* c, int pid, int mode, const double* mom_in, double* mom_out,
              double* tab, double dt, double eps, double tau, const double* tau_cells, int step,
              cudaStream_t st, int check_finite = 0) {
  FinalArgs f = fin_args(c, c->plan[pid]);
  f.check_finite = check_finite;
  f.mode = mode;
  f.mom_in = mom_in;
  f.mom_out = mom_out;
  f.tab = tab;
  f.dt = dt;
  f.eps = eps;
  f.tau = tau;
  f.tau_arr = tau_cells;
  f.step = step;
  ProfScope ps(c, st, 1, 0.0);
  CK(launch_finalize(f, st));
  return 0;
}

int reset_err(pbgk_ctx* c, cudaStream_t st) {
  ++g_launches;
  CK(launch_set_key(c->d_err, kNoError, st));
  return 0;
}

int fetch_err(pbgk_ctx* c, cudaStream_t st, long long* code) {
  if (!code) return 0;
  CK(cudaMemcpyAsync(c->h_err, c->d_err, sizeof(ErrKey), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *code = (*c->h_err == kNoError) ? -1 : (long long)*c->h_err;
  return 0;
}

}  // namespace

extern "C" {

int pbgk_version(void) { return 1; }

const char* pbgk_last_error(void) { return g_last_error.c_str(); }

int pbgk_ctx_create(const pbgk_grid_desc* g, pbgk_ctx** out) {
  if (!g || !out) return fail("null argument");
  if (g->nx < 1 || g->nvx < 1 || g->nvy < 1 || g->nvz < 1) return fail("bad grid sizes");
  if (g->nvx > 4096 || g->nvy > 4096 || g->nvz > 4096) return fail("velocity axis too long");
  if (g->bc < 0 || g->bc > 3) return fail("bc must be 0 (absorbing), 1 (periodic), 2 (outflow) or 3 (slab)");
  pbgk_ctx* c = new pbgk_ctx();
  c->g = *g;
  c->dx = (g->x_max - g->x_min) / g->nx;  // ref/grid.py:95
  const int nv[3] = {g->nvx, g->nvy, g->nvz};
  for (int a = 0; a < 3; ++a) c->dv[a] = 2.0 * g->v_max / nv[a];  // ref/grid.py:114
  c->dvol = c->dv[0] * c->dv[1] * c->dv[2];
  auto bail = [&](int rc) {
    pbgk_ctx_destroy(c);
    return rc;
  };
  c->dev = g->device;
  if (cudaSetDevice(c->dev) != cudaSuccess) return bail(fail("cannot select CUDA device"));
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c->dev) != cudaSuccess) return bail(fail("device query failed"));
  c->nsm = prop.multiProcessorCount;
  if (const char* k = getenv("PBGK_L2KEEP")) c->l2_keep = atoi(k);  // development knob
  c->smem_optin = prop.sharedMemPerBlockOptin;
  c->smem_per_sm = prop.sharedMemPerMultiprocessor;
  // table row: [r, ls, gx(nvx), gy(nvy), gz(nvz)] padded to 16 bytes
  c->gxo = 2;
  c->gyo = c->gxo + g->nvx;
  c->gzo = (c->gyo + g->nvy + 1) & ~1;  // 16-byte aligned for vector reads
  c->TL = (c->gzo + g->nvz + 1) & ~1;
  // the multi-step sweep: 16-wide boxes whenever v_z allows (same-box A/B:
  // 64^3 -4.7 %, 32^3 -3 %, 48^3 -23 % window time against the upwind
  // sweep's 64- / 32- / 48-wide boxes; 8-wide boxes +35 %), else the upwind
  // tiling
  if (!make_plan(c, false, false, c->plan[0]) || !make_plan(c, true, false, c->plan[1]) ||
      !make_plan(c, false, true, c->plan[2]) ||
      !make_plan(c, false, false, c->plan[3],
                 getenv("PBGK_FPLAN_CFG") ? atoi(getenv("PBGK_FPLAN_CFG"))  // dev knob
                                          : (g->nvz % 16 == 0 ? 3 : c->plan[0].cfg)))
    return bail(fail("no tiling fits this velocity grid"));
  if (!msweep_tiling(g->nvx, g->nvy, g->nvz, &c->ms_t)) c->ms_t.NT = 0;
  for (int a = 0; a < 3; ++a) {
    std::vector<double> h(nv[a]);
    for (int j = 0; j < nv[a]; ++j) h[j] = ((double)j - (nv[a] - 1) / 2.0) * c->dv[a];  // ref/grid.py:100-103
    if (cudaMalloc(&c->d_c[a], nv[a] * sizeof(double)) != cudaSuccess) return bail(fail("cudaMalloc"));
    cudaMemcpy(c->d_c[a], h.data(), nv[a] * sizeof(double), cudaMemcpyHostToDevice);
  }
  c->part_elems = 0;
  for (int f = 0; f < 3; ++f)
    c->part_elems = std::max(c->part_elems, (size_t)g->nx * c->plan[f].t.NT * c->plan[f].t.PS);
  size_t bytes = c->part_elems * 8 + 2 * (size_t)g->nx * c->TL * 8 + (size_t)5 * g->nx * 8 + 64;
  if (cudaMalloc(&c->d_part, c->part_elems * 8) != cudaSuccess ||
      cudaMalloc(&c->d_tab[0], (size_t)g->nx * c->TL * 8) != cudaSuccess ||
      cudaMalloc(&c->d_tab[1], (size_t)g->nx * c->TL * 8) != cudaSuccess ||
      cudaMalloc(&c->d_scratch, (size_t)5 * g->nx * 8) != cudaSuccess ||
      cudaMalloc(&c->d_err, 64) != cudaSuccess)
    return bail(fail("cudaMalloc workspace"));
  if (cudaMallocHost(&c->h_err, 64) != cudaSuccess || cudaMallocHost(&c->h_dbl, 64) != cudaSuccess)
    return bail(fail("cudaMallocHost"));
  c->ws_bytes = bytes;
  *out = c;
  return 0;
}

void pbgk_ctx_destroy(pbgk_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->dev);
  for (auto* v : {&c->ev_pool, &c->ev_used})
    for (auto& e : *v) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
  for (int a = 0; a < 3; ++a) cudaFree(c->d_c[a]);
  cudaFree(c->d_part);
  cudaFree(c->d_tab[0]);
  cudaFree(c->d_tab[1]);
  cudaFree(c->d_q0);
  cudaFree(c->d_bt);
  cudaFree(c->d_bq);
  cudaFree(c->d_bg);
  cudaFree(c->d_bdts);
  cudaFree(c->d_bnst);
  cudaFree(c->d_gbar);
  cudaFree(c->d_prog);
  cudaFree(c->d_mpart);
  cudaFree(c->d_trip);
  cudaFree(c->d_fb[0]);
  cudaFree(c->d_fb[1]);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->st_side) cudaStreamDestroy(c->st_side);
  cudaFree(c->d_scratch);
  cudaFree(c->d_err);
  cudaFree(c->d_keys);
  cudaFreeHost(c->h_keys);
  cudaFree(c->d_times);
  cudaFree(c->d_times2);
  if (c->h_err) cudaFreeHost(c->h_err);
  if (c->h_dbl) cudaFreeHost(c->h_dbl);
  delete c;
}

size_t pbgk_ctx_workspace_bytes(const pbgk_ctx* c) { return c ? c->ws_bytes : 0; }

long long pbgk_launch_count(void) { return g_launches.load(); }

int pbgk_ctx_describe(const pbgk_ctx* c, char* buf, size_t n) {
  if (!c || !buf || n == 0) return fail("null argument");
  const char* names[3] = {"plain", "field", "muscl"};
  int off = 0;
  for (int f = 0; f < 3; ++f) {
    const Plan& p = c->plan[f];
    const CfgShape& s = kCfg[p.cfg];
    off += snprintf(buf + off, n - off > 0 ? n - off : 0,
                    "%s: cfg=%d V=%d LZ=%d K=%d T=%d tma=%d box=%dx%dx%d rows_load=%d NT=%d PS=%d "
                    "grid=%d ns=%d; ",
                    names[f], p.cfg, s.V, s.LZ, s.K, s.NTHR, (int)s.tma, p.t.A, p.t.By, p.t.Bz,
                    p.t.rows_load, p.t.NT, p.t.PS, p.grid, p.ns);
    if (off >= (int)n) break;
  }
  return 0;
}

int pbgk_profile_enable(pbgk_ctx* c, int on) {
  if (!c) return fail("null context");
  c->prof = on != 0;
  return 0;
}

int pbgk_profile_read(pbgk_ctx* c, pbgk_profile* out) {
  if (!c || !out) return fail("null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  std::memset(out, 0, sizeof *out);
  for (auto& e : c->ev_used) {
    CK(cudaEventSynchronize(e.b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e.a, e.b));
    if (e.kind == 0) {
      out->sweep_ms += ms;
      out->sweep_bytes += e.bytes;
      out->sweeps += 1;
    } else if (e.kind == 2) {
      out->msweep_ms += ms;
      out->msweep_bytes += e.bytes;
      out->msweeps += 1;
      out->msweep_steps += e.steps;
    } else if (e.kind == 3) {
      out->marg_ms += ms;
      out->margs += 1;
    } else {
      out->finalize_ms += ms;
      out->finalizes += 1;
    }
    c->ev_pool.push_back(e);
  }
  c->ev_used.clear();
  return 0;
}

int pbgk_lift(pbgk_ctx* c, const double* mom, int normalize, double* f_out, void* stream,
              long long* h_code) {
  if (!c || !mom || !f_out) return fail("pbgk_lift: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  if (reset_err(c, st)) return -1;
  if (run_final(c, 0, normalize ? kFinSynthNorm : kFinSynthRaw, mom, nullptr, c->d_tab[0], 0, 1,
                1, nullptr, 0, st))
    return -1;
  if (run_sweep(c, 0, false, nullptr, c->d_tab[0], f_out, 0.0, nullptr, 0.0, 0.0, 0, st)) return -1;
  return fetch_err(c, st, h_code);
}

int pbgk_project(pbgk_ctx* c, const double* f, double* mom_out, void* stream, long long* h_code) {
  if (!c || !f || !mom_out) return fail("pbgk_project: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  if (reset_err(c, st)) return -1;
  if (run_final(c, 0, kFinIdentity, nullptr, nullptr, c->d_tab[0], 0, 1, 1, nullptr, 0, st)) return -1;
  if (run_sweep(c, 0, false, f, c->d_tab[0], nullptr, 0.0, nullptr, 0.0, 0.0, 0, st)) return -1;
  if (run_final(c, 0, kFinProject, nullptr, mom_out, nullptr, 0, 1, 1, nullptr, 0, st)) return -1;
  return fetch_err(c, st, h_code);
}

int pbgk_transport(pbgk_ctx* c, const double* f, double* f_out, double dt, const double* E,
                   double e_max, void* stream) {
  if (!c || !f || !f_out) return fail("pbgk_transport: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  const bool field = (E != nullptr && e_max > 0.0);
  const int pid = field ? 1 : (c->x_scheme == 1 ? 2 : 0);
  if (run_final(c, pid, kFinIdentity, nullptr, nullptr, c->d_tab[0], 0, 1, 1, nullptr, 0, st)) return -1;
  return run_sweep(c, pid, field, f, c->d_tab[0], f_out, dt / c->dx, E, 0.5 * e_max, dt / c->dv[0], 0,
                   st);
}

int pbgk_relax(pbgk_ctx* c, const double* f, double* f_out, double dt, double eps, double tau,
               const double* tau_cells, void* stream, long long* h_code) {
  if (!c || !f || !f_out) return fail("pbgk_relax: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  if (reset_err(c, st)) return -1;
  if (run_final(c, 0, kFinIdentity, nullptr, nullptr, c->d_tab[0], 0, 1, 1, nullptr, 0, st)) return -1;
  if (run_sweep(c, 0, false, f, c->d_tab[0], nullptr, 0.0, nullptr, 0.0, 0.0, 0, st)) return -1;
  if (run_final(c, 0, kFinRelax, nullptr, nullptr, c->d_tab[1], dt, eps, tau, tau_cells, 1, st))
    return -1;
  if (run_sweep(c, 0, false, f, c->d_tab[1], f_out, 0.0, nullptr, 0.0, 0.0, 0, st)) return -1;
  return fetch_err(c, st, h_code);
}

int pbgk_check_finite(pbgk_ctx* c, const double* f, int step, void* stream, long long* h_code) {
  if (!c || !f) return fail("pbgk_check_finite: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  if (reset_err(c, st)) return -1;
  if (run_final(c, 0, kFinIdentity, nullptr, nullptr, c->d_tab[0], 0, 1, 1, nullptr, 0, st)) return -1;
  if (run_sweep(c, 0, false, f, c->d_tab[0], nullptr, 0.0, nullptr, 0.0, 0.0, step, st)) return -1;
  if (run_final(c, 0, kFinProject, nullptr, nullptr, nullptr, 0, 1, 1, nullptr, step, st, 1)) return -1;
  return fetch_err(c, st, h_code);
}

namespace {
bool fused_ok(pbgk_ctx* c, bool field);
int propagate_body_fused(pbgk_ctx* c, const double* f0, const double* mom0, double* f_out,
                         double* f_tmp, int write_final, double* mom_out, int S, const double* h_dts,
                         double eps, double tau, const double* E, double e_max, cudaStream_t st);

// One propagation on the stream, failures atomicMin-ed into the current
// error slot; no reset, no host synchronisation.
int propagate_body(pbgk_ctx* c, const double* f0, const double* mom0, double* f_out, double* f_tmp,
                   int write_final, double* mom_out, int S, const double* h_dts, double eps,
                   double tau, const double* E, double e_max, cudaStream_t st) {
  const bool field = (E != nullptr && e_max > 0.0);
  // (the multi-step path keeps the tables of every step: a very long single
  // propagation whose tables exceed PBGK_BATCH_BYTES stays one-step)
  if (S > 0 && !c->one_step && fused_ok(c, field) &&
      8.0 * (S + 1) * (double)c->g.nx * c->TL <= batch_budget(c))
    return propagate_body_fused(c, f0, mom0, f_out, f_tmp, write_final, mom_out, S, h_dts, eps, tau,
                                E, e_max, st);
  const int pid = field ? 1 : (c->x_scheme == 1 ? 2 : 0);
  const int W = S + (write_final ? 1 : 0);
  auto buf = [&](int w) { return ((W - w) % 2 == 0) ? f_out : f_tmp; };
  // f_0: the given distribution (identity tables) or the raw lift of mom0
  if (f0) {
    if (run_final(c, pid, kFinIdentity, nullptr, nullptr, c->d_tab[0], 0, 1, 1, nullptr, 0, st)) return -1;
  } else {
    if (run_final(c, pid, kFinSynthRaw, mom0, nullptr, c->d_tab[0], 0, 1, 1, nullptr, 0, st)) return -1;
  }
  for (int s = 1; s <= S; ++s) {
    const double dt = h_dts[s - 1];
    const double* in = (s == 1) ? f0 : buf(s - 1);
    if (run_sweep(c, pid, field, in, c->d_tab[(s - 1) & 1], buf(s), dt / c->dx, E, 0.5 * e_max,
                  dt / c->dv[0], s == 1 ? 0 : s - 1, st))
      return -1;
    if (run_final(c, pid, kFinRelax, nullptr, nullptr, c->d_tab[s & 1], dt, eps, tau, nullptr, s, st))
      return -1;
  }
  if (S > 0) {
    if (run_sweep(c, pid, false, buf(S), c->d_tab[S & 1], write_final ? f_out : nullptr, 0.0, nullptr,
                  0.0, 0.0, S, st))
      return -1;
    if (mom_out &&
        run_final(c, pid, kFinProject, nullptr, mom_out, nullptr, 0, 1, 1, nullptr, S + 1, st))
      return -1;
  }
  return 0;
}
}  // namespace

namespace {
// Multi-step path usable on this context: the upwind scheme (the moment
// recursion is closed for it, with or without the v_x field term -- the field
// runs one step per pass, see propagate_body_fused; MUSCL's limiter is not
// linear), bc 0..2 (slabs exchange halos per step).
int fuse_levels(pbgk_ctx* c);

bool fused_ok(pbgk_ctx* c, bool field) {
  (void)field;
  if (fuse_levels(c) < 1 || c->x_scheme != 0 || c->g.bc == 3) return false;
  if (!fsweep_has_cfg(c->plan[3].cfg)) return false;
  if (marg_smem_bytes(c->g.nvx, c->g.nvy, c->g.nvz, c->TL) > c->smem_optin) return false;
  if (!c->d_q0) {
    const size_t ms = (size_t)c->g.nx * marg_state_doubles(c->g.nvx) * sizeof(double);
    if (cudaMalloc(&c->d_q0, ms) != cudaSuccess) return false;
    c->ws_bytes += ms;
  }
  return true;
}

// Levels per pass: the context's setting, or (auto, -1) the measured best
// per shape (round 1, one B200): 4 for the 2-wide lane layouts (run as
// 4-wide lanes, 255 registers), 3 for the 48-wide V = 6 one (its fourth level
// spills heavily).  The same for single propagations and batched windows,
// so a window gives bitwise the same moments either way (the pipelined
// parareal schedule propagates windows one by one, the phased one batched).
int fuse_levels(pbgk_ctx* c) {
  static const int env = getenv("PBGK_FUSE") ? atoi(getenv("PBGK_FUSE")) : -2;
  int L = env >= -1 ? env : c->fuse;
  if (L < 0) {
    L = kCfg[c->plan[3].cfg].V == 6 ? 3 : 4;
  }
  return std::min(L, 4);
}

// One pass of n <= 4 fine steps (steps s0+1 .. s0+n) over f.
int run_fsweep(pbgk_ctx* c, int n, const double* in, double* out, const double* const* tabs,
               const double* dtdx, int step0, cudaStream_t st, const unsigned* prog = nullptr,
               unsigned need = 0) {
  const Plan& p = c->plan[3];
  const CfgShape& s = kCfg[p.cfg];
  FSweepArgs a{};
  a.nx = c->g.nx;
  a.nvx = c->g.nvx;
  a.nvy = c->g.nvy;
  a.nvz = c->g.nvz;
  a.plane = (long long)c->g.nvx * c->g.nvy * c->g.nvz;
  a.t = p.t;
  a.total = (long long)p.t.NT * c->g.nx;
  a.fin = in;
  a.fout = out;
  for (int l = 0; l < n; ++l) {
    a.tab[l] = tabs[l];
    a.dtdx[l] = dtdx[l];
  }
  a.TL = c->TL;
  a.gxo = c->gxo;
  a.gyo = c->gyo;
  a.gzo = c->gzo;
  a.cx = c->d_c[0];
  a.bc = c->g.bc;
  a.err = c->err_slot ? c->err_slot : c->d_err;
  a.step0 = step0;
  a.prog = prog;
  a.need = need;
  const bool synth = (in == nullptr);
  const CUtensorMap* map = tensor_map(c, synth ? nullptr : in, p.t, p.cfg);
  if (!map) return fail("tensor map: " + g_last_error);
  // ring depth: the plan's, fewer stages if the L table rows per stage do not
  // fit the plan's CTAs per SM
  const int per_sm = std::min(p.per_sm, fsweep_ctas_per_sm(n));
  const size_t budget = (per_sm == 2) ? (c->smem_per_sm / 2) - 2048 : c->smem_optin;
  // (L >= 2 consumes two planes per round: at least 4 stages)
  static const int pr = getenv("PBGK_FS_NS") ? atoi(getenv("PBGK_FS_NS")) : 6;  // dev knob
  int ns = per_sm == 2 ? p.ns : std::max(p.ns, pr);
  const int ns_min = per_sm == 2 ? 2 : 4;
  while (ns > ns_min && fsweep_smem_bytes(a, s.V, s.LZ, synth, n, ns) > budget) --ns;
  if (fsweep_smem_bytes(a, s.V, s.LZ, synth, n, ns) > budget) return fail("multi-step sweep: ring does not fit");
  const size_t smem = fsweep_smem_bytes(a, s.V, s.LZ, synth, n, ns);
  const double fbytes = 8.0 * (double)a.plane * a.nx;
  ProfScope ps(c, st, 2, (synth ? 0.0 : fbytes) + fbytes, n);
  // persistent grid minus the CTA slots left to side-stream work AND the SMs
  // of a concurrent recursion (both can be active at once)
  int grid = (int)std::min<long long>(a.total, (long long)c->nsm * per_sm);
  const int reserve = c->slot_reserve + (prog != nullptr ? c->rec_reserve * per_sm : 0);
  grid = std::max(1, std::min(grid, c->nsm * per_sm - reserve));
  CK(launch_fsweep(p.cfg, *map, a, synth, n, grid, ns, smem, st));
  return 0;
}

// Round-2 multi-step sweep (msweep.cu): levels per pass (8, or 4 on request), or 0 when the
// context's velocity grid / quadrature / scheme does not run on it.
int ms_levels(pbgk_ctx* c) {
  static const int env = getenv("PBGK_MS") ? atoi(getenv("PBGK_MS")) : -1;  // dev A/B knob
  if (!(env >= 0 ? env : c->ms) || c->quad != 0 || c->x_scheme != 0 || c->g.bc == 3) return 0;
  if (c->fuse > 0) return 0;  // an explicit pbgk_set_fusion level count selects the round-1 kernel
  static const int envl = getenv("PBGK_MS_L") ? atoi(getenv("PBGK_MS_L")) : 0;  // dev A/B knob
  const int L = envl ? envl : (c->ms_levels ? c->ms_levels : 8);
  if (L != 4 && L != 8) return 0;
  if (c->ms_t.NT == 0) return 0;
  return L;
}

// One msweep pass: n <= L fine steps (steps step0 .. step0+n-1) from `in`
// (null: SYNTH, level 0 lifts tabs[0]), writing the last level to `out`
// (may be null); FINAL (`tabR` non-null): R_S applied, partial records of
// P(f_S) into d_mpart.
// A batch of windows in one msweep launch (grid.y = window): `in` / `out` hold
// the windows' f back to back, tabs / tabR / d_mpart are window 0's with
// stride t_ws / the record block, keys at errw[window], dt of step s0 + l of
// window k on the device at dts[(s0 + l) * nwin + k].
struct MsBatch {
  int nwin;
  long long t_ws;
  ErrKey* errw;
  const double* dts;
  int s0;
};

int run_msweep(pbgk_ctx* c, int L, const double* in, double* out, const double* const* tabs,
               const double* tabR, const double* dtdx, int n, int step0, cudaStream_t st,
               const unsigned* prog = nullptr, unsigned need = 0, const MsBatch* mb = nullptr,
               const double* trip = nullptr, long long trip_ws = 0) {
  const Tiling& t = c->ms_t;
  const int nwin = mb ? mb->nwin : 1;
  MSweepArgs a{};
  a.trip = trip;
  a.trip_ls = (long long)c->g.nx * c->g.nvx * 4;
  a.trip_ws = trip_ws;
  a.nx = c->g.nx;
  a.nvx = c->g.nvx;
  a.nvy = c->g.nvy;
  a.nvz = c->g.nvz;
  a.plane = (long long)c->g.nvx * c->g.nvy * c->g.nvz;
  a.t = t;
  a.total = (long long)t.NT * c->g.nx;
  a.fout = out;
  for (int l = 0; l < kMaxL; ++l) {
    a.tab[l] = tabs[std::min(l, n - 1)];  // levels >= n are skipped (their copies land unused)
    a.dtdx[l] = l < n ? dtdx[l] : 0.0;
  }
  a.tabR = tabR;
  a.nlev = n;
  a.TL = c->TL;
  a.gxo = c->gxo;
  a.gyo = c->gyo;
  a.gzo = c->gzo;
  a.cx = c->d_c[0];
  a.bc = c->g.bc;
  a.err = c->err_slot ? c->err_slot : c->d_err;
  a.step0 = step0;
  a.prog = prog;
  a.need = need;
  const int mode = (in == nullptr ? 1 : 0) | (tabR != nullptr ? 2 : 0);
  if (tabR) {
    if (ensure_dev(c->d_mpart, c->mpart_cap, (size_t)nwin * c->g.nx * t.NT * t.PS, st)) return -1;
    a.part = c->d_mpart;
  }
  if (mb) {
    a.f_ws = a.plane * a.nx;
    a.t_ws = mb->t_ws;
    a.p_ws = (long long)c->g.nx * t.NT * t.PS;
    a.errw = mb->errw;
    a.dts = mb->dts;
    a.dts_g = nwin;
    a.s0 = mb->s0;
    a.dx = c->dx;
  }
  const CUtensorMap* map = tensor_map(c, in, t, 3, mb ? nwin * c->g.nx : 0);
  if (!map) return fail("tensor map: " + g_last_error);
  static const int ns_env = getenv("PBGK_MS_NS") ? atoi(getenv("PBGK_MS_NS")) : 0;  // dev knob
  const int per_sm = msweep_ctas_per_sm();
  const size_t budget = per_sm == 1 ? c->smem_optin : c->smem_per_sm / per_sm - 1024;
  int ns = ns_env > 0 ? ns_env : 12;
  while (ns > 3 && msweep_smem_bytes(L, mode, c->g.nvx, ns, trip != nullptr) > budget) --ns;
  const size_t smem = msweep_smem_bytes(L, mode, c->g.nvx, ns, trip != nullptr);
  if (smem > budget) return fail("msweep: ring does not fit");
  const double fbytes = 8.0 * (double)a.plane * a.nx * nwin;
  ProfScope ps(c, st, 2, (in ? fbytes : 0.0) + (out ? fbytes : 0.0), n);
  // one CTA per SM, minus the slots left to side-stream work and the SMs of a
  // concurrent recursion; a batch splits them between its windows
  int grid = (int)std::min<long long>(a.total, (long long)c->nsm * per_sm);
  int reserve = c->slot_reserve + (prog != nullptr ? c->rec_reserve * per_sm : 0);
  grid = std::max(1, std::min(grid, c->nsm * per_sm - reserve));
  if (nwin > 1) grid = std::max(1, grid / nwin);
  CK(launch_msweep(L, mode, *map, a, grid, nwin, ns, smem, st));
  return 0;
}

// The per-row factors of S steps of g windows into d_trip (see msweep.cu
// ms_prep_kernel); dts[s * dts_g + window] on the device.  Returns the
// window stride (doubles), 0 when switched off (PBGK_MS_NOPRE: A/B and test
// knob, read per call), -1 on error.
long long ms_prep(pbgk_ctx* c, int g, const double* T, long long t_ws, int S, const double* d_dts, int dts_g,
                  bool lift0, cudaStream_t st) {
  if (getenv("PBGK_MS_NOPRE") != nullptr || S <= 0) return 0;
  const long long ws = (long long)S * c->g.nx * c->g.nvx * 4;
  if (ensure_dev(c->d_trip, c->trip_cap, (size_t)g * ws, st)) return -1;
  ProfScope ps(c, st, 3, 0.0);
  if (launch_ms_prep(T, t_ws, (long long)c->g.nx * c->TL, c->TL, c->gxo, c->d_c[0], d_dts, dts_g, c->dx, S,
                     c->g.nx, c->g.nvx, lift0 ? 1 : 0, c->d_trip, ws, g, st) != cudaSuccess) {
    fail("ms_prep launch");
    return -1;
  }
  return ws;
}

// The passes and the projection of a batch of g windows with S steps each
// (small grids: one window cannot fill the GPU, its tile runs are shorter than
// their lead-in): every pass is one launch over all windows, f in the
// context's batch buffers; tables at T + k t_ws, moments to mom_out + k * 5 nx.
int ms_windows_batched(pbgk_ctx* c, int L, int g, const double* T, long long t_ws, int S,
                       const double* d_dts, ErrKey* errw, double* mom_out, cudaStream_t st) {
  const size_t tstep = (size_t)c->g.nx * c->TL;
  const size_t fw = (size_t)c->g.nx * c->g.nvx * c->g.nvy * c->g.nvz;
  const int P = (S + L - 1) / L;
  if (P > 1 && ensure_dev(c->d_fb[0], c->fb_cap[0], (size_t)g * fw, st)) return -1;
  if (P > 2 && ensure_dev(c->d_fb[1], c->fb_cap[1], (size_t)g * fw, st)) return -1;
  const double* in = nullptr;
  int wcount = 0;
  const long long trip_ws = ms_prep(c, g, T, t_ws, S, d_dts, g, true, st);
  if (trip_ws < 0) return -1;
  const size_t lstride = (size_t)c->g.nx * c->g.nvx * 4;
  for (int s0 = 0; s0 < S;) {
    const int n = std::min(L, S - s0);
    const bool last = s0 + n == S;
    const double* tabs[kMaxL];
    double dtdx[kMaxL] = {};
    for (int l = 0; l < n; ++l) tabs[l] = T + (size_t)(s0 + l) * tstep;
    double* out = last ? nullptr : c->d_fb[(wcount++) & 1];
    MsBatch mb{g, t_ws, errw, d_dts, s0};
    if (run_msweep(c, L, in, out, tabs, last ? T + (size_t)S * tstep : nullptr, dtdx, n, s0 + 1, st, nullptr, 0,
                   &mb, trip_ws > 0 ? c->d_trip + s0 * lstride : nullptr, trip_ws))
      return -1;
    in = out;
    s0 += n;
  }
  FinalArgs f = fin_args(c, c->plan[0]);
  f.t = c->ms_t;
  f.part = c->d_mpart;
  f.mode = kFinProject;
  f.mom_out = mom_out;
  f.step = S + 1;
  f.relax_tab = T + (size_t)S * tstep;  // the records are those of f*_S
  FinalBatch fb{(long long)c->g.nx * c->ms_t.NT * c->ms_t.PS, 0, (long long)5 * c->g.nx, t_ws, errw};
  ProfScope ps(c, st, 1, 0.0);
  CK(launch_finalize_batch(f, fb, g, st));
  return 0;
}

// The passes of one window on the msweep path, then its projection: tables
// T[s] (R_s; T[0] the lift or identity rows), S steps with h_dts; f0 null:
// the first pass synthesises L(mom); f_S = R_S(f*_S) is stored to f_out only
// when write_final; mom_out (may be null) gets P(f_S).
int ms_window(pbgk_ctx* c, int L, const double* f0, double* f_out, double* f_tmp, int write_final,
              double* mom_out, const double* T, int S, const double* h_dts, cudaStream_t st,
              const unsigned* prog = nullptr, unsigned base = 0, const double* d_dts = nullptr,
              int dts_g = 1) {
  const size_t tstep = (size_t)c->g.nx * c->TL;
  // the per-row factors of every step, once per window (not with a concurrent
  // recursion: its tables arrive pass by pass)
  long long trip_ws = 0;
  if (prog == nullptr && d_dts != nullptr) {
    trip_ws = ms_prep(c, 1, T, 0, S, d_dts, dts_g, f0 == nullptr, st);
    if (trip_ws < 0) return -1;
  }
  const size_t lstride = (size_t)c->g.nx * c->g.nvx * 4;
  const int P = (S + L - 1) / L;
  const int W = P - 1 + (write_final ? 1 : 0);
  auto buf = [&](int w) { return ((W - w) % 2 == 0) ? f_out : f_tmp; };
  const double* in = f0;
  int wcount = 0;
  for (int s0 = 0; s0 < S;) {
    const int n = std::min(L, S - s0);
    const bool last = s0 + n == S;
    const double* tabs[kMaxL];
    double dtdx[kMaxL];
    for (int l = 0; l < n; ++l) {
      tabs[l] = T + (size_t)(s0 + l) * tstep;
      dtdx[l] = h_dts[s0 + l] / c->dx;
    }
    double* out = (!last || write_final) ? buf(++wcount) : nullptr;
    if (run_msweep(c, L, in, out, tabs, last ? T + (size_t)S * tstep : nullptr, dtdx, n, s0 + 1, st, prog,
                   base + (unsigned)(last ? S : s0 + n - 1), nullptr,
                   trip_ws > 0 ? c->d_trip + s0 * lstride : nullptr, 0))
      return -1;
    in = out;
    s0 += n;
  }
  if (mom_out) {
    FinalArgs f = fin_args(c, c->plan[0]);
    f.t = c->ms_t;
    f.part = c->d_mpart;
    f.mode = kFinProject;
    f.mom_out = mom_out;
    f.step = S + 1;
    // f_S not stored: the last pass's records are those of f*_S
    f.relax_tab = write_final ? nullptr : T + (size_t)S * tstep;
    ProfScope ps(c, st, 1, 0.0);
    CK(launch_finalize(f, st));
  }
  return 0;
}

// Levels per pass of the field-term passes (esweep.cu): its compiled maximum
// for this nvx, or fewer under an explicit pbgk_set_fusion; 0 when the shape,
// scheme or boundary does not run on it (the field then runs one step per
// pass on the recursion's tables).
int es_levels(pbgk_ctx* c) {
  static const int env = getenv("PBGK_ES") ? atoi(getenv("PBGK_ES")) : -1;  // dev A/B knob
  if (!(env >= 0 ? env : c->es) || c->x_scheme != 0 || c->g.bc > 2) return 0;
  const int Lmax = esweep_levels(c->g.nvx, c->g.nvz);
  if (Lmax < 1 || esweep_smem_bytes(c->g.nvx, true) > c->smem_optin) return 0;
  if (c->es_per_sm == 0) c->es_per_sm = std::max(0, esweep_ctas_per_sm(c->g.nvx));
  if (c->es_per_sm < 1) return 0;
  return c->fuse > 0 ? std::min(c->fuse, Lmax) : Lmax;
}

// The window's last field-term pass can project (FINAL): midpoint quadrature
// (the partial records carry no quadrature weights).
bool es_final_ok(pbgk_ctx* c) {
  return getenv("PBGK_ES_NOFINAL") == nullptr && c->quad == 0;  // (env: A/B and test knob, read per call)
}

// One field-term pass: n levels (steps step0 .. step0+n-1) from `in` (null:
// SYNTH, level 0 lifts tabs[0]) to `out`; FINAL (`tabR` non-null, out null):
// R_S applied and the partial records of P(f_S) written to d_mpart.
int run_esweep(pbgk_ctx* c, int n, const double* in, double* out, const double* const* tabs,
               const double* dts, const double* E, double e_max, int step0, cudaStream_t st,
               const double* tabR = nullptr) {
  ESweepArgs a{};
  if (tabR) {
    Tiling t;
    esweep_tiling(c->g.nvx, c->g.nvy, c->g.nvz, &t);
    if (ensure_dev(c->d_mpart, c->mpart_cap, (size_t)c->g.nx * t.NT * t.PS, st)) return -1;
    a.tabR = tabR;
    a.part = c->d_mpart;
    a.PS = t.PS;
  }
  a.nx = c->g.nx;
  a.nvx = c->g.nvx;
  a.nvy = c->g.nvy;
  a.nvz = c->g.nvz;
  a.fin = in;
  a.fout = out;
  for (int l = 0; l < kMaxLevels; ++l) {
    a.tab[l] = tabs[std::min(l, n - 1)];
    a.dtdx[l] = l < n ? dts[l] / c->dx : 0.0;
    a.dtdv[l] = l < n ? dts[l] / c->dv[0] : 0.0;
  }
  a.TL = c->TL;
  a.gyo = c->gyo;
  a.gzo = c->gzo;
  a.cx = c->d_c[0];
  a.E = E;
  a.half_emax = 0.5 * e_max;
  a.nlev = n;
  a.bc = c->g.bc;
  a.err = c->err_slot ? c->err_slot : c->d_err;
  a.step0 = step0;
  const int per_sm = c->es_per_sm;
  int grid = c->nsm * per_sm;
  if (c->slot_reserve > 0) grid = std::max(1, grid - (c->slot_reserve + 3) / 4);
  // items: warp columns x x-segments; the segment count minimising the
  // busiest warp's positions (its segments plus their 2n halo positions)
  const int warps = grid * 4;
  a.ncol = a.nvy * (a.nvz / 8);
  int best = 1;
  double best_cost = 1e300;
  const int smax = std::max(1, std::min(a.nx, 256));
  for (int ns = 1; ns <= smax; ++ns) {
    const int len = (a.nx + ns - 1) / ns;
    const long long items = (long long)a.ncol * ns;
    const double rounds = (double)((items + warps - 1) / warps);
    const double cost = rounds * (len + 2 * n);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = ns;
    }
  }
  a.seglen = (a.nx + best - 1) / best;
  a.nseg = (a.nx + a.seglen - 1) / a.seglen;
  const long long items = (long long)a.ncol * a.nseg;
  grid = (int)std::max(1LL, std::min<long long>(grid, (items + 3) / 4));
  const size_t smem = esweep_smem_bytes(c->g.nvx, tabR != nullptr);
  const double fbytes = 8.0 * (double)a.nx * a.nvx * a.nvy * a.nvz;
  ProfScope ps(c, st, 2, (in ? fbytes : 0.0) + (out ? fbytes : 0.0), n);
  CK(launch_esweep(a, in == nullptr, grid, smem, st));
  return 0;
}

// P(f_S) from the partial records (of f*_S) of a FINAL field-term pass
int es_project(pbgk_ctx* c, double* mom_out, const double* tabR, int step, cudaStream_t st) {
  FinalArgs f = fin_args(c, c->plan[0]);
  esweep_tiling(c->g.nvx, c->g.nvy, c->g.nvz, &f.t);
  f.part = c->d_mpart;
  f.relax_tab = tabR;  // the records are those of f*_S
  f.mode = kFinProject;
  f.mom_out = mom_out;
  f.step = step;
  ProfScope ps(c, st, 1, 0.0);
  CK(launch_finalize(f, st));
  return 0;
}

// propagate_body on the multi-step path (one window, from moments or a given
// f0): the moment recursion for all S steps first (one launch when the grid
// is co-resident), per-step tables; then the passes of up to L steps; the
// last relax + projection is the reference-order marginal sweep of f*_S.
int run_recursion(pbgk_ctx* c, int g, const double* q0, double* T, long long t_ws, int S,
                  const double* dts, const int* nst, ErrKey* errw, double eps, double tau,
                  const double* E, double e_max, cudaStream_t st, unsigned* prog = nullptr,
                  unsigned prog_base = 0, int max_ctas = 0);

// A single propagation runs its recursion concurrently when its one-launch
// grid fits <= 16 SMs (the passes lose at most 11 % of their SMs) and it has
// enough steps to matter (PBGK_REC_CONCURRENT=0 disables: dev A/B knob).
bool concurrent_ok(pbgk_ctx* c, int S, int L) {
  static const int env = getenv("PBGK_REC_CONCURRENT") ? atoi(getenv("PBGK_REC_CONCURRENT")) : 1;
  if (!env || S < 8 * L || getenv("PBGK_REC_STEPWISE")) return false;
  int ctas = 0, per = 0;
  marg_all_shape(c->g.nx, c->g.nvx, c->g.nvy, c->g.nvz, c->TL, c->quad != 0, 1, &ctas, &per);
  if (per < 1) return false;
  const int need = (ctas + per - 1) / per;
  if (need > 16) return false;
  if (!c->st_side) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&c->st_side, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&c->d_prog, sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(c->d_prog, 0, sizeof(unsigned)) != cudaSuccess ||
        (!c->d_gbar && cudaMalloc(&c->d_gbar, 2 * sizeof(unsigned)) != cudaSuccess))
      return false;
  }
  c->rec_reserve = need;
  return true;
}

int propagate_body_fused(pbgk_ctx* c, const double* f0, const double* mom0, double* f_out,
                         double* f_tmp, int write_final, double* mom_out, int S, const double* h_dts,
                         double eps, double tau, const double* E, double e_max, cudaStream_t st) {
  const bool field = (E != nullptr && e_max > 0.0);
  const int LE = field ? es_levels(c) : 0;
  const int L = field ? std::max(LE, 1) : fuse_levels(c);
  const int P = (S + L - 1) / L;  // passes
  const int W = P + (write_final ? 1 : 0);
  auto buf = [&](int w) { return ((W - w) % 2 == 0) ? f_out : f_tmp; };
  const size_t tstep = (size_t)c->g.nx * c->TL;
  const size_t qw = (size_t)c->g.nx * marg_state_doubles(c->g.nvx);
  if (ensure_dev(c->d_bt, c->bt_cap, (size_t)(S + 1) * tstep, st) ||
      ensure_dev(c->d_bq, c->bq_cap, 2 * qw, st) ||
      ensure_dev(c->d_bg, c->bg_cap, (size_t)12 * c->g.nx, st) ||
      ensure_dev(c->d_bdts, c->bdts_cap, (size_t)S, st))
    return -1;
  double* T = c->d_bt;
  // (pageable source: the copy completes before the call returns)
  c->sh_bdts.clear();
  CK(cudaMemcpyAsync(c->d_bdts, h_dts, (size_t)S * sizeof(double), cudaMemcpyHostToDevice, st));
  // f_0: the lift of mom0 (synthesised by the first pass), or the given f0
  // with identity tables (r = 1, ls = 0) and the recursion started from Q(f0)
  const double* q0 = nullptr;
  if (f0) {
    if (run_final(c, 0, kFinIdentity, nullptr, nullptr, T, 0, 1, 1, nullptr, 0, st)) return -1;
    MargArgs m{};
    m.nx = c->g.nx;
    m.nvx = c->g.nvx;
    m.nvy = c->g.nvy;
    m.nvz = c->g.nvz;
    m.cy = c->d_c[1];
    m.cz = c->d_c[2];
    m.trap = c->quad;
    m.mout = c->d_q0;
    ++g_launches;
    CK(launch_q_from_f(m, f0, st));
    q0 = c->d_q0;
  } else {
    if (run_final(c, 0, kFinSynthRaw, mom0, nullptr, T, 0, 1, 1, nullptr, 0, st)) return -1;
  }
  // concurrent recursion (long propagations on small grids, where its serial
  // chain of S dependent steps is a large share): the one-launch recursion
  // runs on a side stream on `rec_reserve` SMs, the passes on the others wait
  // per pass on its device progress word
  unsigned* prog = nullptr;
  unsigned base = 0;
  if (!field && !c->no_concurrent && concurrent_ok(c, S, L)) {
    prog = c->d_prog;
    base = c->prog_next;
    c->prog_next += (unsigned)S + 1;
    CK(cudaEventRecord(c->ev_start, st));
    CK(cudaStreamWaitEvent(c->st_side, c->ev_start, 0));
    int ctas = 0, per = 0;
    marg_all_shape(c->g.nx, c->g.nvx, c->g.nvy, c->g.nvz, c->TL, c->quad != 0, 1, &ctas, &per);
    if (run_recursion(c, 1, q0, T, 0, S, c->d_bdts, nullptr, nullptr, eps, tau, nullptr, 0.0, c->st_side,
                      prog, base,
                      c->rec_reserve * per))
      return -1;
    CK(cudaEventRecord(c->ev_done, c->st_side));
  } else if (run_recursion(c, 1, q0, T, 0, S, c->d_bdts, nullptr, nullptr, eps, tau, E, e_max, st)) {
    return -1;
  }
  int rc = 0;
  const int LM = field ? 0 : ms_levels(c);
  if (LM > 0) {
    rc = ms_window(c, LM, f0, f_out, f_tmp, write_final, mom_out, T, S, h_dts, st, prog, base, c->d_bdts, 1);
  } else {
    int w = 0;
    bool projected = false;
    const double* in = f0;
    for (int s0 = 0; s0 < S && rc == 0;) {
      const int n = std::min(L, S - s0);
      const double* tabs[kMaxLevels];
      double dtdx[kMaxLevels];
      for (int l = 0; l < n; ++l) {
        tabs[l] = T + (size_t)(s0 + l) * tstep;
        dtdx[l] = h_dts[s0 + l] / c->dx;
      }
      if (field && LE > 0 && s0 + n == S && !write_final && mom_out && es_final_ok(c)) {
        // the window's last pass: R_S and the projection folded in (no f_S)
        rc = run_esweep(c, n, in, nullptr, tabs, h_dts + s0, E, e_max, s0 + 1, st, T + (size_t)S * tstep);
        if (rc == 0) rc = es_project(c, mom_out, T + (size_t)S * tstep, S + 1, st);
        projected = true;
        break;
      }
      double* out = buf(++w);
      if (field && LE > 0) {
        // the v_x field term, n levels per pass on the recursion's tables
        rc = run_esweep(c, n, in, out, tabs, h_dts + s0, E, e_max, s0 + 1, st);
      } else if (field) {
        // the v_x field term: the one-step sweep (its neighbour-row flux) on
        // the recursion's tables, without the marginal partials
        rc = run_sweep(c, 1, true, in, tabs[0], out, dtdx[0], E, 0.5 * e_max, h_dts[s0] / c->dv[0], s0 + 1,
                       st, 1);
      } else {
        rc = run_fsweep(c, n, in, out, tabs, dtdx, s0 + 1, st, prog, base + (unsigned)(s0 + n - 1));
      }
      in = out;
      s0 += n;
    }
    if (prog && rc == 0) rc = cudaStreamWaitEvent(st, c->ev_done, 0) == cudaSuccess ? 0 : fail("event");
    if (rc == 0 && !projected)
      rc = run_sweep(c, 0, false, in, T + (size_t)S * tstep, write_final ? f_out : nullptr, 0.0, nullptr,
                     0.0, 0.0, S, st);
    if (rc == 0 && mom_out && !projected)
      rc = run_final(c, 0, kFinProject, nullptr, mom_out, nullptr, 0, 1, 1, nullptr, S + 1, st);
  }
  // the side-stream recursion joins the stream on every exit path (its
  // tables and state buffers are reused by the next call)
  if (prog) cudaStreamWaitEvent(st, c->ev_done, 0);
  return rc;
}
}  // namespace

}  // extern "C"

namespace {

// The moment recursion for steps 1..S of `g` windows: per-(window, step)
// tables at T + w t_ws + s (nx TL) (the step-0 tables already there), state
// ping-pong in d_bq, G sums in d_bg, dts[s-1][w] and per-window step counts
// on the device (nst may be null for one window), keys per window (errw, or
// the context's error slot).  One cooperative launch for all steps when the
// grid is co-resident, else one launch per step.
int run_recursion(pbgk_ctx* c, int g, const double* q0, double* T, long long t_ws, int S,
                  const double* dts, const int* nst, ErrKey* errw, double eps, double tau,
                  const double* E, double e_max, cudaStream_t st, unsigned* prog, unsigned prog_base,
                  int max_ctas) {
  const int nx = c->g.nx;
  const size_t tstep = (size_t)nx * c->TL;
  const size_t qw = (size_t)nx * marg_state_doubles(c->g.nvx);
  MargArgs mg{};
  mg.nx = nx;
  mg.nvx = c->g.nvx;
  mg.nvy = c->g.nvy;
  mg.nvz = c->g.nvz;
  mg.bc = c->g.bc;
  mg.cx = c->d_c[0];
  mg.q_ws = (long long)qw;
  mg.t_ws = t_ws;
  mg.g_ws = 12LL * nx;
  mg.nst = nst;
  mg.errw = errw;
  mg.dx = c->dx;
  mg.E = (E != nullptr && e_max > 0.0) ? E : nullptr;
  mg.half_emax = 0.5 * e_max;
  mg.dvx = c->dv[0];
  FinalArgs f = fin_args(c, c->plan[0]);
  f.mode = kFinRelax;
  f.eps = eps;
  f.tau = tau;
  static const bool no_multi = getenv("PBGK_REC_STEPWISE") != nullptr;  // dev A/B knob
  if (!no_multi) {
    if (!c->d_gbar) CK(cudaMalloc(&c->d_gbar, 2 * sizeof(unsigned)));
    mg.tab_in = T;
    mg.dts = dts;
    ProfScope ps(c, st, 3, 0.0);
    ++g_launches;  // + the barrier reset
    const cudaError_t e = launch_marg_all(mg, f, q0, c->d_bq + (size_t)g * qw, c->d_bq, c->d_bg,
                                          (long long)tstep, S, g, c->d_gbar, st, prog, prog_base,
                                          max_ctas);
    if (e == cudaSuccess) return 0;
    if (prog != nullptr) return fail("concurrent recursion: launch refused");
    if (e != cudaErrorCooperativeLaunchTooLarge) return fail(std::string("recursion: ") + cudaGetErrorString(e));
    cudaGetLastError();
  }
  for (int s = 1; s <= S; ++s) {
    MargArgs m = mg;
    m.min = s == 1 ? q0 : c->d_bq + ((s - 1) & 1) * g * qw;
    m.mout = c->d_bq + (s & 1) * g * qw;
    m.tab_in = T + (size_t)(s - 1) * tstep;
    m.dts = dts + (size_t)(s - 1) * g;
    FinalArgs fs = f;
    fs.tab = T + (size_t)s * tstep;
    fs.step = s;
    ProfScope ps(c, st, 3, 0.0);
    if (s == 1) ++g_launches;
    CK(launch_marg(m, fs, c->d_bg, s, g, st));
  }
  return 0;
}

// pbgk_propagate_windows on the multi-step path: the moment recursion of a
// group of windows runs batched (one launch per step for the whole group,
// grid.y = window), then each window's passes read its own per-step tables.
// Groups bound the table memory (PBGK_BATCH_BYTES; default: see default_batch_budget).
int windows_fused(pbgk_ctx* c, int nwin, const double* mom_in, double* mom_out, double* f_a,
                  double* f_b, const int* h_nsteps, const double* h_dts, double eps, double tau,
                  const double* E, double e_max, cudaStream_t st) {
  const bool field = (E != nullptr && e_max > 0.0);
  const int nx = c->g.nx;
  const size_t m5 = (size_t)5 * nx;
  const size_t tstep = (size_t)nx * c->TL;  // one table set
  const size_t qw = (size_t)nx * marg_state_doubles(c->g.nvx);
  int Smax = 0;
  std::vector<size_t> off(nwin + 1, 0);
  for (int w = 0; w < nwin; ++w) {
    Smax = std::max(Smax, h_nsteps[w]);
    off[w + 1] = off[w] + h_nsteps[w];
  }
  const double budget = batch_budget(c);
  const double per_w = 8.0 * ((double)(Smax + 1) * tstep + 2.0 * qw + 12.0 * nx);
  const int G = std::max(1, std::min(nwin, (int)(budget / per_w)));
  const size_t t_ws = (size_t)(Smax + 1) * tstep;
  if ((size_t)std::max(Smax, 1) * G > c->bdts_cap) c->sh_bdts.clear();  // reallocated below
  if ((size_t)G > c->bnst_cap) c->sh_bnst.clear();
  if (ensure_dev(c->d_bt, c->bt_cap, (size_t)G * t_ws, st) ||
      ensure_dev(c->d_bq, c->bq_cap, (size_t)2 * G * qw, st) ||
      ensure_dev(c->d_bg, c->bg_cap, (size_t)G * 12 * nx, st) ||
      ensure_dev(c->d_bdts, c->bdts_cap, (size_t)std::max(Smax, 1) * G, st) ||
      ensure_dev(c->d_bnst, c->bnst_cap, (size_t)G, st))
    return -1;
  const int LE = field ? es_levels(c) : 0;
  const int L = field ? std::max(LE, 1) : fuse_levels(c);
  const int LM = field ? 0 : ms_levels(c);
  std::vector<double> hd((size_t)std::max(Smax, 1) * G);
  std::vector<int> hn(G);
  for (int w0 = 0; w0 < nwin; w0 += G) {
    const int g = std::min(G, nwin - w0);
    for (int k = 0; k < g; ++k) {
      const int w = w0 + k;
      hn[k] = h_nsteps[w];
      for (int s = 0; s < Smax; ++s) hd[(size_t)s * g + k] = s < h_nsteps[w] ? h_dts[off[w] + s] : 0.0;
    }
    // pageable sources: the copies complete before the calls return; an
    // unchanged group (every parareal iteration repeats the schedule) is not
    // uploaded again
    const size_t nd = (size_t)std::max(Smax, 1) * g;
    if (!(c->sh_bnst.size() == (size_t)g && std::memcmp(c->sh_bnst.data(), hn.data(), g * sizeof(int)) == 0)) {
      c->sh_bnst.assign(hn.begin(), hn.begin() + g);
      CK(cudaMemcpyAsync(c->d_bnst, hn.data(), g * sizeof(int), cudaMemcpyHostToDevice, st));
    }
    if (!(c->sh_bdts.size() == nd && std::memcmp(c->sh_bdts.data(), hd.data(), nd * sizeof(double)) == 0)) {
      c->sh_bdts.assign(hd.begin(), hd.begin() + nd);
      CK(cudaMemcpyAsync(c->d_bdts, hd.data(), nd * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    // small grids: the group's windows as one batch per launch (equal step
    // counts; f of the batch in the context's own buffers)
    bool batched = LM > 0 && g >= 2 && g <= c->nsm && h_nsteps[w0] > 0 && !getenv("PBGK_NO_WBATCH") &&
                   8.0 * (double)g * nx * c->g.nvx * c->g.nvy * c->g.nvz <= 256.0 * 1048576.0;
    for (int k = 1; k < g && batched; ++k) batched = h_nsteps[w0 + k] == h_nsteps[w0];
    if (batched) {
      FinalArgs f = fin_args(c, c->plan[0]);
      f.mode = kFinSynthRaw;
      f.mom_in = mom_in + w0 * m5;
      f.tab = c->d_bt;
      FinalBatch fb{0, (long long)m5, 0, (long long)t_ws, c->d_keys + w0};
      {
        ProfScope ps(c, st, 1, 0.0);
        CK(launch_finalize_batch(f, fb, g, st));
      }
      if (run_recursion(c, g, nullptr, c->d_bt, (long long)t_ws, Smax, c->d_bdts, c->d_bnst,
                        c->d_keys + w0, eps, tau, E, e_max, st))
        return -1;
      if (ms_windows_batched(c, LM, g, c->d_bt, (long long)t_ws, h_nsteps[w0], c->d_bdts, c->d_keys + w0,
                             mom_out + w0 * m5, st))
        return -1;
      continue;
    }
    for (int k = 0; k < g; ++k) {
      const int w = w0 + k;
      if (h_nsteps[w] == 0) {  // empty window: the moments themselves
        CK(cudaMemcpyAsync(mom_out + w * m5, mom_in + w * m5, m5 * sizeof(double),
                           cudaMemcpyDeviceToDevice, st));
        continue;
      }
      c->err_slot = c->d_keys + w;
      const int rc = run_final(c, 0, kFinSynthRaw, mom_in + w * m5, nullptr, c->d_bt + k * t_ws, 0, 1,
                               1, nullptr, 0, st);
      c->err_slot = nullptr;
      if (rc) return -1;
    }
    // the batched recursion: steps 1..Smax for the group's windows
    if (run_recursion(c, g, nullptr, c->d_bt, (long long)t_ws, Smax, c->d_bdts, c->d_bnst,
                      c->d_keys + w0, eps, tau, E, e_max, st))
      return -1;
    // each window's passes and its final projection from f
    for (int k = 0; k < g; ++k) {
      const int w = w0 + k, S = h_nsteps[w];
      if (S == 0) continue;
      const double* T = c->d_bt + k * t_ws;
      c->err_slot = c->d_keys + w;
      if (LM > 0) {
        const int rc = ms_window(c, LM, nullptr, f_a, f_b, 0, mom_out + w * m5, T, S, h_dts + off[w], st,
                                 nullptr, 0, c->d_bdts + k, g);
        c->err_slot = nullptr;
        if (rc) return -1;
        continue;
      }
      const int P = (S + L - 1) / L;
      auto buf = [&](int i) { return ((P - i) % 2 == 0) ? f_a : f_b; };
      const double* in = nullptr;
      int s0 = 0, wcount = 0;
      bool projected = false;
      while (s0 < S) {
        const int n = std::min(L, S - s0);
        const double* tabs[kMaxLevels];
        double dtdx[kMaxLevels];
        for (int l = 0; l < n; ++l) {
          tabs[l] = T + (size_t)(s0 + l) * tstep;
          dtdx[l] = h_dts[off[w] + s0 + l] / c->dx;
        }
        if (field && LE > 0 && s0 + n == S && es_final_ok(c)) {
          // the window's last pass: R_S and the projection folded in (no f_S)
          int rcf = run_esweep(c, n, in, nullptr, tabs, h_dts + off[w] + s0, E, e_max, s0 + 1, st,
                               T + (size_t)S * tstep);
          if (rcf == 0) rcf = es_project(c, mom_out + w * m5, T + (size_t)S * tstep, S + 1, st);
          if (rcf) { c->err_slot = nullptr; return -1; }
          projected = true;
          break;
        }
        double* out = buf(++wcount);
        const int rc = (field && LE > 0)
                           ? run_esweep(c, n, in, out, tabs, h_dts + off[w] + s0, E, e_max, s0 + 1, st)
                       : field ? run_sweep(c, 1, true, in, tabs[0], out, dtdx[0], E, 0.5 * e_max,
                                           h_dts[off[w] + s0] / c->dv[0], s0 + 1, st, 1)
                               : run_fsweep(c, n, in, out, tabs, dtdx, s0 + 1, st);
        if (rc) { c->err_slot = nullptr; return -1; }
        in = out;
        s0 += n;
      }
      if (projected) {
        c->err_slot = nullptr;
        continue;
      }
      const int rc1 = run_sweep(c, 0, false, in, T + (size_t)S * tstep, nullptr, 0.0, nullptr, 0.0, 0.0,
                                S, st);
      const int rc2 = rc1 ? rc1 : run_final(c, 0, kFinProject, nullptr, mom_out + w * m5, nullptr, 0, 1, 1,
                                           nullptr, S + 1, st);
      c->err_slot = nullptr;
      if (rc2) return -1;
    }
  }
  return 0;
}
}  // namespace

extern "C" {

int pbgk_propagate(pbgk_ctx* c, const double* f0, const double* mom0, double* f_out, double* f_tmp,
                   int write_final, double* mom_out, int nsteps, const double* h_dts, double eps,
                   double tau, const double* E, double e_max, void* stream, long long* h_code) {
  if (!c || (!f0 && !mom0) || !f_out || !f_tmp || (nsteps > 0 && !h_dts))
    return fail("pbgk_propagate: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  if (f_out == f_tmp || (f0 && (f0 == f_out || f0 == f_tmp)))
    return fail("pbgk_propagate: buffers alias");
  cudaStream_t st = (cudaStream_t)stream;
  if (reset_err(c, st)) return -1;
  c->err_slot = nullptr;
  if (propagate_body(c, f0, mom0, f_out, f_tmp, write_final, mom_out, nsteps, h_dts, eps, tau, E,
                     e_max, st))
    return -1;
  long long code = -1;
  if (fetch_err(c, st, &code)) return -1;
  if (code >= 0 && (int)(code & 0xFF) == kErrSync) {
    // a pass gave up waiting for the concurrent recursion (its SMs were taken
    // by other work): the same propagation with the recursion run serially
    if (reset_err(c, st)) return -1;
    c->no_concurrent = 1;
    const int rc = propagate_body(c, f0, mom0, f_out, f_tmp, write_final, mom_out, nsteps, h_dts, eps,
                                  tau, E, e_max, st);
    c->no_concurrent = 0;
    if (rc) return -1;
    if (fetch_err(c, st, &code)) return -1;
  }
  if (code >= 0 && (int)(code & 0xFF) == kErrNonFiniteMulti) {
    // non-finite somewhere in a multi-step pass: the one-step path finds the step
    if (reset_err(c, st)) return -1;
    c->one_step = 1;
    const int rc = propagate_body(c, f0, mom0, f_out, f_tmp, write_final, mom_out, nsteps, h_dts, eps,
                                  tau, E, e_max, st);
    c->one_step = 0;
    if (rc) return -1;
    if (fetch_err(c, st, &code)) return -1;
  }
  if (h_code) *h_code = code;
  return 0;
}

int pbgk_propagate_windows(pbgk_ctx* c, int nwin, const double* mom_in, double* mom_out,
                           double* f_a, double* f_b, const int* h_nsteps, const double* h_dts,
                           double eps, double tau, const double* E, double e_max, void* stream,
                           long long* h_codes) {
  if (!c || !mom_in || !mom_out || !f_a || !f_b || !h_nsteps || !h_codes)
    return fail("pbgk_propagate_windows: null argument");
  if (f_a == f_b) return fail("pbgk_propagate_windows: buffers alias");
  if (nwin <= 0) return 0;
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  if (nwin > c->keys_cap) {
    CK(cudaStreamSynchronize(st));
    cudaFree(c->d_keys);
    cudaFreeHost(c->h_keys);
    c->d_keys = nullptr;
    c->h_keys = nullptr;
    c->keys_cap = 0;
    CK(cudaMalloc(&c->d_keys, (size_t)nwin * sizeof(ErrKey)));
    CK(cudaMallocHost(&c->h_keys, (size_t)nwin * sizeof(ErrKey)));
    c->keys_cap = nwin;
  }
  CK(cudaMemsetAsync(c->d_keys, 0xFF, (size_t)nwin * sizeof(ErrKey), st));  // kNoError = ~0
  const size_t m = (size_t)5 * c->g.nx;
  const bool field = (E != nullptr && e_max > 0.0);
  int smax = 0;
  for (int w = 0; w < nwin; ++w) smax = std::max(smax, h_nsteps[w]);
  if (fused_ok(c, field) && 8.0 * (smax + 1) * (double)c->g.nx * c->TL <= batch_budget(c)) {
    if (windows_fused(c, nwin, mom_in, mom_out, f_a, f_b, h_nsteps, h_dts, eps, tau, E, e_max, st))
      return -1;
    CK(cudaMemcpyAsync(c->h_keys, c->d_keys, (size_t)nwin * sizeof(ErrKey), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // a window whose first failure is "non-finite somewhere in a multi-step
    // pass" is re-run on the one-step path for its exact key
    std::vector<size_t> offs(nwin + 1, 0);
    for (int w = 0; w < nwin; ++w) offs[w + 1] = offs[w] + h_nsteps[w];
    for (int w = 0; w < nwin; ++w) {
      if (c->h_keys[w] == kNoError || (int)(c->h_keys[w] & 0xFF) != kErrNonFiniteMulti) continue;
      CK(cudaMemsetAsync(c->d_keys + w, 0xFF, sizeof(ErrKey), st));
      c->err_slot = c->d_keys + w;
      c->one_step = 1;
      const int rc = propagate_body(c, nullptr, mom_in + w * m, f_a, f_b, 0, mom_out + w * m,
                                    h_nsteps[w], h_dts + offs[w], eps, tau, E, e_max, st);
      c->one_step = 0;
      c->err_slot = nullptr;
      if (rc) return -1;
      CK(cudaMemcpyAsync(c->h_keys + w, c->d_keys + w, sizeof(ErrKey), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    for (int w = 0; w < nwin; ++w)
      h_codes[w] = (c->h_keys[w] == kNoError) ? -1 : (long long)c->h_keys[w];
    return 0;
  }
  size_t off = 0;
  for (int w = 0; w < nwin; ++w) {
    const int S = h_nsteps[w];
    if (S == 0) {  // empty window: the moments themselves
      CK(cudaMemcpyAsync(mom_out + w * m, mom_in + w * m, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
      continue;
    }
    c->err_slot = c->d_keys + w;
    const int rc = propagate_body(c, nullptr, mom_in + w * m, f_a, f_b, 0, mom_out + w * m, S,
                                  h_dts + off, eps, tau, E, e_max, st);
    c->err_slot = nullptr;
    if (rc) return -1;
    off += S;
  }
  CK(cudaMemcpyAsync(c->h_keys, c->d_keys, (size_t)nwin * sizeof(ErrKey), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int w = 0; w < nwin; ++w)
    h_codes[w] = (c->h_keys[w] == kNoError) ? -1 : (long long)c->h_keys[w];
  return 0;
}

namespace {
// slot 0: window times of the batched G; slot 1: coarse times of the correction
int upload_times(pbgk_ctx* c, int slot, const double* h, size_t n, cudaStream_t st) {
  double*& d = slot == 0 ? c->d_times : c->d_times2;
  size_t& dcap = slot == 0 ? c->times_cap : c->times2_cap;
  std::vector<double>& sh = slot == 0 ? c->sh_times : c->sh_times2;
  if (n > dcap) {
    if (d) {
      CK(cudaStreamSynchronize(st));
      CK(cudaFree(d));
      d = nullptr;
    }
    sh.clear();
    size_t cap = 256;
    while (cap < n) cap *= 2;
    CK(cudaMalloc(&d, cap * sizeof(double)));
    dcap = cap;
  }
  if (sh.size() == n && std::memcmp(sh.data(), h, n * sizeof(double)) == 0) return 0;
  sh.assign(h, h + n);
  // from the context's own copy: it outlives the call
  CK(cudaMemcpyAsync(d, sh.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
  return 0;
}
}  // namespace

int pbgk_fluid_propagate(pbgk_ctx* c, int nwin, const double* mom_in, double* mom_out,
                         const double* minuend, const double* h_t0, const double* h_t1,
                         double dt_max, double cfl, const double* force, void* stream,
                         long long* h_code) {
  if (!c || !mom_in || !mom_out || !h_t0 || !h_t1) return fail("pbgk_fluid_propagate: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  if (nwin <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<double> t(2 * (size_t)nwin);
  for (int w = 0; w < nwin; ++w) {
    t[w] = h_t0[w];
    t[nwin + w] = h_t1[w];
  }
  if (upload_times(c, 0, t.data(), t.size(), st)) return -1;
  if (reset_err(c, st)) return -1;
  FluidArgs a{c->g.nx, c->dx, c->g.bc == 1 ? 1 : 0, dt_max, cfl, force, c->d_err, c->g_model,
              c->g_diff};
  ++g_launches;
  CK(launch_fluid_batch(a, nwin, mom_in, mom_out, minuend, c->d_times, c->d_times + nwin, st));
  return fetch_err(c, st, h_code);
}

int pbgk_parareal_correct(pbgk_ctx* c, int n_g, int start, double* snaps, const double* old,
                          const double* jumps, const double* h_times, double dt_max, double cfl,
                          const double* force, void* stream, double* h_err, long long* h_code) {
  if (!c || !snaps || !old || !jumps || !h_times) return fail("pbgk_parareal_correct: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  if (start < 1) return fail("pbgk_parareal_correct: start < 1");
  cudaStream_t st = (cudaStream_t)stream;
  if (upload_times(c, 1, h_times, (size_t)n_g + 1, st)) return -1;
  if (reset_err(c, st)) return -1;
  FluidArgs a{c->g.nx, c->dx, c->g.bc == 1 ? 1 : 0, dt_max, cfl, force, c->d_err, c->g_model,
              c->g_diff};
  double* d_e = c->d_scratch;
  CK(cudaMemsetAsync(d_e, 0, sizeof(double), st));
  if (start <= n_g) ++g_launches;
  if (start <= n_g) CK(launch_correct(a, n_g, start, snaps, old, jumps, c->d_times2, d_e, st));
  CK(cudaMemcpyAsync(c->h_dbl, d_e, sizeof(double), cudaMemcpyDeviceToHost, st));
  long long code = -1;
  if (fetch_err(c, st, &code)) return -1;
  if (h_code) *h_code = code;
  if (h_err) *h_err = c->h_dbl[0];
  return 0;
}

int pbgk_table_len(const pbgk_ctx* c) { return c ? c->TL : -1; }

int pbgk_ctx_set_quadrature(pbgk_ctx* c, int quadrature) {
  if (!c) return fail("pbgk_ctx_set_quadrature: null context");
  if (quadrature != 0 && quadrature != 1) return fail("pbgk_ctx_set_quadrature: 0 (midpoint) or 1 (trapezoid)");
  const int nv[3] = {c->g.nvx, c->g.nvy, c->g.nvz};
  if (quadrature == 1 && (nv[0] < 2 || nv[1] < 2 || nv[2] < 2))
    return fail("pbgk_ctx_set_quadrature: trapezoidal quadrature needs >= 2 nodes per axis");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  for (int a = 0; a < 3; ++a) {
    c->dv[a] = quadrature == 1 ? 2.0 * c->g.v_max / (nv[a] - 1) : 2.0 * c->g.v_max / nv[a];
    std::vector<double> h(nv[a]);
    for (int j = 0; j < nv[a]; ++j) h[j] = ((double)j - (nv[a] - 1) / 2.0) * c->dv[a];
    if (cudaMemcpy(c->d_c[a], h.data(), nv[a] * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail("cudaMemcpy");
  }
  c->dvol = c->dv[0] * c->dv[1] * c->dv[2];
  c->quad = quadrature;
  return 0;
}

int pbgk_ctx_set_dx(pbgk_ctx* c, double dx) {
  if (!c) return fail("pbgk_ctx_set_dx: null context");
  if (!(dx > 0.0)) return fail("pbgk_ctx_set_dx: dx must be > 0");
  c->dx = dx;
  return 0;
}

namespace {
int slab_check(pbgk_ctx* c, const char* who) {
  if (!c) return fail(std::string(who) + ": null context");
  if (c->g.bc != 3) return fail(std::string(who) + ": needs a slab context (bc 3)");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  return 0;
}
}  // namespace

int pbgk_slab_tables(pbgk_ctx* c, int kind, const double* mom, double* tab_pad, void* stream,
                     long long* h_code) {
  if (slab_check(c, "pbgk_slab_tables")) return -1;
  if (!tab_pad || (kind == 1 && !mom)) return fail("pbgk_slab_tables: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (reset_err(c, st)) return -1;
  // rows 1..nx (row 0 / nx+1 are the halos, filled by the caller)
  if (run_final(c, 0, kind == 1 ? kFinSynthRaw : kFinIdentity, mom, nullptr, tab_pad + c->TL, 0, 1, 1,
                nullptr, 0, st))
    return -1;
  return fetch_err(c, st, h_code);
}

int pbgk_slab_sweep(pbgk_ctx* c, const double* fin_pad, const double* tab_pad, double* fout_pad,
                    double dt, const double* E, double e_max, void* stream) {
  if (slab_check(c, "pbgk_slab_sweep")) return -1;
  if (!tab_pad) return fail("pbgk_slab_sweep: null table");
  if (c->x_scheme == 1 && dt != 0.0) return fail("pbgk_slab_sweep: MUSCL needs two halo planes (upwind only)");
  const bool field = E != nullptr && e_max > 0.0 && dt != 0.0;
  const int pid = field ? 1 : 0;
  return run_sweep(c, pid, field, fin_pad, tab_pad, fout_pad, dt / c->dx, E, 0.5 * e_max,
                   dt / c->dv[0], 0, (cudaStream_t)stream);
}

int pbgk_slab_finalize(pbgk_ctx* c, int mode, int field, double* tab_pad, double* mom_out,
                       double dt, double eps, double tau, int step, void* stream, long long* h_code) {
  if (slab_check(c, "pbgk_slab_finalize")) return -1;
  if ((mode == 0 && !tab_pad) || (mode == 1 && !mom_out)) return fail("pbgk_slab_finalize: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  // no reset: failure keys accumulate (atomicMin) from pbgk_slab_tables on,
  // and are only read back (synchronising) when h_code is given
  const int pid = field ? 1 : 0;
  if (mode == 0) {
    if (run_final(c, pid, kFinRelax, nullptr, nullptr, tab_pad + c->TL, dt, eps, tau, nullptr, step, st))
      return -1;
  } else {
    if (run_final(c, pid, kFinProject, nullptr, mom_out, nullptr, 0, 1, 1, nullptr, step, st))
      return -1;
  }
  return fetch_err(c, st, h_code);
}

int pbgk_set_x_scheme(pbgk_ctx* c, int scheme) {
  if (!c) return fail("pbgk_set_x_scheme: null context");
  if (scheme != 0 && scheme != 1) return fail("pbgk_set_x_scheme: scheme must be 0 (upwind) or 1 (MUSCL)");
  c->x_scheme = scheme;
  return 0;
}

int pbgk_set_fusion(pbgk_ctx* c, int levels) {
  if (!c) return fail("pbgk_set_fusion: null context");
  if (levels < -1 || levels > 4) return fail("pbgk_set_fusion: levels must be -1 (auto), 0 (off) .. 4");
  c->fuse = levels;
  return 0;
}

int pbgk_set_esweep(pbgk_ctx* c, int on) {
  if (!c) return fail("null context");
  c->es = on != 0;
  return 0;
}

int pbgk_esweep_levels(pbgk_ctx* c) { return c ? es_levels(c) : 0; }

int pbgk_set_msweep(pbgk_ctx* c, int on, int levels) {
  if (!c) return fail("null context");
  if (levels != 0 && levels != 4 && levels != 8) return fail("msweep levels must be 0 (auto), 4 or 8");
  c->ms = on != 0;
  c->ms_levels = levels;
  return 0;
}

int pbgk_msweep_levels(pbgk_ctx* c) { return c ? ms_levels(c) : -1; }

int pbgk_set_batch_bytes(pbgk_ctx* c, double bytes) {
  if (!c) return fail("null context");
  if (!(bytes >= 0.0)) return fail("batch bytes must be >= 0");
  c->batch_bytes = bytes;
  return 0;
}

int pbgk_set_grid_reserve(pbgk_ctx* c, int slots) {
  if (!c) return fail("pbgk_set_grid_reserve: null context");
  if (slots < 0 || slots >= c->nsm) return fail("pbgk_set_grid_reserve: need 0 <= slots < SM count");
  c->slot_reserve = slots;
  return 0;
}

int pbgk_fluid_propagate_async(pbgk_ctx* c, int nwin, const double* mom_in, double* mom_out,
                               const double* minuend, const double* d_t0, const double* d_t1,
                               double dt_max, double cfl, const double* force, void* stream,
                               long long* d_status) {
  if (!c || !mom_in || !mom_out || !d_t0 || !d_t1 || !d_status)
    return fail("pbgk_fluid_propagate_async: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  if (nwin <= 0) return 0;
  FluidArgs a{c->g.nx, c->dx, c->g.bc == 1 ? 1 : 0, dt_max, cfl, force,
              reinterpret_cast<ErrKey*>(d_status), c->g_model, c->g_diff};
  ++g_launches;
  CK(launch_fluid_batch(a, nwin, mom_in, mom_out, minuend, d_t0, d_t1, (cudaStream_t)stream, true));
  return 0;
}

int pbgk_parareal_correct_range(pbgk_ctx* c, int first, int last, double* snaps, const double* old,
                                const double* jumps, const double* d_times, double dt_max,
                                double cfl, const double* force, void* stream, double* d_errmax,
                                long long* d_status) {
  if (!c || !snaps || !old || !jumps || !d_times || !d_errmax || !d_status)
    return fail("pbgk_parareal_correct_range: null argument");
  if (cudaSetDevice(c->dev) != cudaSuccess) return fail("cudaSetDevice");
  if (first < 1) return fail("pbgk_parareal_correct_range: first < 1");
  if (last < first) return 0;
  FluidArgs a{c->g.nx, c->dx, c->g.bc == 1 ? 1 : 0, dt_max, cfl, force,
              reinterpret_cast<ErrKey*>(d_status), c->g_model, c->g_diff};
  ++g_launches;
  CK(launch_correct(a, last, first, snaps, old, jumps, d_times, d_errmax, (cudaStream_t)stream, true));
  return 0;
}

int pbgk_fluid_model(pbgk_ctx* c, int model, double diffusivity) {
  if (!c) return fail("pbgk_fluid_model: null context");
  if (model != 0 && model != 1) return fail("pbgk_fluid_model: model must be 0 (Euler) or 1 (drift-diffusion)");
  if (model == 1 && !(diffusivity > 0.0)) return fail("pbgk_fluid_model: diffusivity must be > 0");
  c->g_model = model;
  c->g_diff = diffusivity;
  return 0;
}

}  // extern "C"
