// Multi-step sweep: L fine steps of f per pass, no reductions.
//
// With the relax tables of every step computed beforehand by the marginal
// recursion (marginal.cu), step s+1 of ref/kinetic.py:152-160 needs nothing
// grid-wide: f*_{s+1}(i) = T(R_s(f*_s))(i) depends on the cell itself and its
// upwind neighbour plane only.  A tile marching in x (sweep_impl.cuh) can then
// run L steps at once: every level keeps the upwind flux of the previous plane
// in registers, level l+1 relaxes level l's output with its own table row and
// transports it, and only the last level is stored.  HBM traffic per
// cell-update drops from 16 B to 16/L B.
//
// Halo: a tile run that starts at plane p0 is preceded by L lead items at
// p0-L .. p0-1; lead item k (depth k) completes levels < k and relaxes level k
// (its flux becomes `prev` for the next plane).  Ghost planes: absorbing =
// zero flux at every level; periodic = wrap; outflow = the edge plane again,
// which reproduces the zero-gradient ghost at every level (the edge cell's
// inflow flux difference is exactly zero).
//
// Rounding: the transport is evaluated as (1 -/+ a) x +/- q_neighbour with
// q = a x, a = (dt/dx) c_x (2 ops per element instead of the reference's 4),
// within a few ulps of ref/kinetic.py:110-112; the multi-step path is held to
// the oracle at 1e-12 (tests/test_gpu_fused.py) like every multi-step run.
//
// Finiteness (ref/kinetic.py:157-159): each thread sums its stored (last
// level) values; a non-finite value at any level stays non-finite in the same
// element through the later levels, so a non-finite sum means "some step of
// this pass" -- status kind 6, on which the host re-runs the propagation on
// the one-step path to report the exact BlowUpError(step) (same documented
// corner as the marginal check: finite values whose sum overflows).  Per-level
// sums (PBGK_FS_LASTACC=0) cost 9 % on config 4.
#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"
#include "sweep_impl.cuh"

namespace pbgk {

template <int V, int LZ, int K, int NTHR, int MINB, bool SYNTH, int L>
__global__ void __launch_bounds__(NTHR, MINB)
    fsweep_kernel(const __grid_constant__ CUtensorMap fmap, const FSweepArgs a, int ns) {
  constexpr int NL = NTHR / LZ;
  constexpr int BZ = LZ * V;
#ifndef PBGK_FS_PR
#define PBGK_FS_PR 2
#endif
#ifndef PBGK_FS_LK
#define PBGK_FS_LK 0
#endif
#ifndef PBGK_FS_DECOUPLE
#define PBGK_FS_DECOUPLE 0
#endif
#ifndef PBGK_FS_LASTACC
#define PBGK_FS_LASTACC 1
#endif
#ifndef PBGK_FS_LATE
#define PBGK_FS_LATE 1
#endif
  constexpr int PR = PBGK_FS_PR;  // planes per round of the steady path (needs ns >= 2 PR)
  extern __shared__ __align__(128) unsigned char smem[];

  const Tiling& T = a.t;
  const int tid = threadIdx.x;
  const int lz = tid % LZ;
  const int lg = tid / LZ;
  const int lines = T.A * T.By;
  const int lgBy = __ffs(T.By) - 1;
  const int nx = a.nx;

  const uint32_t box_bytes = SYNTH ? 0u : (uint32_t)(T.A * T.By * BZ) * 8u;
  const uint32_t tab_bytes = (uint32_t)(a.TL * 8);
  const uint32_t stage_bytes = (box_bytes + L * tab_bytes + 127u) & ~127u;
  double* SCX = reinterpret_cast<double*>(smem + (size_t)ns * stage_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(SCX + ((a.nvx + 1) & ~1));

  const int g0 = (int)((a.total * blockIdx.x) / gridDim.x);
  const int g1 = (int)((a.total * (blockIdx.x + 1)) / gridDim.x);

  for (int j = tid; j < a.nvx; j += NTHR) SCX[j] = a.cx[j];
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) mbar_init(&bars[s], 1);
#if PBGK_FS_DECOUPLE
    for (int s = 0; s < ns; ++s) mbar_init(&bars[ns + s], NTHR / 32);  // stage empty: one arrive per warp
#endif
    fence_mbar_init();
  }
  pdl_wait();
  pdl_trigger();
  __syncthreads();

  const int ptid = NTHR - 32;
  ItemIter<L, 0> prod;
  prod.init(g0, g1, nx);
  int pstg = 0, ptile = -1;
  TileGeom ptg{};
  auto issue_next = [&]() {
    int t, p, h;
    prod.next(nx, t, p, h);
    if (t != ptile) {
      ptile = t;
      ptg = tile_geom(T, a.nvx, t);
    }
    const int i = item_plane(nx, a.bc, ptg, p);
    const int s = pstg;
    if (++pstg == ns) pstg = 0;
    uint64_t* bar = &bars[s];
    unsigned char* st = smem + (size_t)s * stage_bytes;
    if (i < 0) {
      mbar_arrive_expect_tx(bar, 0);
      return;
    }
    mbar_arrive_expect_tx(bar, box_bytes + L * tab_bytes);
    if (!SYNTH) tma_load_4d(st, &fmap, ptg.z0, ptg.y0, ptg.r0, i, bar);
#pragma unroll
    for (int l = 0; l < L; ++l)
      tma_load_1d(st + box_bytes + l * tab_bytes, a.tab[l] + (size_t)i * a.TL, tab_bytes, bar);
  };
  if (tid == ptid) {
    prefetch_tensormap(&fmap);
    if (a.prog != nullptr) {
      // the recursion runs concurrently (other SMs): wait for this pass's
      // tables, then order the async-proxy (bulk copy) reads after them.
      // Bounded (~5 s): a stalled recursion becomes an error, not a hang.
      long long spins = 0;
      while (ld_acquire_gpu(a.prog) < a.need) {
        __nanosleep(256);
        if (++spins > 20000000LL) {
          atomicMin(a.err, err_key(0, a.step0, kErrSync));
          break;
        }
      }
      fence_proxy_async();
    }
    for (int s = 0; s < ns && !prod.done(); ++s) issue_next();
  }

  int soff[K], lab[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    int l = lg + k * NL;
    if (l >= lines) l = 0;
    const int aa = l >> lgBy, b = l & (T.By - 1);
    soff[k] = (aa * T.By + b) * BZ + zpos<V, LZ>(lz, 0);
    lab[k] = (aa << 16) | b;
  }
  int gxi[K], gyi[K], goff[K];
  double cvx[K];
  unsigned vmask = 0, zmask = 0;
  bool full = false;
  TileGeom tg{};

  double prev[L][K][V];
#pragma unroll
  for (int l = 0; l < L; ++l)
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int v = 0; v < V; ++v) prev[l][k][v] = 0.0;
  double acc[L];
#pragma unroll
  for (int l = 0; l < L; ++l) acc[l] = 0.0;

  // consumer: the producer's item order (ItemIter<L, 0>), walked as runs of
  // one tile: L lead items (depth 0..L-1, generic path), then the run's
  // planes (depth L) on a lean path with no per-item bookkeeping beyond the
  // stage ring
  int stg = 0;
  uint32_t ph = 0;
  int g = g0;
  while (g < g1) {
    const int t = g / nx;
    const int p0 = g - t * nx;
    const int p1 = min(nx, p0 + (g1 - g));
    g += p1 - p0;
    tg = tile_geom(T, a.nvx, t);
    vmask = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int l = lg + k * NL;
      int jx = tg.r0 + (lab[k] >> 16), jy = tg.y0 + (lab[k] & 0xffff);
      if (l < lines && jx < tg.r1 && jy < a.nvy) vmask |= 1u << k;
      jx = min(jx, a.nvx - 1);
      jy = min(jy, a.nvy - 1);
      gxi[k] = a.gxo + jx;
      gyi[k] = a.gyo + jy;
      goff[k] = (jx * a.nvy + jy) * a.nvz + tg.z0 + zpos<V, LZ>(lz, 0);
      cvx[k] = SCX[jx];
    }
    zmask = 0;
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (tg.z0 + zpos<V, LZ>(lz, v) < a.nvz) zmask |= 1u << v;
    full = (vmask == (1u << K) - 1) && (zmask == (1u << V) - 1);
    // one item: plane i (-1 = absorbing ghost), `depth` levels completed;
    // `sync`: end a round (CTA barrier, the producer refills the `nfree`
    // stages the round consumed)
    auto item = [&](int i, int depth, bool sync, int nfree) {
      const double* SF = reinterpret_cast<const double*>(smem + (size_t)stg * stage_bytes);
      mbar_wait(&bars[stg], ph);
      if (i < 0) {
        // absorbing ghost plane: zero flux at every level
#pragma unroll
        for (int l = 0; l < L; ++l)
#pragma unroll
          for (int k = 0; k < K; ++k)
#pragma unroll
            for (int v = 0; v < V; ++v) prev[l][k][v] = 0.0;
      } else {
        double* gdst = (depth == L) ? a.fout + (size_t)i * a.plane : nullptr;
      // per level: relax factors and this lane's g_z values of the plane's row
#if PBGK_FS_LATE
        // (late variant: each (line, level) step reads its table factors)
        constexpr int LP = 1;
#else
        constexpr int LP = L;
#endif
        double rr[LP], lss[LP], gz[LP][V];
#pragma unroll
        for (int l = 0; l < LP && !PBGK_FS_LATE; ++l) {
          const double* ST = reinterpret_cast<const double*>(
              reinterpret_cast<const unsigned char*>(SF) + box_bytes + l * tab_bytes);
          rr[l] = ST[0];
          lss[l] = ST[1];
          if (zmask == (1u << V) - 1) {
            lds_lane<V, LZ>(ST + a.gzo + tg.z0 + zpos<V, LZ>(lz, 0), gz[l]);
          } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
              gz[l][v] = ((zmask >> v) & 1u) ? ST[a.gzo + tg.z0 + zpos<V, LZ>(lz, v)] : 0.0;
          }
        }
        auto body = [&](auto fast_c, auto down_c) {
          constexpr bool FAST = decltype(fast_c)::value;
          constexpr bool DOWNT = decltype(down_c)::value;
          // level l of line k: relax, transport, carry, store at the last level
          auto step = [&](int k, int l, double (&x)[V]) {
            const double c = cvx[k];
            const double* ST = reinterpret_cast<const double*>(
                reinterpret_cast<const unsigned char*>(SF) + box_bytes + l * tab_bytes);
            const double gxy = ST[gxi[k]] * ST[gyi[k]];
#if PBGK_FS_LATE
            double rl = ST[0], lsl = ST[1], gzl[V];
            if (FAST || zmask == (1u << V) - 1) {
              lds_lane<V, LZ>(ST + a.gzo + tg.z0 + zpos<V, LZ>(lz, 0), gzl);
            } else {
#pragma unroll
              for (int v = 0; v < V; ++v)
                gzl[v] = ((zmask >> v) & 1u) ? ST[a.gzo + tg.z0 + zpos<V, LZ>(lz, v)] : 0.0;
            }
#define PBGK_RR rl
#define PBGK_LS lsl
#define PBGK_GZ(v) gzl[v]
#else
#define PBGK_RR rr[l]
#define PBGK_LS lss[l]
#define PBGK_GZ(v) gz[l][v]
#endif
            // relax R of this level (level 0 of a synthesising pass: f_0 = L(U))
            if (l == 0 && SYNTH) {
#pragma unroll
              for (int v = 0; v < V; ++v) x[v] = (gxy * PBGK_GZ(v)) * PBGK_LS;
            } else {
              double raw[V];
              if (l == 0) {
                lds_lane<V, LZ>(SF + soff[k], raw);
              } else {
#pragma unroll
                for (int v = 0; v < V; ++v) raw[v] = x[v];
              }
              const double w = PBGK_RR * (PBGK_LS * gxy);
#pragma unroll
              for (int v = 0; v < V; ++v) x[v] = fma(w, PBGK_GZ(v), PBGK_RR * raw[v]);
            }
#undef PBGK_RR
#undef PBGK_LS
#undef PBGK_GZ
            // upwind transport of ref/kinetic.py:110-112 with a = (dt/dx) c_x:
            // up (c >= 0)  f* = x - a (x - x_{i-1}) = (1 - a) x + q_{i-1}
            // down (c < 0) f* = x - a (x_{i+1} - x) = (1 + a) x - q_{i+1}
            // with q = a x carried per level (2 fp64 ops per element instead of
            // 4; a few ulps from the reference's order, see the header)
            const double av = a.dtdx[l] * c;
            const double keep = DOWNT ? 1.0 + av : 1.0 - av;
            double q[V];
#pragma unroll
            for (int v = 0; v < V; ++v) q[v] = av * x[v];
            if (FAST || l < depth) {
#pragma unroll
              for (int v = 0; v < V; ++v) x[v] = DOWNT ? fma(keep, x[v], -prev[l][k][v]) : fma(keep, x[v], prev[l][k][v]);
            }
#pragma unroll
            for (int v = 0; v < V; ++v) prev[l][k][v] = q[v];
            if ((FAST || depth == L) && (!PBGK_FS_LASTACC || l == L - 1)) {
              const bool ok = FAST || ((vmask >> k) & 1u);
              double sl = 0.0;
#pragma unroll
              for (int v = 0; v < V; ++v) sl += (FAST || (ok && ((zmask >> v) & 1u))) ? x[v] : 0.0;
              acc[l] += sl;
              if (l == L - 1 && (FAST || ok)) store_line<V, LZ, FAST>(gdst + goff[k], x, zmask);
            }
          };
#if PBGK_FS_LK
          // levels outer, lines inner: the K lines' chains interleave per level
          double x[K][V];
#pragma unroll
          for (int l = 0; l < L; ++l) {
            if (!FAST && l > depth) break;
#pragma unroll
            for (int k = 0; k < K; ++k) step(k, l, x[k]);
          }
#else
#pragma unroll
          for (int k = 0; k < K; ++k) {
            double x[V];
#pragma unroll
            for (int l = 0; l < L; ++l) {
              if (!FAST && l > depth) break;
              step(k, l, x);
            }
          }
#endif
        };
        using T1 = std::integral_constant<bool, true>;
        using F1 = std::integral_constant<bool, false>;
        if (full && depth == L) {
          if (tg.down) body(T1{}, T1{}); else body(T1{}, F1{});
        } else {
          if (tg.down) body(F1{}, T1{}); else body(F1{}, F1{});
        }
      }
#if PBGK_FS_DECOUPLE
      // no CTA barrier: every warp marks the stage consumed; the producer
      // refills it once all warps have (warps run up to ns items apart)
      (void)sync;
      (void)nfree;
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&bars[ns + stg]);
      if (tid == ptid && !prod.done()) {
        mbar_wait(&bars[ns + stg], ph);
        fence_proxy_async();
        issue_next();
      }
#else
      if (sync) {
        __syncthreads();  // the round's stages are consumed: the producer may refill them
        if (tid == ptid) {
          fence_proxy_async();
          for (int q = 0; q < nfree && !prod.done(); ++q) issue_next();
        }
      }
#endif
      if (++stg == ns) {
        stg = 0;
        ph ^= 1u;
      }
    };
    for (int k = 0; k < L; ++k) item(item_plane(nx, a.bc, tg, p0 - L + k), k, true, 1);
    // the run's planes PR per round (one barrier per round; the upwind carry
    // goes from plane to plane in registers)
    int p = p0;
    for (; p + PR <= p1; p += PR) {
#pragma unroll 1
      for (int q = 0; q < PR - 1; ++q) item(tg.down ? nx - 1 - p - q : p + q, L, false, 0);
      item(tg.down ? nx - PR - p : p + PR - 1, L, true, PR);
    }
    for (; p < p1; ++p) item(tg.down ? nx - 1 - p : p, L, true, 1);
  }
#if PBGK_FS_LASTACC
  // only the stored level is summed (a non-finite value at any level stays
  // non-finite in the same element through the later ones): the failing step
  // is one of this pass's, and the host finds it on the one-step path
  if (!isfinite(acc[L - 1]))
    atomicMin(a.err, err_key(0, a.step0, L == 1 ? kErrNonFinite : kErrNonFiniteMulti));
#else
#pragma unroll
  for (int l = 0; l < L; ++l)
    if (!isfinite(acc[l])) atomicMin(a.err, err_key(0, a.step0 + l, kErrNonFinite));
#endif
}

size_t fsweep_smem_bytes(const FSweepArgs& a, int V, int LZ, bool synth, int L, int ns) {
  const int BZ = LZ * V;
  const size_t box = synth ? 0 : (size_t)a.t.A * a.t.By * BZ * 8;
  const size_t stage = (box + (size_t)L * a.TL * 8 + 127) & ~(size_t)127;
  return (size_t)ns * stage + (size_t)((a.nvx + 1) & ~1) * 8 + (size_t)2 * ns * 8 + 16;
}

template <int V, int LZ, int K, int NTHR, int MINB, int L>
static cudaError_t launch_l(const CUtensorMap& map, const FSweepArgs& a, bool synth, int grid, int ns,
                            size_t smem, cudaStream_t st) {
  void (*fn)(const CUtensorMap, const FSweepArgs, int) =
      synth ? fsweep_kernel<V, LZ, K, NTHR, MINB, true, L> : fsweep_kernel<V, LZ, K, NTHR, MINB, false, L>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (a.prog != nullptr) {
    // concurrent recursion: no programmatic early launch -- a second pass's
    // CTAs waiting on the first would take the SMs reserved for the recursion
    fn<<<grid, NTHR, smem, st>>>(map, a, ns);
    return cudaGetLastError();
  }
  return launch_pdl(fn, grid, NTHR, smem, st, map, a, ns);
}

// L = 1: the upwind sweep's CTA shape (256 threads, K lines each, 2 CTAs/SM);
// L >= 2: the same box lines with K/2 lines per thread, one CTA per SM (several
// levels of upwind carries per line do not fit 128 registers at K): 2-wide
// lane layouts as 4-wide lanes on 256 threads (255 registers, 8 elements per
// thread per item: measured 5 % faster than 2-wide on 512 threads), the
// 48-wide V = 6 layout on 512 threads
template <int V, int LZ, int K>
static cudaError_t launch_f(const CUtensorMap& map, const FSweepArgs& a, bool synth, int L, int grid,
                            int ns, size_t smem, cudaStream_t st) {
#ifndef PBGK_FS_WIDE
#define PBGK_FS_WIDE 1
#endif
  // PBGK_FS_WIDE (V = 2 shapes): the same box lines as 2V-wide lanes on 256
  // threads, 1 CTA/SM with up to 255 registers (twice the elements per thread)
  constexpr bool WIDE = PBGK_FS_WIDE && V == 2;
  constexpr int V2 = WIDE ? 2 * V : V, LZ2 = WIDE ? LZ / 2 : LZ, T2 = WIDE ? 256 : 512;
  switch (L) {
    case 1: return launch_l<V, LZ, K, 256, 2, 1>(map, a, synth, grid, ns, smem, st);
    case 2: return launch_l<V2, LZ2, K / 2, T2, 1, 2>(map, a, synth, grid, ns, smem, st);
    case 3: return launch_l<V2, LZ2, K / 2, T2, 1, 3>(map, a, synth, grid, ns, smem, st);
    case 4: return launch_l<V2, LZ2, K / 2, T2, 1, 4>(map, a, synth, grid, ns, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

int fsweep_ctas_per_sm(int L) { return L >= 2 ? 1 : 2; }

// Shapes: the TMA tile shapes of the upwind sweep (capi.cu kCfg ids).
cudaError_t launch_fsweep(int cfg_id, const CUtensorMap& map, const FSweepArgs& a, bool synth, int L,
                          int grid, int ns, size_t smem, cudaStream_t st) {
  switch (cfg_id) {
    case 0: return launch_f<2, 32, 4>(map, a, synth, L, grid, ns, smem, st);
    case 2: return launch_f<2, 16, 4>(map, a, synth, L, grid, ns, smem, st);
    case 3: return launch_f<2, 8, 4>(map, a, synth, L, grid, ns, smem, st);
    case 4: return launch_f<2, 4, 4>(map, a, synth, L, grid, ns, smem, st);
    case 11: return launch_f<6, 8, 2>(map, a, synth, L, grid, ns, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

bool fsweep_has_cfg(int cfg_id) {
  return cfg_id == 0 || cfg_id == 2 || cfg_id == 3 || cfg_id == 4 || cfg_id == 11;
}

}  // namespace pbgk
