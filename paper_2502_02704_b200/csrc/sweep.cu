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
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace pbgk {

cudaError_t launch_sweep_a(int, const CUtensorMap&, const SweepArgs&, bool, bool, int, int, size_t,
                           cudaStream_t);
cudaError_t launch_sweep_b(int, const CUtensorMap&, const SweepArgs&, bool, bool, int, int, size_t,
                           cudaStream_t);
cudaError_t launch_sweep_c(int, const CUtensorMap&, const SweepArgs&, bool, bool, int, int, size_t,
                           cudaStream_t);

size_t sweep_smem_bytes(const SweepArgs& a, int V, int LZ, int NTHR, bool synth, bool tma, int ns) {
  const int BZ = LZ * V;
  const size_t box = synth ? 0 : (size_t)a.t.rows_load * a.t.By * BZ * 8;
  const size_t stage = (box + (size_t)a.TL * 8 + 127) & ~(size_t)127;
  const size_t lines = (size_t)a.t.A * a.t.By;
  if (!tma) ns = 1;
  return (size_t)ns * stage + 2 * lines * 8 + 2 * (size_t)(NTHR / 32) * BZ * 8 +
         (size_t)((a.nvx + 1) & ~1) * 8 + (size_t)ns * 8 + 16;
}

cudaError_t launch_sweep(int cfg_id, const CUtensorMap& map, const SweepArgs& a, bool synth,
                         bool field, int grid, int ns, size_t smem, cudaStream_t st) {
  switch (cfg_id) {
    case 0: return launch_sweep_a(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 1: return launch_sweep_a(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 2: return launch_sweep_a(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 3: return launch_sweep_b(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 4: return launch_sweep_b(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 5: return launch_sweep_b(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 7: return launch_sweep_c(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 8: return launch_sweep_c(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 9: return launch_sweep_c(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 10: return launch_sweep_c(cfg_id, map, a, synth, field, grid, ns, smem, st);
    case 11: return launch_sweep_b(cfg_id, map, a, synth, field, grid, ns, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pbgk
