// Sweep dispatch: shared-memory sizing and the switch from a configuration id
// (capi.cu make_plan) to the translation unit that instantiates that shape
// (sweep_a/b/c.cu).  The kernel itself and its design are in sweep_impl.cuh.
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
