// Sweep kernel instantiations, part a (split for a parallel build; the
// kernel is in sweep_impl.cuh, the dispatch in sweep.cu).
#include "sweep_impl.cuh"

namespace pbgk {

cudaError_t launch_sweep_a(int cfg_id, const CUtensorMap& map, const SweepArgs& a, bool synth,
                           bool field, int grid, int ns, size_t smem, cudaStream_t st) {
  switch (cfg_id) {
    case 0: return launch_cfg<2, 32, 4, 256, 2, true, 15>(map, a, synth, field, grid, ns, smem, st);
    case 1: return launch_cfg<3, 16, 4, 256, 2, true, 5>(map, a, synth, field, grid, ns, smem, st);
    case 2: return launch_cfg<2, 16, 4, 256, 2, true, 13>(map, a, synth, field, grid, ns, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pbgk
