// Sweep kernel instantiations, part c (split for a parallel build; the
// kernel is in sweep_impl.cuh, the dispatch in sweep.cu).
#include "sweep_impl.cuh"

namespace pbgk {

cudaError_t launch_sweep_c(int cfg_id, const CUtensorMap& map, const SweepArgs& a, bool synth,
                           bool field, int grid, int ns, size_t smem, cudaStream_t st) {
  switch (cfg_id) {
    case 7: return launch_cfg<3, 16, 4, 256, 1, true, 11>(map, a, synth, field, grid, ns, smem, st);
    case 8: return launch_cfg<2, 16, 4, 256, 1, true, 11>(map, a, synth, field, grid, ns, smem, st);
    case 9: return launch_cfg<2, 8, 4, 256, 1, true, 11>(map, a, synth, field, grid, ns, smem, st);
    case 10: return launch_cfg<2, 4, 4, 256, 1, true, 11>(map, a, synth, field, grid, ns, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pbgk
