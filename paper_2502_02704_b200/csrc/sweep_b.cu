// Sweep kernel instantiations, part b (split for a parallel build; the
// kernel is in sweep_impl.cuh, the dispatch in sweep.cu).
#include "sweep_impl.cuh"

namespace pbgk {

cudaError_t launch_sweep_b(int cfg_id, const CUtensorMap& map, const SweepArgs& a, bool synth,
                           bool field, int grid, int ns, size_t smem, cudaStream_t st) {
  switch (cfg_id) {
    case 3: return launch_cfg<2, 8, 4, 256, 2, true, 13>(map, a, synth, field, grid, ns, smem, st);
    case 4: return launch_cfg<2, 4, 4, 256, 2, true, 13>(map, a, synth, field, grid, ns, smem, st);
    case 5: return launch_cfg<1, 32, 4, 256, 2, false, 15>(map, a, synth, field, grid, ns, smem, st);
    case 11: return launch_cfg<6, 8, 2, 256, 2, true, 9>(map, a, synth, field, grid, ns, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pbgk
