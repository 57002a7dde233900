// Fused stage kernel instantiations for nf = 6 fields (see hydro_stage.cuh).
#include "hydro_stage.cuh"

namespace tsh {
template cudaError_t launch_stage_n<6>(const StageArgs&, int, int, int, cudaStream_t, bool);
}  // namespace tsh
