// Fused stage kernel instantiations for nf = 6 fields (see hydro_stage.cuh).
#include "hydro_stage.cuh"

namespace tsh {
template cudaError_t launch_stage_n<6>(const StageArgs&, int, int, int, cudaStream_t, bool);
}  // namespace tsh

#ifdef TS_RCP_CHECK
// Diagnostic build only (TS_DEFINES="-DTS_FAST_RCP=1 -DTS_RCP_CHECK"): the
// operands the nf = 6 stage kernels saw where rcp_rn != 1.0 / x.
extern "C" long long ts_debug_rcp_bad(double* out, int cap) {
    unsigned long long n = 0;
    if (cudaMemcpyFromSymbol(&n, tsh::g_rcp_bad_n, sizeof(n)) != cudaSuccess) return -1;
    double buf[64][3];
    if (cudaMemcpyFromSymbol(buf, tsh::g_rcp_bad, sizeof(buf)) != cudaSuccess) return -1;
    for (int i = 0; i < cap && i < 64 && i < (int)n; ++i)
        for (int k = 0; k < 3; ++k) out[3 * i + k] = buf[i][k];
    return (long long)n;
}
#endif
