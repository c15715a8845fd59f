// Stub kernel launchers for the sanitizer build of the host model compiler
// (tests/test_sanitizers.py): odf_capi.cu compiled with -fsanitize=address,undefined
// and linked against these instead of the sm_100a kernels.  On a host without a
// GPU every load returns ODF_E_CUDA after the whole host-side compile has run.
#include "../../paper_2205_07307_b200/csrc/odf_internal.h"

namespace odf {
cudaError_t prepare_kernels(int) { return cudaErrorNotSupported; }
int occupancy_main(int, int, size_t, int) { return 1; }
cudaError_t launch_main(int, int, const KParams &, const CUtensorMap *, int, size_t, cudaStream_t, int, bool)
{
    return cudaErrorNotSupported;
}
cudaError_t launch_index(int, const KParams &, bool, int, size_t, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_latency(int, const KParams &, const CUtensorMap *, int, size_t, size_t, cudaStream_t)
{
    return cudaErrorNotSupported;
}
cudaError_t launch_bits(int, const KParams &, bool, size_t, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace odf
