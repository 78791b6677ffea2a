// The key-centric backward kernels of degree L = 0 (see attention_bwd.cuh).
#define ES_BWD_DEFINE
#include "attention_bwd.cuh"

namespace es {
template es_status bwd_run_L<0>(const AttnArgs&, const int*, const void*, const void*, const void*, const double*,
                                const int32_t*, const int32_t*, const int32_t*, const void*, const float*,
                                const void*, void*, void*, void*, float*, float*, double*, bool, bool, cudaStream_t);
}  // namespace es
