// gs_bin_sort path B placeholder: falls back to path A until the bucketed binning lands.
#include "gs_internal.cuh"

namespace gs {
gs_status run_bin_sort_bucket(WsState* s, int64_t* n_keys, uint32_t flags, cudaStream_t st) {
    return run_bin_sort_keys(s, n_keys, flags | GS_FLAG_BINSORT_KEYS, st);
}
}  // namespace gs
