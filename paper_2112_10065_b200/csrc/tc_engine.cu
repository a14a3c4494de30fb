// tcgen05 engine -- placeholder: no shapes taken yet (all calls go to the
// FFMA engine).  Replaced by the tensor-core implementation.
#include "tc_api.h"

namespace bpx {
bool tc_conv_fwd_ok(int, int, int, int, int) { return false; }
bool tc_conv_dgrad_ok(int, int, int, int, int) { return false; }
bool tc_conv_wgrad_ok(int, int, int, int, int) { return false; }
bool tc_linear_ok(int, int, int) { return false; }
size_t tc_conv_fwd_ws(int, int, int, int, int) { return 0; }
size_t tc_conv_dgrad_ws(int, int, int, int, int) { return 0; }
size_t tc_conv_wgrad_ws(int, int, int, int, int) { return 0; }
size_t tc_linear_fwd_ws(int, int, int) { return 0; }
size_t tc_linear_dgrad_ws(int, int, int) { return 0; }
size_t tc_linear_wgrad_ws(int, int, int) { return 0; }
bpx_status_t tc_conv_fwd(const float*, const float*, const float*, float*, int, int, int,
                         int, int, int, void*, size_t, cudaStream_t) { return BPX_ERR_UNSUPPORTED; }
bpx_status_t tc_conv_dgrad(const float*, const float*, const float*, float*, int, int, int,
                           int, int, void*, size_t, cudaStream_t) { return BPX_ERR_UNSUPPORTED; }
bpx_status_t tc_conv_wgrad(const float*, const float*, float*, float*, int, int, int, int,
                           int, void*, size_t, cudaStream_t) { return BPX_ERR_UNSUPPORTED; }
bpx_status_t tc_linear_fwd(const float*, const float*, const float*, float*, int, int, int,
                           int, void*, size_t, cudaStream_t) { return BPX_ERR_UNSUPPORTED; }
bpx_status_t tc_linear_dgrad(const float*, const float*, const float*, float*, int, int,
                             int, void*, size_t, cudaStream_t) { return BPX_ERR_UNSUPPORTED; }
bpx_status_t tc_linear_wgrad(const float*, const float*, float*, float*, int, int, int,
                             void*, size_t, cudaStream_t) { return BPX_ERR_UNSUPPORTED; }
}  // namespace bpx
