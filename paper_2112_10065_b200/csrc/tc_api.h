// tcgen05 / TMEM tensor-core engine (3xTF32 split, fp32-accurate) for the
// conv3x3 and dense layers.  *_ok() says whether a shape is taken.
#pragma once
#include "common.cuh"

namespace bpx {
bool tc_conv_fwd_ok(int n, int h, int w, int cin, int cout);
bool tc_conv_dgrad_ok(int n, int h, int w, int cin, int cout);
bool tc_conv_wgrad_ok(int n, int h, int w, int cin, int cout);
bool tc_linear_ok(int b, int in, int out);
size_t tc_conv_fwd_ws(int n, int h, int w, int cin, int cout);
size_t tc_conv_dgrad_ws(int n, int h, int w, int cin, int cout);
size_t tc_conv_wgrad_ws(int n, int h, int w, int cin, int cout);
size_t tc_linear_fwd_ws(int b, int in, int out);
size_t tc_linear_dgrad_ws(int b, int in, int out);
size_t tc_linear_wgrad_ws(int b, int in, int out);
bpx_status_t tc_conv_fwd(const float* x, const float* w, const float* bias, float* y,
                         int n, int h, int w_, int cin, int cout, int relu, void* ws,
                         size_t ws_bytes, cudaStream_t st);
bpx_status_t tc_conv_dgrad(const float* dz, const float* w, const float* mask, float* dx,
                           int n, int h, int w_, int cin, int cout, void* ws,
                           size_t ws_bytes, cudaStream_t st);
bpx_status_t tc_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias,
                           int n, int h, int w_, int cin, int cout, void* ws,
                           size_t ws_bytes, cudaStream_t st);
bpx_status_t tc_linear_fwd(const float* x, const float* w, const float* bias, float* y,
                           int b, int in, int out, int relu, void* ws, size_t ws_bytes,
                           cudaStream_t st);
bpx_status_t tc_linear_dgrad(const float* dy, const float* w, const float* mask,
                             float* dx, int b, int in, int out, void* ws,
                             size_t ws_bytes, cudaStream_t st);
bpx_status_t tc_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias,
                             int b, int in, int out, void* ws, size_t ws_bytes,
                             cudaStream_t st);
}  // namespace bpx

// TS engine (tc_ts.cu): conv fwd / dgrad with A in TMEM, B as a pre-split
// weight image loaded by cp.async.bulk.
namespace bpx {
bool ts_conv_ok(int cin, int cout);
size_t ts_conv_ws(int cin, int cout);
bpx_status_t ts_conv_fwd(const float* x, const float* w, const float* bias, float* y, int n,
                         int h, int w_, int cin, int cout, int relu, void* ws,
                         size_t ws_bytes, cudaStream_t st);
bpx_status_t ts_conv_dgrad(const float* dz, const float* w, const float* mask, float* dx,
                           int n, int h, int w_, int cin, int cout, void* ws,
                           size_t ws_bytes, cudaStream_t st);
}  // namespace bpx

// Weight-gradient engine (tc_wgrad.cu): A = dz^T in TMEM, B = im2col(x) in
// the MN-major shared-memory layout, split-K over pixels.
namespace bpx {
bool wg_conv_ok(int cin, int cout);
size_t wg_conv_ws(int n, int h, int w, int cin, int cout);
bpx_status_t wg_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias, int n,
                           int h, int w_, int cin, int cout, void* ws, size_t ws_bytes,
                           cudaStream_t st);
}  // namespace bpx

// TMA-fed weight-gradient engine (tc_wgt.cu): A = im2col(x)^T and B = dz as
// 4-D TMA boxes (MN-major, SWIZZLE_128B_ATOM_32B), A in TMEM, split-K.
namespace bpx {
bool wgt_conv_ok(int cin, int cout);
size_t wgt_conv_ws(int n, int h, int w, int cin, int cout);
bpx_status_t wgt_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias, int n,
                            int h, int w_, int cin, int cout, void* ws, size_t ws_bytes,
                            cudaStream_t st);
}  // namespace bpx

// fp16x3 operand preparation (f16split.cu): *amax = max |x| as bits (memset +
// one launch); f16_split = absmax of the span, then hi/lo fp16 arrays of
// w * 2^s in w's layout (two launches + memset).
namespace bpx {
struct F16Weights {
  const void* hi = nullptr;          // fp16 [cout][3][3][cin]
  const void* lo = nullptr;
  const uint32_t* amax = nullptr;    // max |w| bits of the split span (sets the scale)
};
void absmax(const float* x, size_t n, uint32_t* amax, cudaStream_t st);
void absmax_into(const float* x, size_t n, uint32_t* amax, cudaStream_t st);   // no reset
void f16_split(const float* w, size_t n, void* hi, void* lo, uint32_t* amax, cudaStream_t st);
}  // namespace bpx

// TMA-fed weight-gradient engine, fp16x3 (tc_wgh.cu): Cin % 32, Cout % 64.
// amax_x / amax_dz (nullable): the operands' max |v| bits (bpx_absmax).
namespace bpx {
bool wgh_conv_ok(int cin, int cout);
size_t wgh_conv_ws(int n, int h, int w, int cin, int cout);
bpx_status_t wgh_conv_wgrad(const float* x, const float* dz, const uint32_t* amax_x,
                            const uint32_t* amax_dz, float* dw, float* dbias, int n, int h,
                            int w_, int cin, int cout, void* ws, size_t ws_bytes,
                            cudaStream_t st);
}  // namespace bpx

// Weight gradient of the Cin = 3 -> 64 first conv (tc_wg1.cu).
namespace bpx {
bool wg1_conv_ok(int n, int h, int w, int cin, int cout);
size_t wg1_conv_ws(int n, int h, int w, int cin, int cout);
bpx_status_t wg1_conv_wgrad(const float* x, const float* dz, const uint32_t* amax_x,
                            const uint32_t* amax_dz, float* dw, float* dbias, int n, int h,
                            int w_, void* ws, size_t ws_bytes, cudaStream_t st);
}  // namespace bpx

// Weight gradient for Cin = Cout = 64 with all M tiles resident (tc_wgc.cu).
namespace bpx {
bool wgc_conv_ok(int n, int h, int w, int cin, int cout);
size_t wgc_conv_ws(int n, int h, int w, int cin, int cout);
bpx_status_t wgc_conv_wgrad(const float* x, const float* dz, const uint32_t* amax_x,
                            const uint32_t* amax_dz, float* dw, float* dbias, int n, int h,
                            int w_, void* ws, size_t ws_bytes, cudaStream_t st);
}  // namespace bpx

// TMA-fed persistent forward / data-gradient engine, fp16x3 (tc_fdt.cu).
namespace bpx {
bool fdt_conv_ok(int cin, int cout, int w);
size_t fdt_conv_ws(int n, int h, int w, int cin, int cout);
// wsplit (nullable): the weights split by the caller (bpx_f16_split);
// amax_x / amax_dz (nullable): the A operand's max |v| bits (bpx_absmax)
// amax_y / amax_dx (nullable): atomicMax'ed with the output's max |v| bits
bpx_status_t fdt_conv_fwd(const float* x, const float* w, const F16Weights* wsplit,
                          const uint32_t* amax_x, uint32_t* amax_y, const float* bias, float* y,
                          int n, int h, int w_, int cin, int cout, int relu, void* ws,
                          size_t ws_bytes, cudaStream_t st);
bpx_status_t fdt_conv_dgrad(const float* dz, const float* w, const F16Weights* wsplit,
                            const uint32_t* amax_dz, uint32_t* amax_dx, const float* mask,
                            float* dx, int n, int h, int w_, int cin, int cout, void* ws,
                            size_t ws_bytes, cudaStream_t st);
}  // namespace bpx

// TMA-fed tcgen05 dense fwd / dgrad for batches <= 32 (tc_dense.cu).
namespace bpx {
bool dwt_linear_ok(int b, int in, int out);
size_t dwt_linear_ws(int b, int in, int out);
bpx_status_t dwt_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias, int b,
                              int in, int out, void* ws, size_t ws_bytes, cudaStream_t st);
bool dtc_linear_ok(int b, int in, int out);
size_t dtc_linear_ws(int b, int in, int out);
bpx_status_t dtc_linear_fwd(const float* x, const float* w, const float* bias, float* y, int b,
                            int in, int out, int relu, void* ws, size_t ws_bytes,
                            cudaStream_t st);
bpx_status_t dtc_linear_dgrad(const float* dy, const float* w, const float* mask, float* dx,
                              int b, int in, int out, void* ws, size_t ws_bytes,
                              cudaStream_t st);
}  // namespace bpx

// FFMA thin-GEMM engine (thin.cu): pixel-batched 1x1 convs with 32 outputs.
namespace bpx {
bool thin_linear_ok(int b, int in, int out);
size_t thin_linear_ws(int b, int in, int out);
bpx_status_t thin_linear_fwd(const float* x, const float* w, const float* bias, float* y,
                             int b, int in, int out, int relu, cudaStream_t st);
bpx_status_t thin_linear_dgrad(const float* dy, const float* w, const float* mask, float* dx,
                               int b, int in, int out, cudaStream_t st);
bpx_status_t thin_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias,
                               int b, int in, int out, void* ws, size_t ws_bytes,
                               cudaStream_t st);
}  // namespace bpx
namespace bpx {
bool thin_conv_wgrad_ok(int cin, int cout, int w);
size_t thin_conv_wgrad_ws(int n, int h, int w, int cin, int cout);
bpx_status_t thin_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias, int n,
                             int h, int w_, int cin, int cout, void* ws, size_t ws_bytes,
                             cudaStream_t st);
}  // namespace bpx
