// Internal entry points of the FFMA implicit-GEMM engine (conv_simt.cu).
#pragma once
#include "common.cuh"

namespace bpx {
size_t simt_conv_wgrad_ws(int n, int h, int w, int cin, int cout);
bpx_status_t simt_conv_fwd(const float* x, const float* w, const float* bias, float* y,
                           int n, int h, int w_, int cin, int cout, int relu,
                           cudaStream_t st);
bpx_status_t simt_conv_dgrad(const float* dz, const float* w, const float* mask,
                             float* dx, int n, int h, int w_, int cin, int cout,
                             cudaStream_t st);
bpx_status_t simt_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias,
                             int n, int h, int w_, int cin, int cout, void* ws,
                             size_t ws_bytes, cudaStream_t st);
size_t simt_linear_fwd_ws(int b, int in, int out);
size_t simt_linear_dgrad_ws(int b, int in, int out);
size_t simt_linear_wgrad_ws(int b, int in, int out);
bpx_status_t simt_linear_fwd(const float* x, const float* w, const float* bias, float* y,
                             int b, int in, int out, int relu, void* ws, size_t ws_bytes,
                             cudaStream_t st);
bpx_status_t simt_linear_dgrad(const float* dy, const float* w, const float* mask,
                               float* dx, int b, int in, int out, void* ws,
                               size_t ws_bytes, cudaStream_t st);
bpx_status_t simt_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias,
                               int b, int in, int out, void* ws, size_t ws_bytes,
                               cudaStream_t st);
}  // namespace bpx

// FFMA weight gradient for tiny input depth (conv_small.cu: conv1_1, Cin = 3).
namespace bpx {
bool small_conv_fwd_ok(int cin, int cout);
bpx_status_t small_conv_fwd(const float* x, const float* w, const float* bias, float* y, int n,
                            int h, int w_, int cin, int cout, int relu, cudaStream_t st);
bool small_conv_wgrad_ok(int cin, int cout);
size_t small_conv_wgrad_ws(int n, int h, int w, int cin, int cout);
bpx_status_t small_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias, int n,
                              int h, int w_, int cin, int cout, void* ws, size_t ws_bytes,
                              cudaStream_t st);
}  // namespace bpx

// FFMA dense layers for per-GPU batches <= 32 (dense_ffma.cu).
namespace bpx {
bool dns_linear_ok(int b, int in, int out);
size_t dns_linear_ws(int b, int in, int out);
bpx_status_t dns_linear_fwd(const float* x, const float* w, const float* bias, float* y, int b,
                            int in, int out, int relu, void* ws, size_t ws_bytes,
                            cudaStream_t st);
bpx_status_t dns_linear_dgrad(const float* dy, const float* w, const float* mask, float* dx,
                              int b, int in, int out, void* ws, size_t ws_bytes,
                              cudaStream_t st);
bpx_status_t dns_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias, int b,
                              int in, int out, void* ws, size_t ws_bytes, cudaStream_t st);
}  // namespace bpx

// tcgen05 forward of the first conv (Cin = 3, Cout = 64; conv_first.cu).
namespace bpx {
bool c1_conv_fwd_ok(int cin, int cout);
bpx_status_t c1_conv_fwd(const float* x, const float* w, const float* bias, float* y, int n,
                         int h, int w_, int relu, uint32_t* x_amax, uint32_t* y_amax,
                         cudaStream_t st);
}  // namespace bpx
