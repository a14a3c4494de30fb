// Shared helpers for libbpx kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include "../../include/bpx.h"

#define BPX_CHECK_ARG(cond)                         \
  do {                                              \
    if (!(cond)) return BPX_ERR_INVALID_ARGUMENT;   \
  } while (0)

namespace bpx {

// Host-side count of kernel launches issued by libbpx (exported through
// bpx_launch_count); call sites with k launches report k.
void count_launches(long long k);

inline bpx_status_t launch_status(int kernels = 1) {
  count_launches(kernels);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BPX_OK : BPX_ERR_LAUNCH;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// SM budget of the calling host thread's launches (0 = the whole GPU):
// persistent grids and split-K choices size themselves to it, so a kernel
// launched (or captured) under a budget of k keeps at most k SMs busy with
// its long-lived CTAs -- the background job's share under multiplexing
// (bpx_set_sm_budget, multiplex.BgJob).
int& sm_budget();

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  const int b = sm_budget();
  return (b > 0 && b < n) ? b : n;
}

__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline long long cdivll(long long a, long long b) { return (a + b - 1) / b; }

// Deterministic column sums: out[c] = sum_r in[r*cols + c] (fixed order).
bpx_status_t colsum(const float* in, long long rows, int cols, float* out,
                    float* ws, size_t ws_floats, cudaStream_t st);
size_t colsum_workspace_floats(long long rows, int cols);

// Fixed-order split reduction: out[i] = sum_s parts[s*n + i].
bpx_status_t split_reduce(const float* parts, int splits, size_t n, float* out,
                          cudaStream_t st);
// The same for a weight gradient and its bias gradient in ONE launch:
// dw[i] = sum_s pw[s*nw + i], db[j] = sum_s pb[s*nb + j] (db may be null).
bpx_status_t split_reduce_wb(const float* pw, size_t nw, float* dw, const float* pb, size_t nb,
                             float* db, int splits, cudaStream_t st);

}  // namespace bpx
