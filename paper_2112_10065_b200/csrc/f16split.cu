// Operand preparation for the fp16x3 tensor-core path (tc_ptx.cuh):
//   * absmax: the max |v| of a fp32 tensor as its bit pattern (|v| bits are
//     ordered like the values, so an integer max is exact and
//     order-independent: the result is deterministic);
//   * f16_split: a weight span's max |w|, then w 2^s split into fp16 hi and
//     lo arrays in w's own layout -- the B operand the fwd/dgrad engine
//     loads by TMA.  Run once per weight update, not per call.
#include <cuda_fp16.h>
#include "tc_ptx.cuh"
#include "tc_api.h"

namespace bpx {
namespace f16s {
using namespace tcx;

__device__ __forceinline__ uint32_t absbits(float v) { return __float_as_uint(v) & 0x7fffffffu; }

__global__ void absmax_kernel(const float4* __restrict__ x, long long n4,
                              const float* __restrict__ tail, int ntail, uint32_t* out) {
  uint32_t m = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {       // four loads in flight
    float4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldg(x + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      m = max(m, max(max(absbits(v[k].x), absbits(v[k].y)), max(absbits(v[k].z), absbits(v[k].w))));
  }
  for (; i < n4; i += stride) {
    const float4 v = __ldg(x + i);
    m = max(m, max(max(absbits(v.x), absbits(v.y)), max(absbits(v.z), absbits(v.w))));
  }
  if (blockIdx.x == 0 && (int)threadIdx.x < ntail) m = max(m, absbits(tail[threadIdx.x]));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void split_kernel(const float4* __restrict__ w, long long n4,
                             const float* __restrict__ tail, int ntail,
                             const uint32_t* __restrict__ amax, uint2* __restrict__ hi,
                             uint2* __restrict__ lo) {
  const float s = exp2i(f16_scale_exp(*amax));
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = __ldg(w + i);
    uint2 h, l;
    split_f16x2(v.x * s, v.y * s, h.x, l.x);
    split_f16x2(v.z * s, v.w * s, h.y, l.y);
    hi[i] = h;
    lo[i] = l;
  }
  if (blockIdx.x == 0 && (int)threadIdx.x < ntail) {
    const float v = tail[threadIdx.x] * s;
    const __half h = __float2half_rn(v);
    const __half l = __float2half_rn(v - __half2float(h));
    reinterpret_cast<__half*>(hi + n4)[threadIdx.x] = h;
    reinterpret_cast<__half*>(lo + n4)[threadIdx.x] = l;
  }
}

inline int grid_for(long long n4) {
  long long g = cdivll(n4 > 0 ? n4 : 1, 256);
  const long long cap = 4LL * num_sms();
  return (int)(g < cap ? g : cap);
}

}  // namespace f16s

// *amax = max |x[i]| as bits (a memset and one reduction launch)
void absmax(const float* x, size_t n, uint32_t* amax, cudaStream_t st) {
  cudaMemsetAsync(amax, 0, sizeof(uint32_t), st);
  const long long n4 = (long long)(n / 4);
  f16s::absmax_kernel<<<f16s::grid_for(n4), 256, 0, st>>>(
      reinterpret_cast<const float4*>(x), n4, x + 4 * n4, (int)(n % 4), amax);
}

// hi/lo: n fp16 each (8-B aligned); amax: the span's max |w| bits
void f16_split(const float* w, size_t n, void* hi, void* lo, uint32_t* amax, cudaStream_t st) {
  absmax(w, n, amax, st);
  const long long n4 = (long long)(n / 4);
  f16s::split_kernel<<<f16s::grid_for(n4), 256, 0, st>>>(
      reinterpret_cast<const float4*>(w), n4, w + 4 * n4, (int)(n % 4), amax,
      static_cast<uint2*>(hi), static_cast<uint2*>(lo));
}

}  // namespace bpx

extern "C" bpx_status_t bpx_absmax(const float* x, size_t n, unsigned* amax, void* stream) {
  using namespace bpx;
  BPX_CHECK_ARG(amax && (n == 0 || (x && aligned16(x))));
  absmax(x, n, amax, as_stream(stream));
  return launch_status(1);
}

extern "C" bpx_status_t bpx_f16_split(const float* w, size_t n, void* hi, void* lo,
                                      unsigned* amax, void* stream) {
  using namespace bpx;
  BPX_CHECK_ARG(amax && hi && lo && (n == 0 || (w && aligned16(w))));
  BPX_CHECK_ARG((reinterpret_cast<uintptr_t>(hi) & 7u) == 0 &&
                (reinterpret_cast<uintptr_t>(lo) & 7u) == 0);
  f16_split(w, n, hi, lo, amax, as_stream(stream));
  return launch_status(2);
}
