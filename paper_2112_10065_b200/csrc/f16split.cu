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
    split_f16x2_s(v.x, v.y, s, h.x, l.x);
    split_f16x2_s(v.z, v.w, s, h.y, l.y);
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

// Batched split of several weight tensors (one launch each for the maxima
// and the split, whatever the layer count): block b serves segment k with
// blk0[k] <= b < blk0[k+1], CHUNK float4 per block.
struct Seg {
  const float4* w; uint2* hi; uint2* lo; uint32_t* amax; long long n4, blk0;
};
constexpr int CHUNK = 2048;          // float4 per block: 8 per thread

__device__ __forceinline__ int seg_of(const Seg* segs, int nseg, long long b) {
  int k = 0;
  while (k + 1 < nseg && segs[k + 1].blk0 <= b) ++k;
  return k;
}

__global__ void absmax_batch_kernel(const Seg* __restrict__ segs, int nseg) {
  const int k = seg_of(segs, nseg, blockIdx.x);
  const Seg sg = segs[k];
  const long long i0 = (blockIdx.x - sg.blk0) * (long long)CHUNK;
  uint32_t m = 0;
#pragma unroll 4
  for (int j = threadIdx.x; j < CHUNK; j += blockDim.x) {
    if (i0 + j < sg.n4) {
      const float4 v = __ldg(sg.w + i0 + j);
      m = max(m, max(max(absbits(v.x), absbits(v.y)), max(absbits(v.z), absbits(v.w))));
    }
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(sg.amax, m);
}

__global__ void split_batch_kernel(const Seg* __restrict__ segs, int nseg) {
  const int k = seg_of(segs, nseg, blockIdx.x);
  const Seg sg = segs[k];
  const float s = exp2i(f16_scale_exp(*sg.amax));
  const long long i0 = (blockIdx.x - sg.blk0) * (long long)CHUNK;
#pragma unroll 4
  for (int j = threadIdx.x; j < CHUNK; j += blockDim.x) {
    const long long i = i0 + j;
    if (i < sg.n4) {
      const float4 v = __ldg(sg.w + i);
      uint2 h, l;
      split_f16x2_s(v.x, v.y, s, h.x, l.x);
      split_f16x2_s(v.z, v.w, s, h.y, l.y);
      sg.hi[i] = h;
      sg.lo[i] = l;
    }
  }
}

inline int grid_for(long long n4) {
  long long g = cdivll(n4 > 0 ? n4 : 1, 256);
  const long long cap = 4LL * num_sms();
  return (int)(g < cap ? g : cap);
}

}  // namespace f16s

// *amax = max(*amax, max |x[i]| as bits): one reduction launch
void absmax_into(const float* x, size_t n, uint32_t* amax, cudaStream_t st) {
  const long long n4 = (long long)(n / 4);
  f16s::absmax_kernel<<<f16s::grid_for(n4), 256, 0, st>>>(
      reinterpret_cast<const float4*>(x), n4, x + 4 * n4, (int)(n % 4), amax);
}

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

// segs: a DEVICE array of nseg {w, hi, lo, amax, n4, blk0} records (each
// n = 4 n4 floats, blk0 = the first block of the segment, blocks = the
// total); words/nwords: every amax word of the batch (zeroed here).
extern "C" bpx_status_t bpx_f16_split_batch(const void* segs, int nseg, long long blocks,
                                            unsigned* words, size_t nwords, void* stream) {
  using namespace bpx;
  BPX_CHECK_ARG(nseg >= 0 && blocks >= 0 && (nseg == 0 || (segs && words)));
  if (nseg == 0 || blocks == 0) return BPX_OK;
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(words, 0, nwords * sizeof(unsigned), st);
  const f16s::Seg* sg = static_cast<const f16s::Seg*>(segs);
  f16s::absmax_batch_kernel<<<(unsigned)blocks, 256, 0, st>>>(sg, nseg);
  f16s::split_batch_kernel<<<(unsigned)blocks, 256, 0, st>>>(sg, nseg);
  return launch_status(2);
}

extern "C" int bpx_f16_split_batch_chunk(void) { return bpx::f16s::CHUNK; }

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
