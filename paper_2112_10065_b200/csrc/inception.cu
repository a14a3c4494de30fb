// Branch/join element kernels for the executable net behind the reference's
// `inception_like` family (synth.py:172-226): the parameter-free pool tower
// (3x3 / stride-1 / pad-1 max pool over the first cs channels of the module
// input), the four-tower channel concat, and the stride-2 subsample with an
// offset used where the module resolution drops (35 -> 17 -> 8 keeps pixels
// 1, 3, 5, ...).  All HBM-bound elementwise passes over NHWC float4 groups,
// deterministic (fixed-order gathers, no atomics).
#include "common.cuh"

namespace bpx {
namespace {

int grid_for(long long work) {
  long long g = cdivll(work, 256);
  long long cap = 8LL * num_sms();
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// y[p][c] = max over the 3x3 window (pad 1, out-of-image taps skipped) of
// x[.][c], c < cs4*4; idx = first max position (dy+1)*3 + (dx+1), row-major
__global__ void maxpool3_fwd_kernel(const float4* __restrict__ x, float4* __restrict__ y,
                                    uchar4* __restrict__ idx, long long total, int h, int w,
                                    int C4, int cs4) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(e % cs4);
    const long long pix = e / cs4;
    const int ow = (int)(pix % w);
    const long long r = pix / w;
    const int oh = (int)(r % h);
    const long long img = r / h;
    float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    unsigned char k[4] = {0, 0, 0, 0};
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const int ih = oh + t / 3 - 1, iw = ow + t % 3 - 1;
      if ((unsigned)ih >= (unsigned)h || (unsigned)iw >= (unsigned)w) continue;
      const float4 v = x[((img * h + ih) * w + iw) * C4 + ci];
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (vv[j] > m[j]) { m[j] = vv[j]; k[j] = (unsigned char)t; }
    }
    y[e] = make_float4(m[0], m[1], m[2], m[3]);
    idx[e] = make_uchar4(k[0], k[1], k[2], k[3]);
  }
}

// dx[p][c] = sum over the outputs q whose window holds p (fixed order) of
// dy[q][c] * [idx[q][c] == position of p in q's window]; 0 for c >= cs
__global__ void maxpool3_bwd_kernel(const uchar4* __restrict__ idx, const float4* __restrict__ dy,
                                    float4* __restrict__ dx, long long total, int h, int w,
                                    int C4, int cs4) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(e % C4);
    const long long pix = e / C4;
    const int iw = (int)(pix % w);
    const long long r = pix / w;
    const int ih = (int)(r % h);
    const long long img = r / h;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ci < cs4) {
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        // output q = p - (tap offset); p sits at tap t of q's window
        const int oh = ih - (t / 3 - 1), ow = iw - (t % 3 - 1);
        if ((unsigned)oh >= (unsigned)h || (unsigned)ow >= (unsigned)w) continue;
        const long long q = ((img * h + oh) * w + ow) * cs4 + ci;
        const uchar4 k = idx[q];
        const float4 g = dy[q];
        if (k.x == t) s.x += g.x;
        if (k.y == t) s.y += g.y;
        if (k.z == t) s.z += g.z;
        if (k.w == t) s.w += g.w;
      }
    }
    dx[e] = s;
  }
}

struct Parts {
  const float4* in[4];
  float4* out[4];
  int c4[4];        // float4 groups per part
};

__global__ void concat_fwd_kernel(Parts p, float4* __restrict__ y, long long total, int C4) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int c = (int)(e % C4);
    const long long pix = e / C4;
    int k = 0;
    while (c >= p.c4[k]) { c -= p.c4[k]; ++k; }
    y[e] = p.in[k][pix * p.c4[k] + c];
  }
}

__global__ void concat_bwd_kernel(Parts p, const float4* __restrict__ dy, long long total,
                                  int C4) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int c = (int)(e % C4);
    const long long pix = e / C4;
    int k = 0;
    while (c >= p.c4[k]) { c -= p.c4[k]; ++k; }
    p.out[k][pix * p.c4[k] + c] = dy[e];
  }
}

// y[n][i][j] = x[n][2i+off][2j+off]  (bwd: dx = 0 elsewhere)
__global__ void subsample_fwd_kernel(const float4* __restrict__ x, float4* __restrict__ y,
                                     long long total, int hin, int win, int h, int w, int c4,
                                     int off) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(e % c4);
    const long long pix = e / c4;
    const int ow = (int)(pix % w);
    const long long r = pix / w;
    const int oh = (int)(r % h);
    const long long img = r / h;
    y[e] = x[((img * hin + 2LL * oh + off) * win + 2LL * ow + off) * c4 + ci];
  }
}

__global__ void subsample_bwd_kernel(const float4* __restrict__ dy, float4* __restrict__ dx,
                                     long long total, int hin, int win, int h, int w, int c4,
                                     int off) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(e % c4);
    const long long pix = e / c4;
    const int iw = (int)(pix % win) - off;
    const long long r = pix / win;
    const int ih = (int)(r % hin) - off;
    const long long img = r / hin;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ih >= 0 && iw >= 0 && !(ih & 1) && !(iw & 1) && ih / 2 < h && iw / 2 < w)
      v = dy[((img * h + ih / 2) * w + iw / 2) * c4 + ci];
    dx[e] = v;
  }
}

bool parts_ok(const float* const* ptrs, const int* cs, int k) {
  if (k < 1 || k > 4) return false;
  for (int i = 0; i < k; ++i)
    if (!ptrs[i] || !aligned16(ptrs[i]) || cs[i] <= 0 || cs[i] % 4) return false;
  return true;
}

}  // namespace
}  // namespace bpx

using namespace bpx;

extern "C" {

bpx_status_t bpx_maxpool3x3_fwd_idx(const float* x, float* y, uint8_t* idx, int n, int h,
                                    int w_, int c, int cs, void* stream) {
  BPX_CHECK_ARG(n >= 0 && h >= 0 && w_ >= 0 && c % 4 == 0 && cs % 4 == 0 && cs > 0 && cs <= c);
  const long long total = (long long)n * h * w_ * (cs / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(x && y && idx && aligned16(x) && aligned16(y) &&
                (reinterpret_cast<uintptr_t>(idx) & 3) == 0);
  maxpool3_fwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y),
      reinterpret_cast<uchar4*>(idx), total, h, w_, c / 4, cs / 4);
  return launch_status();
}

bpx_status_t bpx_maxpool3x3_bwd_idx(const uint8_t* idx, const float* dy, float* dx, int n,
                                    int h, int w_, int c, int cs, void* stream) {
  BPX_CHECK_ARG(n >= 0 && h >= 0 && w_ >= 0 && c % 4 == 0 && cs % 4 == 0 && cs > 0 && cs <= c);
  const long long total = (long long)n * h * w_ * (c / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(idx && dy && dx && aligned16(dy) && aligned16(dx) &&
                (reinterpret_cast<uintptr_t>(idx) & 3) == 0);
  maxpool3_bwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const uchar4*>(idx), reinterpret_cast<const float4*>(dy),
      reinterpret_cast<float4*>(dx), total, h, w_, c / 4, cs / 4);
  return launch_status();
}

bpx_status_t bpx_concat_fwd(const float* const* parts, const int* cs, int k, float* y,
                            long long npix, void* stream) {
  BPX_CHECK_ARG(npix >= 0 && parts && cs);
  BPX_CHECK_ARG(parts_ok(parts, cs, k) && y && aligned16(y));
  Parts p{};
  int C = 0;
  for (int i = 0; i < 4; ++i) {
    p.in[i] = i < k ? reinterpret_cast<const float4*>(parts[i]) : nullptr;
    p.c4[i] = i < k ? cs[i] / 4 : 1 << 30;
    C += i < k ? cs[i] : 0;
  }
  const long long total = npix * (C / 4);
  if (total == 0) return BPX_OK;
  concat_fwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      p, reinterpret_cast<float4*>(y), total, C / 4);
  return launch_status();
}

bpx_status_t bpx_concat_bwd(const float* dy, float* const* parts, const int* cs, int k,
                            long long npix, void* stream) {
  BPX_CHECK_ARG(npix >= 0 && parts && cs && dy && aligned16(dy));
  BPX_CHECK_ARG(parts_ok(const_cast<const float* const*>(parts), cs, k));
  Parts p{};
  int C = 0;
  for (int i = 0; i < 4; ++i) {
    p.out[i] = i < k ? reinterpret_cast<float4*>(parts[i]) : nullptr;
    p.c4[i] = i < k ? cs[i] / 4 : 1 << 30;
    C += i < k ? cs[i] : 0;
  }
  const long long total = npix * (C / 4);
  if (total == 0) return BPX_OK;
  concat_bwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      p, reinterpret_cast<const float4*>(dy), total, C / 4);
  return launch_status();
}

bpx_status_t bpx_subsample_fwd(const float* x, float* y, int n, int hin, int win, int h,
                               int w_, int c, int off, void* stream) {
  BPX_CHECK_ARG(n >= 0 && h >= 0 && w_ >= 0 && c % 4 == 0 && (off == 0 || off == 1));
  BPX_CHECK_ARG(2 * h + off <= hin && 2 * w_ + off <= win);
  const long long total = (long long)n * h * w_ * (c / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(x && y && aligned16(x) && aligned16(y));
  subsample_fwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), total, hin, win, h,
      w_, c / 4, off);
  return launch_status();
}

bpx_status_t bpx_subsample_bwd(const float* dy, float* dx, int n, int hin, int win, int h,
                               int w_, int c, int off, void* stream) {
  BPX_CHECK_ARG(n >= 0 && hin >= 0 && win >= 0 && c % 4 == 0 && (off == 0 || off == 1));
  BPX_CHECK_ARG(2 * h + off <= hin && 2 * w_ + off <= win);
  const long long total = (long long)n * hin * win * (c / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(dy && dx && aligned16(dy) && aligned16(dx));
  subsample_bwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(dy), reinterpret_cast<float4*>(dx), total, hin, win, h,
      w_, c / 4, off);
  return launch_status();
}

}  // extern "C"
