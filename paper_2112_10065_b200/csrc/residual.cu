// Branch/join element kernels for the residual (WRN-style) executable net
// behind the reference's `wideresnet_like` family (synth.py:126-169): the
// `add` join of each residual diamond, the stride-2 subsample at stage
// transitions, and the global average pool before the classifier.  All are
// HBM-bound elementwise passes: float4 over NHWC channels, grid-stride,
// fixed-order arithmetic (deterministic).
//
// Residual join (post-activation basic block):
//   y = relu(a + P(s)),  a, y: [n][h][w][c],  s: [n][h*f][w*f][cs], cs <= c
//   P = stride-f subsample (f = 2 at a stage transition, else 1) followed by
//       zero channel padding cs -> c (ResNet "option A" shortcut: no params)
// Its backward to the skip source h (grad wrt h's pre-activation, the
// executor's `dy` convention: the consumer applies the producer's ReLU mask):
//   dh[n][H][W][cs] = (acc ? dh : 0)
//                     + [H%f==0 && W%f==0] * (dmain[n][H/f][W/f][cs]     (if given)
//                                             + (mask > 0) * dz[n][H/f][W/f][c < cs])
// `dmain` is the low-resolution data gradient of the block's first conv
// (already masked by its dgrad) when that conv reads a subsampled copy of h,
// so one pass writes all of dh at a transition; otherwise the first conv's
// dgrad has written dh in place and the skip term is accumulated (acc = 1).
#include "common.cuh"
#include "simt_api.h"
#include "tc_api.h"

namespace bpx {
namespace {

int grid_for(long long work) {
  long long g = cdivll(work, 256);
  long long cap = 8LL * num_sms();
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

__device__ __forceinline__ float4 relu4(float4 v) {
  return make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
}

__global__ void resadd_fwd_kernel(const float4* __restrict__ a, const float4* __restrict__ s,
                                  float4* __restrict__ y, long long total, int h, int w, int c4,
                                  int cs4, int f, int relu) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(e % c4);
    const long long pix = e / c4;
    const int ow = (int)(pix % w);
    const long long r = pix / w;
    const int oh = (int)(r % h);
    const long long img = r / h;
    float4 v = a[e];
    if (ci < cs4) {
      const float4 t = s[((img * (h * f) + (long long)oh * f) * (w * f) + (long long)ow * f) * cs4 + ci];
      v.x += t.x; v.y += t.y; v.z += t.z; v.w += t.w;
    }
    y[e] = relu ? relu4(v) : v;
  }
}

// Same-shape joins (f = 1, cs = c: every diamond but the stage transitions)
// are plain elementwise passes: no per-element index arithmetic, 4 vectors
// in flight per thread; the forward also reduces max |y| for the fp16x3
// scale word of the conv that reads y (amax nullable).
constexpr int UNR = 4;
__global__ void resadd_flat_kernel(const float4* __restrict__ a, const float4* __restrict__ s,
                                   float4* __restrict__ y, long long total, int relu,
                                   uint32_t* __restrict__ amax) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  uint32_t mx = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += UNR * stride) {
    float4 va[UNR], vs[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const bool in = e + u * stride < total;
      va[u] = in ? a[e + u * stride] : make_float4(0.f, 0.f, 0.f, 0.f);
      vs[u] = in ? s[e + u * stride] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (e + u * stride >= total) break;
      float4 v = make_float4(va[u].x + vs[u].x, va[u].y + vs[u].y, va[u].z + vs[u].z,
                             va[u].w + vs[u].w);
      if (relu) v = relu4(v);
      mx = max(mx, max(max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu),
                       max(__float_as_uint(v.z) & 0x7fffffffu, __float_as_uint(v.w) & 0x7fffffffu)));
      y[e + u * stride] = v;
    }
  }
  if (amax) {
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(amax, mx);
  }
}
__global__ void skip_flat_kernel(const float4* __restrict__ dz, const float4* __restrict__ dmain,
                                 const float4* __restrict__ mask, float4* __restrict__ dh,
                                 long long total, int acc) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += UNR * stride) {
    float4 g[UNR], m[UNR], v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const long long q = e + u * stride;
      const bool in = q < total;
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      g[u] = in ? dz[q] : z4;
      m[u] = in ? mask[q] : z4;
      v[u] = in && acc ? dh[q] : z4;
      if (in && dmain) {
        const float4 d = dmain[q];
        v[u].x += d.x; v[u].y += d.y; v[u].z += d.z; v[u].w += d.w;
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (e + u * stride >= total) break;
      v[u].x += m[u].x > 0.f ? g[u].x : 0.f; v[u].y += m[u].y > 0.f ? g[u].y : 0.f;
      v[u].z += m[u].z > 0.f ? g[u].z : 0.f; v[u].w += m[u].w > 0.f ? g[u].w : 0.f;
      dh[e + u * stride] = v[u];
    }
  }
}

__global__ void skip_bwd_kernel(const float4* __restrict__ dz, const float4* __restrict__ dmain,
                                const float4* __restrict__ mask, float4* __restrict__ dh,
                                long long total, int H, int W, int c4, int cs4, int f, int acc) {
  const int h = H / f, w = W / f;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(e % cs4);
    const long long pix = e / cs4;
    const int iw = (int)(pix % W);
    const long long r = pix / W;
    const int ih = (int)(r % H);
    const long long img = r / H;
    float4 v = acc ? dh[e] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (ih % f == 0 && iw % f == 0) {
      const long long lp = (img * h + ih / f) * w + iw / f;      // low-res pixel
      if (dmain) {
        const float4 d = dmain[lp * cs4 + ci];
        v.x += d.x; v.y += d.y; v.z += d.z; v.w += d.w;
      }
      const float4 g = dz[lp * c4 + ci];
      const float4 m = mask[e];
      v.x += m.x > 0.f ? g.x : 0.f; v.y += m.y > 0.f ? g.y : 0.f;
      v.z += m.z > 0.f ? g.z : 0.f; v.w += m.w > 0.f ? g.w : 0.f;
    }
    dh[e] = v;
  }
}

__global__ void subsample2_kernel(const float4* __restrict__ x, float4* __restrict__ y,
                                  long long total, int h, int w, int c4) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(e % c4);
    const long long pix = e / c4;
    const int ow = (int)(pix % w);
    const long long r = pix / w;
    const int oh = (int)(r % h);
    const long long img = r / h;
    y[e] = x[((img * (2 * h) + 2LL * oh) * (2 * w) + 2LL * ow) * c4 + ci];
  }
}

// dx[n][2h][2w][c] = dy at even (row, col), 0 elsewhere
__global__ void subsample2_bwd_kernel(const float4* __restrict__ dy, float4* __restrict__ dx,
                                      long long total, int H, int W, int c4) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(e % c4);
    const long long pix = e / c4;
    const int iw = (int)(pix % W);
    const long long r = pix / W;
    const int ih = (int)(r % H);
    const long long img = r / H;
    dx[e] = ((ih | iw) & 1) ? make_float4(0.f, 0.f, 0.f, 0.f)
                            : dy[((img * (H / 2) + ih / 2) * (W / 2) + iw / 2) * c4 + ci];
  }
}

__global__ void accumulate_kernel(float4* __restrict__ dst, const float4* __restrict__ src,
                                  long long n4) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n4;
       e += (long long)gridDim.x * blockDim.x) {
    float4 a = dst[e];
    const float4 b = src[e];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    dst[e] = a;
  }
}

// one thread per (image, 4 channels): fixed-order sum over the hw pixels
__global__ void gap_fwd_kernel(const float4* __restrict__ x, float4* __restrict__ y, int n,
                               int hw, int c4, float scale) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * c4;
       e += (long long)gridDim.x * blockDim.x) {
    const long long img = e / c4;
    const int ci = (int)(e % c4);
    const float4* p = x + img * hw * c4 + ci;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < hw; ++q) {
      const float4 v = p[(long long)q * c4];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    y[e] = make_float4(s.x * scale, s.y * scale, s.z * scale, s.w * scale);
  }
}

__global__ void gap_bwd_kernel(const float4* __restrict__ dy, const float4* __restrict__ mask,
                               float4* __restrict__ dx, long long total, int hw, int c4,
                               float scale) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ci = (int)(e % c4);
    const long long img = e / ((long long)hw * c4);
    const float4 g = dy[img * c4 + ci];
    float4 v = make_float4(g.x * scale, g.y * scale, g.z * scale, g.w * scale);
    if (mask) {
      const float4 m = mask[e];
      v.x = m.x > 0.f ? v.x : 0.f; v.y = m.y > 0.f ? v.y : 0.f;
      v.z = m.z > 0.f ? v.z : 0.f; v.w = m.w > 0.f ? v.w : 0.f;
    }
    dx[e] = v;
  }
}

}  // namespace
}  // namespace bpx

using namespace bpx;

extern "C" {

bpx_status_t bpx_residual_add_fwd(const float* a, const float* s, float* y, int n, int h,
                                  int w_, int c, int cs, int down, int relu, unsigned* y_amax,
                                  void* stream) {
  BPX_CHECK_ARG(n >= 0 && h >= 0 && w_ >= 0 && c % 4 == 0 && cs % 4 == 0);
  BPX_CHECK_ARG(cs > 0 && cs <= c && (down == 0 || down == 1));
  const long long total = (long long)n * h * w_ * (c / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(a && s && y && aligned16(a) && aligned16(s) && aligned16(y));
  if (!down && cs == c) {
    resadd_flat_kernel<<<grid_for(cdivll(total, UNR)), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const float4*>(a), reinterpret_cast<const float4*>(s),
        reinterpret_cast<float4*>(y), total, relu, y_amax);
    return launch_status();
  }
  resadd_fwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(a), reinterpret_cast<const float4*>(s),
      reinterpret_cast<float4*>(y), total, h, w_, c / 4, cs / 4, down ? 2 : 1, relu);
  if (y_amax) {         // the transition joins: one reduction over y
    absmax_into(y, (size_t)total * 4, y_amax, as_stream(stream));
    return launch_status(2);
  }
  return launch_status();
}

bpx_status_t bpx_residual_skip_bwd(const float* dz, const float* dmain, const float* mask,
                                   float* dh, int n, int h, int w_, int c, int cs, int down,
                                   int accumulate, void* stream) {
  BPX_CHECK_ARG(n >= 0 && h >= 0 && w_ >= 0 && c % 4 == 0 && cs % 4 == 0);
  BPX_CHECK_ARG(cs > 0 && cs <= c && (down == 0 || down == 1));
  BPX_CHECK_ARG(!(dmain && accumulate));
  const int f = down ? 2 : 1;
  const long long total = (long long)n * (h * f) * (w_ * f) * (cs / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(dz && mask && dh && aligned16(dz) && aligned16(mask) && aligned16(dh) &&
                aligned16(dmain));
  if (!down && cs == c) {
    skip_flat_kernel<<<grid_for(cdivll(total, UNR)), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const float4*>(dz), reinterpret_cast<const float4*>(dmain),
        reinterpret_cast<const float4*>(mask), reinterpret_cast<float4*>(dh), total,
        accumulate);
    return launch_status();
  }
  skip_bwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(dz), reinterpret_cast<const float4*>(dmain),
      reinterpret_cast<const float4*>(mask), reinterpret_cast<float4*>(dh), total, h * f,
      w_ * f, c / 4, cs / 4, f, accumulate);
  return launch_status();
}

bpx_status_t bpx_subsample2_fwd(const float* x, float* y, int n, int h, int w_, int c,
                                void* stream) {
  BPX_CHECK_ARG(n >= 0 && h >= 0 && w_ >= 0 && c % 4 == 0);
  const long long total = (long long)n * h * w_ * (c / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(x && y && aligned16(x) && aligned16(y));
  subsample2_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), total, h, w_, c / 4);
  return launch_status();
}

bpx_status_t bpx_subsample2_bwd(const float* dy, float* dx, int n, int h, int w_, int c,
                                void* stream) {
  BPX_CHECK_ARG(n >= 0 && h >= 0 && w_ >= 0 && c % 4 == 0);
  const long long total = (long long)n * (2 * h) * (2 * w_) * (c / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(dy && dx && aligned16(dy) && aligned16(dx));
  subsample2_bwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(dy), reinterpret_cast<float4*>(dx), total, 2 * h,
      2 * w_, c / 4);
  return launch_status();
}

bpx_status_t bpx_accumulate(float* dst, const float* src, size_t n, void* stream) {
  BPX_CHECK_ARG(n % 4 == 0);
  if (n == 0) return BPX_OK;
  BPX_CHECK_ARG(dst && src && aligned16(dst) && aligned16(src));
  const long long n4 = (long long)(n / 4);
  accumulate_kernel<<<grid_for(n4), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<float4*>(dst), reinterpret_cast<const float4*>(src), n4);
  return launch_status();
}

bpx_status_t bpx_global_avgpool_fwd(const float* x, float* y, int n, int h, int w_, int c,
                                    void* stream) {
  BPX_CHECK_ARG(n >= 0 && h > 0 && w_ > 0 && c % 4 == 0);
  const long long total = (long long)n * (c / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(x && y && aligned16(x) && aligned16(y));
  gap_fwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), n, h * w_, c / 4,
      1.0f / (float)(h * w_));
  return launch_status();
}

bpx_status_t bpx_global_avgpool_bwd(const float* dy, const float* mask, float* dx, int n,
                                    int h, int w_, int c, void* stream) {
  BPX_CHECK_ARG(n >= 0 && h > 0 && w_ > 0 && c % 4 == 0);
  const long long total = (long long)n * h * w_ * (c / 4);
  if (total == 0) return BPX_OK;
  BPX_CHECK_ARG(dy && dx && aligned16(dy) && aligned16(dx) && aligned16(mask));
  gap_bwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(dy), reinterpret_cast<const float4*>(mask),
      reinterpret_cast<float4*>(dx), total, h * w_, c / 4, 1.0f / (float)(h * w_));
  return launch_status();
}

}  // extern "C"
