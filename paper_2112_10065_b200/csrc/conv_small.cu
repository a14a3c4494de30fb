// Weight gradient of a 3x3/pad-1 conv with a tiny input depth (conv1_1:
// Cin = 3, so im2col has only R = 27 columns -- far too narrow for a
// tensor-core tile, and TMA boxes need 16-byte rows):
//
//   dW[co][r] = sum_p col[p][r] * dz[p][co],  r = tap*Cin + ci,  db[co] = sum_p dz[p][co]
//
// FFMA outer products.  A CTA walks a contiguous pixel range in tiles of 64
// pixels: the dz tile (64 x Cout) is loaded with coalesced float4s and the
// 27-wide im2col rows are built in shared memory from x (19 MB for the whole
// batch: L2-resident).  Each warp owns every 8th pixel of a tile; lane l
// owns output channels [l*CPL, l*CPL+CPL) for all R columns, so per pixel a
// lane does R*CPL FMAs from 7 broadcast LDS.128 of the col row plus one LDS
// of its dz channels.  Warp partials are combined in a fixed order, CTA
// partials by split_reduce: results are deterministic run to run.
#include "common.cuh"

namespace bpx {
namespace small {

constexpr int PB = 8;            // pixels per batch (loads in flight per lane)

// Coordinates of PB consecutive pixels from (img, oh, ow) of the first.
struct Pix {
  int img, oh, ow;
  __device__ __forceinline__ void step(int H, int W) {
    if (++ow == W) { ow = 0; if (++oh == H) { oh = 0; ++img; } }
  }
};

// Every lane j < R fetches im2col column j of a pixel (its tap/ci is fixed
// per lane, so the index math is a handful of adds); the warp shares the
// row through shared memory and every lane reads it back as R4/4
// broadcast LDS.128.  No CTA-wide synchronisation: each warp streams its
// own contiguous pixel range with PB pixels of loads in flight.
template <int CIN>
__device__ __forceinline__ float col_value(const float* __restrict__ x, const Pix& q, int H,
                                           int W, int lane) {
  constexpr int R = 9 * CIN;
  if (lane >= R) return 0.f;
  const int tap = lane / CIN, ci = lane - tap * CIN;
  const int ih = q.oh + tap / 3 - 1, iw = q.ow + tap % 3 - 1;
  if ((unsigned)ih >= (unsigned)H || (unsigned)iw >= (unsigned)W) return 0.f;
  return __ldg(x + (((long long)q.img * H + ih) * W + iw) * CIN + ci);
}

template <int CIN, int CPL>
__global__ void __launch_bounds__(256, 2)
small_wgrad_kernel(const float* __restrict__ x, const float* __restrict__ dz, int H, int W,
                   long long npix, long long chunk, float* __restrict__ part,
                   float* __restrict__ bias_part) {
  constexpr int R = 9 * CIN, R4 = (R + 3) / 4 * 4, COUT = 32 * CPL;
  static_assert(R <= 32, "one im2col column per lane");
  __shared__ __align__(16) float colw[8][PB][R4];
  __shared__ __align__(16) float red[COUT * R + COUT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long p0 = ((long long)blockIdx.x * 8 + warp) * chunk;
  const long long p1 = min(npix, p0 + chunk);
  const int hw = H * W;

  float acc[R][CPL];
  float bacc[CPL];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[r][c] = 0.f;
#pragma unroll
  for (int c = 0; c < CPL; ++c) bacc[c] = 0.f;

  if (p0 < p1) {
    Pix q;
    q.img = (int)(p0 / hw);
    const int rem = (int)(p0 - (long long)q.img * hw);
    q.oh = rem / W;
    q.ow = rem - q.oh * W;
    for (long long p = p0; p < p1; p += PB) {
      const int nb = (int)min((long long)PB, p1 - p);
      float xv[PB], d[PB][CPL];
#pragma unroll
      for (int b = 0; b < PB; ++b) {
        xv[b] = 0.f;
#pragma unroll
        for (int c = 0; c < CPL; ++c) d[b][c] = 0.f;
        if (b < nb) {
          xv[b] = col_value<CIN>(x, q, H, W, lane);
          const float* src = dz + (p + b) * COUT + lane * CPL;
          if (CPL == 2) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(src));
            d[b][0] = v.x; d[b][CPL - 1] = v.y;
          } else {
#pragma unroll
            for (int c = 0; c < CPL; ++c) d[b][c] = __ldg(src + c);
          }
          q.step(H, W);
        }
      }
#pragma unroll
      for (int b = 0; b < PB; ++b)
        if (lane < R4) colw[warp][b][lane] = xv[b];
      __syncwarp();
#pragma unroll
      for (int b = 0; b < PB; ++b) {
#pragma unroll
        for (int r4 = 0; r4 < R4; r4 += 4) {
          const float4 cv = *reinterpret_cast<const float4*>(&colw[warp][b][r4]);
          const float cr[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (r4 + j < R) {
#pragma unroll
              for (int c = 0; c < CPL; ++c) acc[r4 + j][c] = fmaf(cr[j], d[b][c], acc[r4 + j][c]);
            }
        }
#pragma unroll
        for (int c = 0; c < CPL; ++c) bacc[c] += d[b][c];
      }
      __syncwarp();
    }
  }

  // fixed-order combine of the 8 warps' partials
  for (int w = 0; w < 8; ++w) {
    if (warp == w) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int co = lane * CPL + c;
#pragma unroll
        for (int r = 0; r < R; ++r)
          red[co * R + r] = (w == 0 ? 0.f : red[co * R + r]) + acc[r][c];
        red[COUT * R + co] = (w == 0 ? 0.f : red[COUT * R + co]) + bacc[c];
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < COUT * R; i += 256)
    part[(long long)blockIdx.x * COUT * R + i] = red[i];
  if (bias_part)
    for (int i = threadIdx.x; i < COUT; i += 256)
      bias_part[(long long)blockIdx.x * COUT + i] = red[COUT * R + i];
}

// Forward of the same conv: y[p][co] = act(b[co] + sum_r col[p][r] w[co][r]).
// Lane l keeps w[l*CPL .. +CPL][0..R) in registers; per pixel R4/4
// broadcast LDS.128 of the im2col row, R*CPL FMAs, one coalesced store.
template <int CIN, int CPL>
__global__ void __launch_bounds__(256, 2)
small_fwd_kernel(const float* __restrict__ x, const float* __restrict__ w,
                 const float* __restrict__ bias, float* __restrict__ y, int H, int W,
                 long long npix, long long chunk, int relu) {
  constexpr int R = 9 * CIN, R4 = (R + 3) / 4 * 4, COUT = 32 * CPL;
  __shared__ __align__(16) float colw[8][PB][R4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hw = H * W;
  float wr[R][CPL], b0[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int co = lane * CPL + c;
    b0[c] = bias ? __ldg(bias + co) : 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) wr[r][c] = __ldg(w + co * R + r);
  }
  const long long p0 = ((long long)blockIdx.x * 8 + warp) * chunk;
  const long long p1 = min(npix, p0 + chunk);
  if (p0 >= p1) return;
  Pix q;
  q.img = (int)(p0 / hw);
  const int rem = (int)(p0 - (long long)q.img * hw);
  q.oh = rem / W;
  q.ow = rem - q.oh * W;
  for (long long p = p0; p < p1; p += PB) {
    const int nb = (int)min((long long)PB, p1 - p);
    float xv[PB];
#pragma unroll
    for (int b = 0; b < PB; ++b) {
      xv[b] = 0.f;
      if (b < nb) { xv[b] = col_value<CIN>(x, q, H, W, lane); q.step(H, W); }
    }
#pragma unroll
    for (int b = 0; b < PB; ++b)
      if (lane < R4) colw[warp][b][lane] = xv[b];
    __syncwarp();
#pragma unroll
    for (int b = 0; b < PB; ++b) {
      if (b < nb) {
        float o[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) o[c] = b0[c];
#pragma unroll
        for (int r4 = 0; r4 < R4; r4 += 4) {
          const float4 cv = *reinterpret_cast<const float4*>(&colw[warp][b][r4]);
          const float cr[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (r4 + j < R) {
#pragma unroll
              for (int c = 0; c < CPL; ++c) o[c] = fmaf(cr[j], wr[r4 + j][c], o[c]);
            }
        }
        float* dst = y + (p + b) * COUT + lane * CPL;
#pragma unroll
        for (int c = 0; c < CPL; ++c) dst[c] = relu ? fmaxf(o[c], 0.f) : o[c];
      }
    }
    __syncwarp();
  }
}

inline int grid_for(long long npix) {
  long long g = 2LL * num_sms();
  const long long units = cdivll(npix, 8LL * PB);     // >= one batch per warp
  return (int)(units < g ? units : g);
}

}  // namespace small

bool small_conv_fwd_ok(int cin, int cout) { return cin == 3 && (cout == 32 || cout == 64 || cout == 128); }

bpx_status_t small_conv_fwd(const float* x, const float* w, const float* bias, float* y, int n,
                            int h, int w_, int cin, int cout, int relu, cudaStream_t st) {
  if (!small_conv_fwd_ok(cin, cout)) return BPX_ERR_INVALID_ARGUMENT;
  const long long npix = (long long)n * h * w_;
  if (npix == 0) return launch_status(0);
  const int grid = small::grid_for(npix);
  const long long chunk = cdivll(cdivll(npix, 8LL * grid), small::PB) * small::PB;
  const int g = (int)cdivll(npix, 8 * chunk);
  switch (cout) {
    case 32: small::small_fwd_kernel<3, 1><<<g, 256, 0, st>>>(x, w, bias, y, h, w_, npix, chunk, relu); break;
    case 64: small::small_fwd_kernel<3, 2><<<g, 256, 0, st>>>(x, w, bias, y, h, w_, npix, chunk, relu); break;
    default: small::small_fwd_kernel<3, 4><<<g, 256, 0, st>>>(x, w, bias, y, h, w_, npix, chunk, relu); break;
  }
  return launch_status();
}

bool small_conv_wgrad_ok(int cin, int cout) { return cin == 3 && (cout == 32 || cout == 64 || cout == 128); }

size_t small_conv_wgrad_ws(int n, int h, int w, int cin, int cout) {
  if (!small_conv_wgrad_ok(cin, cout)) return 0;
  const long long npix = (long long)n * h * w;
  const int g = small::grid_for(npix < 1 ? 1 : npix);
  return (size_t)g * (size_t)(cout * 9 * cin + cout) * sizeof(float);
}

bpx_status_t small_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias, int n,
                              int h, int w_, int cin, int cout, void* ws, size_t ws_bytes,
                              cudaStream_t st) {
  if (!small_conv_wgrad_ok(cin, cout) || !aligned16(dz)) return BPX_ERR_INVALID_ARGUMENT;
  if (ws_bytes < small_conv_wgrad_ws(n, h, w_, cin, cout)) return BPX_ERR_WORKSPACE;
  const long long npix = (long long)n * h * w_;
  const size_t slab = (size_t)cout * 9 * cin;
  if (npix == 0) {
    cudaMemsetAsync(dw, 0, sizeof(float) * slab, st);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * cout, st);
    return launch_status(0);
  }
  const int grid = small::grid_for(npix);
  const long long chunk = cdivll(cdivll(npix, 8LL * grid), small::PB) * small::PB;
  const int g = (int)cdivll(npix, 8 * chunk);
  float* part = static_cast<float*>(ws);
  float* bpart = part + (size_t)g * slab;
  switch (cout) {
    case 32: small::small_wgrad_kernel<3, 1><<<g, 256, 0, st>>>(x, dz, h, w_, npix, chunk, part, bpart); break;
    case 64: small::small_wgrad_kernel<3, 2><<<g, 256, 0, st>>>(x, dz, h, w_, npix, chunk, part, bpart); break;
    default: small::small_wgrad_kernel<3, 4><<<g, 256, 0, st>>>(x, dz, h, w_, npix, chunk, part, bpart); break;
  }
  bpx_status_t s = launch_status();
  if (s != BPX_OK) return s;
  s = split_reduce(part, g, slab, dw, st);
  if (s != BPX_OK || !dbias) return s;
  return split_reduce(bpart, g, (size_t)cout, dbias, st);
}

}  // namespace bpx
