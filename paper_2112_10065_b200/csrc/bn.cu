// Synchronised batch normalisation over a layer's GPU group [0, g) for the
// residual nets (wideresnet_like C3, resnet50_like background), SURVEY.md
// §7.4-8: per-shard batch statistics would make the numerics depend on the
// plan's g, so every rank reduces its shard's per-channel sums, the sums
// are allreduced over [0, g) (the executor's small in-graph allreduce), and
// every rank normalises with the statistics of the WHOLE global batch --
// the result is full-batch BN whatever the plan (the CPU oracle is plain
// BatchNorm2d in training mode, eps 1e-5, biased variance).
//
//   fwd : S = [sum z ; sum z^2] (local)  -> allreduce ->  y = act(gamma * (z - mu) * rstd + beta)
//   bwd : T = [sum g ; sum g*xhat] (local) -> allreduce ->
//         dz = gamma * rstd * (g - T0/N - xhat * T1/N)
//   The local T is also the layer's parameter gradient [dbeta ; dgamma]
//   (summed over [0, g) by the gradient-bucket allreduce like every other
//   parameter gradient).
//
// Sums accumulate in fp64 per thread, then in fixed order across rows of a
// block, across blocks (finish kernel): bitwise reproducible.  NHWC: the
// channel is the fastest dimension, so a block reads whole 16-B channel
// groups of consecutive pixels.
#include "common.cuh"

namespace bpx {
namespace bn {

constexpr int NT = 256;
// statistics passes: NB blocks of NTP threads -- a constant (results are
// independent of the GPU), with ~8 MB of loads in flight on a whole B200
// (128 blocks of 256 threads left them at ~25 % of the HBM rate); 256 parts
// keep the fixed-order finish short
constexpr int NB = 256;
constexpr int NTP = 1024;
constexpr int UNR = 4;           // rows (vectors) loaded per thread before their adds

// partial[blk][0..c) = sum a, [c..2c) = sum a * f(b)  where MODE 0: f = a (squares);
// MODE 1: f = (b - mu) * rstd with mu/rstd from stats (xhat of z = b)
template <int MODE>
__global__ void __launch_bounds__(NTP)
partial_kernel(const float* __restrict__ a, const float* __restrict__ b,
               const float* __restrict__ stats, long long npix, long long ntot, int c, float eps,
               double* __restrict__ part) {
  extern __shared__ double sh[];               // [rows in flight][2c]
  const int C4 = c / 4;
  const int tpr = C4 < NTP ? C4 : NTP;         // threads per pixel row
  const int rpi = NTP / tpr;                   // rows in flight
  const int rr = threadIdx.x / tpr, cq = threadIdx.x % tpr;
  const int J = C4 / tpr;                      // channel groups per thread (c <= 4096)
  const long long chunk = (npix + gridDim.x - 1) / gridDim.x;
  const long long p0 = blockIdx.x * chunk, p1 = p0 + chunk < npix ? p0 + chunk : npix;
  for (int j = 0; j < J; ++j) {
    const int c0 = 4 * (cq + j * tpr);
    double s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
    float mu[4], rs[4];
    if (MODE == 1) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double m = (double)stats[c0 + e] / (double)ntot;
        const double v = (double)stats[c + c0 + e] / (double)ntot - m * m;
        mu[e] = (float)m;
        rs[e] = (float)(1.0 / sqrt((v > 0 ? v : 0.0) + (double)eps));
      }
    }
    if (rr < rpi && threadIdx.x < rpi * tpr) {
      // rows p0 + rr + k * rpi in order; UNR loads issued before their adds
      for (long long p = p0 + rr; p < p1; p += (long long)UNR * rpi) {
        float4 va[UNR], vb[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const long long q = p + (long long)u * rpi;
          va[u] = q < p1 ? __ldg(reinterpret_cast<const float4*>(a + q * c + c0))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
          if (MODE == 1)
            vb[u] = q < p1 ? __ldg(reinterpret_cast<const float4*>(b + q * c + c0))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          if (p + (long long)u * rpi >= p1) break;
          const float av[4] = {va[u].x, va[u].y, va[u].z, va[u].w};
          if (MODE == 0) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              s1[e] += av[e];
              s2[e] += (double)av[e] * av[e];
            }
          } else {
            const float bv[4] = {vb[u].x, vb[u].y, vb[u].z, vb[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              s1[e] += av[e];
              s2[e] += (double)av[e] * ((bv[e] - mu[e]) * rs[e]);
            }
          }
        }
      }
    }
    // fixed-order reduction over the rows in flight
    if (threadIdx.x < rpi * tpr) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        sh[(size_t)rr * 2 * c + c0 + e] = s1[e];
        sh[(size_t)rr * 2 * c + c + c0 + e] = s2[e];
      }
    }
    __syncthreads();
    if (rr == 0) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        double t1 = 0, t2 = 0;
        for (int q = 0; q < rpi; ++q) {
          t1 += sh[(size_t)q * 2 * c + c0 + e];
          t2 += sh[(size_t)q * 2 * c + c + c0 + e];
        }
        part[(size_t)blockIdx.x * 2 * c + c0 + e] = t1;
        part[(size_t)blockIdx.x * 2 * c + c + c0 + e] = t2;
      }
    }
    __syncthreads();
  }
}

// out[i] = sum_k part[k][i]: 8 warps per 32 outputs, warp w sums the parts
// k = w, w + 8, ... (4 loads in flight), then a fixed-order combine
__global__ void finish_kernel(const double* __restrict__ part, int nb, int n2,
                              float* __restrict__ out) {
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  double s = 0;
  if (i < n2) {
    int k = w;
    for (; k + 24 < nb; k += 32) {
      const double v0 = part[(size_t)k * n2 + i], v1 = part[(size_t)(k + 8) * n2 + i];
      const double v2 = part[(size_t)(k + 16) * n2 + i], v3 = part[(size_t)(k + 24) * n2 + i];
      s += v0; s += v1; s += v2; s += v3;
    }
    for (; k < nb; k += 8) s += part[(size_t)k * n2 + i];
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && i < n2) {
    for (int q = 1; q < 8; ++q) s += red[q][lane];
    out[i] = (float)s;
  }
}

// Elementwise passes: per-channel coefficients in shared memory, float4
// over NHWC with UNR vectors in flight per thread.  The grid stride is a
// multiple of c/4 whenever NT is (c <= 1024), so a thread's channel group is
// fixed and no 64-bit modulo runs per element.  amax (nullable): atomicMax of
// the output's max |v| bits -- the fp16x3 scale word of the conv reading it.
__device__ __forceinline__ void amax_commit_bn(uint32_t* amax, uint32_t mx) {
  if (!amax) return;
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(amax, mx);
}

__global__ void __launch_bounds__(NT)
apply_kernel(const float* __restrict__ z, const float* __restrict__ stats,
             const float* __restrict__ gb, long long npix, long long ntot, int c, float eps,
             int relu, float* __restrict__ y, uint32_t* __restrict__ amax) {
  extern __shared__ float coef[];               // scale[c], shift[c]
  for (int i = threadIdx.x; i < c; i += NT) {
    const double m = (double)stats[i] / (double)ntot;
    const double v = (double)stats[c + i] / (double)ntot - m * m;
    const double rstd = 1.0 / sqrt((v > 0 ? v : 0.0) + (double)eps);
    const double sc = (double)gb[c + i] * rstd;
    coef[i] = (float)sc;
    coef[c + i] = (float)((double)gb[i] - m * sc);
  }
  __syncthreads();
  const long long n4 = npix * c / 4;
  const int C4 = c / 4;
  const long long stride = (long long)gridDim.x * NT;
  const bool fixed = stride % C4 == 0;
  const long long e0 = blockIdx.x * (long long)NT + threadIdx.x;
  const int cf = 4 * (int)(e0 % C4);
  uint32_t mx = 0;
  for (long long e = e0; e < n4; e += UNR * stride) {
    float4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      v[u] = e + u * stride < n4 ? reinterpret_cast<const float4*>(z)[e + u * stride]
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const long long eu = e + u * stride;
      if (eu >= n4) break;
      const int c0 = fixed ? cf : 4 * (int)(eu % C4);
      float r[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float t = fmaf(r[k], coef[c0 + k], coef[c + c0 + k]);
        r[k] = relu ? fmaxf(t, 0.f) : t;
        mx = max(mx, __float_as_uint(r[k]) & 0x7fffffffu);
      }
      reinterpret_cast<float4*>(y)[eu] = make_float4(r[0], r[1], r[2], r[3]);
    }
  }
  amax_commit_bn(amax, mx);
}

__global__ void __launch_bounds__(NT)
bwd_apply_kernel(const float* __restrict__ g, const float* __restrict__ z,
                 const float* __restrict__ stats, const float* __restrict__ sums,
                 const float* __restrict__ gb, long long npix, long long ntot, int c, float eps,
                 float* __restrict__ dz, uint32_t* __restrict__ amax) {
  extern __shared__ float coef[];               // a = gamma*rstd, mu, rstd, t0, t1
  for (int i = threadIdx.x; i < c; i += NT) {
    const double m = (double)stats[i] / (double)ntot;
    const double v = (double)stats[c + i] / (double)ntot - m * m;
    const double rstd = 1.0 / sqrt((v > 0 ? v : 0.0) + (double)eps);
    coef[i] = (float)((double)gb[c + i] * rstd);
    coef[c + i] = (float)m;
    coef[2 * c + i] = (float)rstd;
    coef[3 * c + i] = (float)((double)sums[i] / (double)ntot);
    coef[4 * c + i] = (float)((double)sums[c + i] / (double)ntot);
  }
  __syncthreads();
  const long long n4 = npix * c / 4;
  const int C4 = c / 4;
  const long long stride = (long long)gridDim.x * NT;
  const bool fixed = stride % C4 == 0;
  const long long e0 = blockIdx.x * (long long)NT + threadIdx.x;
  const int cf = 4 * (int)(e0 % C4);
  uint32_t mx = 0;
  for (long long e = e0; e < n4; e += UNR * stride) {
    float4 gv[UNR], zv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const bool in = e + u * stride < n4;
      gv[u] = in ? reinterpret_cast<const float4*>(g)[e + u * stride] : make_float4(0.f, 0.f, 0.f, 0.f);
      zv[u] = in ? reinterpret_cast<const float4*>(z)[e + u * stride] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const long long eu = e + u * stride;
      if (eu >= n4) break;
      const int c0 = fixed ? cf : 4 * (int)(eu % C4);
      const float gg[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
      const float zz[4] = {zv[u].x, zv[u].y, zv[u].z, zv[u].w};
      float r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int ch = c0 + k;
        const float xh = (zz[k] - coef[c + ch]) * coef[2 * c + ch];
        r[k] = coef[ch] * (gg[k] - coef[3 * c + ch] - xh * coef[4 * c + ch]);
        mx = max(mx, __float_as_uint(r[k]) & 0x7fffffffu);
      }
      reinterpret_cast<float4*>(dz)[eu] = make_float4(r[0], r[1], r[2], r[3]);
    }
  }
  amax_commit_bn(amax, mx);
}

inline int rows_in_flight(int c) {
  const int C4 = c / 4, tpr = C4 < NTP ? C4 : NTP;
  return NTP / tpr;
}

inline int grid_for(long long n4) {
  long long g = (n4 + (long long)NT * UNR - 1) / ((long long)NT * UNR);
  long long cap = 8LL * num_sms();
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

bpx_status_t partial(int mode, const float* a, const float* b, const float* stats,
                     long long npix, long long ntot, int c, float eps, float* out, void* ws,
                     size_t ws_bytes, cudaStream_t st) {
  const size_t need = (size_t)NB * 2 * c * sizeof(double);
  if (ws_bytes < need || !ws) return BPX_ERR_WORKSPACE;
  double* part = static_cast<double*>(ws);
  const size_t sm = (size_t)rows_in_flight(c) * 2 * c * sizeof(double);
  if (sm > 227 * 1024) return BPX_ERR_UNSUPPORTED;
  static size_t attr[2] = {0, 0};
  auto k0 = partial_kernel<0>;
  auto k1 = partial_kernel<1>;
  if (sm > 48 * 1024 && sm > attr[mode]) {
    cudaFuncSetAttribute(mode ? k1 : k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr[mode] = sm;
  }
  if (mode == 0) k0<<<NB, NTP, sm, st>>>(a, b, stats, npix, ntot, c, eps, part);
  else k1<<<NB, NTP, sm, st>>>(a, b, stats, npix, ntot, c, eps, part);
  finish_kernel<<<cdiv(2 * c, 32), 256, 0, st>>>(part, NB, 2 * c, out);
  return launch_status(2);
}

}  // namespace bn
}  // namespace bpx

using namespace bpx;

extern "C" {

size_t bpx_bn_workspace(long long npix, int c) {
  (void)npix;
  return (size_t)bn::NB * 2 * (size_t)c * sizeof(double);
}

bpx_status_t bpx_bn_stats(const float* z, long long npix, int c, float* stats, void* ws,
                          size_t ws_bytes, void* stream) {
  BPX_CHECK_ARG(z && stats && npix >= 0 && c > 0 && c % 4 == 0 && c <= 4096 && aligned16(z));
  BPX_CHECK_ARG(c / 4 <= bn::NTP || (c / 4) % bn::NTP == 0);
  return bn::partial(0, z, nullptr, nullptr, npix, npix, c, 0.f, stats, ws, ws_bytes,
                     as_stream(stream));
}

bpx_status_t bpx_bn_apply(const float* z, const float* stats, const float* gamma_beta,
                          long long npix, long long ntot, int c, float eps, int relu, float* y,
                          unsigned* y_amax, void* stream) {
  BPX_CHECK_ARG(z && stats && gamma_beta && y && c > 0 && c % 4 == 0 && c <= 4096 &&
                ntot > 0 && aligned16(z) && aligned16(y));
  if (npix == 0) return BPX_OK;
  bn::apply_kernel<<<bn::grid_for(npix * c / 4), bn::NT, 2 * c * sizeof(float),
                     as_stream(stream)>>>(z, stats, gamma_beta, npix, ntot, c, eps, relu, y,
                                          y_amax);
  return launch_status();
}

bpx_status_t bpx_bn_bwd_sums(const float* g, const float* z, const float* stats, long long npix,
                             long long ntot, int c, float eps, float* sums, void* ws,
                             size_t ws_bytes, void* stream) {
  BPX_CHECK_ARG(g && z && stats && sums && c > 0 && c % 4 == 0 && c <= 4096 && ntot > 0 &&
                aligned16(g) && aligned16(z));
  BPX_CHECK_ARG(c / 4 <= bn::NTP || (c / 4) % bn::NTP == 0);
  return bn::partial(1, g, z, stats, npix, ntot, c, eps, sums, ws, ws_bytes, as_stream(stream));
}

bpx_status_t bpx_bn_bwd_apply(const float* g, const float* z, const float* stats,
                              const float* sums, const float* gamma_beta, long long npix,
                              long long ntot, int c, float eps, float* dz, unsigned* dz_amax,
                              void* stream) {
  BPX_CHECK_ARG(g && z && stats && sums && gamma_beta && dz && c > 0 && c % 4 == 0 &&
                c <= 4096 && ntot > 0 && aligned16(g) && aligned16(z) && aligned16(dz));
  if (npix == 0) return BPX_OK;
  bn::bwd_apply_kernel<<<bn::grid_for(npix * c / 4), bn::NT, 5 * c * sizeof(float),
                         as_stream(stream)>>>(g, z, stats, sums, gamma_beta, npix, ntot, c, eps,
                                              dz, dz_amax);
  return launch_status();
}

}  // extern "C"
