// FFMA engine for the pixel-batched 1x1 convolutions of the four-tower net
// (inception_like, synth.py:172-226: 128 -> 32 and 64 -> 32 towers, run as
// dense ops with b = pixels): thin GEMMs whose narrow side is 32.
//
//   fwd   y[p][o]  = act(b[o] + sum_i x[p][i] w[o][i])     K = in  <= 128, N = 32
//   dgrad dx[p][i] = mask(p,i) * sum_o dy[p][o] w[o][i]   K = 32,         N = in
//   wgrad dw[o][i] = sum_p dy[p][o] x[p][i],  db[o] = sum_p dy[p][o]   K = pixels
//
// Why FFMA and not the tensor cores: per output element these layers do 32
// to 128 MACs, so a 128-pixel tile is ~0.5 M MACs against 16-64 KB of
// operands; fp32 FFMA at 128 FMA/clk/SM finishes a tile in ~4 k cycles,
// about the time its operands take to arrive, and it is fp32-exact per
// product (no 3xTF32 split, no split-K finish: the whole K sits in shared
// memory).  The tcgen05 SS engine this replaces ran split-K GEMMs plus a
// finish pass and a bias column sum: ~60-75 us per op at b = 39 200 where
// these kernels need ~5-10 (profiles/r2_inception_launches_summary.txt).
//
// Every reduction runs in a fixed order (K ascending inside a thread; the
// wgrad partials of the pixel chunks summed in chunk order by thin_reduce),
// so results are bitwise reproducible.
#include "common.cuh"

namespace bpx {
namespace thin {

// 16-byte global -> shared copies in flight without staging through registers
// (LDGSTS): every tile load issues all its requests at once; src_bytes = 0
// zero-fills (rows past the end).
__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem),
               "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int TM = 128;          // pixels per tile
constexpr int N32 = 32;          // the narrow side
constexpr int PAD = 4;           // floats of row padding: conflict-free LDS.128

// ---- fwd: tile 128 pixels x 32 outputs; thread = 4 rows x 4 outputs
template <int K>
constexpr int fwd_smem() { return (TM + N32) * (K + PAD) * 4; }

template <int K>
__global__ void __launch_bounds__(256)
fwd_kernel(const float* __restrict__ x, const float* __restrict__ w,
           const float* __restrict__ bias, float* __restrict__ y, long long P, int relu) {
  extern __shared__ float4 dsmem[];
  auto xs = reinterpret_cast<float(*)[K + PAD]>(dsmem);
  auto wsm = reinterpret_cast<float(*)[K + PAD]>(reinterpret_cast<float*>(dsmem) + TM * (K + PAD));
  const int tid = threadIdx.x;
  const long long p0 = (long long)blockIdx.x * TM;
  constexpr int KH = K / 2;                     // two K halves: compute on the first
#pragma unroll                                  // while the second is in flight
  for (int h = 0; h < 2; ++h) {
    for (int e = tid; e < N32 * KH / 4; e += 256) {
      const int o = e / (KH / 4), k = h * KH + 4 * (e % (KH / 4));
      cp16(&wsm[o][k], w + (long long)o * K + k, true);
    }
    for (int e = tid; e < TM * KH / 4; e += 256) {
      const int r = e / (KH / 4), k = h * KH + 4 * (e % (KH / 4));
      const bool ok = p0 + r < P;
      cp16(&xs[r][k], x + (ok ? (p0 + r) * K + k : 0), ok);
    }
    cp_commit();
  }
  const int cg = tid & 7, rg = tid >> 3;        // 8 output groups x 32 row groups
  float acc[4][4] = {};
  cp_wait<1>();
  __syncthreads();
#pragma unroll 4
  for (int k = 0; k < K; k += 4) {
    if (k == KH) {
      cp_wait<0>();
      __syncthreads();
    }
    float4 a[4], b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = *reinterpret_cast<const float4*>(&xs[rg + 32 * j][k]);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = *reinterpret_cast<const float4*>(&wsm[cg + 8 * i][k]);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[j][i] = fmaf(a[j].x, b[i].x, acc[j][i]);
        acc[j][i] = fmaf(a[j].y, b[i].y, acc[j][i]);
        acc[j][i] = fmaf(a[j].z, b[i].z, acc[j][i]);
        acc[j][i] = fmaf(a[j].w, b[i].w, acc[j][i]);
      }
  }
  // thread holds outputs cg + 8i (i = 0..3) of rows rg + 32j: scalar stores,
  // a warp's 8 lanes of one row covering 8 consecutive outputs (32 B) per i
  float bb[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) bb[i] = bias ? __ldg(bias + cg + 8 * i) : 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const long long p = p0 + rg + 32 * j;
    if (p >= P) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float t = acc[j][i] + bb[i];
      y[p * N32 + cg + 8 * i] = relu ? fmaxf(t, 0.f) : t;
    }
  }
}

// ---- dgrad: tile 128 pixels x N inputs; thread = 8 rows x (N/16) inputs
template <int N>
__global__ void __launch_bounds__(256)
dgrad_kernel(const float* __restrict__ dy, const float* __restrict__ w,
             const float* __restrict__ mask, float* __restrict__ dx, long long P) {
  constexpr int CW = N / 16;                    // inputs per thread (8 or 4)
  __shared__ __align__(16) float ds[TM][N32 + PAD];
  __shared__ __align__(16) float wsm[N32][N];
  const int tid = threadIdx.x;
  const long long p0 = (long long)blockIdx.x * TM;
  for (int e = tid; e < N32 * N / 4; e += 256) cp16(&wsm[0][0] + 4 * e, w + 4 * e, true);
  for (int e = tid; e < TM * N32 / 4; e += 256) {
    const int r = e / (N32 / 4), k = 4 * (e % (N32 / 4));
    const bool ok = p0 + r < P;
    cp16(&ds[r][k], dy + (ok ? (p0 + r) * N32 + k : 0), ok);
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  const int rg = tid & 15, cg = tid >> 4;       // 16 row groups x 16 input groups
  float acc[8][CW] = {};
#pragma unroll 2
  for (int k = 0; k < N32; k += 4) {
    float4 a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = *reinterpret_cast<const float4*>(&ds[rg + 16 * j][k]);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      float b[CW];
#pragma unroll
      for (int c = 0; c < CW; c += 4) {
        const float4 t = *reinterpret_cast<const float4*>(&wsm[k + kk][cg * CW + c]);
        b[c] = t.x; b[c + 1] = t.y; b[c + 2] = t.z; b[c + 3] = t.w;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float av = kk == 0 ? a[j].x : kk == 1 ? a[j].y : kk == 2 ? a[j].z : a[j].w;
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[j][c] = fmaf(av, b[c], acc[j][c]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const long long p = p0 + rg + 16 * j;
    if (p >= P) continue;
#pragma unroll
    for (int c = 0; c < CW; c += 4) {
      float4 v = make_float4(acc[j][c], acc[j][c + 1], acc[j][c + 2], acc[j][c + 3]);
      const long long off = p * N + cg * CW + c;
      if (mask) {
        const float4 m = __ldg(reinterpret_cast<const float4*>(mask + off));
        v.x = m.x > 0.f ? v.x : 0.f; v.y = m.y > 0.f ? v.y : 0.f;
        v.z = m.z > 0.f ? v.z : 0.f; v.w = m.w > 0.f ? v.w : 0.f;
      }
      *reinterpret_cast<float4*>(dx + off) = v;
    }
  }
}

// ---- wgrad: each CTA sums a contiguous pixel chunk into a [32][K] partial
// (+ the [32] bias partial); thread = 8 outputs x 4 inputs.  The chunk is
// walked in 64-pixel tiles, double-buffered: the next tile's cp.async loads
// are in flight while this one is summed.
constexpr int TW = 64;

template <int K>
constexpr int wgrad_smem() { return 2 * (TW * (K + PAD) + TW * (N32 + PAD)) * 4; }

template <int K>
__global__ void __launch_bounds__(K)
wgrad_kernel(const float* __restrict__ x, const float* __restrict__ dy,
             float* __restrict__ part, float* __restrict__ bpart, long long P, long long chunk) {
  constexpr int NT = K;                         // K/4 input groups x 4 groups of 8 outputs
  constexpr int IG = K / 4;
  constexpr int XF = TW * (K + PAD), DF = TW * (N32 + PAD);   // floats per buffer
  extern __shared__ float4 dsmem[];
  float* sm = reinterpret_cast<float*>(dsmem);
  const int tid = threadIdx.x;
  const int ig = tid % IG, og = tid / IG;
  const long long a0 = (long long)blockIdx.x * chunk;
  const long long a1 = a0 + chunk < P ? a0 + chunk : P;
  const int ntiles = a1 > a0 ? (int)cdivll(a1 - a0, TW) : 0;
  auto load = [&](int t) {
    float* xs = sm + (t & 1) * (XF + DF);
    float* ds = xs + XF;
    const long long t0 = a0 + (long long)t * TW;
    for (int e = tid; e < TW * K / 4; e += NT) {
      const int r = e / (K / 4), k = 4 * (e % (K / 4));
      const bool ok = t0 + r < a1;
      cp16(xs + r * (K + PAD) + k, x + (ok ? (t0 + r) * K + k : 0), ok);
    }
    for (int e = tid; e < TW * N32 / 4; e += NT) {
      const int r = e / (N32 / 4), k = 4 * (e % (N32 / 4));
      const bool ok = t0 + r < a1;
      cp16(ds + r * (N32 + PAD) + k, dy + (ok ? (t0 + r) * N32 + k : 0), ok);
    }
    cp_commit();
  };
  float acc[8][4] = {};
  float bacc[8] = {};
  if (ntiles > 0) load(0);
  for (int t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) {
      load(t + 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const float* xs = sm + (t & 1) * (XF + DF);
    const float* ds = xs + XF;
    const long long t0 = a0 + (long long)t * TW;
    const int rows = (int)(a1 - t0 < TW ? a1 - t0 : TW);
    for (int r = 0; r < rows; ++r) {
      const float4 xv = *reinterpret_cast<const float4*>(xs + r * (K + PAD) + 4 * ig);
      const float4 d0 = *reinterpret_cast<const float4*>(ds + r * (N32 + PAD) + 8 * og);
      const float4 d1 = *reinterpret_cast<const float4*>(ds + r * (N32 + PAD) + 8 * og + 4);
      const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        acc[o][0] = fmaf(dv[o], xv.x, acc[o][0]);
        acc[o][1] = fmaf(dv[o], xv.y, acc[o][1]);
        acc[o][2] = fmaf(dv[o], xv.z, acc[o][2]);
        acc[o][3] = fmaf(dv[o], xv.w, acc[o][3]);
        bacc[o] += dv[o];
      }
    }
    __syncthreads();                            // buffer t & 1 is refilled at t + 2
  }
  float* pp = part + (long long)blockIdx.x * N32 * K;
#pragma unroll
  for (int o = 0; o < 8; ++o)
    *reinterpret_cast<float4*>(pp + (8 * og + o) * K + 4 * ig) =
        make_float4(acc[o][0], acc[o][1], acc[o][2], acc[o][3]);
  if (ig == 0) {
#pragma unroll
    for (int o = 0; o < 8; ++o) bpart[(long long)blockIdx.x * N32 + 8 * og + o] = bacc[o];
  }
}

// out[i] = sum_s part[s][i], fixed order: a block owns 32 outputs (the bias
// partials ride along as outputs n..n+31); its warp q sums splits
// [q*S/8, (q+1)*S/8) in order (coalesced 128-B rows, 8 loads in flight), and
// the eight warp sums are added in warp order.
__global__ void __launch_bounds__(256)
thin_reduce(const float* __restrict__ part, const float* __restrict__ bpart, int splits, int n,
            float* __restrict__ dw, float* __restrict__ db) {
  __shared__ float red[8][32];
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const int k0 = (int)((long long)splits * q / 8), k1 = (int)((long long)splits * (q + 1) / 8);
  float s = 0.f;
  if (i < n) {
#pragma unroll 8
    for (int k = k0; k < k1; ++k) s += part[(long long)k * n + i];
  } else if (i < n + N32) {
#pragma unroll 8
    for (int k = k0; k < k1; ++k) s += bpart[k * N32 + (i - n)];
  }
  red[q][lane] = s;
  __syncthreads();
  if (q == 0) {
    float t = red[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) t += red[w][lane];
    if (i < n) dw[i] = t;
    else if (i < n + N32 && db) db[i - n] = t;
  }
}

// ---- 3x3 / pad-1 weight gradient for 32 -> 32 convs (the four-tower net's
// tower convs): dw[o][tap][i] = sum_p dy[p][o] x[p + s_tap][i] (zero
// padding), db[o] = sum_p dy[p][o].  M = 32, N = 9 * 32 = 288, K = pixels.
// A CTA walks its pixel chunk in 64-pixel tiles of the flattened NHWC
// tensor; per tile it stages the x rows [t0 - W - 1, t0 + 64 + W + 1) (every
// tap's shifted window) and a 9-bit per-pixel tap mask (the padding and the
// image-row wrap), double-buffered by cp.async.  Thread = 8 outputs x one
// (tap, 4 inputs) group: 288 threads.
constexpr int C3 = 32;

__host__ __device__ constexpr int c3_halo(int W) { return TW + 2 * W + 2; }
inline int c3_smem(int W) { return 2 * (c3_halo(W) * (C3 + PAD) + TW * (N32 + PAD) + TW) * 4; }

__global__ void __launch_bounds__(288)
wgrad3_kernel(const float* __restrict__ x, const float* __restrict__ dy,
              float* __restrict__ part, float* __restrict__ bpart, long long P, int H, int W,
              long long chunk) {
  constexpr int NT = 288;
  const int HR = c3_halo(W);
  const int XF = HR * (C3 + PAD), DF = TW * (N32 + PAD), BUF = XF + DF + TW;
  extern __shared__ float4 dsmem[];
  float* sm = reinterpret_cast<float*>(dsmem);
  const int tid = threadIdx.x;
  const int ig = tid % 72, og = tid / 72;       // (tap, 4 inputs) group, 8-output group
  const int tap = ig >> 3, dyt = tap / 3 - 1, dxt = tap % 3 - 1;
  const long long a0 = (long long)blockIdx.x * chunk;
  const long long a1 = a0 + chunk < P ? a0 + chunk : P;
  const int ntiles = a1 > a0 ? (int)cdivll(a1 - a0, TW) : 0;
  const int HWp = H * W;
  auto load = [&](int t) {
    float* xs = sm + (t & 1) * BUF;
    float* ds = xs + XF;
    const long long t0 = a0 + (long long)t * TW;
    const long long h0 = t0 - W - 1;
    for (int e = tid; e < HR * (C3 / 4); e += NT) {
      const int r = e >> 3, k = 4 * (e & 7);
      const long long p = h0 + r;
      const bool ok = p >= 0 && p < P;
      cp16(xs + r * (C3 + PAD) + k, x + (ok ? p * C3 + k : 0), ok);
    }
    for (int e = tid; e < TW * (N32 / 4); e += NT) {
      const int r = e >> 3, k = 4 * (e & 7);
      const bool ok = t0 + r < a1;
      cp16(ds + r * (N32 + PAD) + k, dy + (ok ? (t0 + r) * N32 + k : 0), ok);
    }
    cp_commit();
    if (tid < TW) {                             // tap mask of pixel t0 + tid
      int* msk = reinterpret_cast<int*>(ds + DF);
      const long long p = t0 + tid;
      int m = 0;
      if (p < a1) {
        const int rem = (int)(p % HWp), oh = rem / W, ow = rem - oh * W;
#pragma unroll
        for (int tp = 0; tp < 9; ++tp) {
          const int ih = oh + tp / 3 - 1, iw = ow + tp % 3 - 1;
          if ((unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W) m |= 1 << tp;
        }
      }
      msk[tid] = m;
    }
  };
  float acc[8][4] = {};
  float bacc[8] = {};
  const int xoff = (W + 1 + dyt * W + dxt) * (C3 + PAD) + 4 * (ig & 7);
  if (ntiles > 0) load(0);
  for (int t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) {
      load(t + 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const float* xs = sm + (t & 1) * BUF;
    const float* ds = xs + XF;
    const int* msk = reinterpret_cast<const int*>(ds + DF);
    const long long t0 = a0 + (long long)t * TW;
    const int rows = (int)(a1 - t0 < TW ? a1 - t0 : TW);
    for (int r = 0; r < rows; ++r) {
      float4 xv = *reinterpret_cast<const float4*>(xs + r * (C3 + PAD) + xoff);
      if (!((msk[r] >> tap) & 1)) xv = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 d0 = *reinterpret_cast<const float4*>(ds + r * (N32 + PAD) + 8 * og);
      const float4 d1 = *reinterpret_cast<const float4*>(ds + r * (N32 + PAD) + 8 * og + 4);
      const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        acc[o][0] = fmaf(dv[o], xv.x, acc[o][0]);
        acc[o][1] = fmaf(dv[o], xv.y, acc[o][1]);
        acc[o][2] = fmaf(dv[o], xv.z, acc[o][2]);
        acc[o][3] = fmaf(dv[o], xv.w, acc[o][3]);
        bacc[o] += dv[o];
      }
    }
    __syncthreads();
  }
  constexpr int NO = 9 * C3;                    // 288 weights per output channel
  float* pp = part + (long long)blockIdx.x * N32 * NO;
#pragma unroll
  for (int o = 0; o < 8; ++o)
    *reinterpret_cast<float4*>(pp + (8 * og + o) * NO + 4 * ig) =
        make_float4(acc[o][0], acc[o][1], acc[o][2], acc[o][3]);
  if (ig == 0) {
#pragma unroll
    for (int o = 0; o < 8; ++o) bpart[(long long)blockIdx.x * N32 + 8 * og + o] = bacc[o];
  }
}

inline int wgrad_splits(long long P) {
  long long tiles = cdivll(P, 32);
  long long s = 2LL * num_sms();
  return (int)(tiles < s ? tiles : s);
}

}  // namespace thin

// Pixel-batched (b > 256) dense ops with 32 outputs and 64 or 128 inputs.
bool thin_linear_ok(int b, int in, int out) {
  return b > 256 && out == 32 && (in == 64 || in == 128);
}

size_t thin_linear_ws(int b, int in, int out) {
  if (!thin_linear_ok(b, in, out)) return 0;
  const int s = thin::wgrad_splits(b);
  return (size_t)s * (32 * (size_t)in + 32) * sizeof(float);
}

bpx_status_t thin_linear_fwd(const float* x, const float* w, const float* bias, float* y,
                             int b, int in, int out, int relu, cudaStream_t st) {
  if (!thin_linear_ok(b, in, out) || !aligned16(x) || !aligned16(w) || !aligned16(y))
    return BPX_ERR_UNSUPPORTED;
  const int grid = cdiv(b, thin::TM);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(thin::fwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         thin::fwd_smem<128>());
    cudaFuncSetAttribute(thin::fwd_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         thin::fwd_smem<64>());
    attr = true;
  }
  if (in == 128)
    thin::fwd_kernel<128><<<grid, 256, thin::fwd_smem<128>(), st>>>(x, w, bias, y, b, relu);
  else
    thin::fwd_kernel<64><<<grid, 256, thin::fwd_smem<64>(), st>>>(x, w, bias, y, b, relu);
  return launch_status();
}

bpx_status_t thin_linear_dgrad(const float* dy, const float* w, const float* mask, float* dx,
                               int b, int in, int out, cudaStream_t st) {
  if (!thin_linear_ok(b, in, out) || !aligned16(dy) || !aligned16(w) || !aligned16(dx) ||
      (mask && !aligned16(mask)))
    return BPX_ERR_UNSUPPORTED;
  const int grid = cdiv(b, thin::TM);
  if (in == 128) thin::dgrad_kernel<128><<<grid, 256, 0, st>>>(dy, w, mask, dx, b);
  else thin::dgrad_kernel<64><<<grid, 256, 0, st>>>(dy, w, mask, dx, b);
  return launch_status();
}

bpx_status_t thin_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias,
                               int b, int in, int out, void* ws, size_t ws_bytes,
                               cudaStream_t st) {
  if (!thin_linear_ok(b, in, out) || !aligned16(x) || !aligned16(dy) || !aligned16(dw))
    return BPX_ERR_UNSUPPORTED;
  if (ws_bytes < thin_linear_ws(b, in, out) || !aligned16(ws)) return BPX_ERR_WORKSPACE;
  const int splits = thin::wgrad_splits(b);
  const long long chunk = cdivll(cdivll(b, splits), 32) * 32;
  const int used = (int)cdivll(b, chunk);
  float* part = static_cast<float*>(ws);
  float* bpart = part + (size_t)used * 32 * in;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(thin::wgrad_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         thin::wgrad_smem<128>());
    cudaFuncSetAttribute(thin::wgrad_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         thin::wgrad_smem<64>());
    attr = true;
  }
  if (in == 128)
    thin::wgrad_kernel<128><<<used, 128, thin::wgrad_smem<128>(), st>>>(x, dy, part, bpart, b,
                                                                        chunk);
  else
    thin::wgrad_kernel<64><<<used, 64, thin::wgrad_smem<64>(), st>>>(x, dy, part, bpart, b,
                                                                     chunk);
  const int n = 32 * in;
  thin::thin_reduce<<<cdiv(n + 32, 32), 256, 0, st>>>(part, bpart, used, n, dw, dbias);
  return launch_status(2);
}

}  // namespace bpx

namespace bpx {

// 3x3 weight gradient of 32 -> 32 convs, W <= 64 (the halo fits).
bool thin_conv_wgrad_ok(int cin, int cout, int w) { return cin == 32 && cout == 32 && w <= 64; }

size_t thin_conv_wgrad_ws(int n, int h, int w, int cin, int cout) {
  if (!thin_conv_wgrad_ok(cin, cout, w)) return 0;
  const int s = thin::wgrad_splits((long long)n * h * w);
  return (size_t)s * (32 * 288 + 32) * sizeof(float);
}

bpx_status_t thin_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias, int n,
                             int h, int w_, int cin, int cout, void* ws, size_t ws_bytes,
                             cudaStream_t st) {
  if (!thin_conv_wgrad_ok(cin, cout, w_) || !aligned16(x) || !aligned16(dz) || !aligned16(dw))
    return BPX_ERR_UNSUPPORTED;
  const long long P = (long long)n * h * w_;
  if (P == 0) return launch_status(0);
  if (ws_bytes < thin_conv_wgrad_ws(n, h, w_, cin, cout) || !aligned16(ws)) return BPX_ERR_WORKSPACE;
  const int splits = thin::wgrad_splits(P);
  const long long chunk = cdivll(cdivll(P, splits), 32) * 32;
  const int used = (int)cdivll(P, chunk);
  float* part = static_cast<float*>(ws);
  float* bpart = part + (size_t)used * 32 * 288;
  const int smem = thin::c3_smem(w_);
  static int attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(thin::wgrad3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = smem;
  }
  thin::wgrad3_kernel<<<used, 288, smem, st>>>(x, dz, part, bpart, P, h, w_, chunk);
  const int nn = 32 * 288;
  thin::thin_reduce<<<cdiv(nn + 32, 32), 256, 0, st>>>(part, bpart, used, nn, dw, dbias);
  return launch_status(2);
}

}  // namespace bpx
