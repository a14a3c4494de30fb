// FFMA (CUDA-core) implicit GEMM used for the layers that do not map onto
// the tcgen05 path (conv1_1: K = 27, Cin = 3) and as an independent
// on-device cross-check of the tensor-core kernels in the GPU tests.
//
// C[m][n] = sum_k A(m,k) * B(n,k); 128 x BN x 8 tiles, 256 threads,
// register-prefetched double-buffered shared memory, split-K over grid.z.
// Operand "loaders" turn (row, k) into addresses: plain K-major / M-major
// matrices and the 3x3/pad-1 im2col gathers of the conv layers (NHWC).
#pragma once
#include "common.cuh"

namespace bpx {
namespace simt {

constexpr int BK = 8;
constexpr int NT = 256;

// ---------------------------------------------------------------- loaders
// ROWS = 128: one float4 per thread per k-step; ROWS = 32: one float.

// Row-major over k (A(m,k) = p[m*ld + k]); needs ld, K % 4 == 0 for ROWS=128.
template <int ROWS>
struct KMajor {
  const float* p; long long ld; int nrows;
  int r, kk; float4 v;
  __device__ void init(int tid) {
    if (ROWS == 128) { r = tid >> 1; kk = (tid & 1) * 4; }
    else { r = tid >> 3; kk = tid & 7; }
  }
  __device__ void load(int row0, int k0, int kend) {
    int row = row0 + r, k = k0 + kk;
    if (ROWS == 128) {
      v = (row < nrows && k < kend)
              ? __ldg(reinterpret_cast<const float4*>(p + row * ld + k))
              : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      v.x = (row < nrows && k < kend) ? __ldg(p + row * ld + k) : 0.f;
    }
  }
  __device__ void store(float* s) const {
    if (ROWS == 128) {
      s[(kk + 0) * ROWS + r] = v.x; s[(kk + 1) * ROWS + r] = v.y;
      s[(kk + 2) * ROWS + r] = v.z; s[(kk + 3) * ROWS + r] = v.w;
    } else {
      s[kk * ROWS + r] = v.x;
    }
  }
};

// Scalar K-major (row stride not a multiple of 4, e.g. conv1_1's 27).
struct KMajorScalar {
  const float* p; long long ld; int nrows;
  int r, kk; float v[4];
  __device__ void init(int tid) { r = tid >> 1; kk = (tid & 1) * 4; }
  __device__ void load(int row0, int k0, int kend) {
    int row = row0 + r;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int k = k0 + kk + j;
      v[j] = (row < nrows && k < kend) ? __ldg(p + row * ld + k) : 0.f;
    }
  }
  __device__ void store(float* s) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) s[(kk + j) * 128 + r] = v[j];
  }
};

// Column-major over rows (A(m,k) = p[k*ld + m]); nrows % 4 == 0 for ROWS=128.
template <int ROWS>
struct MMajor {
  const float* p; long long ld; int nrows;
  int r, kk; float4 v;
  __device__ void init(int tid) {
    kk = tid >> 5;
    r = (ROWS == 128) ? (tid & 31) * 4 : (tid & 31);
  }
  __device__ void load(int row0, int k0, int kend) {
    int row = row0 + r, k = k0 + kk;
    if (ROWS == 128) {
      v = (row < nrows && k < kend)
              ? __ldg(reinterpret_cast<const float4*>(p + (long long)k * ld + row))
              : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      v.x = (row < nrows && k < kend) ? __ldg(p + (long long)k * ld + row) : 0.f;
    }
  }
  __device__ void store(float* s) const {
    if (ROWS == 128) *reinterpret_cast<float4*>(s + kk * ROWS + r) = v;
    else s[kk * ROWS + r] = v.x;
  }
};

// im2col of an NHWC tensor for a 3x3 / pad-1 conv, rows = output pixels,
// k = tap*C + c.  C % 8 == 0 so a BK block never straddles a tap.
struct Im2colK {
  const float* x; int H, W, C; int npix;
  int r, kk; int img, oh, ow; bool rowok; float4 v;
  __device__ void init(int tid) { r = tid >> 1; kk = (tid & 1) * 4; }
  __device__ void set_row0(int row0) {
    int m = row0 + r;
    rowok = m < npix;
    int hw = H * W;
    img = m / hw; int rem = m - img * hw;
    oh = rem / W; ow = rem - oh * W;
  }
  __device__ void load(int /*row0*/, int k0, int kend) {
    int k = k0 + kk;
    int tap = k0 / C;                       // block-uniform
    int c = k - tap * C;
    int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
    bool ok = rowok && k < kend && (unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W;
    v = ok ? __ldg(reinterpret_cast<const float4*>(
                 x + ((long long)(img * H + ih) * W + iw) * C + c))
           : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __device__ void store(float* s) const {
    s[(kk + 0) * 128 + r] = v.x; s[(kk + 1) * 128 + r] = v.y;
    s[(kk + 2) * 128 + r] = v.z; s[(kk + 3) * 128 + r] = v.w;
  }
};

// Scalar im2col for tiny channel counts (conv1_1: C = 3, K = 27).
struct Im2colScalar {
  const float* x; int H, W, C; int npix;
  int r, kk; int img, oh, ow; bool rowok; float v[4];
  __device__ void init(int tid) { r = tid >> 1; kk = (tid & 1) * 4; }
  __device__ void set_row0(int row0) {
    int m = row0 + r;
    rowok = m < npix;
    int hw = H * W;
    img = m / hw; int rem = m - img * hw;
    oh = rem / W; ow = rem - oh * W;
  }
  __device__ void load(int, int k0, int kend) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int k = k0 + kk + j;
      int tap = k / C, c = k - tap * C;
      int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
      bool ok = rowok && k < kend && (unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W;
      v[j] = ok ? __ldg(x + ((long long)(img * H + ih) * W + iw) * C + c) : 0.f;
    }
  }
  __device__ void store(float* s) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) s[(kk + j) * 128 + r] = v[j];
  }
};

// wgrad B operand: rows n = tap*C + c (N = 9C), k = output pixel.
struct Im2colN {
  const float* x; int H, W, C; int npix;
  int r, kk; int tap, c, dy, dx; bool rowok; float4 v;
  __device__ void init(int tid) { kk = tid >> 5; r = (tid & 31) * 4; }
  __device__ void set_row0(int row0) {
    int n = row0 + r;
    rowok = n < 9 * C;
    tap = n / C; c = n - tap * C;
    dy = tap / 3 - 1; dx = tap % 3 - 1;
  }
  __device__ void load(int, int k0, int kend) {
    int p = k0 + kk;
    bool ok = rowok && p < kend;
    if (ok) {
      int hw = H * W;
      int img = p / hw; int rem = p - img * hw;
      int oh = rem / W, ow = rem - oh * W;
      int ih = oh + dy, iw = ow + dx;
      ok = (unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W;
      if (ok) {
        v = __ldg(reinterpret_cast<const float4*>(
            x + ((long long)(img * H + ih) * W + iw) * C + c));
        return;
      }
    }
    v = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __device__ void store(float* s) const {
    *reinterpret_cast<float4*>(s + kk * 128 + r) = v;
  }
};

// Scalar variant of Im2colN for C % 4 != 0 (conv1_1 wgrad).
struct Im2colNScalar {
  const float* x; int H, W, C; int npix;
  int r, kk; int n0; float v[4];
  __device__ void init(int tid) { kk = tid >> 5; r = (tid & 31) * 4; }
  __device__ void set_row0(int row0) { n0 = row0 + r; }
  __device__ void load(int, int k0, int kend) {
    int p = k0 + kk;
    int hw = H * W;
    int img = p / hw; int rem = p - img * hw;
    int oh = rem / W, ow = rem - oh * W;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + j;
      int tap = n / C, c = n - tap * C;
      int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
      bool ok = n < 9 * C && p < kend && (unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W;
      v[j] = ok ? __ldg(x + ((long long)(img * H + ih) * W + iw) * C + c) : 0.f;
    }
  }
  __device__ void store(float* s) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) s[kk * 128 + r + j] = v[j];
  }
};

// dgrad B operand: B(ci, k = tap'*Cout + co) = w[co][8 - tap'][ci] (flipped).
struct DgradW {
  const float* w; int Cin, Cout;
  int r, kk; float4 v;
  __device__ void init(int tid) { kk = tid >> 5; r = (tid & 31) * 4; }
  __device__ void load(int row0, int k0, int kend) {
    int ci = row0 + r, k = k0 + kk;
    if (ci < Cin && k < kend) {
      int tp = k / Cout, co = k - tp * Cout;
      v = __ldg(reinterpret_cast<const float4*>(
          w + ((long long)co * 9 + (8 - tp)) * Cin + ci));
    } else {
      v = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  __device__ void store(float* s) const {
    *reinterpret_cast<float4*>(s + kk * 128 + r) = v;
  }
};

template <class L> __device__ inline void set_row0_if(L& l, int row0) {}
__device__ inline void set_row0_if(Im2colK& l, int row0) { l.set_row0(row0); }
__device__ inline void set_row0_if(Im2colScalar& l, int row0) { l.set_row0(row0); }
__device__ inline void set_row0_if(Im2colN& l, int row0) { l.set_row0(row0); }
__device__ inline void set_row0_if(Im2colNScalar& l, int row0) { l.set_row0(row0); }

// ---------------------------------------------------------------- epilogues

// out[m*ldo + n] = relu?(acc + bias[n])  (conv fwd: m = pixel, n = cout)
struct EpiBiasAct {
  float* out; const float* bias; long long ldo; int relu;
  __device__ void operator()(int m, int n, float a) const {
    a += bias ? bias[n] : 0.f;
    out[m * ldo + n] = relu ? fmaxf(a, 0.f) : a;
  }
};
// out[n*ldo + m] = relu?(acc + bias[m])  (dense fwd computed as W . x^T)
struct EpiBiasActT {
  float* out; const float* bias; long long ldo; int relu;
  __device__ void operator()(int m, int n, float a) const {
    a += bias ? bias[m] : 0.f;
    out[n * ldo + m] = relu ? fmaxf(a, 0.f) : a;
  }
};
// out[m*ldo + n] = acc * (mask[m*ldo+n] > 0)
struct EpiMask {
  float* out; const float* mask; long long ldo;
  __device__ void operator()(int m, int n, float a) const {
    long long i = m * ldo + n;
    out[i] = (mask && !(mask[i] > 0.f)) ? 0.f : a;
  }
};
// transposed variant (dense dgrad computed as W^T . dy^T)
struct EpiMaskT {
  float* out; const float* mask; long long ldo;
  __device__ void operator()(int m, int n, float a) const {
    long long i = n * ldo + m;
    out[i] = (mask && !(mask[i] > 0.f)) ? 0.f : a;
  }
};
// split-K partial: ws[z][m][n]
struct EpiPartial {
  float* ws; long long ldo; long long slab;
  __device__ void operator()(int m, int n, float a) const {
    ws[blockIdx.z * slab + m * ldo + n] = a;
  }
};

// ---------------------------------------------------------------- kernel

template <int BN, class LA, class LB, class EPI>
__global__ void __launch_bounds__(NT)
sgemm_kernel(LA la, LB lb, EPI epi, int M, int N, int K, int kchunk) {
  constexpr int BM = 128;
  constexpr int TN = BN / 16;
  __shared__ __align__(16) float As[2][BK * BM];
  __shared__ __align__(16) float Bs[2][BK * BN];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * kchunk;
  const int kend = min(K, kbeg + kchunk);
  la.init(tid); lb.init(tid);
  set_row0_if(la, m0); set_row0_if(lb, n0);
  const int ty = tid >> 4, tx = tid & 15;
  float acc[8][TN];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  if (kbeg < kend) {
    la.load(m0, kbeg, kend); lb.load(n0, kbeg, kend);
    la.store(As[0]); lb.store(Bs[0]);
    __syncthreads();
    int buf = 0;
    for (int k0 = kbeg; k0 < kend; k0 += BK) {
      const bool more = k0 + BK < kend;
      if (more) { la.load(m0, k0 + BK, kend); lb.load(n0, k0 + BK, kend); }
      const float* as = As[buf];
      const float* bs = Bs[buf];
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float a[8], b[TN];
        float4 a0 = *reinterpret_cast<const float4*>(as + kk * BM + ty * 4);
        float4 a1 = *reinterpret_cast<const float4*>(as + kk * BM + 64 + ty * 4);
        a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
        a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
        if constexpr (TN == 8) {
          float4 b0 = *reinterpret_cast<const float4*>(bs + kk * BN + tx * 4);
          float4 b1 = *reinterpret_cast<const float4*>(bs + kk * BN + 64 + tx * 4);
          b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
          b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
        } else {
          float2 b0 = *reinterpret_cast<const float2*>(bs + kk * BN + tx * 2);
          b[0] = b0.x; b[1] = b0.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      if (more) { la.store(As[buf ^ 1]); lb.store(Bs[buf ^ 1]); }
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int n = n0 + (TN == 8 ? (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4)) : tx * 2 + j);
      if (n < N) epi(m, n, acc[i][j]);
    }
  }
}

// Split-K factor so that tiles * splits covers ~2 waves of the GPU while
// each split keeps >= min_k of reduction depth.
inline int pick_splits(long long tiles, long long K, int min_k) {
  long long want = (2LL * num_sms() + tiles - 1) / tiles;
  long long cap = K / (min_k > 0 ? min_k : 1);
  if (cap < 1) cap = 1;
  if (want > cap) want = cap;
  if (want > 256) want = 256;
  return (int)(want < 1 ? 1 : want);
}

// Launch; `splits` is rounded so every split gets whole BK blocks and is
// updated to the number of K slabs actually launched.
template <int BN, class LA, class LB, class EPI>
inline bpx_status_t run_gemm(LA la, LB lb, EPI epi, int M, int N, int K,
                             int& splits, cudaStream_t st) {
  int kchunk = (int)cdivll(cdivll(K, splits), BK) * BK;
  splits = (int)cdivll(K, kchunk);
  if (splits < 1) splits = 1;
  dim3 grid(cdiv(M, 128), cdiv(N, BN), splits);
  sgemm_kernel<BN><<<grid, NT, 0, st>>>(la, lb, epi, M, N, K, kchunk);
  return launch_status();
}

}  // namespace simt
}  // namespace bpx
