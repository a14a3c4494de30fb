// Dense layers (fc1/fc2/fc3) at per-GPU batches of 1..32: every weight is
// used by at most 32 samples, so the layer is a weight stream (fc1 fwd reads
// 411 MB of weights for 6.6 GFLOP) and fp32 FFMA at ~60 TF/s keeps up with
// HBM; tensor-core tiles would idle on a 32-wide N.  Three kernels:
//
//   fwd   y[n][o]  = act(b[o] + sum_k x[n][k]  W[o][k])     M = out,  K = in
//   dgrad dx[n][i] = mask(n,i) * sum_o dy[n][o] W[o][i]    M = in,   K = out
//   wgrad dW[o][i] = sum_n dy[n][o] x[n][i]                 (K = batch)
//
// fwd / dgrad (fwd_kernel, dgrad_kernel): a CTA owns 256 weight rows (M) x
// all samples and one K slice; W slices stream through a cp.async double
// buffer in their natural layout, and each thread accumulates a 4(m) x 8(n)
// register tile (12 LDS.128 per 128 FMAs).  Split-K partials are summed in a fixed order by the
// epilogue kernel, which also applies bias + ReLU (fwd) or the ReLU mask
// (dgrad): results are deterministic run to run.
// wgrad (outer_kernel / outer64_kernel): 64x256 tiles with 8x8 per thread
// for N <= 16 (dW-store bound), 64x64 tiles with 4x4 per thread above (FMA
// bound); the batch loop reads dy and x rows in their natural layouts.
#include "common.cuh"
#include "simt_api.h"

namespace bpx {
namespace dns {

constexpr int KC = 32;          // K per stage
constexpr int NT = 256;         // threads

// ---------------------------------------------------------------- fwd/dgrad
__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  const int n = ok ? 16 : 0;                  // zero-fill when out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

constexpr int BM = 256;                       // weight rows (M) per CTA
constexpr int WP = KC + 4;                    // padded [m][k] row (floats)
constexpr int XP = KC + 4;                    // padded [n][k] row
constexpr int FWD_STAGE = BM * WP + 32 * XP;  // floats
constexpr int DG_STAGE = KC * (BM + 4) + KC * (32 + 4);

// fwd: W[m][k], X[n][k] both natural (cp.async 16 B along k); thread tile
// rows m = tm + 64 i, samples n = tn + 4 j (conflict-free LDS.128 along k).
__global__ void __launch_bounds__(NT, 2)
fwd_kernel(const float* __restrict__ W, const float* __restrict__ X, int M, int N, int K,
           int kslice, float* __restrict__ part) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, tn = tid & 3, tm = tid >> 2;
  const int m0 = blockIdx.x * BM;
  const int k0 = blockIdx.y * kslice, k1 = min(K, k0 + kslice);
  const int nst = (k1 - k0 + KC - 1) / KC;
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  auto load = [&](int st, int buf) {
    float* ws = sm + buf * FWD_STAGE;
    float* xs = ws + BM * WP;
    const int kb = k0 + st * KC;
    for (int e = tid; e < BM * (KC / 4); e += NT) {
      const int r = e >> 3, c = (e & 7) * 4, m = m0 + r, k = kb + c;
      const bool ok = m < M && k < k1;
      cp16(ws + r * WP + c, ok ? W + (long long)m * K + k : W, ok);
    }
    for (int e = tid; e < 32 * (KC / 4); e += NT) {
      const int n = e >> 3, c = (e & 7) * 4, k = kb + c;
      const bool ok = n < N && k < k1;
      cp16(xs + n * XP + c, ok ? X + (long long)n * K + k : X, ok);
    }
    cp_commit();
  };
  load(0, 0);
  for (int st = 0; st < nst; ++st) {
    if (st + 1 < nst) load(st + 1, (st + 1) & 1); else cp_commit();
    cp_wait1();
    __syncthreads();
    const float* ws = sm + (st & 1) * FWD_STAGE;
    const float* xs = ws + BM * WP;
#pragma unroll 2
    for (int k4 = 0; k4 < KC; k4 += 4) {
      float4 a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const float4*>(ws + (tm + 64 * i) * WP + k4);
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = *reinterpret_cast<const float4*>(xs + (tn + 4 * j) * XP + k4);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[i][j] = fmaf(a[i].x, b[j].x, acc[i][j]);
          acc[i][j] = fmaf(a[i].y, b[j].y, acc[i][j]);
          acc[i][j] = fmaf(a[i].z, b[j].z, acc[i][j]);
          acc[i][j] = fmaf(a[i].w, b[j].w, acc[i][j]);
        }
    }
    __syncthreads();
  }
  float* out = part + (long long)blockIdx.y * N * M;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int n = tn + 4 * j;
    if (n >= N) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + tm + 64 * i;
      if (m < M) out[(long long)n * M + m] = acc[i][j];
    }
  }
}

// dgrad: W[k][m] natural (cp.async 16 B along m), X[n][k] -> [k][n] (small
// transpose); thread tile m = tm*4 .. +3 (LDS.128), samples n = tn*8 .. +7.
__global__ void __launch_bounds__(NT, 2)
dgrad_kernel(const float* __restrict__ W, const float* __restrict__ X, int M, int N, int K,
             int kslice, float* __restrict__ part) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, tn = tid & 3, tm = tid >> 2;
  const int m0 = blockIdx.x * BM;
  const int k0 = blockIdx.y * kslice, k1 = min(K, k0 + kslice);
  const int nst = (k1 - k0 + KC - 1) / KC;
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  auto load = [&](int st, int buf) {
    float* ws = sm + buf * DG_STAGE;
    float* xs = ws + KC * (BM + 4);
    const int kb = k0 + st * KC;
    for (int e = tid; e < KC * (BM / 4); e += NT) {
      const int kk = e / (BM / 4), c = (e % (BM / 4)) * 4, k = kb + kk, m = m0 + c;
      const bool ok = k < k1 && m < M;
      cp16(ws + kk * (BM + 4) + c, ok ? W + (long long)k * M + m : W, ok);
    }
    for (int e = tid; e < 32 * KC; e += NT) {
      const int n = e / KC, kk = e % KC, k = kb + kk;
      xs[kk * 36 + n] = (n < N && k < k1) ? __ldg(X + (long long)n * K + k) : 0.f;
    }
    cp_commit();
  };
  load(0, 0);
  for (int st = 0; st < nst; ++st) {
    if (st + 1 < nst) load(st + 1, (st + 1) & 1); else cp_commit();
    cp_wait1();
    __syncthreads();
    const float* ws = sm + (st & 1) * DG_STAGE;
    const float* xs = ws + KC * (BM + 4);
#pragma unroll 8
    for (int kk = 0; kk < KC; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(ws + kk * (BM + 4) + tm * 4);
      const float4 b0 = *reinterpret_cast<const float4*>(xs + kk * 36 + tn * 8);
      const float4 b1 = *reinterpret_cast<const float4*>(xs + kk * 36 + tn * 8 + 4);
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* out = part + (long long)blockIdx.y * N * M;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int n = tn * 8 + j;
    if (n >= N) continue;
    const int m = m0 + tm * 4;
    if (m + 3 < M) {
      *reinterpret_cast<float4*>(out + (long long)n * M + m) =
          make_float4(acc[0][j], acc[1][j], acc[2][j], acc[3][j]);
    } else {
      for (int i = 0; i < 4 && m + i < M; ++i) out[(long long)n * M + m + i] = acc[i][j];
    }
  }
}

// sum of the K-slice partials in fixed order + epilogue.
// mode 0: y = act(sum + bias); mode 1: dx = sum * (mask > 0) (mask may be null)
__global__ void skinny_finish(const float* __restrict__ part, int splits, long long NM,
                              int M, const float* __restrict__ bias, int relu,
                              const float* __restrict__ mask, int mode,
                              float* __restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < NM;
       e += (long long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += part[k * NM + e];
    if (mode == 0) {
      if (bias) s += __ldg(bias + (int)(e % M));
      if (relu) s = fmaxf(s, 0.f);
    } else if (mask && !(__ldg(mask + e) > 0.f)) {
      s = 0.f;
    }
    out[e] = s;
  }
}

// ---------------------------------------------------------------- wgrad
// dW[o][i] = sum_n dy[n][o] x[n][i] (N <= 32).  Small-batch variant (N <= 16,
// bound by writing dW: 411 MB for fc1): a CTA keeps one 64-row dy tile in
// shared memory and streams 256-column x tiles through a cp.async double
// buffer; 8x8 outputs per thread, so each warp stores 1 KB runs of a dW row.
// 2 CTAs per SM walk an even share of the flattened tile grid (B200 A/B at
// fc1: 0.08 ms vs 0.19 ms for 64x64 tiles at N = 1..4).
constexpr int WO = 64, WI = 256;
constexpr int WSMEM = (32 * WO + 2 * 32 * WI) * 4;
__global__ void __launch_bounds__(NT)
outer_kernel(const float* __restrict__ dy, const float* __restrict__ x, int N, int O, int I,
             float* __restrict__ dw) {
  extern __shared__ __align__(16) float wsm[];
  float* ds = wsm;                       // [32][WO]
  float* xs = wsm + 32 * WO;             // [2][32][WI]
  const int tid = threadIdx.x;
  const int ti = tid & 31, to = tid >> 5;       // 8 columns x 8 rows per thread
  // the (row tile, column tile) grid, flattened row-major, split evenly over
  // the CTAs; the dy tile is reloaded when a CTA crosses into the next row tile
  const int itiles = cdiv(I, WI);
  const long long total = (long long)itiles * cdiv(O, WO);
  const int f0 = (int)(total * blockIdx.x / gridDim.x);
  const int f1 = (int)(total * (blockIdx.x + 1) / gridDim.x);
  const int nn = min(N, 32);
  auto load_dy = [&](int o0) {
    for (int e = tid; e < 32 * (WO / 4); e += NT) {
      const int n = e / (WO / 4), c = (e % (WO / 4)) * 4, o = o0 + c;
      const bool ok = n < N && o < O;
      cp16(ds + n * WO + c, ok ? dy + (long long)n * O + o : dy, ok);
    }
  };
  auto load = [&](int f, int buf) {
    const int it = f % itiles;
    if (f == f0 || it == 0) load_dy((f / itiles) * WO);
    for (int e = tid; e < nn * (WI / 4); e += NT) {
      const int n = e / (WI / 4), c = (e % (WI / 4)) * 4, i = it * WI + c;
      const bool ok = i < I;
      cp16(xs + (buf * 32 + n) * WI + c, ok ? x + (long long)n * I + i : x, ok);
    }
    cp_commit();
  };
  if (f0 < f1) load(f0, 0);
  for (int f = f0; f < f1; ++f) {
    const int buf = (f - f0) & 1;
    const int it = f % itiles, o0 = (f / itiles) * WO;
    // the next tile's dy reload may only overwrite ds after this tile is done
    const bool next_dy = f + 1 < f1 && (f + 1) % itiles == 0;
    if (f + 1 < f1 && !next_dy) load(f + 1, buf ^ 1); else cp_commit();
    cp_wait1();
    __syncthreads();
    float acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
    for (int n = 0; n < nn; ++n) {
      const float4 d0 = *reinterpret_cast<const float4*>(ds + n * WO + to * 8);
      const float4 d1 = *reinterpret_cast<const float4*>(ds + n * WO + to * 8 + 4);
      const float4 v0 = *reinterpret_cast<const float4*>(xs + (buf * 32 + n) * WI + ti * 4);
      const float4 v1 = *reinterpret_cast<const float4*>(xs + (buf * 32 + n) * WI + 128 + ti * 4);
      const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
      const float xv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = fmaf(dv[a], xv[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int o = o0 + to * 8 + a;
      if (o >= O) continue;
      float* p = dw + (long long)o * I + it * WI;
      const int i = it * WI + ti * 4;
      if (i + 3 < I)
        *reinterpret_cast<float4*>(p + ti * 4) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
      if (i + 131 < I)
        *reinterpret_cast<float4*>(p + 128 + ti * 4) =
            make_float4(acc[a][4], acc[a][5], acc[a][6], acc[a][7]);
    }
    __syncthreads();
    if (next_dy) {          // row-tile crossing: dy and x of the next tile together
      load(f + 1, buf ^ 1);
      cp_wait0();
      __syncthreads();
    }
  }
}

// Large-batch variant (N > 16, where the FMAs, not the dW stores, bound the
// kernel): 64x64 tiles, 4x4 outputs per thread, the dy tile in shared memory
// and 64-column x tiles through a cp.async double buffer.
__global__ void __launch_bounds__(NT)
outer64_kernel(const float* __restrict__ dy, const float* __restrict__ x, int N, int O, int I,
             int tiles_per_cta, float* __restrict__ dw) {
  __shared__ __align__(16) float ds[32][64];
  __shared__ __align__(16) float xs[2][32][64];
  const int tid = threadIdx.x;
  const int o0 = blockIdx.y * 64;
  const int ti = tid % 16, to = tid / 16;
  const int it0 = blockIdx.x * tiles_per_cta;
  const int it1 = min(cdiv(I, 64), it0 + tiles_per_cta);
  for (int e = tid; e < 32 * 16; e += NT) {
    const int n = e / 16, c = (e % 16) * 4, o = o0 + c;
    const bool ok = n < N && o < O;
    cp16(&ds[n][c], ok ? dy + (long long)n * O + o : dy, ok);
  }
  auto load = [&](int it, int buf) {
    for (int e = tid; e < 32 * 16; e += NT) {
      const int n = e / 16, c = (e % 16) * 4, i = it * 64 + c;
      const bool ok = n < N && i < I;
      cp16(&xs[buf][n][c], ok ? x + (long long)n * I + i : x, ok);
    }
    cp_commit();
  };
  if (it0 < it1) load(it0, 0);
  for (int it = it0; it < it1; ++it) {
    const int buf = (it - it0) & 1;
    if (it + 1 < it1) load(it + 1, buf ^ 1); else cp_commit();
    cp_wait1();
    __syncthreads();
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
#pragma unroll 8
    for (int n = 0; n < 32; ++n) {
      const float4 d = *reinterpret_cast<const float4*>(&ds[n][to * 4]);
      const float4 v = *reinterpret_cast<const float4*>(&xs[buf][n][ti * 4]);
      const float dv[4] = {d.x, d.y, d.z, d.w};
      const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(dv[a], xv[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int o = o0 + to * 4 + a, i = it * 64 + ti * 4;
      if (o < O && i < I)
        *reinterpret_cast<float4*>(dw + (long long)o * I + i) =
            make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
    }
    __syncthreads();
  }
}

inline void geometry(int N, int M, int K, int& bm, int& splits, int& kslice) {
  (void)N;
  bm = BM;
  const int mt = cdiv(M, bm);
  int want = (2 * num_sms()) / mt;           // one wave at 2 CTAs per SM
  const int maxs = cdiv(K, KC);
  if (want > maxs) want = maxs;
  if (want < 1) want = 1;
  kslice = cdiv(cdiv(K, want), KC) * KC;
  splits = cdiv(K, kslice);
}

bpx_status_t skinny(const float* W, const float* X, int M, int N, int K, bool trans_w,
                    float* ws, size_t ws_bytes, const float* bias, int relu,
                    const float* mask, int mode, float* out, cudaStream_t st) {
  int bm, splits, kslice;
  geometry(N, M, K, bm, splits, kslice);
  if (ws_bytes < (size_t)splits * N * M * sizeof(float)) return BPX_ERR_WORKSPACE;
  dim3 grid(cdiv(M, bm), splits);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * FWD_STAGE * 4);
    cudaFuncSetAttribute(dgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * DG_STAGE * 4);
    attr = true;
  }
  if (trans_w)
    fwd_kernel<<<grid, NT, 2 * FWD_STAGE * 4, st>>>(W, X, M, N, K, kslice, ws);
  else
    dgrad_kernel<<<grid, NT, 2 * DG_STAGE * 4, st>>>(W, X, M, N, K, kslice, ws);
  const long long NM = (long long)N * M;
  int g = (int)cdivll(NM, 256);
  if (g > 8 * num_sms()) g = 8 * num_sms();
  skinny_finish<<<g, 256, 0, st>>>(ws, splits, NM, M, bias, relu, mask, mode, out);
  return launch_status(2);
}

}  // namespace dns

bool dns_linear_ok(int b, int in, int out) { return b >= 1 && b <= 32 && in % 4 == 0 && out % 4 == 0; }

size_t dns_linear_ws(int b, int in, int out) {
  if (!dns_linear_ok(b, in, out)) return 0;
  int bm, s1, ks, s2;
  dns::geometry(b, out, in, bm, s1, ks);      // fwd: M = out, K = in
  dns::geometry(b, in, out, bm, s2, ks);      // dgrad: M = in, K = out
  const size_t a = (size_t)s1 * b * out, c = (size_t)s2 * b * in;
  const size_t cs = colsum_workspace_floats(b, out);
  size_t m = a > c ? a : c;
  return (m > cs ? m : cs) * sizeof(float);
}

bpx_status_t dns_linear_fwd(const float* x, const float* w, const float* bias, float* y, int b,
                            int in, int out, int relu, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  if (b == 0) return launch_status(0);
  return dns::skinny(w, x, out, b, in, true, static_cast<float*>(ws), ws_bytes, bias, relu,
                     nullptr, 0, y, st);
}

bpx_status_t dns_linear_dgrad(const float* dy, const float* w, const float* mask, float* dx,
                              int b, int in, int out, void* ws, size_t ws_bytes,
                              cudaStream_t st) {
  if (b == 0) return launch_status(0);
  return dns::skinny(w, dy, in, b, out, false, static_cast<float*>(ws), ws_bytes, nullptr, 0,
                     mask, 1, dx, st);
}

bpx_status_t dns_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias, int b,
                              int in, int out, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (b == 0) {
    cudaMemsetAsync(dw, 0, sizeof(float) * (size_t)in * out, st);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * out, st);
    return launch_status(0);
  }
  if (b > 16) {
    const int itiles = cdiv(in, 64), otiles = cdiv(out, 64);
    int per = cdiv(itiles * otiles, 8 * num_sms());      // ~8 CTAs per SM in total
    if (per < 1) per = 1;
    dim3 grid(cdiv(itiles, per), otiles);
    dns::outer64_kernel<<<grid, dns::NT, 0, st>>>(dy, x, b, out, in, per, dw);
  } else {
    const int tiles = cdiv(in, dns::WI) * cdiv(out, dns::WO);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(dns::outer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           dns::WSMEM);
      attr = true;
    }
    const int grid = tiles < 2 * num_sms() ? tiles : 2 * num_sms();   // 2 CTAs per SM
    dns::outer_kernel<<<grid, dns::NT, dns::WSMEM, st>>>(dy, x, b, out, in, dw);
  }
  bpx_status_t s = launch_status();
  if (s != BPX_OK || !dbias) return s;
  return colsum(dy, b, out, dbias, static_cast<float*>(ws),
                ws_bytes / sizeof(float), st);
}

}  // namespace bpx
