// 3x3 / pad-1 conv and dense layers on the FFMA implicit-GEMM engine
// (simt_gemm.cuh).  These back the C-ABI for shapes the tcgen05 engine does
// not take (Cin % 8 != 0, i.e. conv1_1) and are exported under
// bpx_simt_* for on-device cross-checks.
#include "simt_gemm.cuh"
#include "simt_api.h"

namespace bpx {
using namespace simt;

static int wgrad_splits(int M, int N, long long K) {
  long long tiles = (long long)cdiv(M, 128) * cdiv(N, 128);
  return pick_splits(tiles, K, 2048);
}

size_t simt_conv_wgrad_ws(int n, int h, int w, int cin, int cout) {
  long long npix = (long long)n * h * w;
  int splits = wgrad_splits(cout, 9 * cin, npix);
  return ((size_t)splits * cout * 9 * cin + colsum_workspace_floats(npix, cout)) *
         sizeof(float);
}

bpx_status_t simt_conv_fwd(const float* x, const float* w, const float* bias, float* y,
                           int n, int h, int w_, int cin, int cout, int relu,
                           cudaStream_t st) {
  int npix = n * h * w_;
  if (npix == 0) return BPX_OK;
  EpiBiasAct epi{y, bias, cout, relu};
  KMajor<128> lb{w, 9LL * cin, cout};
  int splits = 1;
  if (cin % 8 == 0) {
    Im2colK la{x, h, w_, cin, npix};
    return run_gemm<128>(la, lb, epi, npix, cout, 9 * cin, splits, st);
  }
  // tiny Cin (conv1_1: K = 27): scalar gathers on both operands
  Im2colScalar la{x, h, w_, cin, npix};
  KMajorScalar lbs{w, 9LL * cin, cout};
  return run_gemm<128>(la, lbs, epi, npix, cout, 9 * cin, splits, st);
}

bpx_status_t simt_conv_dgrad(const float* dz, const float* w, const float* mask,
                             float* dx, int n, int h, int w_, int cin, int cout,
                             cudaStream_t st) {
  int npix = n * h * w_;
  if (npix == 0) return BPX_OK;
  if (cout % 8 != 0 || cin % 4 != 0) return BPX_ERR_UNSUPPORTED;
  Im2colK la{dz, h, w_, cout, npix};
  DgradW lb{w, cin, cout};
  EpiMask epi{dx, mask, cin};
  int splits = 1;
  return run_gemm<128>(la, lb, epi, npix, cin, 9 * cout, splits, st);
}

bpx_status_t simt_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias,
                             int n, int h, int w_, int cin, int cout, void* ws,
                             size_t ws_bytes, cudaStream_t st) {
  long long npix = (long long)n * h * w_;
  int M = cout, N = 9 * cin;
  if (ws_bytes < simt_conv_wgrad_ws(n, h, w_, cin, cout)) return BPX_ERR_WORKSPACE;
  if (cout % 4 != 0) return BPX_ERR_UNSUPPORTED;
  if (npix == 0) {
    cudaMemsetAsync(dw, 0, sizeof(float) * (size_t)M * N, st);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * cout, st);
    return launch_status();
  }
  int splits = wgrad_splits(M, N, npix);
  float* part = static_cast<float*>(ws);
  size_t slab = (size_t)M * N;
  MMajor<128> la{dz, cout, cout};
  EpiPartial epi{part, N, (long long)slab};
  bpx_status_t s;
  if (cin % 4 == 0) {
    Im2colN lb{x, h, w_, cin, (int)npix};
    s = run_gemm<128>(la, lb, epi, M, N, (int)npix, splits, st);
  } else {
    Im2colNScalar lb{x, h, w_, cin, (int)npix};
    s = run_gemm<128>(la, lb, epi, M, N, (int)npix, splits, st);
  }
  if (s != BPX_OK) return s;
  s = split_reduce(part, splits, slab, dw, st);
  if (s != BPX_OK) return s;
  if (dbias) {
    float* cws = part + (size_t)wgrad_splits(M, N, npix) * slab;
    s = colsum(dz, npix, cout, dbias, cws, colsum_workspace_floats(npix, cout), st);
  }
  return s;
}

// ------------------------------------------------------------------ dense
// fwd:   Yt[o][b]  = sum_i W[o][i] x[b][i]       (M=out, N=b, K=in)
// dgrad: dXt[i][b] = sum_o W[o][i] dy[b][o]      (M=in,  N=b, K=out)
// wgrad: dW[o][i]  = sum_b dy[b][o] x[b][i]      (M=out, N=in, K=b)

static int dense_splits(int M, int N, int K) {
  long long tiles = (long long)cdiv(M, 128) * cdiv(N, N <= 32 ? 32 : 128);
  if (tiles <= 0) return 1;                   // empty shard: nothing to split
  return pick_splits(tiles, K, 512);
}

size_t simt_linear_fwd_ws(int b, int in, int out) {
  return (size_t)dense_splits(out, b, in) * out * b * sizeof(float);
}
size_t simt_linear_dgrad_ws(int b, int in, int out) {
  return (size_t)dense_splits(in, b, out) * in * b * sizeof(float);
}
size_t simt_linear_wgrad_ws(int b, int in, int out) {
  return colsum_workspace_floats(b, out) * sizeof(float);
}

// finish a split-K dense result: out[n][m] (+bias[m], relu / mask)
__global__ void dense_finish(const float* __restrict__ part, int splits, int M, int N,
                             const float* __restrict__ bias, const float* __restrict__ mask,
                             int relu, float* __restrict__ out) {
  long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int n = (int)(i / M), m = (int)(i - (long long)n * M);
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += part[(long long)k * total + (long long)m * N + n];
    if (bias) s += bias[m];
    if (relu) s = fmaxf(s, 0.f);
    if (mask && !(mask[i] > 0.f)) s = 0.f;
    out[i] = s;
  }
}

template <class LA, class LB>
static bpx_status_t dense_splitk(LA la, LB lb, int M, int N, int K, const float* bias,
                                 const float* mask, int relu, float* out, void* ws,
                                 size_t ws_bytes, cudaStream_t st) {
  int splits = dense_splits(M, N, K);
  if (ws_bytes < (size_t)splits * M * N * sizeof(float)) return BPX_ERR_WORKSPACE;
  float* part = static_cast<float*>(ws);
  EpiPartial epi{part, N, (long long)M * N};
  bpx_status_t s = (N <= 32) ? run_gemm<32>(la, lb, epi, M, N, K, splits, st)
                             : run_gemm<128>(la, lb, epi, M, N, K, splits, st);
  if (s != BPX_OK) return s;
  long long total = (long long)M * N;
  int grid = (int)std::min<long long>(cdivll(total, 256), 4LL * num_sms());
  dense_finish<<<grid, 256, 0, st>>>(part, splits, M, N, bias, mask, relu, out);
  return launch_status();
}

bpx_status_t simt_linear_fwd(const float* x, const float* w, const float* bias, float* y,
                             int b, int in, int out, int relu, void* ws, size_t ws_bytes,
                             cudaStream_t st) {
  if (b == 0) return BPX_OK;
  if (in % 4 != 0) return BPX_ERR_UNSUPPORTED;
  KMajor<128> la{w, in, out};
  if (b <= 32) {
    KMajor<32> lb{x, in, b};
    return dense_splitk(la, lb, out, b, in, bias, nullptr, relu, y, ws, ws_bytes, st);
  }
  KMajor<128> lb{x, in, b};
  return dense_splitk(la, lb, out, b, in, bias, nullptr, relu, y, ws, ws_bytes, st);
}

bpx_status_t simt_linear_dgrad(const float* dy, const float* w, const float* mask,
                               float* dx, int b, int in, int out, void* ws,
                               size_t ws_bytes, cudaStream_t st) {
  if (b == 0) return BPX_OK;
  if (in % 4 != 0) return BPX_ERR_UNSUPPORTED;
  MMajor<128> la{w, in, in};
  if (b <= 32) {
    KMajor<32> lb{dy, out, b};
    return dense_splitk(la, lb, in, b, out, nullptr, mask, 0, dx, ws, ws_bytes, st);
  }
  if (out % 4 != 0) return BPX_ERR_UNSUPPORTED;
  KMajor<128> lb{dy, out, b};
  return dense_splitk(la, lb, in, b, out, nullptr, mask, 0, dx, ws, ws_bytes, st);
}

bpx_status_t simt_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias,
                               int b, int in, int out, void* ws, size_t ws_bytes,
                               cudaStream_t st) {
  if (out % 4 != 0 || in % 4 != 0) return BPX_ERR_UNSUPPORTED;
  if (ws_bytes < simt_linear_wgrad_ws(b, in, out)) return BPX_ERR_WORKSPACE;
  if (b == 0) {
    cudaMemsetAsync(dw, 0, sizeof(float) * (size_t)out * in, st);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * out, st);
    return launch_status();
  }
  MMajor<128> la{dy, out, out};
  MMajor<128> lb{x, in, in};
  EpiBiasAct epi{dw, nullptr, in, 0};
  int splits = 1;
  bpx_status_t s = run_gemm<128>(la, lb, epi, out, in, b, splits, st);
  if (s != BPX_OK || !dbias) return s;
  return colsum(dy, b, out, dbias, static_cast<float*>(ws),
                colsum_workspace_floats(b, out), st);
}

}  // namespace bpx
