// tcgen05 weight-gradient engine for the 3x3/pad-1 convolutions:
//
//   dW[co][tap*Cin + ci] = sum_pixels dz[p][co] * x[p + tap][ci]
//   M = Cout, N = 9*Cin, K = pixels (split-K over CTAs, fixed-order reduce)
//
//   * A = dz^T goes registers -> TMEM: one thread per output channel row
//     loads 16 consecutive pixels (coalesced across the warp's 32 channels),
//     splits into TF32 hi/lo and tcgen05.st's them; the MMA reads A from TMEM.
//   * B = im2col(x) is produced into shared memory in the UMMA K-major
//     no-swizzle layout with 4x4 register transposes (4 channels x 4
//     pixels per thread).  (Fallback engine: tc_wgt.cu reads MN-major tiles
//     directly -- kind::tf32 takes MN-major operands only in the
//     SWIZZLE_128B_BASE32B layout, see tools/probes/probe_mn.cu.)
//   * hi*hi + hi*lo + lo*hi accumulate in 64-K chunks in ping-pong TMEM
//     buffers, promoted to RN fp32 registers by drain warps (see tc_engine.cu
//     for why: the tensor core's fp32 accumulate truncates).
//
// CTA (672 threads): warps 0-7 A producers (two groups alternating k-blocks),
// warps 8-11 B producers, warps 12-19 drain/epilogue, warp 20 MMA + TMEM.
#include "tc_ptx.cuh"
#include "tc_api.h"

namespace bpx {
namespace wg {
using namespace tcx;

constexpr int BK = 16;
constexpr int P = 4;
constexpr int S = 6;
constexpr int NB = 128;                   // B producer threads
constexpr int ND = 256;                   // drain threads
constexpr int MMA_WARP = 20;
constexpr int NTHREADS = 21 * 32;
// B tile: K-major, no swizzle; 8-row groups padded to 144 B (SBO) so the
// transposed chunk stores of a quarter-warp are bank-conflict free.
constexpr int SBO = 144;

template <int BN>
struct Cfg {
  static_assert(BN == 64 || BN == 128, "BN");
  static constexpr int NG = BN / 4;                  // n-groups (4 channels each)
  static constexpr int LBO = (BN / 8) * SBO;         // k-chunk (4 pixels) stride
  static constexpr int HALF = 4 * LBO;               // 16 pixels, hi or lo
  static constexpr int STAGE = 2 * HALF;
  static constexpr int SMEM = S * STAGE + 1024;
  static constexpr int A_COL = 2 * BN;
  static constexpr int TMEM_COLS = 512;
  static constexpr int CW = BN / 2;
  static_assert(NG * (BK / 4) <= NB, "one B unit per producer thread");
  static_assert(A_COL + S * 2 * BK <= TMEM_COLS, "TMEM budget");
};

template <int BN>
__global__ void __launch_bounds__(NTHREADS, 1)
wgrad_kernel(const float* __restrict__ x, const float* __restrict__ dz, int H, int W,
             int Cin, int Cout, int npix, int kchunk, float* __restrict__ part,
             long long slab) {
  using Cf = Cfg<BN>;
  extern __shared__ __align__(1024) char smem[];
  char* bst = smem;
  uint64_t* afull = reinterpret_cast<uint64_t*>(smem + S * Cf::STAGE);
  uint64_t* bfull = afull + S;
  uint64_t* empty = bfull + S;
  uint64_t* hfull = empty + S;
  uint64_t* hfree = hfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int N = 9 * Cin;
  const int kbeg = blockIdx.z * kchunk;
  const int kend = min(npix, kbeg + kchunk);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  const int nc = (nk + P - 1) / P;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&afull[s], 128);
      mbar_init(&bfull[s], NB);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hfree[b], ND);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) tmem_alloc(tmem_slot, Cf::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // -------------------------------------------- A = dz^T rows -> TMEM
    const int q = warp & 3, grp = warp >> 2;
    const int co = m0 + q * 32 + lane;
    const bool rowok = co < Cout;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + Cf::A_COL;
    auto load = [&](int kb, float (&v)[16]) {
      const int p0 = kbeg + kb * BK;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int p = p0 + j;
        v[j] = (rowok && p < kend) ? __ldg(dz + (long long)p * Cout + co) : 0.f;
      }
    };
    float cur[16], nxt[16];
    int kb = grp;
    if (kb < nk) load(kb, cur);
    for (; kb < nk; kb += 2) {
      if (kb + 2 < nk) load(kb + 2, nxt);
      const int s = kb % S;
      if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
      tc_fence_after();
      float hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split(cur[j], hi[j], lo[j]);
      const uint32_t a = lanebase + s * 2 * BK;
      tmem_st16(a, hi);
      tmem_st16(a + BK, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&afull[s]);
#pragma unroll
      for (int j = 0; j < 16; ++j) cur[j] = nxt[j];
    }
  } else if (warp < 12) {
    // -------------------------------------------- B = im2col(x) -> smem (K-major)
    // unit = 4 channels (n-group) x 4 consecutive pixels: four float4 loads
    // (one per pixel, coalesced across the warp's n-groups), a 4x4 register
    // transpose, four 16-byte chunk stores per hi/lo tile.
    const int bt = tid - 256;
    const int ng = bt % Cf::NG;
    const int kq = bt / Cf::NG;               // pixel quad within the stage
    const bool active = kq < BK / 4;
    const int n = n0 + 4 * ng;
    const bool nok = active && n < N;
    const int tap = nok ? n / Cin : 0, ci = nok ? n - tap * Cin : 0;
    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
    const int hw = H * W;
    auto load = [&](int kb, float4 (&v)[4]) {
      int p = kbeg + kb * BK + 4 * kq;
      int img = p / hw, rem = p - img * hw;
      int oh = rem / W, ow = rem - oh * W;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j) {
          ++p;
          if (++ow == W) { ow = 0; if (++oh == H) { oh = 0; ++img; } }
        }
        const int ih = oh + dy, iw = ow + dx;
        if (nok && p < kend && (unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W)
          v[j] = __ldg(reinterpret_cast<const float4*>(
              x + (((long long)img * H + ih) * W + iw) * Cin + ci));
        else
          v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    float4 cur[4], nxt[4];
    if (nk > 0 && active) load(0, cur);
    for (int kb = 0; kb < nk; ++kb) {
      if (active && kb + 1 < nk) load(kb + 1, nxt);
      const int s = kb % S;
      if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
      if (active) {
        char* hi = bst + s * Cf::STAGE;
        char* lo = hi + Cf::HALF;
        const float4 rows[4] = {make_float4(cur[0].x, cur[1].x, cur[2].x, cur[3].x),
                                make_float4(cur[0].y, cur[1].y, cur[2].y, cur[3].y),
                                make_float4(cur[0].z, cur[1].z, cur[2].z, cur[3].z),
                                make_float4(cur[0].w, cur[1].w, cur[2].w, cur[3].w)};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int row = 4 * ng + r;
          const int off = kq * Cf::LBO + (row >> 3) * SBO + (row & 7) * 16;
          float4 h, l;
          split(rows[r].x, h.x, l.x); split(rows[r].y, h.y, l.y);
          split(rows[r].z, h.z, l.z); split(rows[r].w, h.w, l.w);
          *reinterpret_cast<float4*>(hi + off) = h;
          *reinterpret_cast<float4*>(lo + off) = l;
        }
      }
      fence_proxy_async();
      mbar_arrive(&bfull[s]);
#pragma unroll
      for (int j = 0; j < 4; ++j) cur[j] = nxt[j];
    }
  } else if (warp < MMA_WARP) {
    // -------------------------------------------- drain + epilogue
    const int q = warp & 3;
    const int half = (warp - 12) >> 2;
    const int m = m0 + q * 32 + lane;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16);
    const int cbase = half * Cf::CW;
    float acc[Cf::CW];
#pragma unroll
    for (int j = 0; j < Cf::CW; ++j) acc[j] = 0.f;
    for (int c = 0; c < nc; ++c) {
      const int b = c & 1;
      mbar_wait(&hfull[b], (c >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < Cf::CW; j += 8) {
        uint32_t r[8];
        tmem_ld8(lanebase + b * BN + cbase + j, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[j + t] += __uint_as_float(r[t]);
      }
      tc_fence_before();
      mbar_arrive(&hfree[b]);
    }
    if (m < Cout) {
      float* o = part + blockIdx.z * slab + (long long)m * N;
#pragma unroll
      for (int j = 0; j < Cf::CW; j += 4) {
        const int n = n0 + cbase + j;
        if (n + 4 <= N)
          *reinterpret_cast<float4*>(o + n) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        else
          for (int t = 0; t < 4 && n + t < N; ++t) o[n + t] = acc[j + t];
      }
    }
  } else if (warp == MMA_WARP && lane == 0) {
    // -------------------------------------------- MMA issuer
    constexpr uint32_t idesc = make_idesc(BN);
    for (int c = 0; c < nc; ++c) {
      const int b = c & 1;
      const uint32_t d = tmem + b * BN;
      if (c >= 2) {
        mbar_wait(&hfree[b], ((c >> 1) - 1) & 1);
        tc_fence_after();
      }
      const int kb1 = min(nk, (c + 1) * P);
      for (int kb = c * P; kb < kb1; ++kb) {
        const int s = kb % S;
        const uint32_t ph = (kb / S) & 1;
        mbar_wait(&afull[s], ph);
        mbar_wait(&bfull[s], ph);
        tc_fence_after();
        const uint32_t bh = smem_u32(bst + s * Cf::STAGE);
        const uint32_t bl = bh + Cf::HALF;
        const uint32_t ah = tmem + Cf::A_COL + s * 2 * BK;
        const uint32_t al = ah + BK;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint64_t dbh = make_desc(bh + ks * 2 * Cf::LBO, Cf::LBO, SBO);
          const uint64_t dbl = make_desc(bl + ks * 2 * Cf::LBO, Cf::LBO, SBO);
          const uint32_t first = (kb > c * P || ks > 0) ? 1u : 0u;
          mma_ts(d, al + 8 * ks, dbh, idesc, first);
          mma_ts(d, ah + 8 * ks, dbl, idesc, 1u);
          mma_ts(d, ah + 8 * ks, dbh, idesc, 1u);
        }
        tc_commit(&empty[s]);
      }
      tc_commit(&hfull[b]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_free(tmem, Cf::TMEM_COLS);
  }
}

inline int bn_for(int N) { return (N % 128 == 0) ? 128 : 64; }

inline int splits_for(int Cout, int N, long long npix) {
  const int bn = bn_for(N);
  long long tiles = (long long)cdiv(Cout, BM) * cdiv(N, bn);
  long long want = (num_sms() + tiles - 1) / tiles;
  long long cap = npix / 256;
  if (cap < 1) cap = 1;
  if (want > cap) want = cap;
  if (want > 128) want = 128;
  return (int)(want < 1 ? 1 : want);
}

template <int BN>
bpx_status_t launch(const float* x, const float* dz, int n, int H, int W, int Cin, int Cout,
                    float* part, int splits, long long slab, int kchunk, cudaStream_t st) {
  using Cf = Cfg<BN>;
  auto kern = wgrad_kernel<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    attr = true;
  }
  dim3 grid(cdiv(Cout, BM), cdiv(9 * Cin, BN), splits);
  kern<<<grid, NTHREADS, Cf::SMEM, st>>>(x, dz, H, W, Cin, Cout, n * H * W, kchunk, part, slab);
  return launch_status();
}

}  // namespace wg

// ============================================================ entry points

bool wg_conv_ok(int cin, int cout) { return cin % 4 == 0 && cout % 4 == 0; }

size_t wg_conv_ws(int n, int h, int w, int cin, int cout) {
  long long npix = (long long)n * h * w;
  const int N = 9 * cin;
  return ((size_t)wg::splits_for(cout, N, npix) * cout * N +
          colsum_workspace_floats(npix, cout)) * sizeof(float);
}

bpx_status_t wg_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias, int n,
                           int h, int w_, int cin, int cout, void* ws, size_t ws_bytes,
                           cudaStream_t st) {
  const long long npix = (long long)n * h * w_;
  const int N = 9 * cin;
  if (ws_bytes < wg_conv_ws(n, h, w_, cin, cout)) return BPX_ERR_WORKSPACE;
  if (npix == 0) {
    cudaMemsetAsync(dw, 0, sizeof(float) * (size_t)cout * N, st);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * cout, st);
    return launch_status(0);
  }
  int splits = wg::splits_for(cout, N, npix);
  int kchunk = (int)(cdivll(cdivll(npix, splits), wg::BK) * wg::BK);
  splits = (int)cdivll(npix, kchunk);
  const long long slab = (long long)cout * N;
  float* part = splits == 1 ? dw : static_cast<float*>(ws);
  bpx_status_t s = wg::bn_for(N) == 128
      ? wg::launch<128>(x, dz, n, h, w_, cin, cout, part, splits, slab, kchunk, st)
      : wg::launch<64>(x, dz, n, h, w_, cin, cout, part, splits, slab, kchunk, st);
  if (s == BPX_OK && splits > 1) s = split_reduce(part, splits, (size_t)slab, dw, st);
  if (s != BPX_OK || !dbias) return s;
  float* cws = static_cast<float*>(ws) +
               (size_t)wg::splits_for(cout, N, npix) * (size_t)slab;
  return colsum(dz, npix, cout, dbias, cws, colsum_workspace_floats(npix, cout), st);
}

}  // namespace bpx
