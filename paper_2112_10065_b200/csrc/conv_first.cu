// Forward of the first conv (Cin = 3, Cout = 64) on tcgen05: K = 27 taps x
// channels, padded to 32, is ONE MMA stage, so the layer is a stream of
// 128-pixel tiles bounded by writing y (411 MB at B = 32):
//
//   y[p][co] = relu(b[co] + sum_{r<27} col[p][r] * w[co][r])
//
// Persistent CTAs, two TMEM buffers (A hi|lo 64 columns + D 64 columns each)
// so tile t+1 is gathered and multiplied while tile t drains:
//   * gather warps (thread = pixel = TMEM lane) load the 27 im2col values
//     straight from x (19 MB, L2-resident), split them into TF32 hi/lo and
//     tcgen05.st them;
//   * one warp issues the 3xTF32 MMAs (B = the 64 x 32 weight tile, hi and
//     lo, built once per CTA in shared memory, K-major 128-B swizzle);
//   * drain warps add the bias, apply the ReLU and write the tile into a
//     double-buffered, 128-B-swizzled staging area; one thread stores it
//     with two TMA tensor stores (32 channels x 128 pixels each) -- the
//     128-pixel output tile is contiguous in y, and per-thread 256-byte row
//     stores reached only ~2.7 TB/s.
// One 32-K MMA chain per tile needs no chunk promotion.
#include "tma_host.h"
#include "tc_ptx.cuh"
#include "simt_api.h"

namespace bpx {
namespace c1 {
using namespace tcx;

constexpr int COUT = 64, R = 27, KP = 32;

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr int NTHREADS = 9 * 32;       // warp 0 MMA, 1-4 gather, 5-8 drain
// two CTAs per SM (82 KB smem, 256 TMEM columns each): twice the output
// tiles in flight per SM.  B200 A/B against one: 0.120 -> 0.089 ms at B=32,
// 0.038 -> 0.030 ms at B=8.
#ifndef C1_CPS
#define C1_CPS 2
#endif
constexpr int CPS = C1_CPS;            // CTAs per SM
constexpr int STAGE_OUT = 128 * COUT * 4;      // one output tile (two 16 KB boxes)
constexpr int SMEM = 1024 + 2 * COUT * KP * 4 + 2 * STAGE_OUT + 128;

__global__ void __launch_bounds__(NTHREADS, CPS)
c1_fwd_kernel(const float* __restrict__ x, const float* __restrict__ w,
              const float* __restrict__ bias, const __grid_constant__ CUtensorMap ty, int H,
              int W, long long npix, int relu, uint32_t* __restrict__ x_amax,
              uint32_t* __restrict__ amax) {
  extern __shared__ char smem_raw[];
  // offset from smem_raw (not a uintptr_t round trip) keeps the shared address space: LDS/STS, not generic LD/ST
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  char* bh = smem;                        // 64 rows x 128 B, 128-B swizzle
  char* bl = smem + COUT * KP * 4;
  char* ostage = bl + COUT * KP * 4;      // 2 x (2 boxes of 128 pixels x 128 B), swizzled
  uint64_t* aready = reinterpret_cast<uint64_t*>(ostage + 2 * STAGE_OUT);
  uint64_t* dfull = aready + 2;
  uint64_t* tfree = dfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfree + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long tiles = (npix + 127) / 128;

  // weights, K-major with the 128-B swizzle: row co, 16-B granule j at j ^ (co & 7)
  for (int e = tid; e < COUT * KP; e += NTHREADS) {
    const int co = e / KP, k = e % KP;
    const float v = k < R ? __ldg(w + co * R + k) : 0.f;
    float h, l;
    split(v, h, l);
    const int off = co * 128 + (((k >> 2) ^ (co & 7)) << 4) + (k & 3) * 4;
    *reinterpret_cast<float*>(bh + off) = v;
    *reinterpret_cast<float*>(bl + off) = l;
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&aready[b], 4);
      mbar_init(&dfull[b], 1);
      mbar_init(&tfree[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;       // buffer b: A at 128*b, D at 128*b + 64

  if (warp == 0) {
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                               ((uint32_t)(COUT >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t dbh0 = make_desc_sw128(smem_u32(bh), 16, 1024);
    const uint64_t dbl0 = make_desc_sw128(smem_u32(bl), 16, 1024);
    int it = 0;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      mbar_wait(&aready[b], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t ah = tmem + 128 * b, al = ah + KP, d = ah + 64;
#pragma unroll
      for (int ks = 0; ks < KP / 8; ++ks) {
        const uint64_t dbh = dbh0 + ks * 2, dbl = dbl0 + ks * 2;     // +32 B
        mma_ts_elect(d, al + 8 * ks, dbh, idesc, ks > 0 ? 1u : 0u);
        mma_ts_elect(d, ah + 8 * ks, dbl, idesc, 1u);
        mma_ts_elect(d, ah + 8 * ks, dbh, idesc, 1u);
      }
      tc_commit_elect(&dfull[b]);
    }
  } else if (warp < 5) {
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16);
    const int hw = H * W;
    uint32_t xm = 0;                      // max |x| bits: each pixel is one tile row's centre
    int it = 0;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      const long long p = t * 128 + r;
      float v[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) v[k] = 0.f;
      if (p < npix) {
        const int img = (int)(p / hw), rem = (int)(p - (long long)img * hw);
        const int oh = rem / W, ow = rem - oh * W;
        const float* xi = x + (long long)img * hw * 3;
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
          if ((unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W) {
            const float* s = xi + ((long long)ih * W + iw) * 3;
            v[3 * tap] = __ldg(s);
            v[3 * tap + 1] = __ldg(s + 1);
            v[3 * tap + 2] = __ldg(s + 2);
          }
        }
      }
      xm = max(xm, max(__float_as_uint(v[12]) & 0x7fffffffu,
                       max(__float_as_uint(v[13]) & 0x7fffffffu, __float_as_uint(v[14]) & 0x7fffffffu)));
      float hi[KP], lo[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) split(v[k], hi[k], lo[k]);
      if (it >= 2) mbar_wait(&tfree[b], ((it >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t a = lanebase + 128 * b;
      tmem_st16(a, *reinterpret_cast<float(*)[16]>(hi));
      tmem_st16(a + 16, *reinterpret_cast<float(*)[16]>(hi + 16));
      tmem_st16(a + KP, *reinterpret_cast<float(*)[16]>(lo));
      tmem_st16(a + KP + 16, *reinterpret_cast<float(*)[16]>(lo + 16));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&aready[b]);
    }
    if (x_amax) {
      xm = __reduce_max_sync(0xffffffffu, xm);
      if (lane == 0 && xm) atomicMax(x_amax, xm);
    }
  } else {
    const int q = warp & 3, r = q * 32 + lane;
    const int dtid = (warp - 5) * 32 + lane;          // 0..127 within the drain warps
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16);
    float bv[COUT];
#pragma unroll
    for (int j = 0; j < COUT; ++j) bv[j] = bias ? __ldg(bias + j) : 0.f;
    if (dtid == 0) tma_prefetch_desc(&ty);
    uint32_t mx = 0;                      // max |y| bits of this thread's valid rows
    int it = 0;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      char* st = ostage + b * STAGE_OUT;
      if (it >= 2) {            // the store issued from this staging buffer 2 tiles ago
        if (dtid == 0) bulk_wait_read<1>();
        named_bar(1, 128);
      }
      mbar_wait(&dfull[b], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < COUT; j += 8) {
        uint32_t rr[8];
        tmem_ld8(lanebase + 128 * b + 64 + j, rr);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float o[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float s = __uint_as_float(rr[u]) + bv[j + u];
          o[u] = relu ? fmaxf(s, 0.f) : s;
          if (t * 128 + r < npix) mx = max(mx, __float_as_uint(o[u]) & 0x7fffffffu);
        }
        // box j/32, row r, 16-B granule (j%32)/4 (+1), 128-B swizzle
        char* row = st + (j >> 5) * (STAGE_OUT / 2) + r * 128;
        const int g0 = (j & 31) >> 2;
        *reinterpret_cast<float4*>(row + ((g0 ^ (r & 7)) << 4)) =
            make_float4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<float4*>(row + (((g0 + 1) ^ (r & 7)) << 4)) =
            make_float4(o[4], o[5], o[6], o[7]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tfree[b]);
      fence_proxy_async();
      named_bar(1, 128);
      if (dtid == 0) {
        tma_store_2d(&ty, 0, (int)(t * 128), st);
        tma_store_2d(&ty, 32, (int)(t * 128), st + STAGE_OUT / 2);
        bulk_commit();
      }
    }
    if (dtid == 0) bulk_wait_all();
    if (amax) {
      mx = __reduce_max_sync(0xffffffffu, mx);
      if (lane == 0 && mx) atomicMax(amax, mx);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free(tmem, 256);
  }
}

}  // namespace c1

bool c1_conv_fwd_ok(int cin, int cout) { return cin == 3 && cout == c1::COUT; }

bpx_status_t c1_conv_fwd(const float* x, const float* w, const float* bias, float* y, int n,
                         int h, int w_, int relu, uint32_t* x_amax, uint32_t* y_amax,
                         cudaStream_t st) {
  const long long npix = (long long)n * h * w_;
  if (npix == 0) return launch_status(0);
  if (!aligned16(y) || npix > 0x7fffffffLL) return BPX_ERR_UNSUPPORTED;
  CUtensorMap ty;                  // y as [pixels][64]: box 32 channels x 128 pixels
  {
    const cuuint64_t dims[2] = {(cuuint64_t)c1::COUT, (cuuint64_t)npix};
    const cuuint64_t strides[1] = {(cuuint64_t)c1::COUT * 4};
    const cuuint32_t box[2] = {32, 128};
    const cuuint32_t es[2] = {1, 1};
    if (encode_tiled(&ty, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return BPX_ERR_UNSUPPORTED;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(c1::c1_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         c1::SMEM);
    attr = true;
  }
  const long long tiles = (npix + 127) / 128;
  const int grid = (int)(tiles < c1::CPS * num_sms() ? tiles : c1::CPS * num_sms());
  c1::c1_fwd_kernel<<<grid, c1::NTHREADS, c1::SMEM, st>>>(x, w, bias, ty, h, w_, npix, relu,
                                                               x_amax, y_amax);
  return launch_status();
}

}  // namespace bpx
