// fp16x3 weight gradient of the first convolution (Cin = 3, Cout = 64:
// VGG's conv1_1), an HBM-bound op: 411 MB of dz against 5.5 GFLOP.
//
//   dW^T[r][co] = sum_p im2col(x)[p][r] * dz[p][co],  r = tap*3 + ci < 27
//
// Walks 16 x 4 pixel blocks (K = 64 per block).  Per block TMA brings the
// dz block (two 32-channel 4-D boxes, 16 KB, split in place into an fp16
// MN-major atom by the B converters, which also sum the bias gradient) and
// the 18 x 6 x 3 x-halo as one box of x viewed [n][H][W*3] (its out-of-
// bounds elements are the conv's zero padding).  The 27 im2col rows live in
// EVERY TMEM lane quadrant: quadrant q's converter warp builds them for the
// block's pixel row q only (16 pixels = 8 columns of hi and of lo; the other
// columns of its lanes stay zero), so four warps gather in parallel and the
// drain sums the four quadrants' partial rows at the end.  One M = 128 (27
// live rows) x N = 64 kind::f16 MMA triple per 16-pixel k-step; 128-pixel
// promotion chunks as in the other engines.  Each CTA owns a contiguous
// block range and a partial slab; split_reduce sums the slabs in order.
//
// CTA: 14 warps.  warp 0 TMA, warp 1 MMA + TMEM owner, 2-5 A converters
// (one per lane quadrant), 6-9 B converters, 10-13 drain.
#include <cstdio>
#include "tma_host.h"
#include "tc_ptx.cuh"
#include "tc_api.h"

namespace bpx {
namespace wg1 {
using namespace tcx;

constexpr int TMA_WARP = 0, MMA_WARP = 1, CA0 = 2, CB0 = 6, DR0 = 10, NT = 14 * 32;
constexpr int CI = 3, R = 27, CO = 64;
constexpr int BW = 16, BH = 4, BKP = BW * BH;
// the halo row starts one float before pixel px0 - 1 (TMA wants the start of
// the innermost dimension 16-B aligned): floats [3 px0 - 4, +60)
constexpr int XW = 60;                        // halo row: (16 + 2) * 3 = 54 floats, box 56
constexpr int XB = BH + 2;                       // halo rows
constexpr int XBYTES = XB * XW * 4;              // 1344 B
constexpr int DZB = BKP * 128;                   // one 32-channel dz box
constexpr int STAGE = 2 * DZB + 2048;            // dz boxes | x halo
constexpr int S = 6, SA = 4;
constexpr int ACC = 2 * CO;                      // two 64-column chunk buffers
constexpr int A_COL = ACC, A_STAGE = BKP;        // 32 hi | 32 lo columns
constexpr int PCH = 2;                           // blocks per promotion chunk (K = 128)
constexpr int SMEM = 1024 + S * STAGE + 512 + 128 * 16 * 4;
static_assert(ACC + SA * A_STAGE <= 512, "TMEM budget");

struct Geo {
  int nblk, bpi, bpr, tps;
  const uint32_t* amax_x;
  const uint32_t* amax_dz;
};

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(NT, 1)
wg1_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tdz,
           Geo g, float* __restrict__ part, float* __restrict__ bias_part) {
  extern __shared__ char smem_raw[];
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  uint64_t* ready = full + S;              // A slot (4 warps) + B split (4 warps)
  uint64_t* empty = ready + S;             // MMA done with the stage and its A slot
  uint64_t* hfull = empty + S;
  uint64_t* hfree = hfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + 2);
  float* scr = reinterpret_cast<float*>(smem + S * STAGE + 512);   // bias partials

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b0 = blockIdx.x * g.tps;
  const int nb = max(0, min(g.nblk, b0 + g.tps) - b0);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], 8);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hfree[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int sx = f16_scale_exp(*g.amax_x), sd = f16_scale_exp(*g.amax_dz);

  if (warp == TMA_WARP) {
    if (lane == 0) {
      tma_prefetch_desc(&tx);
      tma_prefetch_desc(&tdz);
      for (int bi = 0; bi < nb; ++bi) {
        const int s = bi % S;
        if (bi >= S) mbar_wait(&empty[s], ((bi / S) - 1) & 1);
        const int blk = b0 + bi, img = blk / g.bpi, rem = blk - img * g.bpi;
        const int py0 = (rem / g.bpr) * BH, px0 = (rem % g.bpr) * BW;
        char* st = smem + s * STAGE;
        mbar_expect_tx(&full[s], (uint32_t)(2 * DZB + XBYTES));
        tma_load_4d(st, &tdz, 0, px0, py0, img, &full[s]);
        tma_load_4d(st + DZB, &tdz, 32, px0, py0, img, &full[s]);
        tma_load_3d(st + 2 * DZB, &tx, px0 * CI - 4, py0 - 1, img, &full[s]);
      }
    }
  } else if (warp == MMA_WARP) {
    constexpr uint32_t idesc = make_idesc_f16(CO) | (1u << 16);       // B MN-major
    for (int bi = 0; bi < nb; ++bi) {
      const int s = bi % S, sa = bi % SA, c = bi / PCH, b = c & 1;
      if (bi % PCH == 0 && c >= 2) {
        mbar_wait(&hfree[b], ((c >> 1) - 1) & 1);
        tc_fence_after();
      }
      mbar_wait(&ready[s], (bi / S) & 1);
      tc_fence_after();
      const uint32_t d = tmem + b * CO;
      const uint32_t ah = tmem + A_COL + sa * A_STAGE, al = ah + BKP / 2;
      const uint32_t bx = smem_u32(smem + s * STAGE);
#pragma unroll
      for (int ks = 0; ks < BKP / 16; ++ks) {
        const uint64_t dbh = make_desc_sw128(bx + ks * 2048, 2 * DZB, 1024);
        const uint64_t dbl = make_desc_sw128(bx + DZB + ks * 2048, 2 * DZB, 1024);
        const uint32_t acc = (bi % PCH != 0 || ks > 0) ? 1u : 0u;
        mma_ts_f16_elect(d, al + 8 * ks, dbh, idesc, acc);
        mma_ts_f16_elect(d, ah + 8 * ks, dbl, idesc, 1u);
        mma_ts_f16_elect(d, ah + 8 * ks, dbh, idesc, 1u);
      }
      tc_commit_elect(&empty[s]);
      if (bi % PCH == PCH - 1 || bi == nb - 1) tc_commit_elect(&hfull[b]);
    }
  } else if (warp < CB0) {
    // ------------------------------------------------------------ A converters
    // lane = im2col row r; quadrant q builds the block's pixel row q
    const int q = warp & 3;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + A_COL;
    const float scale = exp2i(sx);
    const bool live = lane < R;
    const int tap = live ? lane / CI : 0, ci = live ? lane % CI : 0;
    const int dy = tap / 3, dx = tap % 3;            // halo offsets (padding folded in)
    {   // the columns of the other pixel rows stay zero in every slot
      uint32_t z[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) z[k] = 0u;
      for (int sa = 0; sa < SA; ++sa)
        for (int c8 = 0; c8 < 8; ++c8)
          if ((c8 & 3) != q) tmem_st8u(lanebase + sa * A_STAGE + 8 * c8, z);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    for (int bi = 0; bi < nb; ++bi) {
      const int s = bi % S, sa = bi % SA;
      uint32_t hi[8], lo[8];
      mbar_wait(&full[s], (bi / S) & 1);
      const float* xh = reinterpret_cast<const float*>(smem + s * STAGE + 2 * DZB) +
                        (q + dy) * XW + dx * CI + ci + 1;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float v0 = live ? xh[(2 * k) * CI] : 0.f;
        const float v1 = live ? xh[(2 * k + 1) * CI] : 0.f;
        split_f16x2_s(v0, v1, scale, hi[k], lo[k]);
      }
      if (bi >= SA) {      // the MMA of block bi - SA read this slot
        mbar_wait(&empty[(bi - SA) % S], ((bi - SA) / S) & 1);
      }
      tc_fence_after();
      tmem_st8u(lanebase + sa * A_STAGE + 8 * q, hi);
      tmem_st8u(lanebase + sa * A_STAGE + BKP / 2 + 8 * q, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[s]);
    }
  } else if (warp < DR0) {
    // ------------------------------------------------------------ B converters
    const int wb = warp - CB0, c16 = lane >> 3;
    const float scale = exp2i(sd);
    float bs[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) bs[k] = 0.f;
    for (int bi = 0; bi < nb; ++bi) {
      const int s = bi % S;
      mbar_wait(&full[s], (bi / S) & 1);
      char* bt = smem + s * STAGE;
      char* raw = bt + (c16 >> 1) * DZB;
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int pr = 16 * wb + 8 * it + (lane & 7), sw = pr & 7;
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = *reinterpret_cast<const float4*>(raw + pr * 128 + (((4 * (c16 & 1) + u) ^ sw) << 4));
        __syncwarp();
        uint32_t h[8], l[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          split_f16x2_s(v[u].x, v[u].y, scale, h[2 * u], l[2 * u]);
          split_f16x2_s(v[u].z, v[u].w, scale, h[2 * u + 1], l[2 * u + 1]);
          bs[4 * u] += v[u].x; bs[4 * u + 1] += v[u].y;
          bs[4 * u + 2] += v[u].z; bs[4 * u + 3] += v[u].w;
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int off = pr * 128 + (((2 * c16 + e) ^ sw) << 4);
          *reinterpret_cast<uint4*>(bt + off) = make_uint4(h[4 * e], h[4 * e + 1], h[4 * e + 2], h[4 * e + 3]);
          *reinterpret_cast<uint4*>(bt + DZB + off) = make_uint4(l[4 * e], l[4 * e + 1], l[4 * e + 2], l[4 * e + 3]);
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[s]);
    }
    if (bias_part != nullptr) {
      const int bt = tid - CB0 * 32;
#pragma unroll
      for (int k = 0; k < 16; ++k) scr[bt * 16 + k] = bs[k];
      named_sync(1, 128);
      if (bt < CO) {
        const int cc = bt / 16, k = bt % 16;
        float t = 0.f;
        for (int w = 0; w < 4; ++w)
          for (int l8 = 0; l8 < 8; ++l8) t += scr[(w * 32 + cc * 8 + l8) * 16 + k];
        bias_part[(long long)blockIdx.x * CO + bt] = t;
      }
    }
  } else {
    // ------------------------------------------------------------ drain
    const int q = warp & 3;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16);
    const float unscale = exp2i(-sx) * exp2i(-sd);
    float acc[CO];
#pragma unroll
    for (int j = 0; j < CO; ++j) acc[j] = 0.f;
    const int nch = (nb + PCH - 1) / PCH;
    for (int c = 0; c < nch; ++c) {
      const int b = c & 1;
      mbar_wait(&hfull[b], (c >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < CO; j += 8) {
        uint32_t rr[8];
        tmem_ld8(lanebase + b * CO + j, rr);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[j + u] += __uint_as_float(rr[u]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&hfree[b]);
    }
    // sum the four quadrants' partial rows through shared memory (the
    // stage ring is idle once the last chunk drained), fixed order
    float* red = reinterpret_cast<float*>(smem);            // [4][32][64]
    for (int j = 0; j < CO; ++j) red[(q * 32 + lane) * CO + j] = acc[j];
    named_sync(2, 128);
    if (q == 0 && lane < R) {
      float* o = part + (long long)blockIdx.x * (CO * R) + lane;
      for (int j = 0; j < CO; ++j)
        o[j * R] = (red[lane * CO + j] + red[(32 + lane) * CO + j] + red[(64 + lane) * CO + j] +
                    red[(96 + lane) * CO + j]) * unscale;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_free(tmem, 512);
  }
}

inline void plan(int n, int H, int W, Geo& g, int& grid) {
  g.bpr = W / BW;
  g.bpi = (H / BH) * g.bpr;
  g.nblk = n * g.bpi;
  grid = g.nblk < num_sms() ? g.nblk : num_sms();
  g.tps = cdiv(g.nblk, grid);
  grid = cdiv(g.nblk, g.tps);
}

}  // namespace wg1

#ifndef WG1_ON
#define WG1_ON 1
#endif
bool wg1_conv_ok(int n, int h, int w, int cin, int cout) {
  return WG1_ON && cin == wg1::CI && cout == wg1::CO && h % wg1::BH == 0 && w % wg1::BW == 0 &&
         n > 0 && ((size_t)w * wg1::CI * 4) % 16 == 0;
}

size_t wg1_conv_ws(int n, int h, int w, int cin, int cout) {
  if (!wg1_conv_ok(n, h, w, cin, cout)) return 0;
  wg1::Geo g;
  int grid;
  wg1::plan(n, h, w, g, grid);
  return 16 + ((size_t)grid * wg1::CO * wg1::R + (size_t)grid * wg1::CO) * sizeof(float);
}

bpx_status_t wg1_conv_wgrad(const float* x, const float* dz, const uint32_t* amax_x,
                            const uint32_t* amax_dz, float* dw, float* dbias, int n, int h,
                            int w_, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!aligned16(x) || !aligned16(dz) || !aligned16(dw) || (dbias && !aligned16(dbias)))
    return BPX_ERR_INVALID_ARGUMENT;
  if (ws_bytes < wg1_conv_ws(n, h, w_, wg1::CI, wg1::CO) || !aligned16(ws))
    return BPX_ERR_WORKSPACE;
  wg1::Geo g;
  int grid;
  wg1::plan(n, h, w_, g, grid);
  uint32_t* words = static_cast<uint32_t*>(ws);
  int k = 0;
  const size_t npx = (size_t)n * h * w_;
  if (!amax_x) { absmax(x, npx * wg1::CI, words, st); amax_x = words; ++k; }
  if (!amax_dz) { absmax(dz, npx * wg1::CO, words + 1, st); amax_dz = words + 1; ++k; }
  count_launches(k);
  g.amax_x = amax_x;
  g.amax_dz = amax_dz;
  CUtensorMap tx, tdz;
  {   // x as [n][H][W*3]: box 56 floats x 6 rows x 1 image, no swizzle
    const cuuint64_t dims[3] = {(cuuint64_t)w_ * wg1::CI, (cuuint64_t)h, (cuuint64_t)n};
    const cuuint64_t strides[2] = {(cuuint64_t)w_ * wg1::CI * 4, (cuuint64_t)h * w_ * wg1::CI * 4};
    const cuuint32_t box[3] = {(cuuint32_t)wg1::XW, (cuuint32_t)wg1::XB, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (encode_tiled(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return BPX_ERR_INVALID_ARGUMENT;
  }
  {   // dz as [n][H][W][64]: box 32 channels x 16 x 4 x 1, 128-B swizzle
    const cuuint64_t dims[4] = {(cuuint64_t)wg1::CO, (cuuint64_t)w_, (cuuint64_t)h, (cuuint64_t)n};
    const cuuint64_t strides[3] = {(cuuint64_t)wg1::CO * 4, (cuuint64_t)w_ * wg1::CO * 4,
                                   (cuuint64_t)h * w_ * wg1::CO * 4};
    const cuuint32_t box[4] = {32, (cuuint32_t)wg1::BW, (cuuint32_t)wg1::BH, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode_tiled(&tdz, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(dz), dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return BPX_ERR_INVALID_ARGUMENT;
  }
  float* part = reinterpret_cast<float*>(static_cast<char*>(ws) + 16);
  float* bpart = dbias ? part + (size_t)grid * wg1::CO * wg1::R : nullptr;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(wg1::wg1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, wg1::SMEM);
    attr = true;
  }
  wg1::wg1_kernel<<<grid, wg1::NT, wg1::SMEM, st>>>(tx, tdz, g, part, bpart);
  bpx_status_t s = launch_status();
  if (s != BPX_OK) return s;
  return split_reduce_wb(part, (size_t)wg1::CO * wg1::R, dw, bpart, (size_t)wg1::CO, dbias, grid,
                         st);
}

}  // namespace bpx
