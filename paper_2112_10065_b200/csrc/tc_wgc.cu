// fp16x3 weight-gradient engine for Cin = Cout = 64 convolutions (VGG's
// conv1_2 at 224x224), the one wgrad shape whose 64-wide N tiles leave the
// general engine (tc_wgh.cu) bound by its TMA feed: there every 64-pixel K
// block re-loads x once per tap (18 x boxes + 10 dz boxes, 224 KB) for
// 4.5 M tiles held by different CTAs.  Here ONE CTA keeps all five M tiles
// of dW^T (576 rows x 64) as five TMEM accumulators and walks 16 x 4 pixel
// blocks: per block it loads one x halo (18 x 6 pixels, 27 KB; the 4-D
// TMA box's out-of-bounds rows are the conv's zero padding) that serves
// all nine taps, plus the dz block (16 KB): 43 KB per block.
//
//   dW^T[r][co] = sum_p x[p + s_tap][ci] * dz[p][co],  r = tap*64 + ci
//
// Per block and M tile k (rows 128k .. 128k+127 = chunks (tap, 32 ci)), the
// A converters read each row's 64 shifted pixels out of the halo, split
// them into fp16 hi/lo (tc_ptx.cuh) and tcgen05.st them into one of three
// TMEM A slots; the B converters split the dz block in place into an fp16
// MN-major atom (as in tc_wgh.cu) and sum the bias gradient; the MMA warp
// issues a_lo*b_hi + a_hi*b_lo + a_hi*b_hi (kind::f16, N = 64) into
// accumulator k.  Every PB blocks (K = 64 PB pixels) each accumulator is
// promoted: the drain warps read it as soon as its last MMA committed
// (accfull[k]), release it (accfree[k]) and add it in round-to-nearest fp32
// into this CTA's partial dW^T slab in global memory (L2), so the five
// accumulators need no second TMEM buffer.  The slabs of the CTAs (each a
// contiguous range of blocks) meet in the fixed-order split_reduce.
//
// CTA: 22 warps.  warp 0 TMA, warp 1 MMA + TMEM owner, 2-9 A converters
// (lane quadrant = chunk of the M tile; two per quadrant, two pixel rows
// each), 10-13 B converters, 14-21 drain.
#include "tma_host.h"
#include "tc_ptx.cuh"
#include "tc_api.h"

namespace bpx {
namespace wgc {
using namespace tcx;

constexpr int TMA_WARP = 0, MMA_WARP = 1, CA0 = 2, NCA = 8, CB0 = CA0 + NCA, DR0 = CB0 + 4;
constexpr int NT = (DR0 + 8) * 32;
constexpr int C = 64;                         // Cin = Cout
constexpr int MT = 5;                         // M tiles: 9 * 64 = 576 rows (4.5 x 128)
constexpr int NROWS = 9 * C;
constexpr int BW = 16, BH = 4, BKP = BW * BH; // pixel block (K = 64 per block)
constexpr int HX = BW + 2, HY = BH + 2, HROWS = HX * HY;
constexpr int XH = 14336;                     // one 32-channel halo half (108 x 128 B, 1 KB aligned)
constexpr int DZB = BKP * 128;                // one 32-channel dz box (64 x 128 B)
constexpr int STAGE = 2 * XH + 2 * DZB;
constexpr int S = 4, SA = 3;                  // smem stages, TMEM A slots
constexpr int ACC = MT * C;                   // 320 accumulator columns
constexpr int A_COL = ACC, A_STAGE = BKP;     // A slot: 32 hi | 32 lo columns
constexpr int SMEM = 1024 + S * STAGE + 512 + 128 * 16 * 4;
static_assert(ACC + SA * A_STAGE <= 512, "TMEM budget");
static_assert(SMEM <= 227 * 1024, "smem budget");
#ifndef WGC_PB
#define WGC_PB 8                              // blocks per promotion chunk (K = 512)
#endif
constexpr int PB = WGC_PB;
// ALT: the two A-converter warps of a lane quadrant take alternate A slots
// (all four pixel rows each) instead of two rows of every slot, so one
// warp's conversion overlaps the other's wait::st and hand-off (as in fdt)
#ifndef WGC_ALT
#define WGC_ALT 1
#endif

struct Geo {
  int H, W;
  int nblk, bpi, bpr;        // blocks: total, per image, per block row
  int tps;                   // blocks per CTA
  long long slab;            // 64 * 576
  const uint32_t* amax_x;
  const uint32_t* amax_dz;
};

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(NT, 1)
wgc_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tdz,
           Geo g, float* __restrict__ part, float* __restrict__ bias_part) {
  extern __shared__ char smem_raw[];
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);   // stage landed
  uint64_t* bready = full + S;             // dz split
  uint64_t* sempty = bready + S;           // MMA done with B + A converters done with the halo
  uint64_t* aready = sempty + S;           // TMEM A slot written
  uint64_t* aempty = aready + SA;          // TMEM A slot consumed
  uint64_t* accfull = aempty + SA;         // accumulator k: chunk complete
  uint64_t* accfree = accfull + MT;        // accumulator k: drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfree + MT);
  float* bias_scr = reinterpret_cast<float*>(smem + S * STAGE + 512);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b0 = blockIdx.x * g.tps;
  const int nb = max(0, min(g.nblk, b0 + g.tps) - b0);
  const int nch = (nb + PB - 1) / PB;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&bready[s], 4);
      mbar_init(&sempty[s], 1 + NCA);      // MMA commit + the A converter warps
    }
    for (int a = 0; a < SA; ++a) {
      mbar_init(&aready[a], WGC_ALT ? NCA / 2 : NCA);   // the warps that wrote the slot
      mbar_init(&aempty[a], 1);
    }
    for (int k = 0; k < MT; ++k) {
      mbar_init(&accfull[k], 1);
      mbar_init(&accfree[k], 8);
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
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tx);
      tma_prefetch_desc(&tdz);
      for (int bi = 0; bi < nb; ++bi) {
        const int s = bi % S;
        if (bi >= S) mbar_wait(&sempty[s], ((bi / S) - 1) & 1);
        const int blk = b0 + bi, img = blk / g.bpi, rem = blk - img * g.bpi;
        const int py0 = (rem / g.bpr) * BH, px0 = (rem % g.bpr) * BW;
        char* st = smem + s * STAGE;
        mbar_expect_tx(&full[s], (uint32_t)(2 * HROWS * 128 + 2 * DZB));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tma_load_4d(st + h * XH, &tx, 32 * h, px0 - 1, py0 - 1, img, &full[s]);
          tma_load_4d(st + 2 * XH + h * DZB, &tdz, 32 * h, px0, py0, img, &full[s]);
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc_f16(C) | (1u << 16);      // B MN-major
    int ai = 0;
    for (int bi = 0; bi < nb; ++bi) {
      const int s = bi % S, ch = bi / PB;
      const bool first = bi % PB == 0, last = bi % PB == PB - 1 || bi == nb - 1;
      mbar_wait(&bready[s], (bi / S) & 1);
      const uint32_t bx = smem_u32(smem + s * STAGE + 2 * XH);
      for (int k = 0; k < MT; ++k, ++ai) {
        const int sa = ai % SA;
        mbar_wait(&aready[sa], (ai / SA) & 1);
        if (first && ch >= 1) mbar_wait(&accfree[k], (ch - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + k * C;
        const uint32_t ah = tmem + A_COL + sa * A_STAGE, al = ah + BKP / 2;
#pragma unroll
        for (int ks = 0; ks < BKP / 16; ++ks) {
          const uint64_t dbh = make_desc_sw128(bx + ks * 2048, 2 * DZB, 1024);
          const uint64_t dbl = make_desc_sw128(bx + DZB + ks * 2048, 2 * DZB, 1024);
          const uint32_t acc = (!first || ks > 0) ? 1u : 0u;
#ifndef WGC_NOMMA
          mma_ts_f16_elect(d, al + 8 * ks, dbh, idesc, acc);
          mma_ts_f16_elect(d, ah + 8 * ks, dbl, idesc, 1u);
          mma_ts_f16_elect(d, ah + 8 * ks, dbh, idesc, 1u);
#endif
        }
        tc_commit_elect(&aempty[sa]);
        if (last) tc_commit_elect(&accfull[k]);
      }
      tc_commit_elect(&sempty[s]);
    }
  } else if (warp < CB0) {
    // ------------------------------------------------------------ A converters
    // thread = TMEM lane = row r of M tile k = channel `lane` of chunk
    // gc = 4k + q = (tap, 32-channel half); its 64 pixels are the block's
    // 16 x 4 pixels shifted by the tap, read out of the halo
    const int q = warp & 3, ph = (warp - CA0) >> 2;   // quadrant, pixel-row half
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + A_COL;
    const float scale = exp2i(sx);
    const int cofs = ((lane >> 2) << 4) + (lane & 3) * 4;     // logical chunk, word
    int ai = 0;
    for (int bi = 0; bi < nb; ++bi) {
      const int s = bi % S;
      mbar_wait(&full[s], (bi / S) & 1);
      const char* st = smem + s * STAGE;
      for (int k = 0; k < MT; ++k, ++ai) {
        const int sa = ai % SA;
        const int gc = 4 * k + q;
#if WGC_ALT
        if ((ai & 1) != ph) continue;            // the quadrant's other warp takes this slot
#endif
        if (ai >= SA) mbar_wait(&aempty[sa], ((ai / SA) - 1) & 1);
        tc_fence_after();
#ifdef WGC_NOCONV
        if (false) {
#else
        if (gc < 2 * 9) {                        // rows past 576 stay garbage, never stored
#endif
          const int tap = gc >> 1, dy = tap / 3, dx = tap % 3;   // halo offsets (+1 folded in)
          const char* hb = st + (gc & 1) * XH;
          const uint32_t a = lanebase + sa * A_STAGE;
#pragma unroll
          for (int pp = 0; pp < (WGC_ALT ? BH : BH / 2); ++pp) {   // a 16-pixel row = 8 columns
            const int py = WGC_ALT ? pp : 2 * ph + pp;
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2) {
              float v[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int hr = (py + dy) * HX + 2 * k2 + e + dx;
                v[e] = *reinterpret_cast<const float*>(hb + hr * 128 + (cofs ^ ((hr & 7) << 4)));
              }
              split_f16x2_s(v[0], v[1], scale, hi[k2], lo[k2]);
            }
            tmem_st8u(a + 8 * py, hi);
            tmem_st8u(a + BKP / 2 + 8 * py, lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&aready[sa]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[s]);      // done reading this halo
    }
  } else if (warp < DR0) {
    // ------------------------------------------------------------ B converters
    // the dz block's two fp32 boxes become one fp16 MN-major atom in place
    // (hi where box 0 was, lo where box 1 was); four threads (one
    // quarter-warp each, 16 channels) per pixel row pair; warp wb takes
    // pixels [16 wb, +16); bias partials per channel
    const int wb = warp - CB0, c16 = lane >> 3;
    const float scale = exp2i(sd);
    float bs[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) bs[k] = 0.f;
    for (int bi = 0; bi < nb; ++bi) {
      const int s = bi % S;
      mbar_wait(&full[s], (bi / S) & 1);
      char* bt = smem + s * STAGE + 2 * XH;
      char* raw = bt + (c16 >> 1) * DZB;
#pragma unroll
      for (int it = 0; it < 2; ++it) {
#ifdef WGC_NOCONV
        break;
#endif
        const int pr = 16 * wb + 8 * it + (lane & 7), sw = pr & 7;
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = *reinterpret_cast<const float4*>(raw + pr * 128 + (((4 * (c16 & 1) + u) ^ sw) << 4));
        __syncwarp();                     // the row pair is read before anyone overwrites it
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
      fence_proxy_async();                // generic-proxy writes -> the MMA's async reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&bready[s]);
    }
    if (bias_part != nullptr) {
      // fixed-order reduction of the per-thread partials of each channel
      const int bt = tid - CB0 * 32;
#pragma unroll
      for (int k = 0; k < 16; ++k) bias_scr[bt * 16 + k] = bs[k];
      named_sync(1, 128);
      if (bt < C) {
        const int cc = bt / 16, k = bt % 16;
        float t = 0.f;
        for (int w = 0; w < 4; ++w)
          for (int l8 = 0; l8 < 8; ++l8) t += bias_scr[(w * 32 + cc * 8 + l8) * 16 + k];
        bias_part[(long long)blockIdx.x * C + bt] = t;
      }
    }
  } else {
    // ------------------------------------------------------------ drain
    // accumulator k as soon as its chunk completes; rows r = 128k + 32q +
    // lane, columns [32 hf, +32): added in RN fp32 into this CTA's slab
    const int q = warp & 3, hf = (warp - DR0) >> 2;
    const float unscale = exp2i(-sx) * exp2i(-sd);
    float* slab = part + (long long)blockIdx.x * g.slab;
    for (int ch = 0; ch < nch; ++ch) {
      for (int k = 0; k < MT; ++k) {
        mbar_wait(&accfull[k], ch & 1);
        tc_fence_after();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint32_t rr[8];
          tmem_ld8(tmem + ((uint32_t)(q * 32) << 16) + k * C + 32 * hf + j, rr);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 8; ++u) v[j + u] = __uint_as_float(rr[u]) * unscale;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&accfree[k]);
        const int r = 128 * k + 32 * q + lane;
        if (r < NROWS) {
          float* o = slab + (long long)(32 * hf) * NROWS + r;
          if (ch == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) o[(long long)j * NROWS] = v[j];
          } else {
            // fire-and-forget adds in L2; one thread per address, issued in
            // chunk order (same-address order is kept), RN: deterministic
#pragma unroll
            for (int j = 0; j < 32; ++j)
              asm volatile("red.global.add.f32 [%0], %1;" ::"l"(o + (long long)j * NROWS),
                           "f"(v[j]) : "memory");
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_free(tmem, 512);
  }
}

inline bool encode4(CUtensorMap* m, const float* p, int n, int H, int W, int boxw, int boxh) {
  const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n};
  const cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4,
                                 (cuuint64_t)H * W * C * 4};
  const cuuint32_t box[4] = {32, (cuuint32_t)boxw, (cuuint32_t)boxh, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(p), dims, strides,
                      box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline void plan(int n, int H, int W, Geo& g, int& grid) {
  g.H = H; g.W = W;
  g.bpr = W / BW;
  g.bpi = (H / BH) * g.bpr;
  g.nblk = n * g.bpi;
  g.slab = (long long)C * NROWS;
  grid = g.nblk < num_sms() ? g.nblk : num_sms();
  g.tps = cdiv(g.nblk, grid);
  grid = cdiv(g.nblk, g.tps);
}

}  // namespace wgc

#ifndef WGC_ON
#define WGC_ON 1
#endif
bool wgc_conv_ok(int n, int h, int w, int cin, int cout) {
  return WGC_ON && cin == wgc::C && cout == wgc::C && h % wgc::BH == 0 && w % wgc::BW == 0 &&
         (long long)n * h * w >= 64LL * 148;
}

size_t wgc_conv_ws(int n, int h, int w, int cin, int cout) {
  if (!wgc_conv_ok(n, h, w, cin, cout)) return 0;
  wgc::Geo g;
  int grid;
  wgc::plan(n, h, w, g, grid);
  return 16 + ((size_t)grid * (size_t)g.slab + (size_t)grid * wgc::C) * sizeof(float);
}

bpx_status_t wgc_conv_wgrad(const float* x, const float* dz, const uint32_t* amax_x,
                            const uint32_t* amax_dz, float* dw, float* dbias, int n, int h,
                            int w_, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!aligned16(x) || !aligned16(dz) || !aligned16(dw) || (dbias && !aligned16(dbias)))
    return BPX_ERR_INVALID_ARGUMENT;
  if (ws_bytes < wgc_conv_ws(n, h, w_, wgc::C, wgc::C) || !aligned16(ws)) return BPX_ERR_WORKSPACE;
  wgc::Geo g;
  int grid;
  wgc::plan(n, h, w_, g, grid);
  uint32_t* words = static_cast<uint32_t*>(ws);
  int k = 0;
  const size_t npx = (size_t)n * h * w_;
  if (!amax_x) { absmax(x, npx * wgc::C, words, st); amax_x = words; ++k; }
  if (!amax_dz) { absmax(dz, npx * wgc::C, words + 1, st); amax_dz = words + 1; ++k; }
  count_launches(k);
  g.amax_x = amax_x;
  g.amax_dz = amax_dz;
  CUtensorMap tx, tdz;
  if (!wgc::encode4(&tx, x, n, h, w_, wgc::HX, wgc::HY) ||
      !wgc::encode4(&tdz, dz, n, h, w_, wgc::BW, wgc::BH))
    return BPX_ERR_INVALID_ARGUMENT;
  float* part = reinterpret_cast<float*>(static_cast<char*>(ws) + 16);
  float* bpart = dbias ? part + (size_t)grid * g.slab : nullptr;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(wgc::wgc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, wgc::SMEM);
    attr = true;
  }
  wgc::wgc_kernel<<<grid, wgc::NT, wgc::SMEM, st>>>(tx, tdz, g, part, bpart);
  bpx_status_t s = launch_status();
  if (s != BPX_OK) return s;
  return split_reduce_wb(part, (size_t)g.slab, dw, bpart, (size_t)wgc::C, dbias, grid, st);
}

}  // namespace bpx
