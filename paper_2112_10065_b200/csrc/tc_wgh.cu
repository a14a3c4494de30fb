// tcgen05 weight-gradient engine for the 3x3/pad-1 convolutions, fp16x3,
// fed by TMA:
//
//   dW^T[r][co] = sum_p im2col(x)[p][r] * dz[p][co],   r = tap*Cin + ci
//   M = 9*Cin (A = im2col(x)^T), N = Cout (B = dz), K = pixels (split-K)
//
// K = pixels is blocked as 64 consecutive pixels of the flattened NHWC
// tensor (so no tile overhangs an image edge, whatever H and W are).  For a
// 32-channel chunk of one tap the A tile is x[p0+s : +64][ci0 : +32] with
// s = dy*W + dx, the B tile is dz[p0 : +64][co0 : +32]: each is ONE 2-D TMA
// box (fp32, 128-B swizzle, a pixel per 128-B row).  Rows whose shifted
// source pixel wraps across an image row/edge are the conv's zero padding:
// the A converters zero them from a per-tap ballot mask.
//
// fp32 accuracy by fp16x3 (tc_ptx.cuh): x and dz are scaled by powers of two
// from their max |v| words and split into fp16 hi/lo:
//   * A converter warps (one TMEM lane = one row r per thread) read their
//     channel across the stage's 64 pixels, split and tcgen05.st hi and lo
//     (pixel pairs packed per 32-bit column) -> TS-form MMAs;
//   * B converter warps split dz IN PLACE: the two fp32 boxes holding
//     channels [64a, 64a+32) and [64a+32, 64a+64) of a pixel become that
//     pixel's 128-B fp16 hi row and lo row of the 64-channel MN-major atom a
//     (128-B swizzle, the same row XOR as the fp32 boxes), so dz takes no
//     extra shared memory; a warp owns whole row pairs (read, __syncwarp,
//     write).  In CTAs of the first M tile they also sum dz per channel in a
//     fixed order: the bias gradient comes out of the same pass.
// Each 16-pixel k-step issues a_lo*b_hi + a_hi*b_lo + a_hi*b_hi (kind::f16).
// Partial sums live in TMEM in 128-pixel chunks (two ping-pong buffers) and
// are promoted into round-to-nearest fp32 registers by the drain warps
// (the tensor core's fp32 accumulation truncates), which undo the scales.
//
// CTA: 18 warps, one CTA per SM.  warp 0 TMA producer, warp 1 MMA issuer +
// TMEM owner, warps 2-5 A converters, 6-9 B converters (+bias), 10-17 drain.
#include "tma_host.h"
#include "tc_ptx.cuh"
#include "tc_api.h"

namespace bpx {
namespace wgh {
using namespace tcx;

constexpr int TMA_WARP = 0, MMA_WARP = 1, CA0 = 2, CB0 = 6, DR0 = 10, NT = 18 * 32;
constexpr int BK = 64;                          // pixels per stage
constexpr int BOX = 32 * BK * 4;                // 32 channels x 64 pixels, fp32
// promotion chunk K = 256 pixels: fp64 error 9e-7 against the ~3.9e-6 gate
// (K = 128: 4.8e-7), 1.5 % faster (tools/fdt_prec.py, B200 same-box)
#ifndef WGH_PCHK
#define WGH_PCHK 256
#endif
constexpr int PCH = WGH_PCHK / BK;              // stages per promotion chunk
// SSA (experiment, Cin % 64 == 0): A (x^T) is read by the MMA straight from
// shared memory as an MN-major operand -- x's natural [pixel][channel]
// layout -- after the A converters split its boxes IN PLACE into fp16 hi/lo
// atoms (as the B converters do for dz), instead of the column-wise
// transpose into TMEM.  Correct, but 9-14 % slower on every VGG wgrad layer
// (B200 same-box A/B: the three SS-form MMAs re-read A from shared memory,
// 4 KB each): off
#ifndef WGH_SSA
#define WGH_SSA 0
#endif
// ALT (CTA pairs): warps 2-9 are one pool of converters in two groups of
// four taking alternate stages, each warp doing one lane quadrant's x
// conversion and a quarter of its CTA's dz half, so one group's stage
// overlaps the other's hand-off (as the fwd/dgrad engine's converters do).
// B200 same-box: paired layers 3-6 % faster (conv3_2 0.372 -> 0.360 ms,
// conv4_2 0.382 -> 0.363); unpaired ones, whose warps would also split a
// whole 128-channel dz tile, 5-10 % slower -- so pairs only
#ifndef WGH_ALT
#define WGH_ALT 1
#endif

// PAIR (BN = 128): a cluster of two CTAs (M tiles 2m, 2m+1, same N tile and
// pixel split) runs one M = 256 MMA (cta_group::2); each CTA loads and splits
// HALF of the dz tile (64 channels, one fp16 atom), so dz crosses L2 once
// per 256 rows of dW^T instead of once per 128.
template <int BN, bool PAIR = false>
struct Cfg {
  static_assert(BN == 64 || BN == 128, "BN");
  static_assert(!PAIR || BN == 128, "pairs split a 128-channel dz tile");
  static constexpr int BNL = PAIR ? BN / 2 : BN;          // dz channels held by this CTA
  static constexpr int S = BNL == 128 ? 3 : 4;
  static constexpr int A_BYTES = 4 * BOX;                 // 128 rows of A
  static constexpr int B_BYTES = (BNL / 32) * BOX;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int ACC = 2 * BN;                      // two chunk buffers
  static constexpr int A_COL = ACC;                       // + S stages of (hi | lo)
  static constexpr int A_STAGE = BK;                      // 32 hi + 32 lo columns
  static constexpr int BIAS = 256 * 16 * 4;               // converters' bias partials
  static constexpr int SMEM = 1024 + S * STAGE + 512 + BIAS;
  static_assert(ACC + S * A_STAGE <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "smem budget");
};

struct Geo {
  int Cin, Cout, H, W;
  long long npix;
  int tiles, tps;            // 64-pixel tiles in total / per split
  long long slab;            // Cout * 9*Cin
  const uint32_t* amax_x;
  const uint32_t* amax_dz;
};

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int BN, bool PAIR, bool SSA = false>
__global__ void __launch_bounds__(NT, 1)
wgh_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tdz,
           Geo g, float* __restrict__ part, float* __restrict__ bias_part) {
  using Cf = Cfg<BN, PAIR>;
  constexpr int S = Cf::S, BNL = Cf::BNL;
  extern __shared__ char smem_raw[];
  // offset from smem_raw (not a uintptr_t round trip) keeps the shared address space: LDS/STS, not generic LD/ST
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cf::STAGE);   // stage landed
  uint64_t* ready = full + 8;                // A and B converters done
  uint64_t* empty = ready + 8;               // MMA done: stage + TMEM A slot free
  uint64_t* hfull = empty + 8;
  uint64_t* hfree = hfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + 2);
  float* bias_scr = reinterpret_cast<float*>(smem + S * Cf::STAGE + 512);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nrows = 9 * g.Cin;                  // M extent
  const int chunks = nrows / 32;                // 32-row chunks (tap-major)
  const int cpt = g.Cin / 32;                   // chunks per tap
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * BN;
  const int t0 = blockIdx.z * g.tps;
  const int nst = max(0, min(g.tiles, t0 + g.tps) - t0);
  // pairs: the leader (rank 0) issues the MMAs and owns ready / hfree, which
  // both CTAs' converters / drains arrive on; its commits reach both CTAs
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int nl0 = n0 + (int)rank * BNL;         // first dz channel held here

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], (PAIR ? 16 : 8) / (WGH_ALT && !SSA && PAIR ? 2 : 1));   // per converter warp
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hfree[b], PAIR ? 16 : 8);    // one arrival per drain warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    if (PAIR) tmem_alloc2(tmem_slot, 512); else tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t ready_l = PAIR ? mapa_rank(ready, 0) : 0u;
  const uint32_t hfree_l = PAIR ? mapa_rank(hfree, 0) : 0u;
  const int sx = f16_scale_exp(*g.amax_x), sd = f16_scale_exp(*g.amax_dz);

  if (warp == TMA_WARP) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tx);
      tma_prefetch_desc(&tdz);
      int na = 0;
      for (int c = 0; c < 4; ++c) na += (m0 / 32 + c) < chunks;
#ifdef WGH_NOX
      na = 0;
#endif
#ifdef WGH_NODZ
      const uint32_t bytes = (uint32_t)(na * BOX);
#else
      const uint32_t bytes = (uint32_t)(na * BOX + Cf::B_BYTES);
#endif
      for (int i = 0; i < nst; ++i) {
        const int s = i % S;
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        const int p0 = (t0 + i) * BK;
        char* st = smem + s * Cf::STAGE;
        mbar_expect_tx(&full[s], bytes);
        for (int c = 0; c < na; ++c) {
          const int gc = m0 / 32 + c;
          const int tap = gc / cpt, ci0 = (gc - tap * cpt) * 32;
          tma_load_2d(st + c * BOX, &tx, ci0, p0 + (tap / 3 - 1) * g.W + tap % 3 - 1, &full[s]);
        }
#ifndef WGH_NODZ
#pragma unroll
        for (int j = 0; j < BNL / 32; ++j)
          tma_load_2d(st + Cf::A_BYTES + j * BOX, &tdz, nl0 + 32 * j, p0, &full[s]);
#endif
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    // M=128, N=BN, f16 x f16 -> f32, A from TMEM, B MN-major (bit 16): atom a
    // (64 channels) of b_hi sits where box 2a landed, b_lo where box 2a+1 did
    constexpr uint32_t idesc = (PAIR ? ((make_idesc_f16(BN) & ~(0x1Fu << 24)) | (16u << 24))
                                     : make_idesc_f16(BN)) | (1u << 16) |
                               (SSA ? (1u << 15) : 0u);           // A MN-major (SSA)
    for (int i = 0; i < nst && (!PAIR || rank == 0); ++i) {
      const int s = i % S;
      const int c = i / PCH, b = c & 1;
      if (i % PCH == 0 && c >= 2) {
        if (PAIR) mbar_wait_cluster(&hfree[b], ((c >> 1) - 1) & 1);
        else mbar_wait(&hfree[b], ((c >> 1) - 1) & 1);
        tc_fence_after();
      }
      if (PAIR) mbar_wait_cluster(&ready[s], (i / S) & 1); else mbar_wait(&ready[s], (i / S) & 1);
      tc_fence_after();
      const uint32_t d = tmem + b * BN;
      const uint32_t ah = tmem + Cf::A_COL + s * Cf::A_STAGE, al = ah + BK / 2;
      const uint32_t ax = smem_u32(smem + s * Cf::STAGE);
      const uint32_t bx = ax + Cf::A_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / 16; ++ks) {
        const uint64_t dbh = make_desc_sw128(bx + ks * 2048, 2 * BOX, 1024);
        const uint64_t dbl = make_desc_sw128(bx + BOX + ks * 2048, 2 * BOX, 1024);
        const uint32_t acc = (i % PCH != 0 || ks > 0) ? 1u : 0u;
#ifndef WGH_NOMMA
        if (SSA) {         // A atoms a = 0, 1 (64 rows each) where boxes 2a / 2a+1 landed
          const uint64_t dah = make_desc_sw128(ax + ks * 2048, 2 * BOX, 1024);
          const uint64_t dal = make_desc_sw128(ax + BOX + ks * 2048, 2 * BOX, 1024);
          if (PAIR) {
            mma_ss2_f16_elect(d, dal, dbh, idesc, acc);
            mma_ss2_f16_elect(d, dah, dbl, idesc, 1u);
            mma_ss2_f16_elect(d, dah, dbh, idesc, 1u);
          } else {
            mma_ss_f16_elect(d, dal, dbh, idesc, acc);
            mma_ss_f16_elect(d, dah, dbl, idesc, 1u);
            mma_ss_f16_elect(d, dah, dbh, idesc, 1u);
          }
        } else if (PAIR) {
          mma_ts2_f16_elect(d, al + 8 * ks, dbh, idesc, acc);
          mma_ts2_f16_elect(d, ah + 8 * ks, dbl, idesc, 1u);
          mma_ts2_f16_elect(d, ah + 8 * ks, dbh, idesc, 1u);
        } else {
          mma_ts_f16_elect(d, al + 8 * ks, dbh, idesc, acc);
          mma_ts_f16_elect(d, ah + 8 * ks, dbl, idesc, 1u);
          mma_ts_f16_elect(d, ah + 8 * ks, dbh, idesc, 1u);
        }
#endif
      }
      if (PAIR) {
        tc_commit2_elect(&empty[s]);
        if (i % PCH == PCH - 1 || i == nst - 1) tc_commit2_elect(&hfull[b]);
      } else {
        tc_commit_elect(&empty[s]);
        if (i % PCH == PCH - 1 || i == nst - 1) tc_commit_elect(&hfull[b]);
      }
    }
  } else if (warp < DR0 && WGH_ALT && !SSA && PAIR) {
    // ------------------------------------------------------------ converters (ALT)
    // warps 2-9 in two groups of four taking alternate stages; in its stage a
    // warp converts A for lane quadrant q (as the A converters below) AND
    // splits dz rows share q in place (as the B converters below), so one
    // group's work on stage i + 1 overlaps the other's hand-off of stage i
    // (q = warp % 4: a warp reaches only its own TMEM lane quadrant)
    const int cw = warp - CA0, grp = cw >> 2, q = warp & 3;
    // --- A (x^T) for lane quadrant q
    const bool valid = (m0 / 32 + q) < chunks;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + Cf::A_COL;
    const int gc = m0 / 32 + q, tap = valid ? gc / cpt : 4;
    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
    const float scx = exp2i(sx);
    const int cofs = ((lane >> 2) << 4) + (lane & 3) * 4;
    long long p = (long long)t0 * BK + lane;
    int img = (int)(p / ((long long)g.H * g.W));
    int rem = (int)(p - (long long)img * g.H * g.W);
    int oh = rem / g.W, ow = rem - (rem / g.W) * g.W;
    // --- B (dz) rows share q
    const int c16 = lane >> 3;
    const int at = BNL == 128 ? (q & 1) : 0;
    constexpr int PPW = BNL == 128 ? 32 : 16;
    const int pb = (BNL == 128 ? (q >> 1) : q) * PPW;
    const float scd = exp2i(sd);
    const bool do_bias = bias_part != nullptr && blockIdx.x == (PAIR ? rank : 0u);
    float bs[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) bs[k] = 0.f;
    for (int i = 0; i < nst; ++i) {
      const int s = i % S;
      uint32_t vmask[BK / 32];
#pragma unroll
      for (int h = 0; h < BK / 32; ++h) {      // every stage: the coordinates advance
        const bool ok = valid && p < g.npix && (unsigned)(oh + dy) < (unsigned)g.H &&
                        (unsigned)(ow + dx) < (unsigned)g.W;
        vmask[h] = __ballot_sync(0xffffffffu, ok);
        p += 32;
        ow += 32;
        while (ow >= g.W) {
          ow -= g.W;
          if (++oh == g.H) { oh = 0; ++img; }
        }
      }
      if ((i & 1) != grp) continue;
      mbar_wait(&full[s], (i / S) & 1);
      tc_fence_after();
      char* st = smem + s * Cf::STAGE;
#if !defined(WGH_NOCONV) && !defined(WGH_NOACONV)
      {
        const char* box = st + q * BOX;
        const uint32_t a = lanebase + s * Cf::A_STAGE;
#pragma unroll
        for (int ps = 0; ps < BK / 16; ++ps) {
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            float v[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int kk = 16 * ps + 2 * k + e;
              v[e] = ((vmask[kk >> 5] >> (kk & 31)) & 1u)
                         ? *reinterpret_cast<const float*>(box + kk * 128 + (cofs ^ ((kk & 7) << 4)))
                         : 0.f;
            }
            split_f16x2_s(v[0], v[1], scx, hi[k], lo[k]);
          }
          tmem_st8u(a + 8 * ps, hi);
          tmem_st8u(a + BK / 2 + 8 * ps, lo);
        }
      }
#endif
#ifndef WGH_NOCONV
      {
        char* bt = st + Cf::A_BYTES;
        char* raw = bt + (2 * at + (c16 >> 1)) * BOX;
        char* hrow = bt + 2 * at * BOX, *lrow = hrow + BOX;
#pragma unroll
        for (int it = 0; it < PPW / 8; ++it) {
          const int pr = pb + 8 * it + (lane & 7);
          const int sw = pr & 7;
          float4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            v[u] = *reinterpret_cast<const float4*>(raw + pr * 128 + (((4 * (c16 & 1) + u) ^ sw) << 4));
          __syncwarp();
          uint32_t h[8], l[8];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            split_f16x2_s(v[u].x, v[u].y, scd, h[2 * u], l[2 * u]);
            split_f16x2_s(v[u].z, v[u].w, scd, h[2 * u + 1], l[2 * u + 1]);
            if (do_bias) {
              bs[4 * u] += v[u].x; bs[4 * u + 1] += v[u].y;
              bs[4 * u + 2] += v[u].z; bs[4 * u + 3] += v[u].w;
            }
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int off = pr * 128 + (((2 * c16 + e) ^ sw) << 4);
            *reinterpret_cast<uint4*>(hrow + off) = make_uint4(h[4 * e], h[4 * e + 1], h[4 * e + 2], h[4 * e + 3]);
            *reinterpret_cast<uint4*>(lrow + off) = make_uint4(l[4 * e], l[4 * e + 1], l[4 * e + 2], l[4 * e + 3]);
          }
        }
      }
#endif
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      fence_proxy_async();                // generic-proxy writes -> the MMA's async reads
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_remote(ready_l + 8u * s); else mbar_arrive(&ready[s]);
      }
    }
    if (do_bias) {
      // fixed-order reduction of the per-thread partials of both groups
      const int bt = tid - CA0 * 32;                        // 0 .. 255
#pragma unroll
      for (int k = 0; k < 16; ++k) bias_scr[bt * 16 + k] = bs[k];
      named_sync(1, 256);
      if (bt < BNL) {
        const int a = bt / 64, cc = (bt % 64) / 16, k = bt % 16;
        float t = 0.f;
        for (int gg = 0; gg < 2; ++gg)
          for (int w = 0; w < 4; ++w) {
            if (BNL == 128 && (w & 1) != a) continue;
            for (int l8 = 0; l8 < 8; ++l8)
              t += bias_scr[((gg * 4 + w) * 32 + cc * 8 + l8) * 16 + k];
          }
        bias_part[(long long)blockIdx.z * g.Cout + nl0 + bt] = t;
      }
    }
  } else if (warp < CB0 && SSA) {
    // ------------------------------------------------------------ A converters (SSA)
    // split x IN PLACE into MN-major fp16 atoms: atom a = channels [64a, +64)
    // of the M tile (boxes 2a, 2a+1: one tap); warp wa takes atom wa & 1,
    // pixel rows [32 (wa >> 1), +32), four threads (16 channels) per row
    // pair; rows whose tap-shifted pixel is outside the image become zeros
    const int wa = warp - CA0, c16 = lane >> 3, at = wa & 1, pb = (wa >> 1) * 32;
    const bool valid = (m0 / 32 + 2 * at) < chunks;
    const int tap = valid ? (m0 / 32 + 2 * at) / cpt : 4;
    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
    const float scale = exp2i(sx);
    long long p = (long long)t0 * BK + lane;
    int img = (int)(p / ((long long)g.H * g.W));
    int rem = (int)(p - (long long)img * g.H * g.W);
    int oh = rem / g.W, ow = rem - (rem / g.W) * g.W;
    for (int i = 0; i < nst; ++i) {
      const int s = i % S;
      uint32_t vm = 0;                   // validity of pixel rows [pb, pb + 32)
#pragma unroll
      for (int h = 0; h < BK / 32; ++h) {
        const bool ok = valid && p < g.npix && (unsigned)(oh + dy) < (unsigned)g.H &&
                        (unsigned)(ow + dx) < (unsigned)g.W;
        const uint32_t b = __ballot_sync(0xffffffffu, ok);
        if (h == (pb >> 5)) vm = b;
        p += 32;
        ow += 32;
        while (ow >= g.W) {
          ow -= g.W;
          if (++oh == g.H) { oh = 0; ++img; }
        }
      }
      mbar_wait(&full[s], (i / S) & 1);
      char* hrow = smem + s * Cf::STAGE + 2 * at * BOX, *lrow = hrow + BOX;
      const char* raw = hrow + (c16 >> 1) * BOX;          // this thread's 16 fp32 channels
#if !defined(WGH_NOCONV) && !defined(WGH_NOACONV)
      if (valid) {
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int pr = pb + 8 * it + (lane & 7), sw = pr & 7;
          const bool ok = (vm >> (8 * it + (lane & 7))) & 1u;
          float4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            v[u] = *reinterpret_cast<const float4*>(raw + pr * 128 + (((4 * (c16 & 1) + u) ^ sw) << 4));
          __syncwarp();                   // the row pair is read before anyone overwrites it
          uint32_t h[8], l[8];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (!ok) v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            split_f16x2_s(v[u].x, v[u].y, scale, h[2 * u], l[2 * u]);
            split_f16x2_s(v[u].z, v[u].w, scale, h[2 * u + 1], l[2 * u + 1]);
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int off = pr * 128 + (((2 * c16 + e) ^ sw) << 4);
            *reinterpret_cast<uint4*>(hrow + off) = make_uint4(h[4 * e], h[4 * e + 1], h[4 * e + 2], h[4 * e + 3]);
            *reinterpret_cast<uint4*>(lrow + off) = make_uint4(l[4 * e], l[4 * e + 1], l[4 * e + 2], l[4 * e + 3]);
          }
        }
      }
#endif
      fence_proxy_async();                // generic-proxy writes -> the MMA's async reads
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_remote(ready_l + 8u * s); else mbar_arrive(&ready[s]);
      }
    }
  } else if (warp < CB0) {
    // ------------------------------------------------------------ A converters
    // thread = TMEM lane = row r of the M tile = channel `lane` of chunk q
    const int q = warp & 3;
    const bool valid = (m0 / 32 + q) < chunks;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + Cf::A_COL;
    const int gc = m0 / 32 + q, tap = valid ? gc / cpt : 4;
    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
    const float scale = exp2i(sx);
    const int cofs = ((lane >> 2) << 4) + (lane & 3) * 4;     // logical chunk, word
    // coordinates of pixel p0 + lane (+32 per half), advanced by 32 pixels per ballot
    long long p = (long long)t0 * BK + lane;
    int img = (int)(p / ((long long)g.H * g.W));
    int rem = (int)(p - (long long)img * g.H * g.W);
    int oh = rem / g.W, ow = rem - (rem / g.W) * g.W;
    auto advance = [&](int by) {
      p += by;
      ow += by;
      while (ow >= g.W) {
        ow -= g.W;
        if (++oh == g.H) { oh = 0; ++img; }
      }
    };
    for (int i = 0; i < nst; ++i) {
      const int s = i % S;
      uint32_t vmask[BK / 32];
#pragma unroll
      for (int h = 0; h < BK / 32; ++h) {
        const bool ok = valid && p < g.npix && (unsigned)(oh + dy) < (unsigned)g.H &&
                        (unsigned)(ow + dx) < (unsigned)g.W;
        vmask[h] = __ballot_sync(0xffffffffu, ok);
        advance(32);
      }
      // full[s] also means the MMA that last read TMEM slot s has finished
      // (the producer waited for it before refilling the stage)
      mbar_wait(&full[s], (i / S) & 1);
      tc_fence_after();
      const char* box = smem + s * Cf::STAGE + q * BOX;
      const uint32_t a = lanebase + s * Cf::A_STAGE;
#if !defined(WGH_NOCONV) && !defined(WGH_NOACONV)
#pragma unroll
      for (int ps = 0; ps < BK / 16; ++ps) {         // 16 pixels = 8 columns per pass
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float v[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int kk = 16 * ps + 2 * k + e;
            v[e] = ((vmask[kk >> 5] >> (kk & 31)) & 1u)
                       ? *reinterpret_cast<const float*>(box + kk * 128 + (cofs ^ ((kk & 7) << 4)))
                       : 0.f;
          }
          split_f16x2_s(v[0], v[1], scale, hi[k], lo[k]);
        }
        tmem_st8u(a + 8 * ps, hi);
        tmem_st8u(a + BK / 2 + 8 * ps, lo);
      }
#endif
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_remote(ready_l + 8u * s); else mbar_arrive(&ready[s]);
      }
    }
  } else if (warp < DR0) {
    // ------------------------------------------------------------ B converters
    // four threads (c16 = lane >> 3, 16 channels each; one quarter-warp per
    // c16, so each 128-bit access phase hits 8 rows x distinct chunks) per
    // (pixel, 64-channel atom) row pair; BN = 128: warp wb takes atom wb & 1,
    // pixels [32 (wb >> 1), +32); BN = 64: atom 0, pixels [16 wb, +16)
    const int wb = warp - CB0, c16 = lane >> 3;
    const int at = BNL == 128 ? (wb & 1) : 0;
    constexpr int PPW = BNL == 128 ? 32 : 16;                // pixels per warp per stage
    const int pb = (BNL == 128 ? (wb >> 1) : wb) * PPW;
    const float scale = exp2i(sd);
    const bool do_bias = bias_part != nullptr && blockIdx.x == (PAIR ? rank : 0u);
    float bs[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) bs[k] = 0.f;
    for (int i = 0; i < nst; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      char* bt = smem + s * Cf::STAGE + Cf::A_BYTES;
      char* raw = bt + (2 * at + (c16 >> 1)) * BOX;      // this thread's 16 fp32 channels
      char* hrow = bt + 2 * at * BOX, *lrow = hrow + BOX;
#ifndef WGH_NOCONV
#pragma unroll
      for (int it = 0; it < PPW / 8; ++it) {
        const int pr = pb + 8 * it + (lane & 7);
        const int sw = pr & 7;
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
          if (do_bias) {
            bs[4 * u] += v[u].x; bs[4 * u + 1] += v[u].y;
            bs[4 * u + 2] += v[u].z; bs[4 * u + 3] += v[u].w;
          }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int off = pr * 128 + (((2 * c16 + e) ^ sw) << 4);
          *reinterpret_cast<uint4*>(hrow + off) = make_uint4(h[4 * e], h[4 * e + 1], h[4 * e + 2], h[4 * e + 3]);
          *reinterpret_cast<uint4*>(lrow + off) = make_uint4(l[4 * e], l[4 * e + 1], l[4 * e + 2], l[4 * e + 3]);
        }
      }
#endif
      fence_proxy_async();                // generic-proxy writes -> the MMA's async reads
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_remote(ready_l + 8u * s); else mbar_arrive(&ready[s]);
      }
    }
    if (do_bias) {
      // fixed-order reduction of the 16 per-thread partials of each channel
      const int bt = tid - CB0 * 32;
#pragma unroll
      for (int k = 0; k < 16; ++k) bias_scr[bt * 16 + k] = bs[k];
      named_sync(1, 128);
      if (bt < BNL) {
        const int a = bt / 64, cc = (bt % 64) / 16, k = bt % 16;
        float t = 0.f;
        for (int w = 0; w < 4; ++w) {
          if (BNL == 128 && (w & 1) != a) continue;
          for (int l8 = 0; l8 < 8; ++l8) t += bias_scr[(w * 32 + cc * 8 + l8) * 16 + k];
        }
        bias_part[(long long)blockIdx.z * g.Cout + nl0 + bt] = t;
      }
    }
  } else {
    // ------------------------------------------------------------ drain + epilogue
    const int q = warp & 3, hf = (warp - DR0) >> 2;
    constexpr int CW = BN / 2;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + hf * CW;
    const float unscale = exp2i(-sx) * exp2i(-sd);
    float acc[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) acc[j] = 0.f;
    const int nch = (nst + PCH - 1) / PCH;
    for (int c = 0; c < nch; ++c) {
      const int b = c & 1;
      mbar_wait(&hfull[b], (c >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < CW; j += 8) {
        uint32_t r[8];
        tmem_ld8(lanebase + b * BN + j, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[j + t] += __uint_as_float(r[t]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_remote(hfree_l + 8u * b); else mbar_arrive(&hfree[b]);
      }
    }
    const int r = m0 + q * 32 + lane;
    if (r < nrows) {
      float* o = part + (long long)blockIdx.z * g.slab + r;
#pragma unroll
      for (int j = 0; j < CW; ++j) o[(long long)(n0 + hf * CW + j) * nrows] = acc[j] * unscale;
    }
  }

  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    if (PAIR) tmem_free2(tmem, 512); else tmem_free(tmem, 512);
  }
}

// ------------------------------------------------------------------ host side

inline int bn_for(int cout) { return cout % 128 == 0 ? 128 : 64; }
#ifndef WGH_PAIR
#define WGH_PAIR 1
#endif
#ifndef WGH_PAIR_PAD
#define WGH_PAIR_PAD 9
#endif
// pairs for 128-wide N tiles whose M tiles pair up (Cin = 256, 512), and for
// odd counts of at least WGH_PAIR_PAD tiles with a padding tile (A rows
// zero, nothing stored): with the alternating converter groups of pairs,
// Cin = 128 (9 -> 10 tiles) gains 2-3 % (conv2_2 0.418 -> 0.411 ms, conv3_1
// 0.217 -> 0.210), Cin = 64 (5 -> 6) loses 4 %
inline bool paired(int cin, int cout) {
  const int mt = cdiv(9 * cin, 128);
  return WGH_PAIR && bn_for(cout) == 128 && mt >= 2 &&
         (mt % 2 == 0 || (WGH_PAIR_PAD > 0 && mt >= WGH_PAIR_PAD));
}

inline void plan(int n, int H, int W, int cin, int cout, Geo& g, int& mt, int& nt, int& splits) {
  g.Cin = cin; g.Cout = cout; g.H = H; g.W = W;
  g.npix = (long long)n * H * W;
  g.tiles = (int)cdivll(g.npix, BK);
  g.slab = (long long)cout * 9 * cin;
  mt = cdiv(9 * cin, 128);
  if (paired(cin, cout)) mt += mt & 1;           // whole pairs (a padding tile computes zeros)
  nt = cout / bn_for(cout);
  const int tiles_mn = mt * nt;
  int want = num_sms() / tiles_mn;
  if (want < 1) want = 1;
  if (want > g.tiles) want = g.tiles;
  g.tps = cdiv(g.tiles, want);
  splits = cdiv(g.tiles, g.tps);
}

// [pixels][C] fp32, box = 32 channels x 64 pixels, 128-B swizzle
inline bool encode_rows(CUtensorMap* m, const float* p, long long npix, int C) {
  const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)npix};
  const cuuint64_t strides[1] = {(cuuint64_t)C * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)BK};
  const cuuint32_t es[2] = {1, 1};
  return encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p), dims,
                      strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool PAIR, bool SSA>
bpx_status_t launch(const CUtensorMap& tx, const CUtensorMap& tdz, const Geo& g, int mt,
                    int nt, int splits, float* part, float* bias_part, cudaStream_t st) {
  using Cf = Cfg<BN, PAIR>;
  auto kern = wgh_kernel<BN, PAIR, SSA>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    attr = true;
  }
  if (!PAIR) {
    kern<<<dim3(mt, nt, splits), NT, Cf::SMEM, st>>>(tx, tdz, g, part, bias_part);
    return launch_status();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(mt, nt, splits);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = Cf::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, tx, tdz, g, part, bias_part) != cudaSuccess)
    return BPX_ERR_LAUNCH;
  return launch_status();
}

}  // namespace wgh

// ============================================================ entry points

bool wgh_conv_ok(int cin, int cout) { return cin % 32 == 0 && cout % 64 == 0; }

// workspace: amax words (x, dz), then split partials [splits][slab] + [splits][cout]
size_t wgh_conv_ws(int n, int h, int w, int cin, int cout) {
  if (!wgh_conv_ok(cin, cout)) return 0;
  wgh::Geo g;
  int mt, nt, splits;
  wgh::plan(n, h, w, cin, cout, g, mt, nt, splits);
  size_t parts = splits <= 1 ? 0 : ((size_t)splits * (size_t)g.slab + (size_t)splits * cout);
  return 16 + parts * sizeof(float);
}

bpx_status_t wgh_conv_wgrad(const float* x, const float* dz, const uint32_t* amax_x,
                            const uint32_t* amax_dz, float* dw, float* dbias, int n, int h,
                            int w_, int cin, int cout, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  if (!wgh_conv_ok(cin, cout) || !aligned16(x) || !aligned16(dz) || !aligned16(dw))
    return BPX_ERR_INVALID_ARGUMENT;
  if (dbias && !aligned16(dbias)) return BPX_ERR_INVALID_ARGUMENT;
  if (ws_bytes < wgh_conv_ws(n, h, w_, cin, cout) || !aligned16(ws)) return BPX_ERR_WORKSPACE;
  const size_t slab = (size_t)cout * 9 * cin;
  if (n == 0) {
    cudaMemsetAsync(dw, 0, sizeof(float) * slab, st);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * cout, st);
    return launch_status(0);
  }
  wgh::Geo g;
  int mt, nt, splits;
  wgh::plan(n, h, w_, cin, cout, g, mt, nt, splits);
  uint32_t* words = static_cast<uint32_t*>(ws);
  int k = 0;
  if (!amax_x) { absmax(x, (size_t)g.npix * cin, words, st); amax_x = words; ++k; }
  if (!amax_dz) { absmax(dz, (size_t)g.npix * cout, words + 1, st); amax_dz = words + 1; ++k; }
  count_launches(k);
  g.amax_x = amax_x;
  g.amax_dz = amax_dz;
  CUtensorMap tx, tdz;
  if (!wgh::encode_rows(&tx, x, g.npix, cin) || !wgh::encode_rows(&tdz, dz, g.npix, cout))
    return BPX_ERR_INVALID_ARGUMENT;
  float* scratch = reinterpret_cast<float*>(static_cast<char*>(ws) + 16);
  float* part = splits == 1 ? dw : scratch;
  float* bpart = !dbias ? nullptr : (splits == 1 ? dbias : scratch + (size_t)splits * slab);
  const bool ssa = WGH_SSA && cin % 64 == 0;
  bpx_status_t s;
  if (wgh::bn_for(cout) == 128 && wgh::paired(cin, cout))
    s = ssa ? wgh::launch<128, true, true>(tx, tdz, g, mt, nt, splits, part, bpart, st)
            : wgh::launch<128, true, false>(tx, tdz, g, mt, nt, splits, part, bpart, st);
  else if (wgh::bn_for(cout) == 128)
    s = ssa ? wgh::launch<128, false, true>(tx, tdz, g, mt, nt, splits, part, bpart, st)
            : wgh::launch<128, false, false>(tx, tdz, g, mt, nt, splits, part, bpart, st);
  else
    s = ssa ? wgh::launch<64, false, true>(tx, tdz, g, mt, nt, splits, part, bpart, st)
            : wgh::launch<64, false, false>(tx, tdz, g, mt, nt, splits, part, bpart, st);
  if (s != BPX_OK || splits == 1) return s;
  return split_reduce_wb(part, slab, dw, bpart, (size_t)cout, dbias, splits, st);
}

}  // namespace bpx
