// tcgen05 forward / data-gradient engine for the 3x3/pad-1 convolutions,
// fed by TMA, persistent over output tiles:
//
//   fwd   : y[p][co]  = act(b[co] + sum_{tap,ci} x[p + s_tap][ci]  * w[co][tap][ci])
//   dgrad : dx[q][ci] = mask(q) * sum_{tap,co} dz[q - s_tap][co] * w[co][tap][ci]
//   s_tap = dy*W + dx  (flattened-pixel shift of the tap)
//
// M = 128 output pixels per tile, N = output channels, K = (channel chunk,
// tap) stages of 64 channels.  Per channel chunk the CTA loads ONE halo of
// the activations by TMA and all nine taps read their shifted 128-row window
// out of it, so activation traffic is the halo/tile ratio instead of 9x the
// tile:
//   * 2-D tiles (W, H divisible by a TW x TH = 128 block, e.g. 32 x 4 at
//     224x224): the halo is one 4-D box (TW+2) x (TH+2) x 32 channels per
//     32-channel half whose out-of-bounds rows TMA zero-fills -- the conv's
//     padding for free;
//   * otherwise 128 consecutive flattened pixels: the halo is the flattened
//     rows [m0 - W - 1, m0 + 128 + W + 1), and rows whose source pixel wraps
//     across an image row/edge are zeroed by the A converters from a 9-bit
//     per-pixel tap mask computed once per tile.
//
// fp32 accuracy by fp16x3 (tc_ptx.cuh): the activations are scaled by a
// power of two from their absolute maximum (one word written by a reduction
// before the launch) and split by the A converters into fp16 hi/lo pairs
// stored in TMEM (TS form); the weights come pre-split by bpx_conv3x3_wsplit
// (fp16 hi and lo in the layout of w, one power-of-two scale per weight
// span) and are loaded by TMA:
//   fwd   B(co, k) = w16[co][tap][ci]: K-major, 128-B swizzle
//   dgrad B(ci, k) = w16[co][tap][ci]: MN-major, 128-B swizzle, one box per
//                    64 input channels (w viewed [Cout][9][Cin]).
// Each k-step (16 channels) issues a_lo*b_hi + a_hi*b_lo + a_hi*b_hi as
// kind::f16 MMAs: twice the tf32 rate and, at 64-wide N tiles, half the
// TMEM A reads per product.  Partial sums accumulate in 256-K chunks in
// ping-pong TMEM and are promoted into round-to-nearest fp32 registers by
// the drain warps (the tensor core's fp32 accumulation truncates), which
// undo both scales (exact powers of two) before the epilogue.  The kernel is
// persistent: the stage ring and the accumulator ping-pong run straight
// across tiles, so a tile's epilogue (bias + ReLU or ReLU mask, stores)
// overlaps the next tile's main loop.
//
// CTA: 2 + 8 + BN/16 warps.  warp 0 TMA, warp 1 MMA + TMEM owner, 2-9 A
// converters (two per TMEM lane quadrant, one 32-channel half each), then
// the drain + epilogue warps.
#include "tma_host.h"
#include "tc_ptx.cuh"
#include "tc_api.h"

// ALT: the two converter warps of a TMEM lane quadrant take alternate
// stages (all 64 channels each) instead of 32 channels of every stage, so
// one warp's copy of stage i + 1 overlaps the other's tcgen05.wait::st and
// barrier hand-off of stage i (B200 same-box A/B: VGG fwd layers 2.90 ->
// 2.75 ms, dgrad 3.04 -> 2.88 ms, conv1_2 fwd 0.508 -> 0.481 ms)
#ifndef FDT_ALT
#define FDT_ALT 1
#endif
// (a halo split by one converter group alone, overlapping the other group's
// last tap of the previous chunk, measured neutral: not kept)
// 12 converter warps for 64-wide tiles (three stage groups) measured 8-15 %
// slower: the 96-register cap of 18 warps spills
#ifndef FDT_NCONV64
#define FDT_NCONV64 8
#endif

namespace bpx {
namespace fdt {
using namespace tcx;

constexpr int TMA_WARP = 0, MMA_WARP = 1, CV0 = 2;   // A converters from warp 2
constexpr int KS = 64;                               // channels per stage
constexpr int NCH = 2;                               // 32-channel halo halves per stage
// promotion chunk: K = 256 per RN fp32 promotion of the truncating tensor
// core accumulator.  fp64 error (tools/fdt_prec.py, VGG shapes): K = 128
// 4.5e-7, 256 8.6e-7, 512 1.7e-6 against the 2e-6 gate; 256 is 2-5 % faster
// than 128 (conv1_2 fwd 0.478 -> 0.456 ms, B200 same-box) at 2.3x margin
#ifndef FDT_PCHK
#define FDT_PCHK 256
#endif
constexpr int PCH = FDT_PCHK / KS;                   // stages per promotion chunk

// BN output channels per tile, S stages; PAIR: a cluster of two CTAs runs
// M tiles 2m, 2m+1 as one M = 256 MMA (cta_group::2), each CTA holding its
// own A in TMEM and HALF of the B tile (BN/2 channels) in shared memory, so
// the weights cross L2 once per 256 output pixels instead of once per 128.
template <int BN, int S_, bool PAIR = false>
struct Cfg {
  static_assert(BN == 128 || BN == 64, "tile");
  static constexpr int S = S_;
  // converter warps: two per TMEM lane quadrant (FDT_NCONV64 for 64-wide tiles)
  static constexpr int NCONV = (BN == 64 && FDT_ALT) ? FDT_NCONV64 : 8;
  static constexpr int NGRP = NCONV / 4;                  // stage groups (ALT)
  static constexpr int NDRAIN = BN / 16;                  // 64 accumulator columns per thread
  static constexpr int DR0 = CV0 + NCONV;
  static constexpr int NTHREADS = 32 * (2 + NCONV + NDRAIN);
  static constexpr int BNL = PAIR ? BN / 2 : BN;          // B channels held by this CTA
  static constexpr int B_BYTES = BNL * KS * 2;            // one fp16 tile (hi or lo)
  static constexpr int STAGE = 2 * B_BYTES;               // B hi | B lo
  static constexpr int A_COL = 2 * BN;                    // accumulators: 2 x BN columns
  static constexpr int A_STAGE = KS;                      // TMEM columns per stage: hi | lo
  static_assert(A_COL + S * A_STAGE <= 512, "TMEM budget");
  // dynamic smem = 1024 (align) + B stages (S, or the nine resident tiles)
  // + 2 halo slots + 512 (barriers)
  static int smem(int halo_bytes, bool rb) {
    return 1024 + (rb ? 9 : S) * STAGE + 2 * halo_bytes + 512;
  }
};

struct Geo {
  int H, W, C;               // C = gathered channels (Cin fwd, Cout dgrad)
  int N;                     // output channels
  int npix, mt, nt, tiles;
  int tw, th;                // 2-D tile (tw * th <= 128) or 0 = flattened tiles
  int trows;                 // output pixels per tile: tw * th, or 128
  int hbox, nhbox;           // rows per halo TMA box, boxes per 32-channel halo
  int half_bytes;            // smem stride of one 32-channel halo (1 KB aligned)
  int halo_bytes;            // one halo slot (NCH halves)
  int halo_tx;               // bytes TMA delivers per halo slot
  int halo_rows;             // halo pixels (rows) per 32-channel half
  int ksplit, units;         // K parts per tile and work units = tiles (pairs) * ksplit
  float* part;               // ksplit > 1: partial sums [ksplit][npix][N]
  const uint32_t* amax_a;    // max |A| bits (activations / output gradient)
  const uint32_t* amax_w;    // max |w| bits of the weights' span
};

// FDT_PROF builds (tools/fdt_prof.py): per-role cycle counters of warp 0 of
// each role, summed over CTAs into a device buffer (bpx_fdt_prof).
#ifdef FDT_PROF
__device__ unsigned long long g_prof[16];
#define PROF_DECL long long _pt = 0
#define PROF_START() (_pt = clock64())
#define PROF_ADD(slot, first) do { if ((first) && (threadIdx.x & 31) == 0) \
    atomicAdd(&g_prof[slot], (unsigned long long)(clock64() - _pt)); } while (0)
#else
#define PROF_DECL
#define PROF_START()
#define PROF_ADD(slot, first)
#endif

// Epilogues return the max |v| bits of what they stored: the drain reduces
// them into *amax (the output's fp16x3 scale word for its consumers).
__device__ __forceinline__ uint32_t absbits(float v) { return __float_as_uint(v) & 0x7fffffffu; }

struct EBiasAct {
  float* out; const float* bias; int relu; uint32_t* amax;
  __device__ uint32_t operator()(long long m, int n0, int N, const float (&v)[8]) const {
    float* o = out + m * N + n0;
    float r[8];
    uint32_t mx = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float t = v[j] + (bias ? __ldg(bias + n0 + j) : 0.f);
      r[j] = relu ? fmaxf(t, 0.f) : t;
      mx = max(mx, absbits(r[j]));
    }
    *reinterpret_cast<float4*>(o) = make_float4(r[0], r[1], r[2], r[3]);
    *reinterpret_cast<float4*>(o + 4) = make_float4(r[4], r[5], r[6], r[7]);
    return mx;
  }
};
struct EMask {
  float* out; const float* mask; uint32_t* amax;
  __device__ uint32_t operator()(long long m, int n0, int N, const float (&v)[8]) const {
    float* o = out + m * N + n0;
    float4 a = make_float4(v[0], v[1], v[2], v[3]);
    float4 b = make_float4(v[4], v[5], v[6], v[7]);
    if (mask) {
      const float* mk = mask + m * N + n0;
      const float4 p = __ldg(reinterpret_cast<const float4*>(mk));
      const float4 q = __ldg(reinterpret_cast<const float4*>(mk + 4));
      a.x = p.x > 0.f ? a.x : 0.f; a.y = p.y > 0.f ? a.y : 0.f;
      a.z = p.z > 0.f ? a.z : 0.f; a.w = p.w > 0.f ? a.w : 0.f;
      b.x = q.x > 0.f ? b.x : 0.f; b.y = q.y > 0.f ? b.y : 0.f;
      b.z = q.z > 0.f ? b.z : 0.f; b.w = q.w > 0.f ? b.w : 0.f;
    }
    *reinterpret_cast<float4*>(o) = a;
    *reinterpret_cast<float4*>(o + 4) = b;
    return max(max(max(absbits(a.x), absbits(a.y)), max(absbits(a.z), absbits(a.w))),
               max(max(absbits(b.x), absbits(b.y)), max(absbits(b.z), absbits(b.w))));
  }
};
__device__ __forceinline__ void amax_commit(uint32_t* amax, uint32_t mx) {
  if (!amax) return;
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(amax, mx);
}

// Output-tile geometry shared by the producer, converters and epilogue.
struct Tile {
  int m0;                    // flattened tiles: first pixel
  int img, oh0, ow0;         // 2-D tiles: image and block origin
};
__device__ __forceinline__ Tile tile_of(const Geo& g, int mi) {
  Tile t{};
  if (g.tw) {
    const int bw = g.W / g.tw, per = bw * (g.H / g.th);
    t.img = mi / per;
    const int rem = mi - t.img * per;
    t.oh0 = (rem / bw) * g.th;
    t.ow0 = (rem % bw) * g.tw;
  } else {
    t.m0 = mi * 128;
  }
  return t;
}

// Work unit u of this CTA -> its M tile, N tile and K part; pad: a pair's
// second tile past the last M tile (it recomputes the last tile, stores nothing)
template <bool PAIR>
__device__ __forceinline__ void unit_tile(const Geo& g, int u, uint32_t rank, int& mi, int& nti,
                                          int& kh, bool& pad) {
  const int t = u / g.ksplit;
  kh = u % g.ksplit;
  nti = t % g.nt;
  mi = PAIR ? 2 * (t / g.nt) + (int)rank : t / g.nt;
  pad = mi >= g.mt;
  if (pad) mi = g.mt - 1;
}

// MT (dgrad with the mask, no split-K, where the tile fits): the ReLU mask
// tile of the unit (the layer input, 128 pixels x BN channels) comes by
// TMA into shared memory, issued mid-unit, so the epilogue reads it there
// instead of issuing 16 dependent global loads per thread.
// RB (one 64-channel chunk and one N tile per launch, e.g. conv1_2): the nine
// B tiles are loaded once and stay resident; the B ring disappears.
template <int BN, int S_, bool DG, bool PAIR, class EPI, bool MT = false, bool RB = false>
__global__ void __launch_bounds__(Cfg<BN, S_, PAIR>::NTHREADS, 1)
fdt_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
           const __grid_constant__ CUtensorMap tbl, const __grid_constant__ CUtensorMap tm,
           Geo g, EPI epi) {
  using Cf = Cfg<BN, S_, PAIR>;
  constexpr int BNL = Cf::BNL;
  constexpr int S = Cf::S;
  constexpr int NCONV = Cf::NCONV, NDRAIN = Cf::NDRAIN, DR0 = Cf::DR0;
  extern __shared__ char smem_raw[];
  // offset from smem_raw (not a uintptr_t round trip) keeps the shared address space: LDS/STS, not generic LD/ST
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int NBS = RB ? 9 : S;                             // B stages in smem
  char* halo = smem + NBS * Cf::STAGE;                        // 2 slots
  uint64_t* bfull = reinterpret_cast<uint64_t*>(halo + 2 * g.halo_bytes);
  uint64_t* aready = bfull + NBS;
  uint64_t* empty = aready + S;
  uint64_t* hfull = empty + S;       // halo slot loaded
  uint64_t* hempty = hfull + 2;      // halo slot consumed by all nine taps
  uint64_t* accfull = hempty + 2;
  uint64_t* accfree = accfull + 2;
  uint64_t* mfull = accfree + 2;     // MT: mask tile landed
  uint64_t* mfree = mfull + 1;       // MT: mask tile read by the drain
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mfree + 1);
  char* mtile = halo + 2 * g.halo_bytes + 1024;               // MT: BN / 32 x 16 KB, 1 KB aligned

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cpu = g.C / KS / g.ksplit;        // channel chunks per work unit
  const int nk = 9 * cpu;                     // stages per work unit
  // pairs: units are walked per cluster; the leader (rank 0) issues the MMAs
  // and owns aready / accfree, which both CTAs' converters / drains arrive on
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int u0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ustep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (tid == 0) {
    for (int s = 0; s < NBS; ++s) mbar_init(&bfull[s], 1);
    for (int s = 0; s < S; ++s) {
      // one arrival per converter warp that wrote the stage
      mbar_init(&aready[s], (PAIR ? 2 * NCONV : NCONV) / (FDT_ALT ? Cf::NGRP : 1));
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hempty[b], NCONV);
      mbar_init(&accfull[b], 1);
      mbar_init(&accfree[b], PAIR ? 2 * NDRAIN : NDRAIN);  // one arrival per drain warp
    }
    mbar_init(mfull, 1);
    mbar_init(mfree, NDRAIN);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    if (PAIR) tmem_alloc2(tmem_slot, 512); else tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t aready_l = PAIR ? mapa_rank(aready, 0) : 0u;
  const uint32_t accfree_l = PAIR ? mapa_rank(accfree, 0) : 0u;
  const int sa = f16_scale_exp(*g.amax_a), sw = f16_scale_exp(*g.amax_w);

  if (warp == TMA_WARP) {
    // ------------------------------------------------------------ TMA producers
    // lane 1 streams the halos (each waits only for its slot), lane 0 the B
    // tiles and mask tiles: one thread doing both issued a halo only after
    // the previous chunk's nine B tiles, each waiting for an MMA slot
    if (lane == 1) {
      tma_prefetch_desc(&ta);
      int hc = 0;
      for (int u = u0; u < g.units; u += ustep) {
        int mi, nti, kh;
        bool pad;
        unit_tile<PAIR>(g, u, rank, mi, nti, kh, pad);
        const Tile T = tile_of(g, mi);
        for (int cc = kh * cpu; cc < (kh + 1) * cpu; ++cc, ++hc) {
          const int hs = hc & 1;
          if (hc >= 2) mbar_wait(&hempty[hs], ((hc >> 1) - 1) & 1);
          mbar_expect_tx(&hfull[hs], (uint32_t)g.halo_tx);
          char* hb = halo + hs * g.halo_bytes;
#pragma unroll
          for (int c2 = 0; c2 < NCH; ++c2) {
            const int c0 = cc * KS + c2 * 32;
            if (g.tw) {
              tma_load_4d(hb + c2 * g.half_bytes, &ta, c0, T.ow0 - 1, T.oh0 - 1, T.img,
                          &hfull[hs]);
            } else {
              for (int j = 0; j < g.nhbox; ++j)
                tma_load_2d(hb + c2 * g.half_bytes + j * g.hbox * 128, &ta, c0,
                            T.m0 - g.W - 1 + j * g.hbox, &hfull[hs]);
            }
          }
        }
      }
    } else if (lane == 0) {
      tma_prefetch_desc(&ta);
      tma_prefetch_desc(&tb);
      tma_prefetch_desc(&tbl);
      if (MT) tma_prefetch_desc(&tm);
      PROF_DECL;
      int i = 0, hc = 0, mu = 0;
      for (int u = u0; u < g.units; u += ustep) {
        int mi, nti, kh;
        bool pad;
        unit_tile<PAIR>(g, u, rank, mi, nti, kh, pad);
        const Tile T = tile_of(g, mi);
        const int n0 = nti * BN + (int)rank * BNL;          // this CTA's B channels
        for (int cc = kh * cpu; cc < (kh + 1) * cpu; ++cc, ++hc) {
          for (int tap = 0; tap < 9; ++tap, ++i) {
            const int s = RB ? tap : i % S;
            if (!RB || i < 9) {      // resident B: the first unit's nine loads only
            PROF_START();
            if (!RB && i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
            PROF_ADD(12, true);
            char* st = smem + s * Cf::STAGE;
            mbar_expect_tx(&bfull[s], 2 * Cf::B_BYTES);
            if (DG && BNL == 32) {   // a pair's half: 32 ci x KS co rows, 64-B swizzle
              tma_load_3d(st, &tb, n0, tap, cc * KS, &bfull[s]);
              tma_load_3d(st + Cf::B_BYTES, &tbl, n0, tap, cc * KS, &bfull[s]);
            } else if (DG) { // BNL/64 boxes of 64 ci x KS co rows (MN-major)
#pragma unroll
              for (int j = 0; j < BNL / 64; ++j) {
                tma_load_3d(st + j * KS * 128, &tb, n0 + 64 * j, tap, cc * KS, &bfull[s]);
                tma_load_3d(st + Cf::B_BYTES + j * KS * 128, &tbl, n0 + 64 * j, tap, cc * KS,
                            &bfull[s]);
              }
            } else {         // one box of 64 k x BNL rows (K-major)
              const int k0 = tap * g.C + cc * KS;
              tma_load_2d(st, &tb, k0, n0, &bfull[s]);
              tma_load_2d(st + Cf::B_BYTES, &tbl, k0, n0, &bfull[s]);
            }
            }
            if (MT && tap == 4 && cc == (kh + 1) * cpu - 1) {    // the unit's mask tile
              if (mu >= 1) mbar_wait(mfree, (mu - 1) & 1);
              mbar_expect_tx(mfull, (uint32_t)(BN * g.trows * 4));
#pragma unroll
              for (int h = 0; h < BN / 32; ++h) {     // all BN channels of this CTA's rows
                if (g.tw)
                  tma_load_4d(mtile + h * 16384, &tm, nti * BN + 32 * h, T.ow0, T.oh0, T.img,
                              mfull);
                else
                  tma_load_2d(mtile + h * 16384, &tm, nti * BN + 32 * h, T.m0, mfull);
              }
              ++mu;
            }
          }
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    // (the whole warp runs the loop; elect.sync picks the issuing lane)
    // M=128, N=BN, f16 x f16 -> f32, A from TMEM; B K-major (fwd) / MN-major (dgrad)
    // (pairs: M = 256 across the two CTAs, leader only)
    constexpr uint32_t idesc = (PAIR ? ((make_idesc_f16(BN) & ~(0x1Fu << 24)) | (16u << 24))
                                     : make_idesc_f16(BN)) | (DG ? (1u << 16) : 0u);
    int i = 0, c = 0;
    PROF_DECL;
#ifdef FDT_PROF
    const long long _t0 = clock64();
#endif
    for (int u = u0; u < g.units && (!PAIR || rank == 0); u += ustep) {
      for (int kb = 0; kb < nk; ++kb, ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        const int b = c & 1;
        if (kb % PCH == 0 && c >= 2) {
          PROF_START();
          if (PAIR) mbar_wait_cluster(&accfree[b], ((c >> 1) - 1) & 1);
          else mbar_wait(&accfree[b], ((c >> 1) - 1) & 1);
          PROF_ADD(1, true);
          tc_fence_after();
        }
        PROF_START();
        // aready[s] also covers the stage's B tiles: the converters wait for
        // them before arriving, so the issuer makes one barrier check per
        // stage (its checks come straight out of MMA issue time)
        if (PAIR) mbar_wait_cluster(&aready[s], ph); else mbar_wait(&aready[s], ph);
        PROF_ADD(2, true);
        tc_fence_after();
        const uint32_t d = tmem + b * BN;
        const uint32_t ah = tmem + Cf::A_COL + s * Cf::A_STAGE, al = ah + KS / 2;
        const uint32_t bh = smem_u32(smem + (RB ? kb : s) * Cf::STAGE);
        // dgrad B is MN-major: 64-channel atoms with the 128-B swizzle, or a
        // pair's 32-channel halves with the 64-B swizzle (8 k-rows = 512 B)
        const uint64_t dbh0 = !DG ? make_desc_sw128(bh, 16, 1024)
                              : BNL == 32 ? make_desc_sw64(bh, KS * 64, 512)
                                          : make_desc_sw128(bh, KS * 128, 1024);
        const uint64_t dbl0 = dbh0 + (Cf::B_BYTES >> 4);
#pragma unroll
        for (int ks = 0; ks < KS / 16; ++ks) {
          // descriptor start address is (addr >> 4) in bits [0,14): dgrad
          // steps 16 k-rows (2 KB), fwd 16 fp16 of the 128-B K row (32 B)
          const uint32_t off = DG ? ks * (BNL == 32 ? 1024 : 2048) : ks * 32;
          const uint64_t dbh = dbh0 + (off >> 4), dbl = dbl0 + (off >> 4);
          const uint32_t acc = (kb % PCH != 0 || ks > 0) ? 1u : 0u;
#ifndef FDT_NOMMA
          if (PAIR) {
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
        if (PAIR) tc_commit2_elect(&empty[s]); else tc_commit_elect(&empty[s]);
        if (kb % PCH == PCH - 1 || kb == nk - 1) {
          if (PAIR) tc_commit2_elect(&accfull[b]); else tc_commit_elect(&accfull[b]);
          ++c;
        }
      }
    }
#ifdef FDT_PROF
    if (lane == 0 && (!PAIR || rank == 0)) {
      atomicAdd(&g_prof[0], (unsigned long long)(clock64() - _t0));
      atomicAdd(&g_prof[4], (unsigned long long)i);
    }
#endif
  } else if (warp < DR0) {
    // ------------------------------------------------------------ A converters
    // thread = TMEM lane = output pixel r of the tile; warp half c2 converts
    // channels [32 c2, 32 c2 + 32) of each stage, i.e. TMEM columns
    // [16 c2, +16) of the hi half and of the lo half
    const int q = warp & 3, c2 = (warp - CV0) >> 2, r = q * 32 + lane;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + Cf::A_COL;
    const float scale = exp2i(sa);
    const int hw = g.H * g.W;
    const int rr = g.tw ? r / g.tw : 0, rc = g.tw ? r % g.tw : 0;
    int i = 0, hc = 0;
    PROF_DECL;
    const bool pw = warp == CV0;
    for (int u = u0; u < g.units; u += ustep) {
      int mi, nti, kh;
      bool pad;
      unit_tile<PAIR>(g, u, rank, mi, nti, kh, pad);
      // bit tap: source pixel inside the image (2-D tiles: TMA zero-fills
      // the border; rows past tw * th read nothing)
      uint32_t tmask = r < g.trows ? 0x1ffu : 0u;
      if (!g.tw) {
        const int p = mi * 128 + r;
        tmask = 0;
        if (p < g.npix) {
          const int img = p / hw, rem = p - img * hw;
          const int oh = rem / g.W, ow = rem - oh * g.W;
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const int dy = tap / 3 - 1, dx = tap % 3 - 1;
            const int ih = DG ? oh - dy : oh + dy, iw = DG ? ow - dx : ow + dx;
            if ((unsigned)ih < (unsigned)g.H && (unsigned)iw < (unsigned)g.W) tmask |= 1u << tap;
          }
        }
      }
      for (int cc = 0; cc < g.C / KS / g.ksplit; ++cc, ++hc) {
        const int hs = hc & 1;
        PROF_START();
        mbar_wait(&hfull[hs], (hc >> 1) & 1);
        PROF_ADD(6, pw);
        PROF_START();
        char* hb = halo + hs * g.halo_bytes;
        // split the halo ONCE for all nine taps, in place: the fp32 rows of
        // channels [0, 32) and [32, 64) of a halo pixel become its fp16 hi
        // row (64 channels, where the first half was) and lo row (where the
        // second was), same 128-B swizzle.  Four threads (one quarter-warp
        // each, 16 channels) per row pair; a warp reads its 8 row pairs
        // before it overwrites them.
#ifndef FDT_NOCONV
        {
          const int cv = warp - CV0, c16 = lane >> 3;
          char* src = hb + (c16 >> 1) * g.half_bytes;
          for (int base = cv * 8; base < g.halo_rows; base += NCONV * 8) {   // warp-uniform
            const int pr = base + (lane & 7), sw = pr & 7;
            float4 v[4];
#pragma unroll
            for (int uu = 0; uu < 4; ++uu)
              v[uu] = *reinterpret_cast<const float4*>(src + pr * 128 +
                                                       (((4 * (c16 & 1) + uu) ^ sw) << 4));
            __syncwarp();
            uint32_t h[8], l[8];
#pragma unroll
            for (int uu = 0; uu < 4; ++uu) {
              split_f16x2_s(v[uu].x, v[uu].y, scale, h[2 * uu], l[2 * uu]);
              split_f16x2_s(v[uu].z, v[uu].w, scale, h[2 * uu + 1], l[2 * uu + 1]);
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int off = pr * 128 + (((2 * c16 + e) ^ sw) << 4);
              *reinterpret_cast<uint4*>(hb + off) =
                  make_uint4(h[4 * e], h[4 * e + 1], h[4 * e + 2], h[4 * e + 3]);
              *reinterpret_cast<uint4*>(hb + g.half_bytes + off) =
                  make_uint4(l[4 * e], l[4 * e + 1], l[4 * e + 2], l[4 * e + 3]);
            }
          }
          asm volatile("bar.sync 1, %0;" ::"n"(NCONV * 32) : "memory");
        }
#endif
        PROF_ADD(7, pw);
        for (int tap = 0; tap < 9; ++tap, ++i) {
          const int s = i % S;
          const int dy = DG ? 1 - tap / 3 : tap / 3 - 1, dx = DG ? 1 - tap % 3 : tap % 3 - 1;
          const int hr = g.tw ? (rr + 1 + dy) * (g.tw + 2) + rc + 1 + dx
                              : r + g.W + 1 + dy * g.W + dx;
          const bool ok = (tmask >> tap) & 1u;
#if FDT_ALT
          // the two warps of a lane quadrant take alternate stages, all 64
          // channels each: stage i + 1's copy overlaps stage i's
          if (i % Cf::NGRP != c2) continue;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int off = hr * 128 + (((4 * hh + k) ^ (hr & 7)) << 4);
              uint4 vh = make_uint4(0u, 0u, 0u, 0u), vl = vh;
              if (ok) {
                vh = *reinterpret_cast<const uint4*>(hb + off);
                vl = *reinterpret_cast<const uint4*>(hb + g.half_bytes + off);
              }
              hi[4 * k] = vh.x; hi[4 * k + 1] = vh.y; hi[4 * k + 2] = vh.z; hi[4 * k + 3] = vh.w;
              lo[4 * k] = vl.x; lo[4 * k + 1] = vl.y; lo[4 * k + 2] = vl.z; lo[4 * k + 3] = vl.w;
            }
            if (hh == 0) {
              PROF_START();
              if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);   // TMEM A slot free
              PROF_ADD(8, pw);
              tc_fence_after();
            }
            const uint32_t a = lanebase + s * Cf::A_STAGE + 16 * hh;
            tmem_st16u(a, hi);
            tmem_st16u(a + KS / 2, lo);
          }
          PROF_START();
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          PROF_ADD(10, pw);
          PROF_START();
          if (lane == 0) {
            if (RB) mbar_wait(&bfull[tap], 0u); else mbar_wait(&bfull[s], (i / S) & 1);
            if (PAIR) mbar_arrive_remote(aready_l + 8u * s); else mbar_arrive(&aready[s]);
          }
          __syncwarp();
          PROF_ADD(9, pw);
          continue;
#endif
          // this thread's 32 channels: fp16 chunks 4 c2 .. 4 c2 + 3 of the
          // hi row and of the lo row
          uint32_t hi[16], lo[16];
#ifdef FDT_NOCONV
#pragma unroll
          for (int k = 0; k < 16; ++k) hi[k] = lo[k] = 0u;
          if (false)
#endif
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int off = hr * 128 + (((4 * c2 + k) ^ (hr & 7)) << 4);
            uint4 vh = make_uint4(0u, 0u, 0u, 0u), vl = vh;
            if (ok) {
              vh = *reinterpret_cast<const uint4*>(hb + off);
              vl = *reinterpret_cast<const uint4*>(hb + g.half_bytes + off);
            }
            hi[4 * k] = vh.x; hi[4 * k + 1] = vh.y; hi[4 * k + 2] = vh.z; hi[4 * k + 3] = vh.w;
            lo[4 * k] = vl.x; lo[4 * k + 1] = vl.y; lo[4 * k + 2] = vl.z; lo[4 * k + 3] = vl.w;
          }
          PROF_START();
          if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);   // TMEM A slot free
          PROF_ADD(8, pw);
          tc_fence_after();
          const uint32_t a = lanebase + s * Cf::A_STAGE + 16 * c2;
          tmem_st16u(a, hi);
          tmem_st16u(a + KS / 2, lo);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          PROF_START();
          if (lane == 0) {
            // aready[s] implies the B tiles (resident: loaded once, phase 0)
            if (RB) mbar_wait(&bfull[tap], 0u); else mbar_wait(&bfull[s], (i / S) & 1);
            if (PAIR) mbar_arrive_remote(aready_l + 8u * s); else mbar_arrive(&aready[s]);
          }
          PROF_ADD(9, pw);
          __syncwarp();
        }
        fence_proxy_async();                 // our stores before the next TMA fill
        __syncwarp();
        if (lane == 0) mbar_arrive(&hempty[hs]);
      }
    }
  } else {
    // ------------------------------------------------------------ drain + epilogue
    const int q = warp & 3, hf = (warp - DR0) >> 2;
    constexpr int CW = BN * 4 / NDRAIN;                 // 64 columns per drain thread
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + hf * CW;
    const int nch = (nk + PCH - 1) / PCH;
    const int r = q * 32 + lane;
    const float unscale = exp2i(-sa) * exp2i(-sw);
    uint32_t mx = 0;
    int c = 0, mu_d = 0;
    PROF_DECL;
    const bool pw = warp == DR0;
    for (int u = u0; u < g.units; u += ustep) {
      int mi, nti, kh;
      bool pad;
      unit_tile<PAIR>(g, u, rank, mi, nti, kh, pad);
      float acc[CW];
#pragma unroll
      for (int j = 0; j < CW; ++j) acc[j] = 0.f;
      for (int k = 0; k < nch; ++k, ++c) {
        const int b = c & 1;
        PROF_START();
        mbar_wait(&accfull[b], (c >> 1) & 1);
        PROF_ADD(14, pw);
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < CW; j += 8) {
          uint32_t rr[8];
          tmem_ld8(lanebase + b * BN + j, rr);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 8; ++u) acc[j + u] += __uint_as_float(rr[u]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) mbar_arrive_remote(accfree_l + 8u * b); else mbar_arrive(&accfree[b]);
        }
      }
      PROF_START();
      const Tile T = tile_of(g, mi);
      const long long p = r >= g.trows ? (long long)g.npix
                          : g.tw ? ((long long)T.img * g.H + T.oh0 + r / g.tw) * g.W + T.ow0 +
                                       r % g.tw
                                 : (long long)T.m0 + r;
      const int n0 = nti * BN + hf * CW;
      if (MT) {
        // the mask from the staged tile: row r, 128-B swizzled rows per 32 channels
        mbar_wait(mfull, mu_d & 1);
        if (p < g.npix) {
          float* o = epi.out + p * g.N + n0;
#pragma unroll
          for (int j = 0; j < CW; j += 4) {
            const float4 mk = *reinterpret_cast<const float4*>(
                mtile + ((hf * CW + j) >> 5) * 16384 + r * 128 +
                ((((j & 31) >> 2) ^ (r & 7)) << 4));
            float4 v = make_float4(acc[j] * unscale, acc[j + 1] * unscale, acc[j + 2] * unscale,
                                   acc[j + 3] * unscale);
            v.x = mk.x > 0.f ? v.x : 0.f; v.y = mk.y > 0.f ? v.y : 0.f;
            v.z = mk.z > 0.f ? v.z : 0.f; v.w = mk.w > 0.f ? v.w : 0.f;
            *reinterpret_cast<float4*>(o + j) = v;
            mx = max(mx, max(max(absbits(v.x), absbits(v.y)), max(absbits(v.z), absbits(v.w))));
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(mfree);
        ++mu_d;
      } else if (p < g.npix && !pad) {
        if (g.ksplit > 1) {               // partial; fdt_finish applies the epilogue
          float* o = g.part + ((long long)kh * g.npix + p) * g.N + n0;
#pragma unroll
          for (int j = 0; j < CW; j += 4)
            *reinterpret_cast<float4*>(o + j) =
                make_float4(acc[j] * unscale, acc[j + 1] * unscale, acc[j + 2] * unscale,
                            acc[j + 3] * unscale);
        } else {
#pragma unroll
          for (int j = 0; j < CW; j += 8) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = acc[j + e] * unscale;
            mx = max(mx, epi(p, n0 + j, g.N, v));
          }
        }
      }
      PROF_ADD(15, pw);
    }
    if (g.ksplit == 1) amax_commit(epi.amax, mx);
  }

  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    if (PAIR) tmem_free2(tmem, 512); else tmem_free(tmem, 512);
  }
}

// ------------------------------------------------------------------ host side

// Split-K finish: out = epilogue(part[0] + part[1] + ...), fixed order.
template <class EPI>
__global__ void fdt_finish(const float* __restrict__ part, int ksplit, long long npix, int N,
                           EPI epi) {
  const long long groups = npix * (N / 8);
  const long long stride = (long long)gridDim.x * blockDim.x;
  // stride a multiple of N/8 (N a power of two <= 512): a thread keeps its
  // channel group and steps whole pixels -- no 64-bit div/mod per element
  const bool fixed = stride % (N / 8) == 0;
  const long long e0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int nf = (int)(e0 % (N / 8)) * 8;
  const long long pstep = stride / (N / 8);
  uint32_t mx = 0;
  long long pf = e0 / (N / 8);
  for (long long e = e0; e < groups; e += stride, pf += pstep) {
    const long long p = fixed ? pf : e / (N / 8);
    const int n0 = fixed ? nf : (int)(e % (N / 8)) * 8;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < ksplit; ++k) {
      const float4* src = reinterpret_cast<const float4*>(part + ((long long)k * npix + p) * N + n0);
      const float4 a = src[0], b = src[1];
      v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
      v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
    }
    mx = max(mx, epi(p, n0, N, v));
  }
  amax_commit(epi.amax, mx);
}

// Work units: output tiles, split along K (2, 4 or 8 ways) while the tiles
// alone would leave the persistent grid under two waves -- conv5 at 14x14
// (196 tiles on 148 SMs), or any layer at the small per-GPU batches of a
// wide burst plan; the parts' sums meet in fdt_finish.
inline int ksplit_for(long long tiles, int chunks, int slots) {
  int k = 1;
  while (k < 8 && tiles * k < 2LL * slots && chunks % (2 * k) == 0) k *= 2;
  return k;
}

// CTA pairs (cta_group::2) when there are two M tiles to pair (the 64-wide
// dgrad's 32-channel MN-major B halves take the 64-B swizzle)
#ifndef FDT_PAIR
#define FDT_PAIR 1
#endif
#ifndef FDT_PAIR64DG
#define FDT_PAIR64DG 1
#endif
// (64-wide dgrad pairs only where the nine B tiles also stay resident, i.e.
// Cin = Cout = 64: conv1_2 dgrad 0.521 -> 0.511 ms; conv2_1's dgrad, with two
// 64-channel chunks, measured 3 % slower paired -- B200 same-box A/B)
inline bool pair_for(int BN, bool dg, long long mt, int C = 0) {
  return FDT_PAIR && (!dg || BN == 128 || (FDT_PAIR64DG && C == 64)) && mt >= 2 &&
         num_sms() >= 2;
}

// work units of a launch: tiles (M tile pairs) x N tiles x K parts
inline void plan_units(long long mt, int nt, int chunks, bool pair, int& ksplit, int& units) {
  const long long mtu = pair ? (mt + 1) / 2 : mt;
  const int slots = pair ? num_sms() / 2 : num_sms();
  ksplit = ksplit_for(mtu * nt, chunks, slots);
  units = (int)(mtu * nt * ksplit);
}

inline bool encode(CUtensorMap* m, const void* p, CUtensorMapDataType dt, int rank,
                   const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                   CUtensorMapSwizzle sw) {
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return encode_tiled(m, dt, rank, const_cast<void*>(p), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D output tile tw x th that divides the image: tw * th = 128, widest
// first; else, for images 64 pixels wide or more (whose flattened halo,
// 128 + 2W + 2 rows, needs two TMA boxes and crowds the B stages out of
// smem), the tile with the most pixels <= 128 (at least 120, rows past
// tw * th idle), e.g. 25 x 5 at 100 x 100 (189 halo rows instead of 330).
inline void tile2d(int H, int W, int& tw, int& th) {
  tw = th = 0;
  for (int w = 32; w >= 16; w >>= 1)
    if (W % w == 0 && H % (128 / w) == 0) { tw = w; th = 128 / w; return; }
  if (128 + 2 * W + 2 <= 256) return;
  int best = 0;
  for (int w = 8; w <= 64; ++w) {
    if (W % w) continue;
    for (int h = 128 / w; h >= 2; --h)
      if (H % h == 0) {
        if (w * h > best) { best = w * h; tw = w; th = h; }
        break;
      }
  }
  if (best < 120) tw = th = 0;
}

// Workspace: [amax word of A (16 B)] [weights: hi | lo fp16 + amax word when
// the caller did not split them] [split-K partials].
inline size_t wsplit_bytes(long long nw) { return (size_t)(4 * nw + 16 + 15) / 16 * 16; }

inline const float* mask_of(const EBiasAct&) { return nullptr; }
inline const float* mask_of(const EMask& e) { return e.mask; }
#ifndef FDT_MT
#define FDT_MT 1
#endif
#ifndef FDT_RB
#define FDT_RB 1
#endif

template <int BN, int S, bool DG, bool PAIR, class EPI, bool MT, bool RB>
bpx_status_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tbl,
                    const CUtensorMap& tm, const Geo& g, int smem, EPI epi, cudaStream_t st) {
  using Cf = Cfg<BN, S, PAIR>;
  auto kern = fdt_kernel<BN, S, DG, PAIR, EPI, MT, RB>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  if (PAIR) {
    const int clusters = g.units < num_sms() / 2 ? g.units : num_sms() / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(Cf::NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, ta, tb, tbl, tm, g, epi) != cudaSuccess)
      return BPX_ERR_LAUNCH;
  } else {
    const int grid = g.units < num_sms() ? g.units : num_sms();
    kern<<<grid, Cf::NTHREADS, smem, st>>>(ta, tb, tbl, tm, g, epi);
  }
  return BPX_OK;
}

template <int BN, int S, bool DG, bool PAIR, class EPI>
bpx_status_t run(const float* a, const F16Weights& wt, float* part, const uint32_t* amax_a,
                 int n, int H, int W, int Cin, int Cout, EPI epi, cudaStream_t st) {
  using Cf = Cfg<BN, S, PAIR>;
  Geo g;
  g.H = H; g.W = W;
  g.C = DG ? Cout : Cin;
  g.N = DG ? Cin : Cout;
  if (g.C % KS || g.N % BN) return BPX_ERR_UNSUPPORTED;
  g.npix = n * H * W;
  tile2d(H, W, g.tw, g.th);
  g.trows = g.tw ? g.tw * g.th : 128;
  g.mt = g.tw ? n * (H / g.th) * (W / g.tw) : cdiv(g.npix, 128);
  g.nt = g.N / BN;
  g.tiles = g.mt * g.nt;
  plan_units(g.mt, g.nt, g.C / KS, PAIR, g.ksplit, g.units);
  g.part = part;
  g.amax_a = amax_a;
  g.amax_w = wt.amax;
  if (g.tw) {
    g.nhbox = 1;
    g.hbox = cdiv((g.tw + 2) * (g.th + 2), 8) * 8;
  } else {
    const int hrows = 128 + 2 * W + 2;
    g.nhbox = cdiv(hrows, 256);
    g.hbox = cdiv(cdiv(hrows, g.nhbox), 8) * 8;
  }
  g.half_bytes = g.nhbox * g.hbox * 128;
  g.halo_bytes = NCH * g.half_bytes;
  g.halo_tx = NCH * (g.tw ? (g.tw + 2) * (g.th + 2) * 128 : g.half_bytes);
  g.halo_rows = g.tw ? (g.tw + 2) * (g.th + 2) : g.nhbox * g.hbox;
  // shared memory: the MT mask tile where it fits; the nine B tiles resident
  // when one 64-channel chunk and one N tile make up the whole launch
  // (64-wide tiles only: conv1_2) and they fit beside it
  const int cap = 227 * 1024, mt_bytes = 512 + BN * 128 * 4;
  const bool want_mt = FDT_MT && DG && mask_of(epi) && g.ksplit == 1;
  // (the forward measured 4 % slower with B resident: dgrad only)
  const bool rb_shape = FDT_RB && DG && BN == 64 && g.C == KS && g.nt == 1 && g.ksplit == 1;
  bool rb = false, mt;
  if (rb_shape && Cf::smem(g.halo_bytes, true) + (want_mt ? mt_bytes : 0) <= cap) {
    rb = true;
    mt = want_mt;
  } else {
    mt = want_mt && Cf::smem(g.halo_bytes, false) + mt_bytes <= cap;
  }
  const int smem = Cf::smem(g.halo_bytes, rb);
  if (smem > cap) return BPX_ERR_UNSUPPORTED;
  CUtensorMap ta, tb, tbl;
  if (g.tw) {        // activations [n][H][W][C]: box 32 ch x (tw+2) x (th+2) x 1 image
    const cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n};
    const cuuint64_t strides[3] = {(cuuint64_t)g.C * 4, (cuuint64_t)W * g.C * 4,
                                   (cuuint64_t)H * W * g.C * 4};
    const cuuint32_t box[4] = {32, (cuuint32_t)g.tw + 2, (cuuint32_t)g.th + 2, 1};
    if (!encode(&ta, a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dims, strides, box,
                CU_TENSOR_MAP_SWIZZLE_128B))
      return BPX_ERR_INVALID_ARGUMENT;
  } else {           // activations [pixels][C]: box 32 ch x hbox rows
    const cuuint64_t dims[2] = {(cuuint64_t)g.C, (cuuint64_t)g.npix};
    const cuuint64_t strides[1] = {(cuuint64_t)g.C * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)g.hbox};
    if (!encode(&ta, a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dims, strides, box,
                CU_TENSOR_MAP_SWIZZLE_128B))
      return BPX_ERR_INVALID_ARGUMENT;
  }
  for (int v = 0; v < 2; ++v) {
    const void* src = v ? wt.lo : wt.hi;
    CUtensorMap* m = v ? &tbl : &tb;
    if (DG) {       // w16 as [Cout][9][Cin]: box 64 ci x 1 tap x KS co, MN-major
      const cuuint64_t dims[3] = {(cuuint64_t)Cin, 9, (cuuint64_t)Cout};
      const cuuint64_t strides[2] = {(cuuint64_t)Cin * 2, (cuuint64_t)9 * Cin * 2};
      const cuuint32_t box[3] = {Cf::BNL == 32 ? 32u : 64u, 1, (cuuint32_t)KS};
      if (!encode(m, src, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, dims, strides, box,
                  Cf::BNL == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
        return BPX_ERR_INVALID_ARGUMENT;
    } else {        // w16 as [Cout][9*Cin]: box 64 k x BNL rows, K-major
      const cuuint64_t dims[2] = {(cuuint64_t)9 * Cin, (cuuint64_t)Cout};
      const cuuint64_t strides[1] = {(cuuint64_t)9 * Cin * 2};
      const cuuint32_t box[2] = {(cuuint32_t)KS, (cuuint32_t)Cf::BNL};
      if (!encode(m, src, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, dims, strides, box,
                  CU_TENSOR_MAP_SWIZZLE_128B))
        return BPX_ERR_INVALID_ARGUMENT;
    }
  }
  // MT: the dgrad mask staged by TMA
  const float* mptr = mask_of(epi);
  const int smem_mt = smem + mt_bytes;
  CUtensorMap tm = ta;
  if (mt) {
    if (g.tw) {
      const cuuint64_t dims[4] = {(cuuint64_t)g.N, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n};
      const cuuint64_t strides[3] = {(cuuint64_t)g.N * 4, (cuuint64_t)W * g.N * 4,
                                     (cuuint64_t)H * W * g.N * 4};
      const cuuint32_t box[4] = {32, (cuuint32_t)g.tw, (cuuint32_t)g.th, 1};
      if (!encode(&tm, mptr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dims, strides, box,
                  CU_TENSOR_MAP_SWIZZLE_128B))
        return BPX_ERR_INVALID_ARGUMENT;
    } else {
      const cuuint64_t dims[2] = {(cuuint64_t)g.N, (cuuint64_t)g.npix};
      const cuuint64_t strides[1] = {(cuuint64_t)g.N * 4};
      const cuuint32_t box[2] = {32, 128};
      if (!encode(&tm, mptr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dims, strides, box,
                  CU_TENSOR_MAP_SWIZZLE_128B))
        return BPX_ERR_INVALID_ARGUMENT;
    }
  }
  constexpr bool RBT = BN == 64;             // instantiate resident B for 64-wide tiles
  const bpx_status_t ls =
      rb ? (mt ? launch<BN, S, DG, PAIR, EPI, true, RBT>(ta, tb, tbl, tm, g, smem_mt, epi, st)
               : launch<BN, S, DG, PAIR, EPI, false, RBT>(ta, tb, tbl, tm, g, smem, epi, st))
         : (mt ? launch<BN, S, DG, PAIR, EPI, true, false>(ta, tb, tbl, tm, g, smem_mt, epi, st)
               : launch<BN, S, DG, PAIR, EPI, false, false>(ta, tb, tbl, tm, g, smem, epi, st));
  if (ls != BPX_OK) return ls;
  if (g.ksplit == 1) return launch_status(1);
  const long long groups = (long long)g.npix * (g.N / 8);
  int fg = (int)cdivll(groups, 256);
  if (fg > 8 * num_sms()) fg = 8 * num_sms();
  fdt_finish<<<fg, 256, 0, st>>>(part, g.ksplit, g.npix, g.N, epi);
  return launch_status(2);
}

#ifndef FDT_S128
#define FDT_S128 3
#endif
#ifndef FDT_S64
#define FDT_S64 6          // TMEM 2x64 accumulators + 6x64 A slots (S = 5: 0.6 % slower)
#endif
#ifndef FDT_S128P
#define FDT_S128P 4
#endif

template <bool DG, class EPI>
bpx_status_t dispatch(const float* a, const F16Weights& wt, float* part, const uint32_t* amax_a,
                      int n, int H, int W, int Cin, int Cout, EPI epi, cudaStream_t st) {
  const int N = DG ? Cin : Cout;
  int tw, th;
  tile2d(H, W, tw, th);
  const long long mt = tw ? (long long)n * (H / th) * (W / tw) : cdivll((long long)n * H * W, 128);
  if (N % 128 == 0) {
    if (pair_for(128, DG, mt))
      return run<128, FDT_S128P, DG, true>(a, wt, part, amax_a, n, H, W, Cin, Cout, epi, st);
    return run<128, FDT_S128, DG, false>(a, wt, part, amax_a, n, H, W, Cin, Cout, epi, st);
  }
  if (pair_for(64, DG, mt, DG ? Cout : Cin))
    return run<64, FDT_S64, DG, (!DG || FDT_PAIR64DG)>(a, wt, part, amax_a, n, H, W, Cin, Cout,
                                                        epi, st);
  return run<64, FDT_S64, DG, false>(a, wt, part, amax_a, n, H, W, Cin, Cout, epi, st);
}

// The call's operands in fp16x3 form: A's amax (from the caller or reduced
// here into the workspace) and the weights' split (from the caller or made
// here).  Returns the kernel launches issued.
inline int prepare(const float* a, long long na, const uint32_t* amax_a_in, const float* w,
                   long long nw, const F16Weights* wsplit, char* ws, const uint32_t*& amax_a,
                   F16Weights& wt, cudaStream_t st) {
  int k = 0;
  uint32_t* aw = reinterpret_cast<uint32_t*>(ws);
  amax_a = amax_a_in;
  if (!amax_a) {
    absmax(a, (size_t)na, aw, st);
    amax_a = aw;
    ++k;
  }
  if (wsplit && wsplit->hi) {
    wt = *wsplit;
  } else {
    char* wb = ws + 16;
    wt.hi = wb;
    wt.lo = wb + 2 * nw;
    wt.amax = reinterpret_cast<uint32_t*>(wb + 4 * nw);
    f16_split(w, (size_t)nw, const_cast<void*>(wt.hi), const_cast<void*>(wt.lo),
              const_cast<uint32_t*>(wt.amax), st);
    k += 2;
  }
  return k;
}

}  // namespace fdt

// ============================================================ entry points

// Channel counts in multiples of 64, W <= 224 (two halo slots + the B stages
// fit in 227 KB of smem).
bool fdt_conv_ok(int cin, int cout, int w) {
  if (cin % 64 || cout % 64 || w > 224) return false;
  return true;
}

// workspace: A's amax word, the weights' split (when not supplied), then
// split-K partials [ksplit][pixels][N]
size_t fdt_conv_ws(int n, int h, int w, int cin, int cout) {
  const long long nw = (long long)cout * 9 * cin;
  const long long npix = (long long)n * h * w;
  size_t part = 0;
  for (int dg = 0; dg < 2; ++dg) {        // fwd (N = cout) and dgrad (N = cin)
    const int N = dg ? cin : cout, C = dg ? cout : cin;
    const int BN = N % 128 == 0 ? 128 : 64;
    int tw, th;
    fdt::tile2d(h, w, tw, th);
    const long long mt = tw ? (long long)n * (h / th) * (w / tw) : cdivll(npix, 128);
    int k = 1, units;
    if (C % fdt::KS == 0)
      fdt::plan_units(mt, N / BN, C / fdt::KS, fdt::pair_for(BN, dg, mt, C), k, units);
    if (k > 1) {
      const size_t need = (size_t)k * npix * N;
      part = part > need ? part : need;
    }
  }
  return 16 + fdt::wsplit_bytes(nw) + part * sizeof(float);
}

bpx_status_t fdt_conv_fwd(const float* x, const float* w, const F16Weights* wsplit,
                          const uint32_t* amax_x, uint32_t* amax_y, const float* bias, float* y,
                          int n, int h, int w_, int cin, int cout, int relu, void* ws,
                          size_t ws_bytes, cudaStream_t st) {
  if (!fdt_conv_ok(cin, cout, w_) || !aligned16(x) || !aligned16(w) || !aligned16(y))
    return BPX_ERR_INVALID_ARGUMENT;
  if ((long long)n * h * w_ == 0) return launch_status(0);
  if (ws_bytes < fdt_conv_ws(n, h, w_, cin, cout) || !aligned16(ws)) return BPX_ERR_WORKSPACE;
  fdt::EBiasAct epi{y, bias, relu, amax_y};
  const long long nw = (long long)cout * 9 * cin;
  char* scratch = static_cast<char*>(ws);
  const uint32_t* amax_a;
  F16Weights wt;
  const int k = fdt::prepare(x, (long long)n * h * w_ * cin, amax_x, w, nw, wsplit, scratch,
                             amax_a, wt, st);
  count_launches(k);
  float* part = reinterpret_cast<float*>(scratch + 16 + fdt::wsplit_bytes(nw));
  return fdt::dispatch<false>(x, wt, part, amax_a, n, h, w_, cin, cout, epi, st);
}

bpx_status_t fdt_conv_dgrad(const float* dz, const float* w, const F16Weights* wsplit,
                            const uint32_t* amax_dz, uint32_t* amax_dx, const float* mask,
                            float* dx, int n, int h, int w_, int cin, int cout, void* ws,
                            size_t ws_bytes, cudaStream_t st) {
  if (!fdt_conv_ok(cin, cout, w_) || !aligned16(dz) || !aligned16(w) || !aligned16(dx) ||
      (mask && !aligned16(mask)))
    return BPX_ERR_INVALID_ARGUMENT;
  if ((long long)n * h * w_ == 0) return launch_status(0);
  if (ws_bytes < fdt_conv_ws(n, h, w_, cin, cout) || !aligned16(ws)) return BPX_ERR_WORKSPACE;
  fdt::EMask epi{dx, mask, amax_dx};
  const long long nw = (long long)cout * 9 * cin;
  char* scratch = static_cast<char*>(ws);
  const uint32_t* amax_a;
  F16Weights wt;
  const int k = fdt::prepare(dz, (long long)n * h * w_ * cout, amax_dz, w, nw, wsplit, scratch,
                             amax_a, wt, st);
  count_launches(k);
  float* part = reinterpret_cast<float*>(scratch + 16 + fdt::wsplit_bytes(nw));
  return fdt::dispatch<true>(dz, wt, part, amax_a, n, h, w_, cin, cout, epi, st);
}

}  // namespace bpx

#ifdef FDT_PROF
// Profiling builds only (BPX_NVCC_EXTRA=-DFDT_PROF): role cycle counters of
// the fwd/dgrad engine summed over CTAs since the last call (reset here).
extern "C" __attribute__((visibility("default"))) void bpx_fdt_prof(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, bpx::fdt::g_prof, sizeof(unsigned long long) * 16);
  static const unsigned long long z[16] = {};
  cudaMemcpyToSymbol(bpx::fdt::g_prof, z, sizeof(z));
}
#endif
