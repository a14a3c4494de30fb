// tcgen05 weight-gradient engine for the 3x3/pad-1 convolutions, fed by TMA:
//
//   dW^T[r][co] = sum_p im2col(x)[p][r] * dz[p][co],   r = tap*Cin + ci
//   M = 9*Cin (A = im2col(x)^T), N = Cout (B = dz), K = pixels (split-K)
//
// K = pixels is blocked as 32 consecutive pixels of the flattened NHWC
// tensor (so no tile overhangs an image edge, whatever H and W are).  For a
// 32-channel chunk of one tap the A tile is x[p0+s : +32][ci0 : +32] with
// s = dy*W + dx, the B tile is dz[p0 : +32][co0 : +32]: each is ONE 2-D TMA
// box.  Rows whose shifted source pixel wraps across an image row/edge are
// the conv's zero padding: the A converters zero them from a per-tap
// ballot mask.  Channels are contiguous, so both tiles are MN-major: TMA
// lays them out with SWIZZLE_128B_ATOM_32B, the one MN-major layout
// kind::tf32 accepts.
//
// fp32 accuracy: 3xTF32 (a_hi*b_hi + a_hi*b_lo + a_lo*b_hi).  The raw fp32
// tile already IS b_hi for the tensor core (it reads the top 19 bits), so
//   * A converter warps (one TMEM lane = one row r per thread) read their
//     row of the raw A tile, split hi/lo in registers and tcgen05.st both
//     into TMEM -> the MMA takes A from TMEM (TS form);
//   * B converter warps write only b_lo, elementwise in the same swizzled
//     layout, and (in CTAs of the first M tile) sum dz per channel in a
//     fixed order: the bias gradient comes out of the same pass over dz.
// Partial sums live in TMEM in 64-pixel chunks (two ping-pong buffers) and
// are promoted into round-to-nearest fp32 registers by the drain warps,
// because the tensor core's own fp32 accumulation truncates.
//
// CTA: 18 warps, one CTA per SM.  warp 0 TMA producer, warp 1 MMA issuer +
// TMEM owner, warps 2-5 A converters, 6-9 B converters (+bias), 10-17 drain.
#include "tma_host.h"
#include "tc_ptx.cuh"
#include "tc_api.h"

namespace bpx {
namespace wgt {
using namespace tcx;

constexpr int TMA_WARP = 0, MMA_WARP = 1, CB0 = 6, DR0 = 10;   // warps 2-5: A converters
constexpr int TMB_WARP = 18;                    // B (dz) TMA producer (decoupled rings only)

// BN = 128: 32 pixels per stage, 4 stages.  BN = 64 (Cout = 64): 64 pixels
// per stage, 3 stages -- a stage then carries as many MMA cycles as a
// BN = 128 stage, so the per-stage handshakes cost the same fraction.
//
// Two rings.  The B ring (raw dz | dz lo) and the TMEM A slots have S
// stages and are released by the MMA commit.  The raw A tiles have their own
// ring of SA stages, released by the A converters as soon as they hold the
// tile in registers, so the x loads run up to SA stages ahead instead of
// waiting for the MMA: with one shared ring the converters waited on TMA
// ~40% of the time and the MMA on the converters ~44% (ncu, conv3_2).
// BN = 64 (conv1_2) keeps one joint ring (A slot s = stage s, one producer,
// 18 warps): the smem budget leaves no extra A slot there (SA = S = 3), and
// decoupled measured 0.88 vs 0.83 ms.
template <int BN>
struct Cfg {
  static_assert(BN == 64 || BN == 128, "BN");
  static constexpr int BK = BN == 128 ? 32 : 64;          // pixels per stage
  static constexpr int BOX = 32 * BK * 4;                 // 32 channels x BK pixels
  static constexpr int PCH = 128 / BK;                    // stages per promotion chunk (K = 128)
  static constexpr int S = BN == 128 ? 4 : 3;
  static constexpr bool DEC = BN == 128;                  // decoupled A ring
  static constexpr int SA = DEC ? 5 : S;
  static constexpr int NT = DEC ? 19 * 32 : 18 * 32;
  static constexpr int A_BYTES = 4 * BOX;                 // 128 rows of A
  static constexpr int B_BYTES = (BN / 32) * BOX;
  // [A0 | B0 raw | B0 lo] [A1 | B1 ...] ... then the extra A slots (SA > S).
  // Interleaving the A and B tiles measured 3-13% faster than separate A and
  // B regions (conv1_2 0.83 vs 0.95 ms, conv5_x 0.14 vs 0.16 ms).
  static constexpr int STAGE = A_BYTES + 2 * B_BYTES;
  static constexpr int RINGS = S * STAGE + (SA - S) * A_BYTES;
  __device__ static char* a_tile(char* smem, int s) {
    return s < S ? smem + s * STAGE : smem + S * STAGE + (s - S) * A_BYTES;
  }
  __device__ static char* b_tile(char* smem, int s) { return smem + s * STAGE + A_BYTES; }
  static constexpr int ACC = 2 * BN;                      // two chunk buffers
  static constexpr int A_COL = ACC;                       // + S stages of (hi|lo)
  static constexpr int RG = 128 / (BN / 4);               // bias row groups
  static constexpr int SMEM = 1024 + RINGS + 512 + 128 * 16;
  static_assert(ACC + S * 2 * BK <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "smem budget");
};

struct Geo {
  const float* x;            // gather-A mode (9*Cin <= 32): the input itself
  int Cin, Cout, H, W;
  long long npix;
  int tiles, tps;            // 32-pixel tiles in total / per split
  long long slab;            // Cout * 9*Cin
};

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// PAIR: the two CTAs of a cluster (M tiles 2p, 2p+1; same N tile and K
// split) run one M = 256 tcgen05.mma.cta_group::2 per k-step.  Each CTA keeps
// its own 128 A rows in its TMEM and loads / splits only HALF of the dz tile
// (N/2 output channels), which halves the per-SM shared-memory traffic of
// the B operand (TMA fill, lo pass, MMA reads).  The leader (rank 0) issues
// the MMAs; its commits arrive on both CTAs' barriers (multicast); the
// peer's converters and drains arrive on the leader's ready / hfree.
// GA (gather A; 9*Cin <= 32 rows, the first conv): the im2col rows are not
// 32-channel TMA boxes.  Every TMEM lane quadrant q holds all 9*Cin rows but
// only the pixels [16q, 16q+16) of each stage (its other columns stay zero,
// stored once per slot), so four converter warps gather 16 pixels each
// straight from x (L2-resident); the drain sums the four partial rows.
template <int BN, bool PAIR, bool GA = false>
__global__ void __launch_bounds__(Cfg<BN>::NT, 1)
wgt_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tdz,
           Geo g, float* __restrict__ part, float* __restrict__ bias_part) {
  using Cf = Cfg<BN>;
  // N = 64 tiles: both a_hi products as one N = 128 MMA, the accumulator
  // columns (2 x 64) serving as one merged buffer instead of a ping-pong pair
  constexpr bool MG = BN == 64 && !PAIR && !GA;
  constexpr int BK = Cf::BK, BOX = Cf::BOX, PCH = Cf::PCH;
  static_assert(!PAIR || Cf::DEC, "pairs run the decoupled-ring layout");
  static_assert(!GA || (!Cf::DEC && !PAIR && Cf::BK == 64), "gather-A: joint ring, 64 px");
  constexpr int BNL = PAIR ? BN / 2 : BN;                 // dz columns held by this CTA
  // gather-A leaves the x half of every joint slot free: dz gets 2*S ring
  // slots (the extra ones in those halves), the TMEM A slots stay S
  constexpr int SB = GA ? 2 * Cf::S : Cf::S;
  constexpr uint32_t B_BYTES_L = (uint32_t)(BNL / 32) * BOX;
  extern __shared__ char smem_raw[];
  // offset from smem_raw (not a uintptr_t round trip) keeps the shared address space: LDS/STS, not generic LD/ST
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cf::RINGS);   // B stage landed
  uint64_t* ready = full + 8;                // A and B converters done
  uint64_t* empty = ready + 8;               // MMA done: B stage + TMEM A slot free
  uint64_t* afull = empty + 8;               // A tile landed
  uint64_t* afree = afull + 8;               // A tile read by the converters
  uint64_t* hfull = afree + 8;
  uint64_t* hfree = hfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + 2);
  float4* bias_scr = reinterpret_cast<float4*>(smem + Cf::RINGS + 512);
  static_assert(Cf::S <= 8 && Cf::SA <= 8, "barrier slots");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nrows = 9 * g.Cin;                  // M extent
  const int chunks = nrows / 32;                // 32-row chunks (tap-major)
  const int cpt = g.Cin / 32;                   // chunks per tap
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * BN;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  auto btile = [&](int sb) -> char* {
    return (GA && sb >= Cf::S) ? Cf::a_tile(smem, sb - Cf::S) : Cf::b_tile(smem, sb);
  };
  const int nl0 = n0 + (int)rank * BNL;                   // first dz column held here
  const int t0 = blockIdx.z * g.tps;
  const int nst = max(0, min(g.tiles, t0 + g.tps) - t0);

  if (tid == 0) {
    for (int s = 0; s < SB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&ready[s], PAIR ? 16 : 256);     // pairs: one arrival per warp, both CTAs
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < Cf::SA; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&afree[s], GA ? 1 : 128);      // GA: TMEM A slot freed by the MMA
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hfree[b], PAIR ? 16 : 256);
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
  // leader's ready / hfree as shared::cluster addresses (pairs)
  const uint32_t ready_l = PAIR ? mapa_rank(ready, 0) : 0u;
  const uint32_t hfree_l = PAIR ? mapa_rank(hfree, 0) : 0u;

  if (warp == TMA_WARP) {
    // ------------------------------------------------------------ TMA: x (A)
    if (lane == 0) {
      tma_prefetch_desc(&tx);
      if (!Cf::DEC) tma_prefetch_desc(&tdz);
      int na = 0;
      if (!GA)
        for (int c = 0; c < 4; ++c) na += (m0 / 32 + c) < chunks;
      const uint32_t bytes = (uint32_t)(na * BOX) + (Cf::DEC ? 0u : (uint32_t)Cf::B_BYTES);
      for (int i = 0; i < nst && GA; ++i) {       // gather-A: the dz ring only
        const int sb = i % SB;
        if (i >= SB) mbar_wait(&empty[sb], ((i / SB) - 1) & 1);
        mbar_expect_tx(&full[sb], (uint32_t)Cf::B_BYTES);
        for (int j = 0; j < BN / 32; ++j)
          tma_load_2d(btile(sb) + j * BOX, &tdz, n0 + 32 * j, (t0 + i) * BK, &full[sb]);
      }
      for (int i = 0; i < nst && !GA; ++i) {
        const int s = i % Cf::SA;
        uint64_t* bar = Cf::DEC ? &afull[s] : &full[s];
        if (i >= Cf::SA) mbar_wait(Cf::DEC ? &afree[s] : &empty[s], ((i / Cf::SA) - 1) & 1);
        const int p0 = (t0 + i) * BK;
        char* st = Cf::a_tile(smem, s);
        mbar_expect_tx(bar, bytes);
        for (int c = 0; c < 4 && !GA; ++c) {
          const int gc = m0 / 32 + c;
          if (gc >= chunks) break;
          const int tap = gc / cpt, ci0 = (gc - tap * cpt) * 32;
          tma_load_2d(st + c * BOX, &tx, ci0, p0 + (tap / 3 - 1) * g.W + tap % 3 - 1, bar);
        }
        if (!Cf::DEC)
          for (int j = 0; j < BN / 32; ++j)
            tma_load_2d(Cf::b_tile(smem, s) + j * BOX, &tdz, n0 + 32 * j, p0, bar);
      }
    }
  } else if (Cf::DEC && warp == TMB_WARP) {
    // ------------------------------------------------------------ TMA: dz (B)
    if (lane == 0) {
      tma_prefetch_desc(&tdz);
      for (int i = 0; i < nst; ++i) {
        const int s = i % Cf::S;
        if (i >= Cf::S) mbar_wait(&empty[s], ((i / Cf::S) - 1) & 1);
        const int p0 = (t0 + i) * BK;
        char* st = Cf::b_tile(smem, s);
        mbar_expect_tx(&full[s], B_BYTES_L);
        for (int j = 0; j < BNL / 32; ++j)
          tma_load_2d(st + j * BOX, &tdz, nl0 + 32 * j, p0, &full[s]);
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    // (the whole warp runs the loop, elect.sync picks the issuing lane; one
    // barrier check per stage: A and B converters both arrive on ready[s]).
    // (Issuing the dz loads from this warp as well, after a wait for
    // MMA(i-1), measured 8% slower than the separate B producer warp.)
    if (!PAIR || rank == 0) {
      // M=128 (pairs: 256), N=BN, tf32 x tf32 -> f32, A from TMEM, B MN-major (bit 16)
      constexpr uint32_t idesc = PAIR ? ((make_idesc(BN) & ~(0x1Fu << 24)) | (16u << 24) | (1u << 16))
                                      : (make_idesc(BN) | (1u << 16));
      constexpr uint32_t idesc_mg = make_idesc(2 * BN) | (1u << 16);
      for (int i = 0; i < nst; ++i) {
        const int s = i % SB, sa = i % Cf::S;     // dz ring slot, TMEM A slot
        const uint32_t ph = (i / SB) & 1;
        const int c = i / PCH, b = MG ? 0 : c & 1;
        if (MG && i % PCH == 0 && c >= 1) {        // one merged buffer: wait for its drain
          mbar_wait(&hfree[0], (c - 1) & 1);
          tc_fence_after();
        }
        if (!MG && i % PCH == 0 && c >= 2) {
          if (PAIR) mbar_wait_cluster(&hfree[b], ((c >> 1) - 1) & 1);
          else mbar_wait(&hfree[b], ((c >> 1) - 1) & 1);
          tc_fence_after();
        }
        if (PAIR) mbar_wait_cluster(&ready[s], ph); else mbar_wait(&ready[s], ph);
        tc_fence_after();
        const uint32_t d = tmem + b * BN;
        const uint32_t ah = tmem + Cf::A_COL + sa * 2 * BK, al = ah + BK;
        const uint32_t bh = smem_u32(btile(s));
        const uint32_t bl = bh + Cf::B_BYTES;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint64_t dbh = make_desc_mn32(bh + ks * 1024, BOX, 512);
          const uint64_t dbl = make_desc_mn32(bl + ks * 1024, BOX, 512);
          const uint32_t acc = (i % PCH != 0 || ks > 0) ? 1u : 0u;
          if (MG) {
            // [b_hi | b_lo] as one N = 128 operand (the lo tile follows the
            // raw one at the same MN-atom stride): one A read for both a_hi
            // products, then a_lo * b_hi into the left half
            mma_ts_elect(d, ah + 8 * ks, dbh, idesc_mg, acc);
            mma_ts_elect(d, al + 8 * ks, dbh, idesc, 1u);
          } else if (PAIR) {
            mma_ts2_elect(d, al + 8 * ks, dbh, idesc, acc);
            mma_ts2_elect(d, ah + 8 * ks, dbl, idesc, 1u);
            mma_ts2_elect(d, ah + 8 * ks, dbh, idesc, 1u);
          } else {
            mma_ts_elect(d, al + 8 * ks, dbh, idesc, acc);
            mma_ts_elect(d, ah + 8 * ks, dbl, idesc, 1u);
            mma_ts_elect(d, ah + 8 * ks, dbh, idesc, 1u);
          }
        }
        if (PAIR) {
          tc_commit2_elect(&empty[s]);
          if (i % PCH == PCH - 1 || i == nst - 1) tc_commit2_elect(&hfull[b]);
        } else {
          tc_commit_elect(&empty[s]);
          if (GA) tc_commit_elect(&afree[sa]);
          if (i % PCH == PCH - 1 || i == nst - 1) tc_commit_elect(&hfull[b]);
        }
      }
    }
  } else if (GA && warp < CB0) {
    // ------------------------------------------------------------ A gather (GA)
    const int q = warp & 3;
    const bool rv = lane < nrows;
    const int tap = rv ? lane / g.Cin : 4, ci = rv ? lane - (lane / g.Cin) * g.Cin : 0;
    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
    const long long sh = ((long long)dy * g.W + dx) * g.Cin + ci;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + Cf::A_COL;
    const long long hw = (long long)g.H * g.W;
    // software-pipelined: stage i+1's loads are issued right after stage i's
    // TMEM stores, so their latency overlaps the wait for the next slot
    float v[16];
    uint32_t okm = 0;
    auto gather = [&](int i) {
      const long long pb = (long long)(t0 + i) * BK + 16 * q;    // this quadrant's pixels
      const int rem = (int)(pb % hw);
      int oh = rem / g.W, ow = rem - (rem / g.W) * g.W;
      okm = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) {      // all loads unconditional: in flight together
        const long long pp = pb + k;
        const bool ok = rv && pp < g.npix && (unsigned)(oh + dy) < (unsigned)g.H &&
                        (unsigned)(ow + dx) < (unsigned)g.W;
        okm |= (uint32_t)ok << k;
        v[k] = __ldg(g.x + (ok ? pp * g.Cin + sh : 0));
        if (++ow == g.W) { ow = 0; if (++oh == g.H) oh = 0; }
      }
    };
    if (nst > 0) gather(0);
    for (int i = 0; i < nst; ++i) {
      const int s = i % Cf::S;                      // TMEM A slot
      float hi[16], lo[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) split((okm >> k) & 1u ? v[k] : 0.f, hi[k], lo[k]);
      if (i >= Cf::S) mbar_wait(&afree[s], ((i / Cf::S) - 1) & 1);   // MMA(i - S) done
      tc_fence_after();
      const uint32_t a = lanebase + s * 2 * BK;
      if (i < Cf::S) {                              // first use of the slot: zero columns
        float z[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) z[k] = 0.f;
#pragma unroll
        for (int c = 0; c < 2 * BK; c += 16)
          if ((c & (BK - 1)) != 16 * q) tmem_st16(a + c, z);
      }
      tmem_st16(a + 16 * q, hi);
      tmem_st16(a + BK + 16 * q, lo);
      if (i + 1 < nst) gather(i + 1);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&ready[i % SB]);
    }
  } else if (warp < CB0) {
    // ------------------------------------------------------------ A converters
    // thread = TMEM lane = row r of the M tile = channel `lane` of chunk q
    const int q = warp & 3;
    const bool valid = (m0 / 32 + q) < chunks;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + Cf::A_COL;
    const int g8 = lane >> 3, w4 = (lane & 7) * 4;
    const int gc = m0 / 32 + q, tap = valid ? gc / cpt : 4;
    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
    // coordinates of pixel p0 + lane (+32 per half), advanced by BK pixels per stage
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
      const int s = i % Cf::S, sa = i % Cf::SA;
      uint32_t vmask[BK / 32];
#pragma unroll
      for (int h = 0; h < BK / 32; ++h) {
        const bool ok = valid && p < g.npix && (unsigned)(oh + dy) < (unsigned)g.H &&
                        (unsigned)(ow + dx) < (unsigned)g.W;
        vmask[h] = __ballot_sync(0xffffffffu, ok);
        advance(32);
      }
      mbar_wait(Cf::DEC ? &afull[sa] : &full[s], (i / Cf::SA) & 1);
      const char* box = Cf::a_tile(smem, sa) + q * BOX;
      const uint32_t a = lanebase + s * 2 * BK;
#pragma unroll
      for (int h = 0; h < BK / 32; ++h) {
        float hi[32], lo[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int kk = 32 * h + k;
          const float v = ((vmask[h] >> k) & 1u)
                              ? *reinterpret_cast<const float*>(box + kk * 128 +
                                                                ((g8 ^ (kk & 3)) << 5) + w4)
                              : 0.f;
          split(v, hi[k], lo[k]);
        }
        if (Cf::DEC && h == BK / 32 - 1) mbar_arrive(&afree[sa]);   // A tile in registers
        if (Cf::DEC && h == 0 && i >= Cf::S) {              // TMEM slot s: MMA(i - S) done
          mbar_wait(&empty[s], ((i / Cf::S) - 1) & 1);
          tc_fence_after();
        }
        tmem_st16(a + 32 * h, *reinterpret_cast<float(*)[16]>(hi));
        tmem_st16(a + 32 * h + 16, *reinterpret_cast<float(*)[16]>(hi + 16));
        tmem_st16(a + BK + 32 * h, *reinterpret_cast<float(*)[16]>(lo));
        tmem_st16(a + BK + 32 * h + 16, *reinterpret_cast<float(*)[16]>(lo + 16));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      if (PAIR) {
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(ready_l + 8u * s);
      } else {
        mbar_arrive(&ready[s]);
      }
    }
  } else if (warp < DR0) {
    // ------------------------------------------------------------ B converters
    // b_lo = b - tf32(b), elementwise in the swizzled layout; per-channel dz
    // sums (bias gradient) over this split's pixels in CTAs of M tile 0.
    const int bt = tid - CB0 * 32;
    constexpr int NC4 = BNL / 4;               // float4 columns of this CTA's tile
    constexpr int RG = 128 / NC4;              // row groups
    const int c4 = bt % NC4, rg = bt / NC4;    // fixed column, row group
    const int box = c4 / 8, gl = (c4 & 7) >> 1, half = c4 & 1;
    const bool do_bias = bias_part != nullptr && blockIdx.x / (PAIR ? 2 : 1) == 0;
    float4 bs = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = 0; i < nst; ++i) {
      const int s = i % SB;
      mbar_wait(&full[s], (i / SB) & 1);
      const char* raw = btile(s);
      char* lo = const_cast<char*>(raw) + Cf::B_BYTES;
#pragma unroll
      for (int k = rg; k < BK; k += RG) {
        const int off = box * BOX + k * 128 + ((gl ^ (k & 3)) << 5) + half * 16;
        const float4 v = *reinterpret_cast<const float4*>(raw + off);
        float4 h, l;
        split(v.x, h.x, l.x); split(v.y, h.y, l.y);
        split(v.z, h.z, l.z); split(v.w, h.w, l.w);
        *reinterpret_cast<float4*>(lo + off) = l;
        if (do_bias) { bs.x += v.x; bs.y += v.y; bs.z += v.z; bs.w += v.w; }
      }
      fence_proxy_async();
      if (PAIR) {
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(ready_l + 8u * s);
      } else {
        mbar_arrive(&ready[s]);
      }
    }
    if (do_bias) {
      bias_scr[bt] = bs;
      named_sync(1, 128);
      if (bt < NC4) {
        float4 t = bias_scr[bt];
        for (int r = 1; r < RG; ++r) {
          const float4 u = bias_scr[r * NC4 + bt];
          t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
        }
        *reinterpret_cast<float4*>(bias_part + (long long)blockIdx.z * g.Cout + nl0 + 4 * bt) = t;
      }
    }
  } else {
    // ------------------------------------------------------------ drain + epilogue
    const int q = warp & 3, hf = (warp - DR0) >> 2;
    constexpr int CW = BN / 2;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + hf * CW;
    float acc[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) acc[j] = 0.f;
    const int nch = (nst + PCH - 1) / PCH;
    for (int c = 0; c < nch; ++c) {
      const int b = MG ? 0 : c & 1;
      mbar_wait(&hfull[b], MG ? (c & 1) : ((c >> 1) & 1));
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < CW; j += 8) {
        uint32_t r[8];
        tmem_ld8(lanebase + b * BN + j, r);
        if (MG) {                       // + the a_hi * b_lo half
          uint32_t r2[8];
          tmem_ld8(lanebase + BN + j, r2);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[j + t] += __uint_as_float(r[t]) + __uint_as_float(r2[t]);
        } else {
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[j + t] += __uint_as_float(r[t]);
        }
      }
      tc_fence_before();
      if (PAIR) {
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(hfree_l + 8u * b);
      } else {
        mbar_arrive(&hfree[b]);
      }
    }
    if (GA) {
      // sum the four quadrants' partial rows through shared memory (the
      // rings are idle: every MMA has completed once the last hfull fired)
      float* red = reinterpret_cast<float*>(smem);      // [4][32][BN]
#pragma unroll
      for (int j = 0; j < CW; ++j) red[(q * 32 + lane) * BN + hf * CW + j] = acc[j];
      named_sync(2, 32 * (Cf::NT / 32 - DR0));
      if (q == 0 && lane < nrows) {
        float* o = part + (long long)blockIdx.z * g.slab + lane;
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          const int col = hf * CW + j;
          const float t = red[lane * BN + col] + red[(32 + lane) * BN + col] +
                          red[(64 + lane) * BN + col] + red[(96 + lane) * BN + col];
          o[(long long)(n0 + col) * nrows] = t;
        }
      }
    } else {
      const int r = m0 + q * 32 + lane;
      if (r < nrows) {
        float* o = part + (long long)blockIdx.z * g.slab + r;
#pragma unroll
        for (int j = 0; j < CW; ++j) o[(long long)(n0 + hf * CW + j) * nrows] = acc[j];
      }
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
#ifndef WGT_PAIR
#define WGT_PAIR 1
#endif
// N = 128 tiles run as CTA pairs (M = 256 per cluster) when the M tiles pair
// up without a padding tile (Cin = 256, 512: 3-4% faster; with a padding
// tile, Cin = 64, 128, the extra tile costs 10-14%)
inline bool paired(int cin, int cout) {
  return WGT_PAIR && bn_for(cout) == 128 && cdiv(9 * cin, 128) % 2 == 0;
}

inline void plan(int n, int H, int W, int cin, int cout, Geo& g, int& mt, int& nt, int& splits) {
  g.Cin = cin; g.Cout = cout; g.H = H; g.W = W;
  g.npix = (long long)n * H * W;
  g.tiles = (int)cdivll(g.npix, bn_for(cout) == 128 ? Cfg<128>::BK : Cfg<64>::BK);
  g.slab = (long long)cout * 9 * cin;
  mt = cdiv(9 * cin, 128);
  if (paired(cin, cout)) mt += mt & 1;         // whole pairs (a padding tile computes zeros)
  nt = cout / bn_for(cout);
  const int tiles_mn = mt * nt;
  int want = num_sms() / tiles_mn;
  if (want < 1) want = 1;
  if (want > g.tiles) want = g.tiles;
  g.tps = cdiv(g.tiles, want);
  splits = cdiv(g.tiles, g.tps);
}

// [pixels][C] fp32, box = 32 channels x BK pixels, MN-major tf32 layout.
inline bool encode_rows(CUtensorMap* m, const float* p, long long npix, int C, int BK) {
  const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)npix};
  const cuuint64_t strides[1] = {(cuuint64_t)C * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)BK};
  const cuuint32_t es[2] = {1, 1};
  return encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                const_cast<float*>(p), dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool PAIR, bool GA = false>
bpx_status_t launch(const CUtensorMap& tx, const CUtensorMap& tdz, const Geo& g, int mt,
                    int nt, int splits, float* part, float* bias_part, cudaStream_t st) {
  using Cf = Cfg<BN>;
  auto kern = wgt_kernel<BN, PAIR, GA>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    attr = true;
  }
  if (!PAIR) {
    kern<<<dim3(mt, nt, splits), Cf::NT, Cf::SMEM, st>>>(tx, tdz, g, part, bias_part);
    return launch_status();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(mt, nt, splits);
  cfg.blockDim = dim3(Cf::NT);
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

}  // namespace wgt

// ============================================================ entry points

// Cin % 32 == 0: x tiles by TMA; 9*Cin <= 32 (the first conv): gather-A mode
bool wgt_conv_ok(int cin, int cout) {
  if (cin % 32 == 0) return cout % 64 == 0;
  return 9 * cin <= 32 && cout % 64 == 0 && cout % 128 != 0;   // gather-A runs N = 64 tiles
}

size_t wgt_conv_ws(int n, int h, int w, int cin, int cout) {
  if (!wgt_conv_ok(cin, cout)) return 0;      // the planner assumes a supported shape
  wgt::Geo g;
  int mt, nt, splits;
  wgt::plan(n, h, w, cin, cout, g, mt, nt, splits);
  if (splits <= 1) return 0;
  return ((size_t)splits * (size_t)g.slab + (size_t)splits * cout) * sizeof(float);
}

bpx_status_t wgt_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias, int n,
                            int h, int w_, int cin, int cout, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  if (!wgt_conv_ok(cin, cout) || !aligned16(x) || !aligned16(dz) || !aligned16(dw))
    return BPX_ERR_INVALID_ARGUMENT;
  if (dbias && !aligned16(dbias)) return BPX_ERR_INVALID_ARGUMENT;
  if (ws_bytes < wgt_conv_ws(n, h, w_, cin, cout)) return BPX_ERR_WORKSPACE;
  const size_t slab = (size_t)cout * 9 * cin;
  if (n == 0) {
    cudaMemsetAsync(dw, 0, sizeof(float) * slab, st);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * cout, st);
    return launch_status(0);
  }
  wgt::Geo g;
  int mt, nt, splits;
  wgt::plan(n, h, w_, cin, cout, g, mt, nt, splits);
  g.x = x;
  const bool ga = cin % 32 != 0;
  CUtensorMap tx, tdz;
  const int bk = wgt::bn_for(cout) == 128 ? wgt::Cfg<128>::BK : wgt::Cfg<64>::BK;
  if ((!ga && !wgt::encode_rows(&tx, x, g.npix, cin, bk)) ||
      !wgt::encode_rows(&tdz, dz, g.npix, cout, bk))
    return BPX_ERR_INVALID_ARGUMENT;
  if (ga) tx = tdz;                          // unused by the gather path
  float* part = splits == 1 ? dw : static_cast<float*>(ws);
  float* bpart = !dbias ? nullptr
                        : (splits == 1 ? dbias : static_cast<float*>(ws) + (size_t)splits * slab);
  bpx_status_t s = wgt::bn_for(cout) == 128
      ? (wgt::paired(cin, cout) ? wgt::launch<128, true>(tx, tdz, g, mt, nt, splits, part, bpart, st)
                           : wgt::launch<128, false>(tx, tdz, g, mt, nt, splits, part, bpart, st))
      : (ga ? wgt::launch<64, false, true>(tx, tdz, g, mt, nt, splits, part, bpart, st)
            : wgt::launch<64, false>(tx, tdz, g, mt, nt, splits, part, bpart, st));
  if (s != BPX_OK || splits == 1) return s;
  return split_reduce_wb(part, slab, dw, bpart, (size_t)cout, dbias, splits, st);
}

}  // namespace bpx
