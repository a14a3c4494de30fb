// tcgen05 forward / data-gradient engine for the 3x3/pad-1 convolutions,
// fed by TMA, persistent over output tiles:
//
//   fwd   : y[p][co]  = act(b[co] + sum_{tap,ci} x[p + s_tap][ci]  * w[co][tap][ci])
//   dgrad : dx[q][ci] = mask(q) * sum_{tap,co} dz[q - s_tap][co] * w[co][tap][ci]
//   s_tap = dy*W + dx  (flattened-pixel shift of the tap)
//
// M = pixels (128 consecutive flattened pixels per tile), N = output
// channels, K = (32-channel chunk, tap) stages.  Per channel chunk the CTA
// loads ONE halo of the activations by TMA -- flattened rows
// [m0 - W - 1, m0 + 128 + W + 1) x 32 channels -- and all nine taps read
// their shifted 128-row window out of it, so activation traffic is
// (128 + 2W + 2)/128 instead of 9x the tile.  Rows whose shifted source
// pixel falls outside its image (the conv's zero padding, including the
// row wrap of the flattened layout) are zeroed by the A converters from a
// per-thread 9-bit tap mask computed once per tile.
// The B tile is the raw weight tile, straight from w by TMA:
//   fwd   B(co, k) = w[co][tap][ci]: K-major, 128-B swizzle (one box)
//   dgrad B(ci, k) = w[co][tap][ci]: MN-major, SWIZZLE_128B_ATOM_32B, one
//                    box per 32 input channels (w viewed [Cout][9][Cin]).
//
// fp32 accuracy by 3xTF32 (a_hi*b_hi + a_hi*b_lo + a_lo*b_hi); the raw tile
// is b_hi.  A converters split A into TMEM (TS form).  b_lo = w - tf32(w) is
// a pre-split copy of the (small) weight tensor made by one elementwise
// kernel per call, loaded by TMA next to b_hi: shared memory then carries
// only the MMA's B reads, the TMA fills and one LDS pass over A -- a
// converter pass over B in shared memory made this kernel smem-bound.
// TMEM chunk promotion into RN fp32 registers as in the other engines.  The kernel is persistent: the stage ring and the
// accumulator ping-pong run straight across tiles, so a tile's epilogue
// (drain warps: bias + ReLU or ReLU mask, stores) overlaps the next tile's
// main loop.
//
// CTA: 14 warps.  warp 0 TMA, warp 1 MMA + TMEM owner, 2-5 A converters,
// 6-13 drain + epilogue.
#include "tma_host.h"
#include "tc_ptx.cuh"
#include "tc_api.h"

namespace bpx {
namespace fdt {
using namespace tcx;

constexpr int BK = 32;                 // K elements per stage (one channel chunk of a tap)
constexpr int PCH = 4;                 // stages per TMEM promotion chunk (K = 128)
constexpr int NTHREADS = 14 * 32;
constexpr int TMA_WARP = 0, MMA_WARP = 1, DR0 = 6;   // warps 2-5: A converters

template <int BN, int NS = 4>
struct Cfg {
  static_assert(BN == 64 || BN == 128, "BN");
  static constexpr int S = NS;                            // B / TMEM-A stages
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE = 2 * B_BYTES;               // B raw | B lo
  static constexpr int A_COL = 2 * BN;
  static_assert(A_COL + S * 2 * BK <= 512, "TMEM budget");
  // dynamic smem = 1024 (align) + S*STAGE + 2*halo_bytes + 512 (barriers)
  static int smem(int halo_bytes) { return 1024 + S * STAGE + 2 * halo_bytes + 512; }
};

struct Geo {
  int H, W, C;               // C = gathered channels (Cin fwd, Cout dgrad)
  int N;                     // output channels
  int npix, mt, nt, tiles;
  int hrows, hbox, nhbox;    // halo rows used, rows per TMA box, boxes per halo
  int halo_bytes;            // one halo slot (nhbox * hbox * 128)
};

struct EBiasAct {
  float* out; const float* bias; int relu;
  __device__ void operator()(long long m, int n0, int N, const float (&v)[8]) const {
    float* o = out + m * N + n0;
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float t = v[j] + (bias ? __ldg(bias + n0 + j) : 0.f);
      r[j] = relu ? fmaxf(t, 0.f) : t;
    }
    *reinterpret_cast<float4*>(o) = make_float4(r[0], r[1], r[2], r[3]);
    *reinterpret_cast<float4*>(o + 4) = make_float4(r[4], r[5], r[6], r[7]);
  }
};
struct EMask {
  float* out; const float* mask;
  __device__ void operator()(long long m, int n0, int N, const float (&v)[8]) const {
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
  }
};

template <int BN, int NS, bool DG, class EPI>
__global__ void __launch_bounds__(NTHREADS, 1)
fdt_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
           const __grid_constant__ CUtensorMap tbl, Geo g, EPI epi) {
  using Cf = Cfg<BN, NS>;
  constexpr int S = Cf::S;
  extern __shared__ char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  char* halo = smem + S * Cf::STAGE;                          // 2 slots
  uint64_t* bfull = reinterpret_cast<uint64_t*>(halo + 2 * g.halo_bytes);
  uint64_t* aready = bfull + S;
  uint64_t* empty = aready + S;
  uint64_t* hfull = empty + S;       // halo slot loaded
  uint64_t* hempty = hfull + 2;      // halo slot consumed by all nine taps
  uint64_t* accfull = hempty + 2;
  uint64_t* accfree = accfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cpt = g.C / BK;                   // channel chunks
  const int nk = 9 * cpt;                     // stages per tile

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&aready[s], 4);          // one arrival per converter warp
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hempty[b], 4);
      mbar_init(&accfull[b], 1);
      mbar_init(&accfree[b], 8);         // one arrival per drain warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == TMA_WARP) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&ta);
      tma_prefetch_desc(&tb);
      tma_prefetch_desc(&tbl);
      int i = 0, hc = 0;
      for (int t = blockIdx.x; t < g.tiles; t += gridDim.x) {
        const int m0 = (t / g.nt) * 128, n0 = (t % g.nt) * BN;
        for (int cc = 0; cc < cpt; ++cc, ++hc) {
          const int hs = hc & 1;
          if (hc >= 2) mbar_wait(&hempty[hs], ((hc >> 1) - 1) & 1);
          mbar_expect_tx(&hfull[hs], (uint32_t)g.halo_bytes);
          for (int j = 0; j < g.nhbox; ++j)
            tma_load_2d(halo + hs * g.halo_bytes + j * g.hbox * 128, &ta, cc * BK,
                        m0 - g.W - 1 + j * g.hbox, &hfull[hs]);
          for (int tap = 0; tap < 9; ++tap, ++i) {
            const int s = i % S;
            if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
            char* st = smem + s * Cf::STAGE;
            mbar_expect_tx(&bfull[s], 2 * Cf::B_BYTES);
            if (DG) {
              for (int j = 0; j < BN / 32; ++j) {
                tma_load_3d(st + j * 4096, &tb, n0 + 32 * j, tap, cc * BK, &bfull[s]);
                tma_load_3d(st + Cf::B_BYTES + j * 4096, &tbl, n0 + 32 * j, tap, cc * BK,
                            &bfull[s]);
              }
            } else {
              tma_load_2d(st, &tb, tap * g.C + cc * BK, n0, &bfull[s]);
              tma_load_2d(st + Cf::B_BYTES, &tbl, tap * g.C + cc * BK, n0, &bfull[s]);
            }
          }
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // M=128, N=BN, tf32 -> f32, A from TMEM; B K-major (fwd) / MN-major (dgrad)
      constexpr uint32_t idesc = make_idesc(BN) | (DG ? (1u << 16) : 0u);
      int i = 0, c = 0;
      for (int t = blockIdx.x; t < g.tiles; t += gridDim.x) {
        for (int kb = 0; kb < nk; ++kb, ++i) {
          const int s = i % S;
          const uint32_t ph = (i / S) & 1;
          const int b = c & 1;
          if (kb % PCH == 0 && c >= 2) {
            mbar_wait(&accfree[b], ((c >> 1) - 1) & 1);
            tc_fence_after();
          }
          mbar_wait(&aready[s], ph);
          mbar_wait(&bfull[s], ph);
          tc_fence_after();
          const uint32_t d = tmem + b * BN;
          const uint32_t ah = tmem + Cf::A_COL + s * 2 * BK, al = ah + BK;
          const uint32_t bh = smem_u32(smem + s * Cf::STAGE);
          const uint32_t bl = bh + Cf::B_BYTES;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            uint64_t dbh, dbl;
            if (DG) {
              dbh = make_desc_mn32(bh + ks * 1024, 4096, 512);
              dbl = make_desc_mn32(bl + ks * 1024, 4096, 512);
            } else {
              dbh = make_desc_sw128(bh + ks * 32, 16, 1024);
              dbl = make_desc_sw128(bl + ks * 32, 16, 1024);
            }
            const uint32_t acc = (kb % PCH != 0 || ks > 0) ? 1u : 0u;
            mma_ts(d, al + 8 * ks, dbh, idesc, acc);
            mma_ts(d, ah + 8 * ks, dbl, idesc, 1u);
            mma_ts(d, ah + 8 * ks, dbh, idesc, 1u);
          }
          tc_commit(&empty[s]);
          if (kb % PCH == PCH - 1 || kb == nk - 1) {
            tc_commit(&accfull[b]);
            ++c;
          }
        }
      }
    }
  } else if (warp < DR0) {
    // ------------------------------------------------------------ A converters
    // thread = TMEM lane = pixel row of the tile; stage (cc, tap) reads halo
    // row r + W + 1 +/- s_tap
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + Cf::A_COL;
    const int hw = g.H * g.W;
    int i = 0, hc = 0;
    for (int t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      const int p = (t / g.nt) * 128 + r;
      uint32_t tmask = 0;                     // bit tap: source pixel inside the image
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
      for (int cc = 0; cc < cpt; ++cc, ++hc) {
        const int hs = hc & 1;
        mbar_wait(&hfull[hs], (hc >> 1) & 1);
        const char* hbase = halo + hs * g.halo_bytes;
        for (int tap = 0; tap < 9; ++tap, ++i) {
          const int s = i % S;
          if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);   // TMEM A slot free
          const int sh = (tap / 3 - 1) * g.W + (tap % 3 - 1);
          const int hr = r + g.W + 1 + (DG ? -sh : sh);
          const bool ok = (tmask >> tap) & 1u;
          const char* row = hbase + hr * 128;
          float hi[BK], lo[BK];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ok) v = *reinterpret_cast<const float4*>(row + ((j ^ (hr & 7)) << 4));
            split(v.x, hi[4 * j + 0], lo[4 * j + 0]);
            split(v.y, hi[4 * j + 1], lo[4 * j + 1]);
            split(v.z, hi[4 * j + 2], lo[4 * j + 2]);
            split(v.w, hi[4 * j + 3], lo[4 * j + 3]);
          }
          tc_fence_after();
          const uint32_t a = lanebase + s * 2 * BK;
          tmem_st16(a, *reinterpret_cast<float(*)[16]>(hi));
          tmem_st16(a + 16, *reinterpret_cast<float(*)[16]>(hi + 16));
          tmem_st16(a + BK, *reinterpret_cast<float(*)[16]>(lo));
          tmem_st16(a + BK + 16, *reinterpret_cast<float(*)[16]>(lo + 16));
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&aready[s]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&hempty[hs]);
      }
    }
  } else {
    // ------------------------------------------------------------ drain + epilogue
    const int q = warp & 3, hf = (warp - DR0) >> 2;
    constexpr int CW = BN / 2;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + hf * CW;
    const int nch = (nk + PCH - 1) / PCH;
    int c = 0;
    for (int t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      float acc[CW];
#pragma unroll
      for (int j = 0; j < CW; ++j) acc[j] = 0.f;
      for (int k = 0; k < nch; ++k, ++c) {
        const int b = c & 1;
        mbar_wait(&accfull[b], (c >> 1) & 1);
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
        if (lane == 0) mbar_arrive(&accfree[b]);
      }
      const long long p = (long long)(t / g.nt) * 128 + q * 32 + lane;
      const int n0 = (t % g.nt) * BN + hf * CW;
      if (p < g.npix) {
#pragma unroll
        for (int j = 0; j < CW; j += 8) {
          float v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = acc[j + u];
          epi(p, n0 + j, g.N, v);
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

// ------------------------------------------------------------------ host side

__global__ void split_lo_kernel(const float4* __restrict__ w, float4* __restrict__ lo,
                                long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = w[i];
    float4 h, l;
    split(v.x, h.x, l.x); split(v.y, h.y, l.y);
    split(v.z, h.z, l.z); split(v.w, h.w, l.w);
    lo[i] = l;
  }
}

inline bool encode(CUtensorMap* m, const float* p, int rank, const cuuint64_t* dims,
                   const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle sw) {
  const cuuint32_t es[3] = {1, 1, 1};
  return encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank,
                                const_cast<float*>(p), dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, bool DG, class EPI>
bpx_status_t run(const float* a, const float* w, float* wlo, int n, int H, int W, int Cin,
                 int Cout, EPI epi, cudaStream_t st) {
  using Cf = Cfg<BN>;
  // BN = 64 leaves TMEM for 6 A stages (64 + 64 accumulator columns); use
  // them when the halo ring still fits in shared memory.
  using Cf6 = Cfg<64, 6>;
  Geo g;
  g.H = H; g.W = W;
  g.C = DG ? Cout : Cin;
  g.N = DG ? Cin : Cout;
  g.npix = n * H * W;
  g.mt = cdiv(g.npix, 128);
  g.nt = g.N / BN;
  g.tiles = g.mt * g.nt;
  g.hrows = 128 + 2 * W + 2;
  g.nhbox = cdiv(g.hrows, 256);
  g.hbox = cdiv(cdiv(g.hrows, g.nhbox), 8) * 8;
  g.halo_bytes = g.nhbox * g.hbox * 128;
  const bool deep = BN == 64 && Cf6::smem(g.halo_bytes) <= 227 * 1024;
  const int smem = deep ? Cf6::smem(g.halo_bytes) : Cf::smem(g.halo_bytes);
  if (smem > 227 * 1024) return BPX_ERR_INVALID_ARGUMENT;
  CUtensorMap ta, tb;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)g.C, (cuuint64_t)g.npix};
    const cuuint64_t strides[1] = {(cuuint64_t)g.C * 4};
    const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)g.hbox};
    if (!encode(&ta, a, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return BPX_ERR_INVALID_ARGUMENT;
  }
  CUtensorMap tbl;
  for (int v = 0; v < 2; ++v) {
    const float* src = v ? wlo : w;
    CUtensorMap* m = v ? &tbl : &tb;
    if (DG) {       // w as [Cout][9][Cin]: box 32 ci x 1 tap x 32 co, MN-major
      const cuuint64_t dims[3] = {(cuuint64_t)Cin, 9, (cuuint64_t)Cout};
      const cuuint64_t strides[2] = {(cuuint64_t)Cin * 4, (cuuint64_t)9 * Cin * 4};
      const cuuint32_t box[3] = {32, 1, (cuuint32_t)BK};
      if (!encode(m, src, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
        return BPX_ERR_INVALID_ARGUMENT;
    } else {        // w as [Cout][9*Cin]: box 32 k x BN rows, K-major
      const cuuint64_t dims[2] = {(cuuint64_t)9 * Cin, (cuuint64_t)Cout};
      const cuuint64_t strides[1] = {(cuuint64_t)9 * Cin * 4};
      const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)BN};
      if (!encode(m, src, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
        return BPX_ERR_INVALID_ARGUMENT;
    }
  }
  const long long n4 = (long long)Cout * 9 * Cin / 4;
  int sgrid = (int)cdivll(n4, 256);
  if (sgrid > 4 * num_sms()) sgrid = 4 * num_sms();
  split_lo_kernel<<<sgrid, 256, 0, st>>>(reinterpret_cast<const float4*>(w),
                                         reinterpret_cast<float4*>(wlo), n4);
  constexpr int DEEP = BN == 64 ? 6 : 4;
  auto kern = deep ? fdt_kernel<BN, DEEP, DG, EPI> : fdt_kernel<BN, 4, DG, EPI>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fdt_kernel<BN, 4, DG, EPI>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(fdt_kernel<BN, DEEP, DG, EPI>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int grid = g.tiles < num_sms() ? g.tiles : num_sms();
  kern<<<grid, NTHREADS, smem, st>>>(ta, tb, tbl, g, epi);
  return launch_status(2);
}

inline int bn_for(int N) { return N % 128 == 0 ? 128 : 64; }

}  // namespace fdt

// ============================================================ entry points

// W <= 224 keeps two halo slots + four B stages inside 227 KB of smem.
bool fdt_conv_ok(int cin, int cout, int w) { return cin % 64 == 0 && cout % 64 == 0 && w <= 224; }

size_t fdt_conv_ws(int cin, int cout) { return (size_t)cout * 9 * cin * sizeof(float); }

bpx_status_t fdt_conv_fwd(const float* x, const float* w, const float* bias, float* y, int n,
                          int h, int w_, int cin, int cout, int relu, void* ws,
                          size_t ws_bytes, cudaStream_t st) {
  if (!fdt_conv_ok(cin, cout, w_) || !aligned16(x) || !aligned16(w) || !aligned16(y))
    return BPX_ERR_INVALID_ARGUMENT;
  if ((long long)n * h * w_ == 0) return launch_status(0);
  if (ws_bytes < fdt_conv_ws(cin, cout) || !aligned16(ws)) return BPX_ERR_WORKSPACE;
  float* wlo = static_cast<float*>(ws);
  fdt::EBiasAct epi{y, bias, relu};
  if (fdt::bn_for(cout) == 64)
    return fdt::run<64, false>(x, w, wlo, n, h, w_, cin, cout, epi, st);
  return fdt::run<128, false>(x, w, wlo, n, h, w_, cin, cout, epi, st);
}

bpx_status_t fdt_conv_dgrad(const float* dz, const float* w, const float* mask, float* dx,
                            int n, int h, int w_, int cin, int cout, void* ws,
                            size_t ws_bytes, cudaStream_t st) {
  if (!fdt_conv_ok(cin, cout, w_) || !aligned16(dz) || !aligned16(w) || !aligned16(dx) ||
      (mask && !aligned16(mask)))
    return BPX_ERR_INVALID_ARGUMENT;
  if ((long long)n * h * w_ == 0) return launch_status(0);
  if (ws_bytes < fdt_conv_ws(cin, cout) || !aligned16(ws)) return BPX_ERR_WORKSPACE;
  float* wlo = static_cast<float*>(ws);
  fdt::EMask epi{dx, mask};
  if (fdt::bn_for(cin) == 64)
    return fdt::run<64, true>(dz, w, wlo, n, h, w_, cin, cout, epi, st);
  return fdt::run<128, true>(dz, w, wlo, n, h, w_, cin, cout, epi, st);
}

}  // namespace bpx
