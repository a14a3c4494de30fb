// tcgen05 engine for the dense layers' forward and data gradient at
// per-GPU batches <= 32 -- a weight stream (fc1: 411 MB of weights per pass)
// that tensor cores keep at the TMA/L2 rate instead of the FFMA rate:
//
//   fwd   D[o][n] = sum_k W[o][k]  x[n][k]     A = W (K-major)   -> y  = act(D^T + b)
//   dgrad D[i][n] = sum_o W[o][i] dy[n][o]     A = W^T (MN-major) -> dx = D^T * mask
//
// M = weight rows/columns in 128-row tiles, N = the batch padded to 16 or 32,
// K split over CTAs (fixed-order finish kernel applies the epilogue).  A is
// one TMA box (fwd: 32 k x 128 rows, 128-B swizzle) or four (dgrad: 32 i x
// 32 o, 128-B swizzle) per 32-K stage; A converter warps split it into TF32
// hi/lo in TMEM (TS form) and write the activations' lo split next to their
// TMA tile in shared memory.  3xTF32 with 128-K chunk promotion into RN fp32
// registers, as in the conv engines.
//
// CTA: 10 warps.  warp 0 TMA, warp 1 MMA + TMEM owner, 2-5 A converters,
// 6-9 drain.
#include "tma_host.h"
#include "tc_ptx.cuh"
#include "tc_api.h"

namespace bpx {
namespace dtc {
using namespace tcx;

constexpr int BK = 32;
// 3 stages so that two CTAs share an SM (TMEM 2 x 256 columns, smem 2 x
// 73 KB): twice the weight streams in flight per SM.  B200 A/B against one
// CTA with 7 stages: fc1 fwd 0.097 -> 0.084 ms, dgrad 0.118 -> 0.093 ms,
// fc2 0.028 / 0.036 -> 0.023 / 0.031 ms (B=32).
#ifndef DTC_S
#define DTC_S 3
#endif
constexpr int S = DTC_S;                  // stages (TMEM: 2*32 acc + S*64 A columns)
constexpr int CPS = S <= 3 ? 2 : 1;       // CTAs per SM
constexpr int PCH = 4;                    // stages per promotion chunk (K = 128)
constexpr int A_BYTES = 128 * BK * 4;     // 16 KB
constexpr int NTHREADS = 10 * 32;
constexpr int TMA_WARP = 0, MMA_WARP = 1, DR0 = 6;

template <int NB>
struct Cfg {
  static constexpr int B_BYTES = NB * BK * 4;
  static constexpr int STAGE = A_BYTES + 2 * B_BYTES;
  static constexpr int A_COL = 2 * NB;
  static constexpr int SMEM = 1024 + S * STAGE + 256;
  static_assert(A_COL + S * 2 * BK <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "smem budget");
};

struct Geo {
  int M, K, batch;
  int kslice;                // K elements per split (multiple of BK)
  int dgrad;
  float* part;               // [splits][batch][M]
};

template <int NB, bool DG>
__global__ void __launch_bounds__(NTHREADS, CPS)
dtc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
           Geo g) {
  using Cf = Cfg<NB>;
  extern __shared__ char smem_raw[];
  // offset from smem_raw (not a uintptr_t round trip) keeps the shared address space: LDS/STS, not generic LD/ST
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cf::STAGE);
  uint64_t* aready = full + S;
  uint64_t* empty = aready + S;
  uint64_t* hfull = empty + S;
  uint64_t* hfree = hfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * 128;
  const int k0 = blockIdx.y * g.kslice;
  const int nst = max(0, min(g.K, k0 + g.kslice) - k0 + BK - 1) / BK;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&aready[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hfree[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) tmem_alloc(tmem_slot, 512 / CPS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == TMA_WARP) {
    if (lane == 0) {
      tma_prefetch_desc(&ta);
      tma_prefetch_desc(&tb);
      for (int i = 0; i < nst; ++i) {
        const int s = i % S;
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        const int k = k0 + i * BK;
        char* st = smem + s * Cf::STAGE;
        mbar_expect_tx(&full[s], A_BYTES + Cf::B_BYTES);
        if (DG) {           // W[o][i] rows o = k..k+31, columns i = m0 + 32j
          for (int j = 0; j < 4; ++j) tma_load_2d(st + j * 4096, &ta, m0 + 32 * j, k, &full[s]);
        } else {            // W[o][k] rows o = m0..m0+127, columns k..k+31
          tma_load_2d(st, &ta, k, m0, &full[s]);
        }
        tma_load_2d(st + A_BYTES, &tb, k, 0, &full[s]);
      }
    }
  } else if (warp == MMA_WARP) {
    {                                   // whole warp; elect.sync issues
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                                 ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      for (int i = 0; i < nst; ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        const int c = i / PCH, b = c & 1;
        if (i % PCH == 0 && c >= 2) {
          mbar_wait(&hfree[b], ((c >> 1) - 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&aready[s], ph);
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t d = tmem + b * NB;
        const uint32_t ah = tmem + Cf::A_COL + s * 2 * BK, al = ah + BK;
        const uint32_t bh = smem_u32(smem + s * Cf::STAGE + A_BYTES);
        const uint32_t bl = bh + Cf::B_BYTES;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint64_t dbh = make_desc_sw128(bh + ks * 32, 16, 1024);
          const uint64_t dbl = make_desc_sw128(bl + ks * 32, 16, 1024);
          const uint32_t acc = (i % PCH != 0 || ks > 0) ? 1u : 0u;
          mma_ts_elect(d, al + 8 * ks, dbh, idesc, acc);
          mma_ts_elect(d, ah + 8 * ks, dbl, idesc, 1u);
          mma_ts_elect(d, ah + 8 * ks, dbh, idesc, 1u);
        }
        tc_commit_elect(&empty[s]);
        if (i % PCH == PCH - 1 || i == nst - 1) tc_commit_elect(&hfull[b]);
      }
    }
  } else if (warp < DR0) {
    // A converters: thread = TMEM lane = weight row/column r of the tile
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + Cf::A_COL;
    for (int i = 0; i < nst; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      char* st = smem + s * Cf::STAGE;
      {   // the activations' lo split, granule for granule (same swizzle)
        const int t = (warp - 2) * 32 + lane;
#pragma unroll
        for (int j = t; j < Cf::B_BYTES / 16; j += 128) {
          const float4 v = *reinterpret_cast<const float4*>(st + A_BYTES + 16 * j);
          float h, l0, l1, l2, l3;
          split(v.x, h, l0); split(v.y, h, l1); split(v.z, h, l2); split(v.w, h, l3);
          *reinterpret_cast<float4*>(st + A_BYTES + Cf::B_BYTES + 16 * j) =
              make_float4(l0, l1, l2, l3);
        }
        fence_proxy_async();        // generic stores -> the MMA's async-proxy reads
      }
      float hi[BK], lo[BK];
      if (DG) {     // box q holds rows k (o) x 32 columns (i); lane reads column `lane`
        const char* box = st + q * 4096;
#pragma unroll
        for (int k = 0; k < BK; ++k) {
          const float v = *reinterpret_cast<const float*>(
              box + k * 128 + ((((lane >> 2) ^ (k & 7))) << 4) + (lane & 3) * 4);
          split(v, hi[k], lo[k]);
        }
      } else {      // row r: 32 k values, 128-B swizzled granules
        const char* row = st + r * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = *reinterpret_cast<const float4*>(row + ((j ^ (r & 7)) << 4));
          split(v.x, hi[4 * j + 0], lo[4 * j + 0]);
          split(v.y, hi[4 * j + 1], lo[4 * j + 1]);
          split(v.z, hi[4 * j + 2], lo[4 * j + 2]);
          split(v.w, hi[4 * j + 3], lo[4 * j + 3]);
        }
      }
      if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);   // (implied by full; explicit for TMEM)
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
  } else {
    // drain: TMEM chunks -> RN fp32 registers; write D^T partial [split][n][m]
    const int q = warp & 3;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16);
    float acc[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[j] = 0.f;
    const int nch = (nst + PCH - 1) / PCH;
    for (int c = 0; c < nch; ++c) {
      const int b = c & 1;
      mbar_wait(&hfull[b], (c >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < NB; j += 8) {
        uint32_t rr[8];
        tmem_ld8(lanebase + b * NB + j, rr);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[j + u] += __uint_as_float(rr[u]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&hfree[b]);
    }
    const int m = m0 + q * 32 + lane;
    if (m < g.M) {
      float* o = g.part + (long long)blockIdx.y * g.batch * g.M + m;
#pragma unroll
      for (int n = 0; n < NB; ++n)
        if (n < g.batch) o[(long long)n * g.M] = acc[n];
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_free(tmem, 512 / CPS);
  }
}

// out[n][m] = epilogue(sum_s part[s][n][m]); mode 0: + bias, ReLU; mode 1: mask.
// (Folded into the GEMM as a last-CTA-per-tile finish it measured slower:
// one CTA per M tile sums all the parts at the kernel's tail.)
__global__ void dtc_finish(const float* __restrict__ part, int splits, long long NM, int M,
                           const float* __restrict__ bias, int relu,
                           const float* __restrict__ mask, int mode, float* __restrict__ out) {
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

inline bool encode2d(CUtensorMap* m, const float* p, long long inner, long long outer,
                     int box_inner, int box_outer) {
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)inner * 4};
  const cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  const cuuint32_t es[2] = {1, 1};
  return encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p), dims,
                      strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifndef DTC_DGW
#define DTC_DGW 2          // dgrad: waves of CTA slots
#endif
#ifndef DTC_MINST
#define DTC_MINST 8        // stages per split, at least (4: fc2 dgrad 0.028 vs 0.025 ms)
#endif
inline int nb_for(int batch) { return batch <= 16 ? 16 : 32; }   // M=128 MMAs take N % 16 == 0

// split count: one wave of CTA slots (CPS per SM) for the forward, two for the data gradient
// (its four MN-major boxes per stage keep more CTAs busy), at least 4
// stages each (B200 A/B at fc1/fc2, B = 4 and 32: 4 waves was 8-25 % slower)
inline void geometry(int M, int K, bool dg, int& splits, int& kslice) {
  const int mt = cdiv(M, 128);
  const int kst = cdiv(K, BK);
  const int slots = CPS * num_sms();
  int want = dg ? cdiv(DTC_DGW * slots, mt) : slots / mt;
  if (want > kst / DTC_MINST) want = kst / DTC_MINST;
  if (want < 1) want = 1;
  kslice = cdiv(kst, want) * BK;
  splits = cdiv(K, kslice);
}

template <int NB, bool DG>
bpx_status_t launch(const CUtensorMap& ta, const CUtensorMap& tb, Geo g, int mt, int splits,
                    cudaStream_t st) {
  auto kern = dtc_kernel<NB, DG>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<NB>::SMEM);
    attr = true;
  }
  kern<<<dim3(mt, splits), NTHREADS, Cfg<NB>::SMEM, st>>>(ta, tb, g);
  return launch_status();
}

// fwd: out[b][M] with W [M][K], act [b][K];  dgrad: W [K][M] (i.e. W[o][i], M = in)
bpx_status_t run(bool dg, const float* W, const float* act, int batch, int M, int K,
                 const float* bias, int relu, const float* mask, float* out, float* ws,
                 size_t ws_floats, cudaStream_t st) {
  int splits, kslice;
  geometry(M, K, dg, splits, kslice);
  const int mt = cdiv(M, 128);
  const int nb = nb_for(batch);
  const size_t need = (size_t)splits * batch * M + 4;
  if (ws_floats < need) return BPX_ERR_WORKSPACE;
  float* part = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(ws) + 15) & ~uintptr_t(15));
  CUtensorMap ta, tb;
  const bool ok = (dg ? encode2d(&ta, W, M, K, 32, 32) : encode2d(&ta, W, K, M, 32, 128)) &&
                  encode2d(&tb, act, K, batch, 32, nb);
  if (!ok) return BPX_ERR_INVALID_ARGUMENT;
  Geo g{M, K, batch, kslice, dg ? 1 : 0, part};
  bpx_status_t s;
  if (nb == 16) s = dg ? launch<16, true>(ta, tb, g, mt, splits, st)
                            : launch<16, false>(ta, tb, g, mt, splits, st);
  else s = dg ? launch<32, true>(ta, tb, g, mt, splits, st)
              : launch<32, false>(ta, tb, g, mt, splits, st);
  if (s != BPX_OK) return s;
  const long long NM = (long long)batch * M;
  int fg = (int)cdivll(NM, 256);
  if (fg > 8 * num_sms()) fg = 8 * num_sms();
  dtc_finish<<<fg, 256, 0, st>>>(part, splits, NM, M, bias, relu, mask, dg ? 1 : 0, out);
  return launch_status();
}

}  // namespace dtc

// Shapes: batch 1..32, features multiples of 32 (TMA rows of 128 B).
bool dtc_linear_ok(int b, int in, int out) {
  return b >= 1 && b <= 32 && in % 32 == 0 && out % 32 == 0;
}

size_t dtc_linear_ws(int b, int in, int out) {
  if (!dtc_linear_ok(b, in, out)) return 0;
  int s1, k1, s2, k2;
  dtc::geometry(out, in, false, s1, k1);    // fwd: M = out, K = in
  dtc::geometry(in, out, true, s2, k2);     // dgrad: M = in, K = out
  const size_t a = (size_t)s1 * b * out;
  const size_t c = (size_t)s2 * b * in;
  return ((a > c ? a : c) + 4) * sizeof(float);
}

bpx_status_t dtc_linear_fwd(const float* x, const float* w, const float* bias, float* y, int b,
                            int in, int out, int relu, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  if (b == 0) return launch_status(0);
  if (!dtc_linear_ok(b, in, out) || !aligned16(x) || !aligned16(w) || !aligned16(ws))
    return BPX_ERR_UNSUPPORTED;
  return dtc::run(false, w, x, b, out, in, bias, relu, nullptr, y, static_cast<float*>(ws),
                  ws_bytes / sizeof(float), st);
}

bpx_status_t dtc_linear_dgrad(const float* dy, const float* w, const float* mask, float* dx,
                              int b, int in, int out, void* ws, size_t ws_bytes,
                              cudaStream_t st) {
  if (b == 0) return launch_status(0);
  if (!dtc_linear_ok(b, in, out) || !aligned16(dy) || !aligned16(w) || !aligned16(ws))
    return BPX_ERR_UNSUPPORTED;
  return dtc::run(true, w, dy, b, in, out, nullptr, 0, mask, dx, static_cast<float*>(ws),
                  ws_bytes / sizeof(float), st);
}

}  // namespace bpx
