// tcgen05 "TS" engine for the conv forward and data-gradient GEMMs:
//
//   D[m][n] = sum_k A(m,k) B(n,k),  A = im2col rows (pixels x tap*C),
//                                   B = weights (pre-split, pre-tiled)
//
// Why a second engine: in the all-shared-memory design every operand byte
// crosses the L1/LSU pipe three times (LDG + st.shared hi + st.shared lo)
// and ncu shows that pipe at ~80% with the tensor pipe at ~20%.  Here
//   * A (the im2col gather, the only operand with reuse in L1) is loaded
//     row-per-thread, split into TF32 hi/lo in registers and written
//     straight into TMEM with tcgen05.st -- no shared-memory traffic;
//     the MMA reads A from TMEM (`tcgen05.mma ... [d], [a_tmem], b_desc`);
//   * B is a weight tensor: one tiny prep kernel per call splits it into
//     hi/lo and lays it out as the exact shared-memory image of every
//     (n-tile, k-block) stage, so a stage is ONE contiguous cp.async.bulk
//     (TMA engine) with mbarrier complete_tx -- no LSU work at all;
//   * accumulation uses the same two-buffer TMEM chunk promotion into RN
//     fp32 registers as tc_engine.cu (fp32-level accuracy vs fp64).
//
// CTA (576 threads, one per SM): warps 0-7 A producers (two groups of four
// warps, one lane quadrant each, alternating k-blocks), warps 8-15 drain +
// epilogue, warp 16 MMA issuer + TMEM allocator, warp 17 B bulk loader.
#include "common.cuh"
#include "tc_api.h"

namespace bpx {
namespace ts {

constexpr int BM = 128;
constexpr int BK = 16;          // K per stage (2 MMA k-steps of 8)
constexpr int P = 4;            // k-blocks per promotion chunk
constexpr int S = 6;            // pipeline stages (A in TMEM, B in smem)
constexpr int ND = 256;         // drain threads (warps 8-15)
constexpr int MMA_WARP = 16;   // warp 17 = B bulk loader
constexpr int NTHREADS = 18 * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(bar)) : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T, kind::tf32
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d), "r"(a), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])),
        "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])),
        "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7])
      : "r"(taddr));
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void split(float a, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
  lo = a - hi;
}

// ---------------------------------------------------------------- B image
// Stage image of one (n-tile, k-block): [hi | lo], each 4 k-chunks x
// (BN/8) row groups x 8 rows x 16 B (K-major, no swizzle; SBO = 128 B,
// LBO = BN*16 B).  Image order: n-tile major, then k-block.
template <int BN>
struct Img {
  static constexpr int HALF = BN * BK * 4;
  static constexpr int STAGE = 2 * HALF;
};

// B(n, k) source for the two conv GEMMs:
//   fwd   : B(co, tap*Cin + ci)   = w[co][tap][ci]       (N = Cout, K = 9 Cin)
//   dgrad : B(ci, tap*Cout + co)  = w[co][8 - tap][ci]   (N = Cin,  K = 9 Cout)
template <int BN>
__global__ void prep_weights(const float* __restrict__ w, int Cin, int Cout, int dgrad,
                             char* __restrict__ img) {
  const int N = dgrad ? Cin : Cout;
  const int Kd = dgrad ? Cout : Cin;        // inner (contiguous in k) dim
  const int K = 9 * Kd;
  const int ntile = (N + BN - 1) / BN, nkb = K / BK;
  const long long units = (long long)ntile * BN * (K / 4);
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < units;
       u += (long long)gridDim.x * blockDim.x) {
    const int kc = (int)(u % (K / 4));
    const int n = (int)(u / (K / 4));
    const int k = kc * 4;
    float v[4];
    if (n < N) {
      const int tap = k / Kd, c = k - tap * Kd;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[j] = dgrad ? w[((long long)(c + j) * 9 + (8 - tap)) * Cin + n]
                     : w[((long long)n * 9 + tap) * Cin + c + j];
      }
    } else {
      v[0] = v[1] = v[2] = v[3] = 0.f;
    }
    float4 h, l;
    split(v[0], h.x, l.x); split(v[1], h.y, l.y);
    split(v[2], h.z, l.z); split(v[3], h.w, l.w);
    const int nt = n / BN, r = n - nt * BN;
    const int kb = k / BK, chunk = (k % BK) / 4;
    char* st = img + ((long long)nt * nkb + kb) * Img<BN>::STAGE;
    const int off = chunk * (BN * 16) + (r >> 3) * 128 + (r & 7) * 16;
    *reinterpret_cast<float4*>(st + off) = h;
    *reinterpret_cast<float4*>(st + Img<BN>::HALF + off) = l;
  }
}

// ---------------------------------------------------------------- epilogues
struct EBiasAct {
  float* out; const float* bias; long long ld; int relu;
  __device__ void operator()(int m, int n0, int N, const float (&v)[8]) const {
    float* o = out + m * ld + n0;
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float t = v[j] + ((bias && n0 + j < N) ? __ldg(bias + n0 + j) : 0.f);
      r[j] = relu ? fmaxf(t, 0.f) : t;
    }
    if (n0 + 8 <= N) {
      *reinterpret_cast<float4*>(o) = make_float4(r[0], r[1], r[2], r[3]);
      *reinterpret_cast<float4*>(o + 4) = make_float4(r[4], r[5], r[6], r[7]);
    } else {
      for (int j = 0; j < 8 && n0 + j < N; ++j) o[j] = r[j];
    }
  }
};
struct EMask {
  float* out; const float* mask; long long ld;
  __device__ void operator()(int m, int n0, int N, const float (&v)[8]) const {
    float* o = out + m * ld + n0;
    const float* mk = mask ? mask + m * ld + n0 : nullptr;
    if (n0 + 8 <= N) {
      float4 a = make_float4(v[0], v[1], v[2], v[3]);
      float4 b = make_float4(v[4], v[5], v[6], v[7]);
      if (mk) {
        float4 p = __ldg(reinterpret_cast<const float4*>(mk));
        float4 q = __ldg(reinterpret_cast<const float4*>(mk + 4));
        a.x = p.x > 0.f ? a.x : 0.f; a.y = p.y > 0.f ? a.y : 0.f;
        a.z = p.z > 0.f ? a.z : 0.f; a.w = p.w > 0.f ? a.w : 0.f;
        b.x = q.x > 0.f ? b.x : 0.f; b.y = q.y > 0.f ? b.y : 0.f;
        b.z = q.z > 0.f ? b.z : 0.f; b.w = q.w > 0.f ? b.w : 0.f;
      }
      *reinterpret_cast<float4*>(o) = a;
      *reinterpret_cast<float4*>(o + 4) = b;
    } else {
      for (int j = 0; j < 8 && n0 + j < N; ++j)
        o[j] = (mk && !(mk[j] > 0.f)) ? 0.f : v[j];
    }
  }
};

// ---------------------------------------------------------------- kernel
template <int BN>
struct Cfg {
  static_assert(BN == 64 || BN == 128, "BN");
  static constexpr int B_STAGE = Img<BN>::STAGE;
  static constexpr int SMEM = S * B_STAGE + 1024;
  static constexpr int A_COL = 2 * BN;                 // A stages after H0, H1
  static constexpr int TMEM_COLS = 512;
  static constexpr int CW = BN / 2;
  static_assert(A_COL + S * 2 * BK <= TMEM_COLS, "TMEM budget");
};

// im2col A rows: x NHWC [n,H,W,C], row m = output pixel, k = tap*C + c.
// C % 16 == 0, so a 16-wide k-block lies inside one tap.
template <int BN, class EPI>
__global__ void __launch_bounds__(NTHREADS, 1)
ts_kernel(const float* __restrict__ x, int H, int W, int C, int npix,
          const char* __restrict__ bimg, EPI epi, int N, int K) {
  using Cf = Cfg<BN>;
  extern __shared__ __align__(1024) char smem[];
  char* bst = smem;
  uint64_t* afull = reinterpret_cast<uint64_t*>(smem + S * Cf::B_STAGE);
  uint64_t* bfull = afull + S;
  uint64_t* empty = bfull + S;
  uint64_t* hfull = empty + S;
  uint64_t* hfree = hfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * BM, nt = blockIdx.y, n0 = nt * BN;
  const int nk = K / BK;
  const int nc = (nk + P - 1) / P;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&afull[s], 128);
      mbar_init(&bfull[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hfree[b], ND);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(Cf::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // -------------------------------------------- A producers
    const int q = warp & 3, grp = warp >> 2;
    const int m = m0 + q * 32 + lane;
    const bool rowok = m < npix;
    int img = 0, oh = 0, ow = 0;
    if (rowok) {
      const int hw = H * W;
      img = m / hw;
      const int rem = m - img * hw;
      oh = rem / W;
      ow = rem - oh * W;
    }
    const float* xrow = x + (long long)img * H * W * C;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + Cf::A_COL;
    auto load = [&](int kb, float4 (&v)[4]) {
      const int k0 = kb * BK;
      const int tap = k0 / C, c0 = k0 - tap * C;
      const int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
      if (rowok && (unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W) {
        const float4* p = reinterpret_cast<const float4*>(xrow + ((long long)ih * W + iw) * C + c0);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = __ldg(p + j);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    float4 cur[4], nxt[4];
    int kb = grp;
    if (kb < nk) load(kb, cur);
    for (; kb < nk; kb += 2) {
      if (kb + 2 < nk) load(kb + 2, nxt);
      const int s = kb % S;
      if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
      tc_fence_after();
      float hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        split(cur[j].x, hi[4 * j + 0], lo[4 * j + 0]);
        split(cur[j].y, hi[4 * j + 1], lo[4 * j + 1]);
        split(cur[j].z, hi[4 * j + 2], lo[4 * j + 2]);
        split(cur[j].w, hi[4 * j + 3], lo[4 * j + 3]);
      }
      const uint32_t a = lanebase + s * 2 * BK;
      tmem_st16(a, hi);
      tmem_st16(a + BK, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&afull[s]);
#pragma unroll
      for (int j = 0; j < 4; ++j) cur[j] = nxt[j];
    }
  } else if (warp < MMA_WARP) {
    // -------------------------------------------- drain + epilogue
    const int q = warp & 3;
    const int half = (warp - 8) >> 2;
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
    if (m < npix) {
#pragma unroll
      for (int j = 0; j < Cf::CW; j += 8) {
        const int n = n0 + cbase + j;
        if (n < N) {
          float v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) v[t] = acc[j + t];
          epi(m, n, N, v);
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // -------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(BN);
      constexpr uint32_t LBO = BN * 16, SBO = 128;
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
          const uint32_t bh = smem_u32(bst + s * Cf::B_STAGE);
          const uint32_t bl = bh + Img<BN>::HALF;
          const uint32_t ah = tmem + Cf::A_COL + s * 2 * BK;
          const uint32_t al = ah + BK;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint64_t dbh = make_desc(bh + ks * 2 * LBO, LBO, SBO);
            const uint64_t dbl = make_desc(bl + ks * 2 * LBO, LBO, SBO);
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
  } else {
    // -------------------------------------------- B bulk loader
    if (lane == 0) {
      const char* src = bimg + (long long)nt * nk * Cf::B_STAGE;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % S;
        if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
        mbar_expect_tx(&bfull[s], Cf::B_STAGE);
        bulk_g2s(bst + s * Cf::B_STAGE, src + (long long)kb * Cf::B_STAGE, Cf::B_STAGE,
                 &bfull[s]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                 ::"r"(tmem), "r"(Cf::TMEM_COLS));
  }
}

template <int BN, class EPI>
bpx_status_t run(const float* x, int n, int H, int W, int C, const float* w, int Cin,
                 int Cout, int dgrad, EPI epi, int N, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  using Cf = Cfg<BN>;
  const int K = 9 * C;
  const int ntile = (N + BN - 1) / BN;
  const size_t img_bytes = (size_t)ntile * (K / BK) * Cf::B_STAGE;
  if (ws_bytes < img_bytes) return BPX_ERR_WORKSPACE;
  char* img = static_cast<char*>(ws);
  long long units = (long long)ntile * BN * (K / 4);
  int pgrid = (int)std::min<long long>(cdivll(units, 256), 8LL * num_sms());
  prep_weights<BN><<<pgrid, 256, 0, st>>>(w, Cin, Cout, dgrad, img);
  auto kern = ts_kernel<BN, EPI>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM);
    attr = true;
  }
  const int npix = n * H * W;
  dim3 grid(cdiv(npix, BM), ntile, 1);
  kern<<<grid, NTHREADS, Cf::SMEM, st>>>(x, H, W, C, npix, img, epi, N, K);
  return launch_status(2);
}

inline int bn_for(int N) { return N <= 64 ? 64 : 128; }

}  // namespace ts

// ============================================================ entry points
// Shapes taken: the gathered channel count (Cin for fwd, Cout for dgrad) a
// multiple of 16 and the output channel count a multiple of 8.

bool ts_conv_ok(int cin, int cout) { return cin % 16 == 0 && cout % 16 == 0; }

size_t ts_conv_ws(int cin, int cout) {
  // weight image: 2 (hi/lo) x N_padded x K floats, for either orientation
  auto img = [](int N, int K) {
    int bn = ts::bn_for(N);
    return (size_t)((N + bn - 1) / bn) * bn * K * 8;
  };
  size_t a = img(cout, 9 * cin), b = img(cin, 9 * cout);
  return a > b ? a : b;
}

bpx_status_t ts_conv_fwd(const float* x, const float* w, const float* bias, float* y, int n,
                         int h, int w_, int cin, int cout, int relu, void* ws,
                         size_t ws_bytes, cudaStream_t st) {
  if ((long long)n * h * w_ == 0) return BPX_OK;
  ts::EBiasAct epi{y, bias, cout, relu};
  if (ts::bn_for(cout) == 64)
    return ts::run<64>(x, n, h, w_, cin, w, cin, cout, 0, epi, cout, ws, ws_bytes, st);
  return ts::run<128>(x, n, h, w_, cin, w, cin, cout, 0, epi, cout, ws, ws_bytes, st);
}

bpx_status_t ts_conv_dgrad(const float* dz, const float* w, const float* mask, float* dx,
                           int n, int h, int w_, int cin, int cout, void* ws,
                           size_t ws_bytes, cudaStream_t st) {
  if ((long long)n * h * w_ == 0) return BPX_OK;
  ts::EMask epi{dx, mask, cin};
  if (ts::bn_for(cin) == 64)
    return ts::run<64>(dz, n, h, w_, cout, w, cin, cout, 1, epi, cin, ws, ws_bytes, st);
  return ts::run<128>(dz, n, h, w_, cout, w, cin, cout, 1, epi, cin, ws, ws_bytes, st);
}

}  // namespace bpx
