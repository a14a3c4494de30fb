// tcgen05 / TMEM implicit-GEMM engine, fp32-accurate via a 3xTF32 split.
//
//   D[m][n] = sum_k A(m,k) B(n,k)    (fp32 in / out)
//
// Split: every operand value a becomes hi = a with the low 13 mantissa bits
// cleared (exact in TF32) and lo = a - hi (exact in fp32); the tensor core
// computes hi*hi + (hi*lo + lo*hi), dropping lo*lo (~2^-22 relative).
//
// Accumulation: the tensor core's fp32 accumulate truncates (measured on
// B200: error grows linearly with K, ~6.7e-9*K normwise, ~20x the CPU fp32
// error at K=4608).  So the big hi*hi term is accumulated in short K-chunks
// (P k-blocks = 64 K) into two ping-pong TMEM buffers, and dedicated "drain"
// warps promote each finished chunk into fp32 registers with round-to-
// nearest adds (the Blackwell analogue of DeepGEMM's FP8 promotion).  The
// cross terms, ~2^-11 smaller, go to a third TMEM accumulator where the
// truncation is negligible.  Result: CPU-fp32-level accuracy vs fp64.
//
// CTA (544 threads, one CTA per SM):
//   warps 0-7   producers: global -> registers (im2col gathers; 4x4 register
//               transposes for MN-major sources) -> hi/lo split -> st.shared
//               in the UMMA K-major no-swizzle layout (8-row groups padded to
//               144 B so MN-major stores are bank-conflict free) ->
//               fence.proxy.async -> mbarrier arrive.
//   warps 8-15  drain + epilogue: tcgen05.ld their TMEM lane quadrant, fp32
//               RN accumulate in registers, then bias/ReLU/mask + stores.
//   warp 16     TMEM alloc + single-thread tcgen05.mma issue; stages are
//               released with tcgen05.commit onto per-stage empty barriers.
#include "common.cuh"
#include "tc_api.h"

namespace bpx {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 16;                 // tf32 elements per stage (2 MMA k-steps)
constexpr int P = 4;                   // k-blocks per promotion chunk (K = 64)
constexpr int NPROD = 256;             // producer threads (warps 0-7)
constexpr int NDRAIN = 256;            // drain / epilogue threads (warps 8-15)
constexpr int MMA_WARP = 16;
constexpr int NTHREADS = NPROD + NDRAIN + 32;
constexpr int SBO = 144;               // 8-row group stride (128 B + 16 B pad)

// ---------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// 8 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_NONE canonical layout
// ((8,m),2):((16B,SBO),LBO); descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// instruction descriptor: D=F32, A=B=TF32, both K-major, M=128, N=n
__host__ __device__ constexpr uint32_t make_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void split(float a, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
  lo = a - hi;
}

// ---------------------------------------------------------------- loaders
// K-major sources: chunk(row, k) = float4 of A(row, k..k+3).
// MN-major sources: quad(row, k) = float4 of A(row..row+3, k).
// Zero outside [0, rows) x [0, kend).

struct MatK {                 // A(r, k) = p[r*ld + k]
  static constexpr bool KMAJOR = true;
  const float* p; long long ld; int rows;
  __device__ float4 chunk(int r, int k, int kend) const {
    if (r < rows && k < kend) return __ldg(reinterpret_cast<const float4*>(p + r * ld + k));
    return make_float4(0.f, 0.f, 0.f, 0.f);
  }
};
struct MatMN {                // A(r, k) = p[k*ld + r]
  static constexpr bool KMAJOR = false;
  const float* p; long long ld; int rows;
  __device__ float4 quad(int r, int k, int kend) const {
    if (r < rows && k < kend) return __ldg(reinterpret_cast<const float4*>(p + (long long)k * ld + r));
    return make_float4(0.f, 0.f, 0.f, 0.f);
  }
};
// conv fwd A / dgrad A: rows = output pixels, k = tap*C + c (C % 16 == 0)
struct Im2colRows {
  static constexpr bool KMAJOR = true;
  const float* x; int H, W, C, npix;
  __device__ float4 chunk(int m, int k, int kend) const {
    if (m >= npix || k >= kend) return make_float4(0.f, 0.f, 0.f, 0.f);
    int hw = H * W;
    int img = m / hw, rem = m - img * hw;
    int oh = rem / W, ow = rem - oh * W;
    int tap = k / C, c = k - tap * C;
    int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
    if ((unsigned)ih >= (unsigned)H || (unsigned)iw >= (unsigned)W)
      return make_float4(0.f, 0.f, 0.f, 0.f);
    return __ldg(reinterpret_cast<const float4*>(x + ((long long)(img * H + ih) * W + iw) * C + c));
  }
};
// wgrad B: rows n = tap*C + c (N = 9C), k = pixel (MN-major along c)
struct Im2colCols {
  static constexpr bool KMAJOR = false;
  const float* x; int H, W, C, npix;
  __device__ float4 quad(int n, int p, int kend) const {
    if (n >= 9 * C || p >= kend) return make_float4(0.f, 0.f, 0.f, 0.f);
    int tap = n / C, c = n - tap * C;
    int hw = H * W;
    int img = p / hw, rem = p - img * hw;
    int oh = rem / W, ow = rem - oh * W;
    int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
    if ((unsigned)ih >= (unsigned)H || (unsigned)iw >= (unsigned)W)
      return make_float4(0.f, 0.f, 0.f, 0.f);
    return __ldg(reinterpret_cast<const float4*>(x + ((long long)(img * H + ih) * W + iw) * C + c));
  }
};
// dgrad B: B(ci, k = tap'*Cout + co) = w[co][8 - tap'][ci] (MN-major along ci)
struct FlipW {
  static constexpr bool KMAJOR = false;
  const float* w; int Cin, Cout;
  __device__ float4 quad(int ci, int k, int kend) const {
    if (ci >= Cin || k >= kend) return make_float4(0.f, 0.f, 0.f, 0.f);
    int tp = k / Cout, co = k - tp * Cout;
    return __ldg(reinterpret_cast<const float4*>(w + ((long long)co * 9 + (8 - tp)) * Cin + ci));
  }
};


// ---------------------------------------------------------------- epilogues
// called with 8 consecutive columns n0..n0+7 of row m (n0 < N, m < M)
struct EBiasAct {            // out[m*ld + n] = relu?(acc + bias[n])
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
struct EMask {               // out[m*ld + n] = acc * (mask > 0)
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
struct EPartial {            // ws[z][m][n] = acc
  float* ws; long long ld; long long slab;
  __device__ void operator()(int m, int n0, int N, const float (&v)[8]) const {
    float* o = ws + blockIdx.z * slab + m * ld + n0;
    if (n0 + 8 <= N) {
      *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(o + 4) = make_float4(v[4], v[5], v[6], v[7]);
    } else {
      for (int j = 0; j < 8 && n0 + j < N; ++j) o[j] = v[j];
    }
  }
};

// ---------------------------------------------------------------- kernel

template <int BN>
struct Cfg {
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 128, "BN");
  static constexpr int A_BYTES = 4 * (BM / 8) * SBO;   // one of hi / lo
  static constexpr int B_BYTES = 4 * (BN / 8) * SBO;
  static constexpr int STAGE = 2 * (A_BYTES + B_BYTES);
  static constexpr int STAGES = (196608 / STAGE) > 8 ? 8 : (196608 / STAGE);
  static constexpr int SMEM = STAGES * STAGE + 1024;   // + barriers / tmem slot
  static constexpr int TMEM_COLS = 3 * BN <= 64 ? 64 : 3 * BN <= 128 ? 128
                                   : 3 * BN <= 256 ? 256 : 512;
  static constexpr int CW = BN / 2;                    // columns per drain thread
};

// Registers of one operand tile for one stage, owned by one producer thread.
template <class L, int ROWS>
struct Frag {
  static constexpr int UNITS = L::KMAJOR ? ROWS * BK / 4 : ROWS * BK / 16;
  static constexpr int PER = (UNITS + NPROD - 1) / NPROD;
  static constexpr int V = L::KMAJOR ? PER : 4 * PER;
  static constexpr int LBO = (ROWS / 8) * SBO;        // k-chunk stride
  float4 v[V];

  __device__ void load(const L& l, int row0, int k0, int kend, int tid) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      int u = tid + i * NPROD;
      if (u >= UNITS) continue;
      if constexpr (L::KMAJOR) {
        int row = (u & 7) + 8 * (u >> 5);     // 8 threads = 8 rows of one chunk
        int c = (u >> 3) & 3;
        v[i] = l.chunk(row0 + row, k0 + 4 * c, kend);
      } else {
        int rq = u % (ROWS / 4), kq = u / (ROWS / 4);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[4 * i + j] = l.quad(row0 + 4 * rq, k0 + 4 * kq + j, kend);
      }
    }
  }

  // split into hi/lo and store; layout [kchunk 4][rows/8 (stride SBO)][8][16 B]
  __device__ void store(char* hi, char* lo, int tid) const {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      int u = tid + i * NPROD;
      if (u >= UNITS) continue;
      if constexpr (L::KMAJOR) {
        int row = (u & 7) + 8 * (u >> 5);
        int c = (u >> 3) & 3;
        int off = c * LBO + (row >> 3) * SBO + (row & 7) * 16;
        float4 h, o;
        split(v[i].x, h.x, o.x); split(v[i].y, h.y, o.y);
        split(v[i].z, h.z, o.z); split(v[i].w, h.w, o.w);
        *reinterpret_cast<float4*>(hi + off) = h;
        *reinterpret_cast<float4*>(lo + off) = o;
      } else {
        int rq = u % (ROWS / 4), kq = u / (ROWS / 4);
        const float4* q = v + 4 * i;
        // 4x4 transpose: row 4rq+r receives (q[0].r, q[1].r, q[2].r, q[3].r)
        float4 rows[4] = {make_float4(q[0].x, q[1].x, q[2].x, q[3].x),
                          make_float4(q[0].y, q[1].y, q[2].y, q[3].y),
                          make_float4(q[0].z, q[1].z, q[2].z, q[3].z),
                          make_float4(q[0].w, q[1].w, q[2].w, q[3].w)};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          int row = 4 * rq + r;
          int off = kq * LBO + (row >> 3) * SBO + (row & 7) * 16;
          float4 h, o;
          split(rows[r].x, h.x, o.x); split(rows[r].y, h.y, o.y);
          split(rows[r].z, h.z, o.z); split(rows[r].w, h.w, o.w);
          *reinterpret_cast<float4*>(hi + off) = h;
          *reinterpret_cast<float4*>(lo + off) = o;
        }
      }
    }
  }
};

template <int BN, class LA, class LB, class EPI>
__global__ void __launch_bounds__(NTHREADS, 1)
gemm_kernel(LA la, LB lb, EPI epi, int M, int N, int K, int kchunk) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) char smem[];
  char* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* hfull = empty + C::STAGES;      // [2] chunk accumulated (MMA -> drain)
  uint64_t* hfree = hfull + 2;              // [2] chunk drained (drain -> MMA)
  uint64_t* sfull = hfree + 2;              // cross-term accumulator final
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfull + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * kchunk;
  const int kend = min(K, kbeg + kchunk);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  const int nc = (nk + P - 1) / P;

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], NPROD);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hfree[b], NDRAIN);
    }
    mbar_init(sfull, 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(tmem_slot)), "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ------------------------------------------------ producers
    Frag<LA, BM> fa[2];
    Frag<LB, BN> fb[2];
    if (nk > 0) {
      fa[0].load(la, m0, kbeg, kend, tid);
      fb[0].load(lb, n0, kbeg, kend, tid);
    }
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::STAGES;
      const int cur = kb & 1;
      if (kb + 1 < nk) {
        const int k1 = kbeg + (kb + 1) * BK;
        if (cur == 0) { fa[1].load(la, m0, k1, kend, tid); fb[1].load(lb, n0, k1, kend, tid); }
        else { fa[0].load(la, m0, k1, kend, tid); fb[0].load(lb, n0, k1, kend, tid); }
      }
      if (kb >= C::STAGES) mbar_wait(&empty[s], ((kb / C::STAGES) - 1) & 1);
      char* st = stages + s * C::STAGE;
      char* a_hi = st;
      char* a_lo = st + C::A_BYTES;
      char* b_hi = st + 2 * C::A_BYTES;
      char* b_lo = b_hi + C::B_BYTES;
      if (cur == 0) { fa[0].store(a_hi, a_lo, tid); fb[0].store(b_hi, b_lo, tid); }
      else { fa[1].store(a_hi, a_lo, tid); fb[1].store(b_hi, b_lo, tid); }
      fence_proxy_async();
      mbar_arrive(&full[s]);
    }
  } else if (warp < MMA_WARP) {
    // ------------------------------------------------ drain + epilogue
    const int dt = tid - NPROD;
    const int q = warp & 3;                  // TMEM lane quadrant (warp % 4)
    const int half = (warp - 8) >> 2;        // column half
    const int m = m0 + q * 32 + (tid & 31);
    const uint32_t lane = tmem + ((uint32_t)(q * 32) << 16);
    const int cbase = half * C::CW;
    float acc[C::CW];
#pragma unroll
    for (int j = 0; j < C::CW; ++j) acc[j] = 0.f;
    (void)dt;
    for (int c = 0; c < nc; ++c) {
      const int b = c & 1;
      mbar_wait(&hfull[b], (c >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < C::CW; j += 8) {
        uint32_t r[8];
        tmem_ld8(lane + b * BN + cbase + j, r);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[j + t] += __uint_as_float(r[t]);
      }
      tc_fence_before();
      mbar_arrive(&hfree[b]);
    }
    if (nk > 0) {
      mbar_wait(sfull, 0);
      tc_fence_after();
#pragma unroll
      for (int j = 0; j < C::CW; j += 8) {
        uint32_t r[8];
        tmem_ld8(lane + 2 * BN + cbase + j, r);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[j + t] += __uint_as_float(r[t]);
      }
    }
    if (m < M) {
#pragma unroll
      for (int j = 0; j < C::CW; j += 8) {
        const int n = n0 + cbase + j;
        if (n < N) {
          float v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) v[t] = acc[j + t];
          epi(m, n, N, v);
        }
      }
    }
  } else if (tid == MMA_WARP * 32) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc(BN);
    constexpr uint32_t LBO_A = (BM / 8) * SBO, LBO_B = (BN / 8) * SBO;
    const uint32_t s_acc = tmem + 2 * BN;
    for (int c = 0; c < nc; ++c) {
      const int b = c & 1;
      const uint32_t h_acc = tmem + b * BN;
      if (c >= 2) {                           // drain finished with this buffer
        mbar_wait(&hfree[b], ((c >> 1) - 1) & 1);
        tc_fence_after();
      }
      const int kb1 = min(nk, (c + 1) * P);
      for (int kb = c * P; kb < kb1; ++kb) {
        const int s = kb % C::STAGES;
        mbar_wait(&full[s], (kb / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t base = smem_u32(stages + s * C::STAGE);
        const uint32_t a_hi = base, a_lo = base + C::A_BYTES;
        const uint32_t b_hi = base + 2 * C::A_BYTES, b_lo = b_hi + C::B_BYTES;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint32_t ka = ks * 2 * LBO_A, kb2 = ks * 2 * LBO_B;
          const uint64_t dah = make_desc(a_hi + ka, LBO_A, SBO);
          const uint64_t dal = make_desc(a_lo + ka, LBO_A, SBO);
          const uint64_t dbh = make_desc(b_hi + kb2, LBO_B, SBO);
          const uint64_t dbl = make_desc(b_lo + kb2, LBO_B, SBO);
          mma_tf32(h_acc, dah, dbh, idesc, (kb > c * P || ks > 0) ? 1u : 0u);
          mma_tf32(s_acc, dal, dbh, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
          mma_tf32(s_acc, dah, dbl, idesc, 1u);
        }
        tc_commit(&empty[s]);
      }
      tc_commit(&hfull[b]);
    }
    if (nk > 0) tc_commit(sfull);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                 ::"r"(tmem), "r"(C::TMEM_COLS));
  }
}

template <int BN, class LA, class LB, class EPI>
bpx_status_t launch(LA la, LB lb, EPI epi, int M, int N, int K, int& splits,
                    cudaStream_t st) {
  using C = Cfg<BN>;
  int kchunk = (int)(cdivll(cdivll(K, splits), BK) * BK);
  splits = (int)cdivll(K, kchunk);
  if (splits < 1) { splits = 1; kchunk = BK; }
  auto kern = gemm_kernel<BN, LA, LB, EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr_set = true;
  }
  dim3 grid(cdiv(M, BM), cdiv(N, BN), splits);
  kern<<<grid, NTHREADS, C::SMEM, st>>>(la, lb, epi, M, N, K, kchunk);
  return launch_status();
}

// split-K so that tiles*splits fills ~1 wave of 148 SMs (1 CTA / SM)
inline int pick_splits(long long tiles, long long K, int min_k) {
  long long want = (num_sms() + tiles - 1) / tiles;
  long long cap = K / (min_k > 0 ? min_k : 1);
  if (cap < 1) cap = 1;
  if (want > cap) want = cap;
  if (want > 64) want = 64;
  return (int)(want < 1 ? 1 : want);
}

}  // namespace tc

using namespace tc;

// ============================================================ entry points

// float4 gathers need 4-channel granularity; tiny Cin (conv1_1) stays on
// the FFMA engine.
bool tc_conv_fwd_ok(int n, int h, int w, int cin, int cout) {
  return cin % 8 == 0 && cout % 4 == 0;
}
bool tc_conv_dgrad_ok(int n, int h, int w, int cin, int cout) {
  return cin % 8 == 0 && cout % 4 == 0;
}
bool tc_conv_wgrad_ok(int n, int h, int w, int cin, int cout) {
  return cin % 8 == 0 && cout % 4 == 0;
}
bool tc_linear_ok(int b, int in, int out) {
  // the [M][b] partials are written as float4 rows: b % 4 == 0
  return in % 4 == 0 && out % 4 == 0 && b <= 256 && b % 4 == 0;
}

size_t tc_conv_fwd_ws(int, int, int, int, int) { return 0; }
size_t tc_conv_dgrad_ws(int, int, int, int, int) { return 0; }

static int wgrad_bn(int N) { return N % 128 == 0 ? 128 : 96; }

static int wg_splits(int n, int h, int w, int cin, int cout) {
  long long npix = (long long)n * h * w;
  long long tiles = (long long)cdiv(cout, BM) * cdiv(9 * cin, wgrad_bn(9 * cin));
  return tc::pick_splits(tiles, npix, 512);
}
size_t tc_conv_wgrad_ws(int n, int h, int w, int cin, int cout) {
  long long npix = (long long)n * h * w;
  return ((size_t)wg_splits(n, h, w, cin, cout) * cout * 9 * cin +
          colsum_workspace_floats(npix, cout)) * sizeof(float);
}

template <class LA, class LB, class EPI>
static bpx_status_t by_bn(int bn, LA la, LB lb, EPI epi, int M, int N, int K, int& splits,
                          cudaStream_t st) {
  switch (bn) {
    case 16: return launch<16>(la, lb, epi, M, N, K, splits, st);
    case 32: return launch<32>(la, lb, epi, M, N, K, splits, st);
    case 64: return launch<64>(la, lb, epi, M, N, K, splits, st);
    case 96: return launch<96>(la, lb, epi, M, N, K, splits, st);
    default: return launch<128>(la, lb, epi, M, N, K, splits, st);
  }
}

static int bn_for(int N) {
  if (N <= 16) return 16;
  if (N <= 32) return 32;
  if (N <= 64) return 64;
  return 128;
}

bpx_status_t tc_conv_fwd(const float* x, const float* w, const float* bias, float* y, int n,
                         int h, int w_, int cin, int cout, int relu, void*, size_t,
                         cudaStream_t st) {
  int npix = n * h * w_;
  if (npix == 0) return BPX_OK;
  Im2colRows la{x, h, w_, cin, npix};
  MatK lb{w, 9LL * cin, cout};
  EBiasAct epi{y, bias, cout, relu};
  int splits = 1;
  return by_bn(bn_for(cout), la, lb, epi, npix, cout, 9 * cin, splits, st);
}

bpx_status_t tc_conv_dgrad(const float* dz, const float* w, const float* mask, float* dx,
                           int n, int h, int w_, int cin, int cout, void*, size_t,
                           cudaStream_t st) {
  int npix = n * h * w_;
  if (npix == 0) return BPX_OK;
  Im2colRows la{dz, h, w_, cout, npix};
  FlipW lb{w, cin, cout};
  EMask epi{dx, mask, cin};
  int splits = 1;
  return by_bn(bn_for(cin), la, lb, epi, npix, cin, 9 * cout, splits, st);
}

bpx_status_t tc_conv_wgrad(const float* x, const float* dz, float* dw, float* dbias, int n,
                           int h, int w_, int cin, int cout, void* ws, size_t ws_bytes,
                           cudaStream_t st) {
  long long npix = (long long)n * h * w_;
  int M = cout, N = 9 * cin;
  if (ws_bytes < tc_conv_wgrad_ws(n, h, w_, cin, cout)) return BPX_ERR_WORKSPACE;
  if (npix == 0) {
    cudaMemsetAsync(dw, 0, sizeof(float) * (size_t)M * N, st);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * cout, st);
    return launch_status(0);
  }
  int splits = wg_splits(n, h, w_, cin, cout);
  const int planned = splits;
  float* part = static_cast<float*>(ws);
  size_t slab = (size_t)M * N;
  MatMN la{dz, cout, cout};
  Im2colCols lb{x, h, w_, cin, (int)npix};
  bpx_status_t s;
  if (splits == 1) {
    EPartial epi{dw, N, 0};
    s = by_bn(wgrad_bn(N), la, lb, epi, M, N, (int)npix, splits, st);
  } else {
    EPartial epi{part, N, (long long)slab};
    s = by_bn(wgrad_bn(N), la, lb, epi, M, N, (int)npix, splits, st);
    if (s == BPX_OK) s = split_reduce(part, splits, slab, dw, st);
  }
  if (s != BPX_OK || !dbias) return s;
  float* cws = part + (size_t)planned * slab;
  return colsum(dz, npix, cout, dbias, cws, colsum_workspace_floats(npix, cout), st);
}

// ------------------------------------------------------------------ dense
// fwd:   D[o][b] = W[o][:] . x[b][:]   (M=out, N=b, K=in)  -> y[b][o]
// dgrad: D[i][b] = W[:][i] . dy[b][:]  (M=in,  N=b, K=out) -> dx[b][i]
// wgrad: D[o][i] = dy[:][o] . x[:][i]  (M=out, N=in, K=b)

static int dense_splits(int M, int N, int K) {
  long long tiles = (long long)cdiv(M, BM) * cdiv(N, bn_for(N));
  if (tiles <= 0) return 1;                   // empty shard: nothing to split
  return tc::pick_splits(tiles, K, 256);
}
size_t tc_linear_fwd_ws(int b, int in, int out) {
  return (size_t)dense_splits(out, b, in) * out * b * sizeof(float);
}
size_t tc_linear_dgrad_ws(int b, int in, int out) {
  return (size_t)dense_splits(in, b, out) * in * b * sizeof(float);
}
// split-K partials over the batch (pixel-batched 1x1 convs: b = pixels),
// then the bias column sums (which reuse the space after the reduce)
static int wgrad_dense_splits(int b, int in, int out) {
  return pick_splits((long long)cdiv(out, BM) * cdiv(in, 128), b, 512);
}
size_t tc_linear_wgrad_ws(int b, int in, int out) {
  const int splits = wgrad_dense_splits(b, in, out);
  const size_t part = splits > 1 ? (size_t)splits * out * in : 0;
  const size_t cs = colsum_workspace_floats(b, out);
  return (part > cs ? part : cs) * sizeof(float);
}

// out[n][m] = act(sum_z part[z][m][n] + bias[m]) * mask
__global__ void dense_finish_t(const float* __restrict__ part, int splits, int M, int N,
                               const float* __restrict__ bias, const float* __restrict__ mask,
                               int relu, float* __restrict__ out) {
  long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int nn = (int)(i / M), m = (int)(i - (long long)nn * M);
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += part[(long long)k * total + (long long)m * N + nn];
    if (bias) s += bias[m];
    if (relu) s = fmaxf(s, 0.f);
    if (mask && !(mask[i] > 0.f)) s = 0.f;
    out[i] = s;
  }
}

template <class LA, class LB>
static bpx_status_t dense_run(LA la, LB lb, int M, int N, int K, const float* bias,
                              const float* mask, int relu, float* out, void* ws,
                              size_t ws_bytes, cudaStream_t st) {
  int splits = dense_splits(M, N, K);
  if (ws_bytes < (size_t)splits * M * N * sizeof(float)) return BPX_ERR_WORKSPACE;
  float* part = static_cast<float*>(ws);
  EPartial epi{part, N, (long long)M * N};
  bpx_status_t s = by_bn(bn_for(N), la, lb, epi, M, N, K, splits, st);
  if (s != BPX_OK) return s;
  long long total = (long long)M * N;
  int grid = (int)std::min<long long>(cdivll(total, 256), 4LL * num_sms());
  dense_finish_t<<<grid, 256, 0, st>>>(part, splits, M, N, bias, mask, relu, out);
  return launch_status();
}

bpx_status_t tc_linear_fwd(const float* x, const float* w, const float* bias, float* y, int b,
                           int in, int out, int relu, void* ws, size_t ws_bytes,
                           cudaStream_t st) {
  if (b == 0) return BPX_OK;
  MatK la{w, in, out};
  MatK lb{x, in, b};
  return dense_run(la, lb, out, b, in, bias, nullptr, relu, y, ws, ws_bytes, st);
}

bpx_status_t tc_linear_dgrad(const float* dy, const float* w, const float* mask, float* dx,
                             int b, int in, int out, void* ws, size_t ws_bytes,
                             cudaStream_t st) {
  if (b == 0) return BPX_OK;
  MatMN la{w, in, in};
  MatK lb{dy, out, b};
  return dense_run(la, lb, in, b, out, nullptr, mask, 0, dx, ws, ws_bytes, st);
}

bpx_status_t tc_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias, int b,
                             int in, int out, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (ws_bytes < tc_linear_wgrad_ws(b, in, out)) return BPX_ERR_WORKSPACE;
  if (b == 0) {
    cudaMemsetAsync(dw, 0, sizeof(float) * (size_t)out * in, st);
    if (dbias) cudaMemsetAsync(dbias, 0, sizeof(float) * out, st);
    return launch_status(0);
  }
  MatMN la{dy, out, out};
  MatMN lb{x, in, in};
  int splits = wgrad_dense_splits(b, in, out);
  bpx_status_t s;
  if (splits == 1) {
    EPartial epi{dw, in, 0};
    s = launch<128>(la, lb, epi, out, in, b, splits, st);
  } else {
    float* part = static_cast<float*>(ws);
    const size_t slab = (size_t)out * in;
    EPartial epi{part, in, (long long)slab};
    s = launch<128>(la, lb, epi, out, in, b, splits, st);
    if (s == BPX_OK) s = split_reduce(part, splits, slab, dw, st);
  }
  if (s != BPX_OK || !dbias) return s;
  return colsum(dy, b, out, dbias, static_cast<float*>(ws),
                colsum_workspace_floats(b, out), st);
}

}  // namespace bpx
