// tcgen05 engine for the dense layers' weight gradient at per-GPU batches
// <= 32:  dW[o][i] = sum_n dy[n][o] x[n][i].
//
// K = the batch (<= 32), so the GEMM is one 32-K step per output tile and the
// kernel is bound by WRITING dW (fc1: 411 MB per pass), not by math.  A prep
// kernel transposes dy and x into K-major rows of 32 floats (zero-padded
// past the batch) and splits them into TF32 hi/lo once (the same launch
// emits the bias gradient, the column sums of dy, from its smem tile); the
// persistent main kernel then streams 128 x 256 output tiles:
//
//   warp 0  TMA: A hi/lo (128 x 32) + B hi/lo (256 x 32) per tile
//   warp 1  MMA (SS form, 3xTF32: 4 k-steps x 3 products into one TMEM
//           accumulator) + TMEM owner; accumulators double-buffered
//           (2 x 256 columns) so tile t+1's MMA runs under tile t's drain
//   2-9     drain (two warps per TMEM lane quadrant, 128 columns each):
//           TMEM -> registers -> 128-B-swizzled smem transpose -> coalesced
//           16-B stores, four full 128-B rows of dW per store instruction
//           (TMA tensor stores of 32 x 32 boxes issue-stalled at ~5 TB/s)
//
// This is the weight gradient of the reference's dense layers (the VGG
// model's fc1-fc3).  Batches <= 8 stay on the FFMA outer
// product (dns::outer_kernel, dense_ffma.cu), which writes faster when the
// math is that small (routing: bpx_linear_wgrad, abi_layers.cu).
#include "tma_host.h"
#include "tc_ptx.cuh"
#include "tc_api.h"

namespace bpx {
namespace dwt {
using namespace tcx;

constexpr int BM_ = 128, BN_ = 256, KP = 32;      // tile and padded K
constexpr int A_BYTES = BM_ * KP * 4;             // 16 KB
constexpr int B_BYTES = BN_ * KP * 4;             // 32 KB
constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // 96 KB
constexpr int S = 1;                              // the drain, not the load, paces a tile
static_assert(S == 1, "B reuse across tiles assumes one stage");
constexpr int DRAIN = 8;                          // 2 warps per TMEM lane quadrant
constexpr int OUT_BOX = 32 * 32 * 4;              // 4 KB per warp-box
constexpr int OUT_BYTES = DRAIN * OUT_BOX;
constexpr int SMEM = 1024 + S * STAGE + OUT_BYTES + 256;
constexpr int NTHREADS = (2 + DRAIN) * 32;
static_assert(SMEM <= 227 * 1024, "smem budget");

__global__ void __launch_bounds__(NTHREADS, 1)
dwt_kernel(const __grid_constant__ CUtensorMap tah, const __grid_constant__ CUtensorMap tal,
           const __grid_constant__ CUtensorMap tbh, const __grid_constant__ CUtensorMap tbl,
           float* __restrict__ dw, int M, int N, int nt, int ntiles) {
  extern __shared__ char smem_raw[];
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  char* obuf = smem + S * STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(obuf + OUT_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tfree = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfree + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // row-tile-major, strided over CTAs: the CTAs in flight together write
  // neighbouring column tiles of the same 128 rows of dW (long DRAM runs)
  const int nmine = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / gridDim.x + 1 : 0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tfree[b], DRAIN);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tah);
      tma_prefetch_desc(&tal);
      tma_prefetch_desc(&tbh);
      tma_prefetch_desc(&tbl);
      int have_n = -1;
      for (int i = 0; i < nmine; ++i) {
        const int t = blockIdx.x + i * gridDim.x;
        const int m0 = (t / nt) * BM_, n0 = (t % nt) * BN_;
        const int s = i % S;
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        char* st = smem + s * STAGE;
        const bool newb = n0 != have_n;
        mbar_expect_tx(&full[s], newb ? STAGE : 2 * A_BYTES);
        tma_load_2d(st, &tah, 0, m0, &full[s]);
        tma_load_2d(st + A_BYTES, &tal, 0, m0, &full[s]);
        if (newb) {
          tma_load_2d(st + 2 * A_BYTES, &tbh, 0, n0, &full[s]);
          tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tbl, 0, n0, &full[s]);
          have_n = n0;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                               ((uint32_t)(BN_ >> 3) << 17) | ((uint32_t)(BM_ >> 4) << 24);
    for (int i = 0; i < nmine; ++i) {
      const int s = i % S, b = i & 1;
      if (i >= 2) {
        mbar_wait(&tfree[b], ((i >> 1) - 1) & 1);
        tc_fence_after();
      }
      mbar_wait(&full[s], (i / S) & 1);
      tc_fence_after();
      const uint32_t ah = smem_u32(smem + s * STAGE), al = ah + A_BYTES;
      const uint32_t bh = al + A_BYTES, bl = bh + B_BYTES;
      const uint32_t d = tmem + b * BN_;
#pragma unroll
      for (int ks = 0; ks < KP / 8; ++ks) {
        const uint64_t dah = make_desc_sw128(ah + ks * 32, 16, 1024);
        const uint64_t dal = make_desc_sw128(al + ks * 32, 16, 1024);
        const uint64_t dbh = make_desc_sw128(bh + ks * 32, 16, 1024);
        const uint64_t dbl = make_desc_sw128(bl + ks * 32, 16, 1024);
        mma_ss_elect(d, dal, dbh, idesc, ks > 0 ? 1u : 0u);
        mma_ss_elect(d, dah, dbl, idesc, 1u);
        mma_ss_elect(d, dah, dbh, idesc, 1u);
      }
      tc_commit_elect(&empty[s]);
      tc_commit_elect(&tfull[b]);
    }
  } else {
    // drain warp: TMEM lanes 32q..32q+31 (tile rows m0 + 32q + lane), columns
    // 128h..128h+127 of the accumulator
    const int q = warp & 3, h = (warp - 2) >> 2;
    const uint32_t lanebase = tmem + ((uint32_t)(q * 32) << 16) + 128 * h;
    char* mybuf = obuf + (warp - 2) * OUT_BOX;
    for (int i = 0; i < nmine; ++i) {
      const int t = blockIdx.x + i * gridDim.x;
      const int m0 = (t / nt) * BM_, n0 = (t % nt) * BN_;
      const int b = i & 1;
      mbar_wait(&tfull[b], (i >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN_ / 64; ++c) {
        uint32_t r[32];
        tmem_ld8(lanebase + b * BN_ + 32 * c, *reinterpret_cast<uint32_t(*)[8]>(r));
        tmem_ld8(lanebase + b * BN_ + 32 * c + 8, *reinterpret_cast<uint32_t(*)[8]>(r + 8));
        tmem_ld8(lanebase + b * BN_ + 32 * c + 16, *reinterpret_cast<uint32_t(*)[8]>(r + 16));
        tmem_ld8(lanebase + b * BN_ + 32 * c + 24, *reinterpret_cast<uint32_t(*)[8]>(r + 24));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c == BN_ / 64 - 1) {        // accumulator buffer b fully read
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tfree[b]);
        }
        // transpose through the warp's swizzled box: lane = row on the way
        // in, four full 128-B rows per store instruction on the way out
        char* box = mybuf;
        char* row = box + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(row + ((j ^ (lane & 7)) << 4)) =
              make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
        __syncwarp();
        const int g = lane & 7;
        const int col = n0 + 128 * h + 32 * c + 4 * g;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int rr = 4 * j + (lane >> 3);
          const uint4 v = *reinterpret_cast<const uint4*>(box + rr * 128 + ((g ^ (rr & 7)) << 4));
          const int m = m0 + 32 * q + rr;
          if (m < M && col < N)
            *reinterpret_cast<uint4*>(dw + (long long)m * N + col) = v;
        }
        __syncwarp();
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, 512);
  }
}

// One launch for both operands: blocks [0, ma) take dy [b][M] -> A hi/lo
// [M][KP] (and dbias = the column sums of dy, from the same smem tile), the
// rest take x [b][N] -> B hi/lo [N][KP]; K-major, zero past b, 32 x 32 tiles.
__global__ void prep_kernel(const float* __restrict__ dy, const float* __restrict__ x, int b,
                            int M, int N, int ma, float* __restrict__ ah, float* __restrict__ al,
                            float* __restrict__ bh, float* __restrict__ bl,
                            float* __restrict__ dbias) {
  __shared__ float t[KP][33];
  const bool isa = (int)blockIdx.x < ma;
  const float* src = isa ? dy : x;
  const int R = isa ? M : N;
  float* hi = isa ? ah : bh;
  float* lo = isa ? al : bl;
  const int r0 = (isa ? blockIdx.x : blockIdx.x - ma) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;    // 256 threads: ty 0..7
  for (int k = ty; k < KP; k += 8) {
    const int r = r0 + tx;
    t[k][tx] = (k < b && r < R) ? src[(long long)k * R + r] : 0.f;
  }
  __syncthreads();
  if (isa && dbias && ty == 0 && r0 + tx < R) {
    float s = 0.f;
    for (int k = 0; k < b; ++k) s += t[k][tx];
    dbias[r0 + tx] = s;
  }
  for (int rr = ty; rr < 32; rr += 8) {
    const int r = r0 + rr;
    if (r < R) {
      float h, l;
      split(t[tx][rr], h, l);
      hi[(long long)r * KP + tx] = h;
      lo[(long long)r * KP + tx] = l;
    }
  }
}

inline bool encode(CUtensorMap* m, const float* p, long long inner, long long outer,
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

}  // namespace dwt

bool dwt_linear_ok(int b, int in, int out) {
  return b >= 1 && b <= 32 && in % 4 == 0 && out % 4 == 0;
}

size_t dwt_linear_ws(int b, int in, int out) {
  if (!dwt_linear_ok(b, in, out)) return 0;
  return (2 * (size_t)dwt::KP * ((size_t)in + out) + 64) * sizeof(float);
}

bpx_status_t dwt_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias, int b,
                              int in, int out, void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace dwt;
  if (!dwt_linear_ok(b, in, out) || !aligned16(dw) || !aligned16(ws))
    return BPX_ERR_UNSUPPORTED;
  if (ws_bytes < dwt_linear_ws(b, in, out)) return BPX_ERR_WORKSPACE;
  float* ah = static_cast<float*>(ws);
  float* al = ah + (size_t)KP * out;
  float* bh = al + (size_t)KP * out;
  float* bl = bh + (size_t)KP * in;
  CUtensorMap tah, tal, tbh, tbl;
  if (!(encode(&tah, ah, KP, out, KP, BM_) && encode(&tal, al, KP, out, KP, BM_) &&
        encode(&tbh, bh, KP, in, KP, BN_) && encode(&tbl, bl, KP, in, KP, BN_)))
    return BPX_ERR_INVALID_ARGUMENT;
  const int ma = cdiv(out, 32);
  prep_kernel<<<ma + cdiv(in, 32), 256, 0, st>>>(dy, x, b, out, in, ma, ah, al, bh, bl, dbias);
  const int nt = cdiv(in, BN_);
  const int ntiles = cdiv(out, BM_) * nt;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dwt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  dwt_kernel<<<grid, NTHREADS, SMEM, st>>>(tah, tal, tbh, tbl, dw, out, in, nt, ntiles);
  return launch_status(2);
}

}  // namespace bpx
