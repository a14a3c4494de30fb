// Probe: which operand-major combinations does tcgen05.mma kind::tf32 accept
// on this B200?  Exact small-integer data; prints max |err| per variant.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -I include -o probe_mn probe_mn.cu
#include <cstdio>
#include <cstring>
#include <cmath>
#include <cuda.h>
#include "../../paper_2112_10065_b200/csrc/tc_ptx.cuh"
using namespace bpx::tcx;

constexpr int M = 128, N = 64, K = 8;

__device__ float Av(int m, int k) { return (float)(((m * 3 + k * 5) % 7) - 3); }
__device__ float Bv(int n, int k) { return (float)(((n * 2 + k * 3) % 5) - 2); }

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// variant: 0 TS + B MN sw128 ; 1 SS A K(nosw) + B MN sw128 ; 2 SS A MN sw128 + B K(nosw)
//          3 TS + B MN no-swizzle ; 4 TS + B K nosw (control)
__global__ void probe(int variant, float* out, const __grid_constant__ CUtensorMap tmap, float* dump) {
  __shared__ __align__(1024) char sm[2 * 16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  char* sa = sm;            // A (smem variants)
  char* sb = sm + 16384;    // B
  const int tid = threadIdx.x, warp = tid >> 5;
  // ---- fill B
  for (int i = tid; i < N * K; i += blockDim.x) {
    int n = i / K, k = i % K;
    int off;
    if (variant == 5 || variant == 6) {   // MN-major SW128_BASE32B: atom 32 n x 4 k rows, 32B granules ^ (k%4)
      int atom = n / 32, nn = n % 32;
      int gran = (nn / 8) ^ (k % 4);
      off = atom * 1024 + (k / 4) * 512 + (k % 4) * 128 + gran * 32 + (nn % 8) * 4;
    } else if (variant == 7) {
      continue;
    } else if (variant == 0 || variant == 1) {   // MN-major SW128: atom = 32 n x 8 k rows of 128B
      int atom = n / 32, nn = n % 32;
      int gran = (nn / 4) ^ (k % 8);
      off = atom * 1024 + k * 128 + gran * 16 + (nn % 4) * 4;
    } else if (variant == 3) {            // MN-major interleave: (n/4)*128 + k*16 + (n%4)*4
      off = (n / 4) * 128 + k * 16 + (n % 4) * 4;
    } else {                              // K-major no swizzle: core 8 rows x 16B
      off = (n / 8) * 256 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4;
    }
    *reinterpret_cast<float*>(sb + off) = Bv(n, k);
  }
  for (int i = tid; i < M * K; i += blockDim.x) {
    int m = i / K, k = i % K;
    int off;
    if (variant == 6) {
      int atom = m / 32, mm = m % 32;
      int gran = (mm / 8) ^ (k % 4);
      off = atom * 1024 + (k / 4) * 512 + (k % 4) * 128 + gran * 32 + (mm % 8) * 4;
    } else if (variant == 2) {   // A MN-major sw128: 4 atoms of 32 m
      int atom = m / 32, mm = m % 32;
      int gran = (mm / 4) ^ (k % 8);
      off = atom * 1024 + k * 128 + gran * 16 + (mm % 4) * 4;
    } else {
      off = (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4;
    }
    *reinterpret_cast<float*>(sa + off) = Av(m, k);
  }
  __shared__ uint64_t tbar;
  if (tid == 0) { mbar_init(&bar, 1); mbar_init(&tbar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (variant == 7) {
    if (tid == 0) {
      mbar_expect_tx(&tbar, 2048);
      for (int a = 0; a < 2; ++a)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(smem_u32(sb + a * 1024)), "l"(&tmap), "r"(a * 32), "r"(0), "r"(smem_u32(&tbar)) : "memory");
    }
    mbar_wait(&tbar, 0);
    for (int i = tid; i < 512; i += blockDim.x) dump[i] = reinterpret_cast<float*>(sb)[i];
  }
  if (warp == 0) tmem_alloc(&slot, 128);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t dcol = tmem, acol = tmem + 64;
  if (variant == 0 || variant == 3 || variant == 4 || variant == 5 || variant == 7) {   // A rows -> TMEM
    float v[16];
    int m = tid;
    for (int j = 0; j < 16; ++j) v[j] = j < K ? Av(m, j) : 0.f;
    tmem_st16(acol + ((uint32_t)(warp * 32) << 16), v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                     ((uint32_t)(M >> 4) << 24);
    uint64_t bdesc, adesc;
    uint32_t bs = smem_u32(sb), as = smem_u32(sa);
    if (variant == 5 || variant == 6 || variant == 7) { bdesc = make_desc(bs, 1024, 512) | ((uint64_t)1 << 61); idesc |= 1u << 16; }
    else if (variant == 0 || variant == 1) { bdesc = make_desc_sw128(bs, 1024, 1024); idesc |= 1u << 16; }
    else if (variant == 3) { bdesc = make_desc(bs, 1024, 128); idesc |= 1u << 16; }
    else bdesc = make_desc(bs, 128, 256);
    if (variant == 6) { adesc = make_desc(as, 1024, 512) | ((uint64_t)1 << 61); idesc |= 1u << 15; }
    else if (variant == 2) { adesc = make_desc_sw128(as, 1024, 1024); idesc |= 1u << 15; }
    else adesc = make_desc(as, 128, 256);
    if (variant == 0 || variant == 3 || variant == 4 || variant == 5 || variant == 7) mma_ts(dcol, acol, bdesc, idesc, 0);
    else mma_ss(dcol, adesc, bdesc, idesc, 0);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int j = 0; j < N; j += 8) {
    uint32_t r[8];
    tmem_ld8(dcol + ((uint32_t)(warp * 32) << 16) + j, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int t = 0; t < 8; ++t) out[tid * N + j + t] = __uint_as_float(r[t]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_free(tmem, 128); }
}

int main() {
  float* d; cudaMalloc(&d, M * N * 4);
  float* dump; cudaMalloc(&dump, 512 * 4);
  // global B for TMA: [K=8 rows][N=64] row-major, value Bv(n,k)
  static float hb[8 * 64];
  for (int k = 0; k < 8; ++k) for (int n = 0; n < 64; ++n) hb[k * 64 + n] = (float)(((n * 2 + k * 3) % 5) - 2);
  float* gb; cudaMalloc(&gb, sizeof(hb)); cudaMemcpy(gb, hb, sizeof(hb), cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t gdim[2] = {64, 8}; cuuint64_t gstr[1] = {64 * 4};
  cuuint32_t box[2] = {32, 8}; cuuint32_t es[2] = {1, 1};
  CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, gb, gdim, gstr, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)cr);
  static float h[M * N];
  const char* names[] = {"TS + B MN sw128", "SS A K + B MN sw128", "SS A MN sw128 + B K",
                         "TS + B MN interleave", "TS + B K (control)", "TS + B MN sw128_32B",
                         "SS A,B MN sw128_32B", "TS + B MN TMA 128B_ATOM_32B"};
  for (int v = 0; v < 8; ++v) {
    cudaMemset(d, 0, M * N * 4);
    probe<<<1, 128>>>(v, d, tm, dump);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0, ref_norm = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)(((m * 3 + k * 5) % 7) - 3) * (((n * 2 + k * 3) % 5) - 2);
      err = fmax(err, fabs(s - h[m * N + n])); ref_norm = fmax(ref_norm, fabs(s));
    }
    printf("variant %d %-24s: %s max|err| %.3g (max|ref| %.3g) sample D[1][2]=%g\n", v, names[v],
           cudaGetErrorString(e), err, ref_norm, h[1 * N + 2]);
    if (e != cudaSuccess) return 1;
    if (v == 7) {
      static float hd[512]; cudaMemcpy(hd, dump, sizeof(hd), cudaMemcpyDeviceToHost);
      for (int r = 0; r < 8; ++r) { printf("row %d:", r); for (int j = 0; j < 32; ++j) printf(" %g", hd[r * 32 + j]); printf("\n"); }
      printf("global row0:"); for (int j = 0; j < 32; ++j) printf(" %g", hb[j]); printf("\n");
    }
  }
  return 0;
}
