// Probe: register layout of tcgen05.st.sync.aligned.16x256b.x1 -- which
// (TMEM lane, column) each thread's 4 registers land in.  One warp (warp 0,
// lane quadrant 0) writes v = (thread << 8) | reg, then reads lanes 0-15,
// columns 0-7 back with the 32x32b shape (thread = lane).
#include <cstdio>
#include <cstdint>
__global__ void probe(uint32_t* out) {
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  if (tid < 32) {
    uint32_t r0 = (tid << 8) | 0, r1 = (tid << 8) | 1, r2 = (tid << 8) | 2, r3 = (tid << 8) | 3;
    asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};"
                 ::"r"(t), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7]) : "r"(t));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int c = 0; c < 8; ++c) out[tid * 8 + c] = v[c];
  }
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
}
int main() {
  uint32_t* d; cudaMalloc(&d, 32 * 8 * 4); cudaMemset(d, 0xff, 32 * 8 * 4);
  probe<<<1, 128>>>(d);
  uint32_t h[256]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int lane = 0; lane < 16; ++lane) {
    printf("lane %2d:", lane);
    for (int c = 0; c < 8; ++c) {
      uint32_t v = h[lane * 8 + c];
      if (v == 0xffffffffu) printf("   --  "); else printf(" t%02u.r%u", v >> 8, v & 255);
    }
    printf("\n");
  }
}
