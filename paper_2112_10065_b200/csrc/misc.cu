// Memory-bound kernels of the training step: max-pool fwd/bwd, softmax
// cross-entropy, SGD, deterministic column sums / split reductions, and the
// ABI bookkeeping entry points.  All HBM-bound: 16-byte vector accesses,
// grid sized in multiples of the SM count.
#include "common.cuh"

namespace bpx {

// ----------------------------------------------------------------- colsum
// pass 1: block b sums rows [b*chunk, (b+1)*chunk) of every column (warp
// lanes = 32 adjacent columns -> coalesced; 8 row-lanes, fixed order).
__global__ void colsum_pass1(const float* __restrict__ in, long long rows,
                             int cols, long long chunk, float* __restrict__ part) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const long long r0 = blockIdx.x * chunk;
  const long long r1 = min(rows, r0 + chunk);
  for (int c0 = 0; c0 < cols; c0 += 32) {
    const int c = c0 + lane;
    float s = 0.f;
    if (c < cols)
      for (long long r = r0 + grp; r < r1; r += 8) s += in[r * cols + c];
    red[grp][lane] = s;
    __syncthreads();
    if (grp == 0 && c < cols) {
      float t = 0.f;
#pragma unroll
      for (int g = 0; g < 8; ++g) t += red[g][lane];
      part[blockIdx.x * (long long)cols + c] = t;
    }
    __syncthreads();
  }
}

__global__ void colsum_pass2(const float* __restrict__ part, int nparts, int cols,
                             float* __restrict__ out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int p = 0; p < nparts; ++p) s += part[(long long)p * cols + c];
  out[c] = s;
}

static int colsum_parts(long long rows) {
  long long p = cdivll(rows, 512);
  long long cap = 2LL * num_sms();
  return (int)(p < 1 ? 1 : (p > cap ? cap : p));
}

size_t colsum_workspace_floats(long long rows, int cols) {
  return (size_t)colsum_parts(rows) * (size_t)cols;
}

// Few rows (a dense layer's batch): one thread per column, rows in order.
__global__ void colsum_rows(const float* __restrict__ in, int rows, int cols,
                            float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int r = 0; r < rows; ++r) s += in[(long long)r * cols + c];
  out[c] = s;
}

bpx_status_t colsum(const float* in, long long rows, int cols, float* out,
                    float* ws, size_t ws_floats, cudaStream_t st) {
  if (rows <= 512) {
    colsum_rows<<<cdiv(cols, 128), 128, 0, st>>>(in, (int)rows, cols, out);
    return launch_status();
  }
  int parts = colsum_parts(rows);
  if (ws_floats < (size_t)parts * cols) return BPX_ERR_WORKSPACE;
  long long chunk = cdivll(rows, parts);
  colsum_pass1<<<parts, 256, 0, st>>>(in, rows, cols, chunk, ws);
  colsum_pass2<<<cdiv(cols, 256), 256, 0, st>>>(ws, parts, cols, out);
  return launch_status(2);
}

__global__ void split_reduce_kernel(const float4* __restrict__ parts, int splits,
                                    long long n4, float4* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 s = parts[i];
    int k = 1;
    for (; k + 8 <= splits; k += 8) {       // 8 loads in flight, adds in order
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = parts[(k + j) * n4 + i];
#pragma unroll
      for (int j = 0; j < 8; ++j) { s.x += v[j].x; s.y += v[j].y; s.z += v[j].z; s.w += v[j].w; }
    }
    for (; k < splits; ++k) {
      float4 v = parts[k * n4 + i];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    out[i] = s;
  }
}
// Many splits of a short vector: 8 warps per block each sum every 8th split
// of 32 float4 columns, then fixed-order combine in shared memory.
__global__ void split_reduce_wide(const float4* __restrict__ parts, int splits, long long n4,
                                  float4* __restrict__ out) {
  __shared__ float4 red[8][32];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * 32 + lane;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < n4) {
    for (int k = grp; k < splits; k += 8) {
      float4 v = parts[k * n4 + i];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
  }
  red[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && i < n4) {
    for (int g = 1; g < 8; ++g) {
      const float4 v = red[g][lane];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    out[i] = s;
  }
}
__global__ void split_reduce_scalar(const float* __restrict__ parts, int splits,
                                    long long n, float* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float s = parts[i];
    for (int k = 1; k < splits; ++k) s += parts[k * n + i];
    out[i] = s;
  }
}

bpx_status_t split_reduce(const float* parts, int splits, size_t n, float* out,
                          cudaStream_t st) {
  int grid = 4 * num_sms();
  if (n % 4 == 0 && aligned16(parts) && aligned16(out) && splits >= 32 &&
      (long long)(n / 4) <= 64LL * num_sms()) {
    const long long n4 = (long long)(n / 4);
    split_reduce_wide<<<(int)cdivll(n4, 32), 256, 0, st>>>(
        reinterpret_cast<const float4*>(parts), splits, n4, reinterpret_cast<float4*>(out));
  } else if (n % 4 == 0 && aligned16(parts) && aligned16(out)) {
    long long n4 = (long long)(n / 4);
    if (cdivll(n4, 256) < grid) grid = (int)cdivll(n4, 256);
    split_reduce_kernel<<<grid, 256, 0, st>>>(
        reinterpret_cast<const float4*>(parts), splits, n4,
        reinterpret_cast<float4*>(out));
  } else {
    if (cdivll(n, 256) < grid) grid = (int)cdivll(n, 256);
    split_reduce_scalar<<<grid, 256, 0, st>>>(parts, splits, (long long)n, out);
  }
  return launch_status();
}

// Two segments (weight and bias partials) of the same split count.  Block b
// of the wide form takes 32 float4 columns of segment b < ba ? w : b; the
// flat form strides over the concatenated index.  Summation order as above.
struct Seg2 {
  const float4* p[2];
  float4* o[2];
  long long n4[2];
};
__global__ void split_reduce2_kernel(Seg2 g, int splits) {
  const long long tot = g.n4[0] + g.n4[1];
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < tot;
       j += (long long)gridDim.x * blockDim.x) {
    const int sg = j >= g.n4[0];
    const long long i = sg ? j - g.n4[0] : j, n4 = g.n4[sg];
    const float4* parts = g.p[sg];
    float4 s = parts[i];
    int k = 1;
    for (; k + 8 <= splits; k += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = parts[(k + u) * n4 + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) { s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w; }
    }
    for (; k < splits; ++k) {
      float4 v = parts[k * n4 + i];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    g.o[sg][i] = s;
  }
}
__global__ void split_reduce2_wide(Seg2 g, int splits, int ba) {
  __shared__ float4 red[8][32];
  const int sg = (int)blockIdx.x >= ba;
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const long long i = (long long)(sg ? blockIdx.x - ba : blockIdx.x) * 32 + lane;
  const long long n4 = g.n4[sg];
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < n4) {
    for (int k = grp; k < splits; k += 8) {
      float4 v = g.p[sg][k * n4 + i];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
  }
  red[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && i < n4) {
    for (int q = 1; q < 8; ++q) {
      const float4 v = red[q][lane];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    g.o[sg][i] = s;
  }
}

bpx_status_t split_reduce_wb(const float* pw, size_t nw, float* dw, const float* pb, size_t nb,
                             float* db, int splits, cudaStream_t st) {
  const bool vec = nw % 4 == 0 && nb % 4 == 0 && aligned16(pw) && aligned16(dw) &&
                   (!db || (aligned16(pb) && aligned16(db)));
  if (!db || !vec) {          // one segment, or the scalar forms
    bpx_status_t s = split_reduce(pw, splits, nw, dw, st);
    if (s != BPX_OK || !db) return s;
    return split_reduce(pb, splits, nb, db, st);
  }
  Seg2 g;
  g.p[0] = reinterpret_cast<const float4*>(pw);
  g.p[1] = reinterpret_cast<const float4*>(pb);
  g.o[0] = reinterpret_cast<float4*>(dw);
  g.o[1] = reinterpret_cast<float4*>(db);
  g.n4[0] = (long long)(nw / 4);
  g.n4[1] = (long long)(nb / 4);
  if (splits >= 32 && g.n4[0] <= 64LL * num_sms()) {
    const int ba = (int)cdivll(g.n4[0], 32), bb = (int)cdivll(g.n4[1], 32);
    split_reduce2_wide<<<ba + bb, 256, 0, st>>>(g, splits, ba);
  } else {
    int grid = 4 * num_sms();
    const long long tot = g.n4[0] + g.n4[1];
    if (cdivll(tot, 256) < grid) grid = (int)cdivll(tot, 256);
    split_reduce2_kernel<<<grid, 256, 0, st>>>(g, splits);
  }
  return launch_status();
}

// ----------------------------------------------------------------- maxpool
// NHWC, 2x2 stride 2, float4 over channels (C % 4 == 0).
__global__ void maxpool_fwd_kernel(const float4* __restrict__ x, float4* __restrict__ y,
                                   int n, int h, int w, int c4) {
  const int oh = h / 2, ow = w / 2;
  const long long total = (long long)n * oh * ow * c4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % c4); long long p = i / c4;
    int xo = (int)(p % ow); p /= ow;
    int yo = (int)(p % oh); int b = (int)(p / oh);
    const float4* base = x + (((long long)b * h + 2 * yo) * w + 2 * xo) * c4 + c;
    float4 a = base[0], bb = base[c4], cc = base[(long long)w * c4],
           d = base[(long long)w * c4 + c4];
    float4 r;
    r.x = fmaxf(fmaxf(a.x, bb.x), fmaxf(cc.x, d.x));
    r.y = fmaxf(fmaxf(a.y, bb.y), fmaxf(cc.y, d.y));
    r.z = fmaxf(fmaxf(a.z, bb.z), fmaxf(cc.z, d.z));
    r.w = fmaxf(fmaxf(a.w, bb.w), fmaxf(cc.w, d.w));
    y[i] = r;
  }
}

// Route dy to the first maximum of the window in (row, col) scan order --
// PyTorch's max_pool2d tie rule -- and zero the other three positions.
__device__ __forceinline__ void route(float a, float b, float c, float d, float g,
                                      float& ra, float& rb, float& rc, float& rd) {
  int k = 0; float m = a;
  if (b > m) { m = b; k = 1; }
  if (c > m) { m = c; k = 2; }
  if (d > m) { m = d; k = 3; }
  ra = k == 0 ? g : 0.f; rb = k == 1 ? g : 0.f;
  rc = k == 2 ? g : 0.f; rd = k == 3 ? g : 0.f;
}

__global__ void maxpool_bwd_kernel(const float4* __restrict__ x, const float4* __restrict__ dy,
                                   float4* __restrict__ dx, int n, int h, int w, int c4) {
  const int oh = h / 2, ow = w / 2;
  const long long total = (long long)n * oh * ow * c4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % c4); long long p = i / c4;
    int xo = (int)(p % ow); p /= ow;
    int yo = (int)(p % oh); int b = (int)(p / oh);
    long long o = (((long long)b * h + 2 * yo) * w + 2 * xo) * c4 + c;
    long long rs = (long long)w * c4;
    float4 a = x[o], bb = x[o + c4], cc = x[o + rs], d = x[o + rs + c4];
    float4 g = dy[i];
    float4 ra, rb, rc, rd;
    route(a.x, bb.x, cc.x, d.x, g.x, ra.x, rb.x, rc.x, rd.x);
    route(a.y, bb.y, cc.y, d.y, g.y, ra.y, rb.y, rc.y, rd.y);
    route(a.z, bb.z, cc.z, d.z, g.z, ra.z, rb.z, rc.z, rd.z);
    route(a.w, bb.w, cc.w, d.w, g.w, ra.w, rb.w, rc.w, rd.w);
    dx[o] = ra; dx[o + c4] = rb; dx[o + rs] = rc; dx[o + rs + c4] = rd;
  }
}

// Index variants: the forward also stores each window's first-max position
// (one byte per output channel, PyTorch's tie order), so the backward reads
// 1 byte per output instead of re-reading the 4x larger input.
__device__ __forceinline__ unsigned char argmax4(float a, float b, float c, float d, float& m) {
  unsigned char k = 0; m = a;
  if (b > m) { m = b; k = 1; }
  if (c > m) { m = c; k = 2; }
  if (d > m) { m = d; k = 3; }
  return k;
}

__device__ __forceinline__ uint32_t abs4(float4 v) {
  const uint32_t m = 0x7fffffffu;
  return max(max(__float_as_uint(v.x) & m, __float_as_uint(v.y) & m),
             max(__float_as_uint(v.z) & m, __float_as_uint(v.w) & m));
}
// amax (nullable): atomicMax'ed with the max |v| bits written (fp16x3 scale)
__device__ __forceinline__ void commit_amax(uint32_t* amax, uint32_t mx) {
  if (!amax) return;
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(amax, mx);
}

// A block walks whole output rows (b, yo); within a row, thread j takes
// (xo, channel group) = (j / c4, j % c4) in 32-bit arithmetic -- a flat
// 64-bit index decomposed per element (three 64-bit div/mods) had made the
// pools issue-bound.
__global__ void maxpool_fwd_idx_kernel(const float4* __restrict__ x, float4* __restrict__ y,
                                       uchar4* __restrict__ idx, int n, int h, int w, int c4,
                                       uint32_t* amax) {
  const int oh = h / 2, ow = w / 2, per = ow * c4;
  const long long rs = (long long)w * c4;
  uint32_t mx = 0;
  for (int row = blockIdx.x; row < n * oh; row += gridDim.x) {
    const int b = row / oh, yo = row - b * oh;
    const float4* xr = x + ((long long)b * h + 2 * yo) * rs;
    float4* yr = y + (long long)row * per;
    uchar4* ir = idx + (long long)row * per;
    for (int j = threadIdx.x; j < per; j += blockDim.x) {
      const int xo = j / c4, c = j - xo * c4;
      const float4* base = xr + 2 * xo * c4 + c;
      const float4 a = base[0], bb = base[c4], cc = base[rs], d = base[rs + c4];
      float4 r;
      uchar4 k;
      k.x = argmax4(a.x, bb.x, cc.x, d.x, r.x);
      k.y = argmax4(a.y, bb.y, cc.y, d.y, r.y);
      k.z = argmax4(a.z, bb.z, cc.z, d.z, r.z);
      k.w = argmax4(a.w, bb.w, cc.w, d.w, r.w);
      yr[j] = r;
      ir[j] = k;
      mx = max(mx, abs4(r));
    }
  }
  commit_amax(amax, mx);
}

__global__ void maxpool_bwd_idx_kernel(const uchar4* __restrict__ idx,
                                       const float4* __restrict__ dy, float4* __restrict__ dx,
                                       int n, int h, int w, int c4, uint32_t* amax) {
  const int oh = h / 2, ow = w / 2, per = ow * c4;
  const long long rs = (long long)w * c4;
  uint32_t mx = 0;
  for (int row = blockIdx.x; row < n * oh; row += gridDim.x) {
    const int b = row / oh, yo = row - b * oh;
    float4* xr = dx + ((long long)b * h + 2 * yo) * rs;
    const float4* gr = dy + (long long)row * per;
    const uchar4* ir = idx + (long long)row * per;
    for (int j = threadIdx.x; j < per; j += blockDim.x) {
      const int xo = j / c4, c = j - xo * c4;
      const long long o = 2 * xo * c4 + c;
      const uchar4 k = ir[j];
      const float4 g = gr[j];
      float4 r[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        r[q].x = k.x == q ? g.x : 0.f;
        r[q].y = k.y == q ? g.y : 0.f;
        r[q].z = k.z == q ? g.z : 0.f;
        r[q].w = k.w == q ? g.w : 0.f;
      }
      xr[o] = r[0]; xr[o + c4] = r[1]; xr[o + rs] = r[2]; xr[o + rs + c4] = r[3];
      mx = max(mx, max(max(abs4(r[0]), abs4(r[1])), max(abs4(r[2]), abs4(r[3]))));
    }
  }
  commit_amax(amax, mx);
}

static int pool_grid(int rows) {          // blocks walk output rows
  const int cap = 8 * num_sms();
  return rows < 1 ? 1 : (rows > cap ? cap : rows);
}

static int ew_grid(long long work) {
  long long g = cdivll(work, 256);
  long long cap = 8LL * num_sms();
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// ------------------------------------------------------------ softmax-CE
// One CTA per local row; fixed-order block reduction, per-row loss written
// to a small scratch inside dlogits' row tail is avoided: rows' losses go to
// a shared-memory-free second kernel for a deterministic sum.
__global__ void xent_rows(const float* __restrict__ logits, const int32_t* __restrict__ labels,
                          int classes, float inv_b, float* __restrict__ dlogits,
                          float* __restrict__ row_loss) {
  const int row = blockIdx.x;
  const float* z = logits + (long long)row * classes;
  float* dz = dlogits + (long long)row * classes;
  __shared__ float red[32];
  __shared__ float bcast;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float m = -INFINITY;
  for (int j = threadIdx.x; j < classes; j += blockDim.x) m = fmaxf(m, z[j]);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[wid] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = red[0];
    for (int i = 1; i < nw; ++i) t = fmaxf(t, red[i]);
    bcast = t;
  }
  __syncthreads();
  m = bcast;
  __syncthreads();
  float s = 0.f;
  for (int j = threadIdx.x; j < classes; j += blockDim.x) s += expf(z[j] - m);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[wid] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < nw; ++i) t += red[i];
    bcast = t;
  }
  __syncthreads();
  const float sum = bcast;
  const float lse = m + logf(sum);
  const int y = labels[row];
  for (int j = threadIdx.x; j < classes; j += blockDim.x) {
    float p = expf(z[j] - lse);
    dz[j] = (p - (j == y ? 1.f : 0.f)) * inv_b;
  }
  if (threadIdx.x == 0) row_loss[row] = (lse - z[y]) * inv_b;
}

__global__ void xent_sum(const float* __restrict__ row_loss, int rows, float* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    float s = 0.f;
    for (int i = 0; i < rows; ++i) s += row_loss[i];
    out[0] = s;
    // rows' individual losses stay at out[1..rows] for diagnostics
  }
}

// ------------------------------------------------------------------- SGD
__global__ void sgd_kernel(float4* __restrict__ w, const float4* __restrict__ g,
                           long long n4, float lr) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 a = w[i], b = g[i];
    a.x -= lr * b.x; a.y -= lr * b.y; a.z -= lr * b.z; a.w -= lr * b.w;
    w[i] = a;
  }
}
__global__ void sgd_tail(float* __restrict__ w, const float* __restrict__ g,
                         long long n, float lr) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) w[i] -= lr * g[i];
}

static long long g_launches = 0;
void count_launches(long long k) { __atomic_add_fetch(&g_launches, k, __ATOMIC_RELAXED); }

int& sm_budget() {
  static thread_local int budget = 0;
  return budget;
}

}  // namespace bpx

using namespace bpx;

extern "C" {

int bpx_set_sm_budget(int n) {
  const int prev = sm_budget();
  sm_budget() = n > 0 ? n : 0;
  return prev;
}

const char* bpx_status_string(bpx_status_t s) {
  switch (s) {
    case BPX_OK: return "BPX_OK";
    case BPX_ERR_INVALID_ARGUMENT: return "BPX_ERR_INVALID_ARGUMENT";
    case BPX_ERR_LAUNCH: return "BPX_ERR_LAUNCH";
    case BPX_ERR_UNSUPPORTED: return "BPX_ERR_UNSUPPORTED";
    case BPX_ERR_WORKSPACE: return "BPX_ERR_WORKSPACE";
    case BPX_ERR_ARCH: return "BPX_ERR_ARCH";
    default: return "BPX_ERR_UNKNOWN";
  }
}

int bpx_abi_version(void) { return 1; }

long long bpx_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int bpx_device_supported(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 1 : 0;
}

bpx_status_t bpx_maxpool2x2_fwd(const float* x, float* y, int n, int h, int w_,
                                int c, void* stream) {
  BPX_CHECK_ARG(x && y && n >= 0 && h % 2 == 0 && w_ % 2 == 0 && c % 4 == 0);
  BPX_CHECK_ARG(aligned16(x) && aligned16(y));
  long long total = (long long)n * (h / 2) * (w_ / 2) * (c / 4);
  if (total == 0) return BPX_OK;
  maxpool_fwd_kernel<<<ew_grid(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), n, h, w_, c / 4);
  return launch_status();
}

bpx_status_t bpx_maxpool2x2_bwd(const float* x, const float* dy, float* dx, int n,
                                int h, int w_, int c, void* stream) {
  BPX_CHECK_ARG(x && dy && dx && n >= 0 && h % 2 == 0 && w_ % 2 == 0 && c % 4 == 0);
  BPX_CHECK_ARG(aligned16(x) && aligned16(dy) && aligned16(dx));
  long long total = (long long)n * (h / 2) * (w_ / 2) * (c / 4);
  if (total == 0) return BPX_OK;
  maxpool_bwd_kernel<<<ew_grid(total), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(dy),
      reinterpret_cast<float4*>(dx), n, h, w_, c / 4);
  return launch_status();
}

bpx_status_t bpx_maxpool2x2_fwd_idx(const float* x, float* y, uint8_t* idx, int n, int h,
                                    int w_, int c, unsigned* y_amax, void* stream) {
  BPX_CHECK_ARG(x && y && idx && n >= 0 && h % 2 == 0 && w_ % 2 == 0 && c % 4 == 0);
  BPX_CHECK_ARG(aligned16(x) && aligned16(y) && (reinterpret_cast<uintptr_t>(idx) & 3) == 0);
  long long total = (long long)n * (h / 2) * (w_ / 2) * (c / 4);
  if (total == 0) return BPX_OK;
  maxpool_fwd_idx_kernel<<<pool_grid(n * (h / 2)), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y),
      reinterpret_cast<uchar4*>(idx), n, h, w_, c / 4, y_amax);
  return launch_status();
}

bpx_status_t bpx_maxpool2x2_bwd_idx(const uint8_t* idx, const float* dy, float* dx, int n,
                                    int h, int w_, int c, unsigned* dx_amax, void* stream) {
  BPX_CHECK_ARG(idx && dy && dx && n >= 0 && h % 2 == 0 && w_ % 2 == 0 && c % 4 == 0);
  BPX_CHECK_ARG(aligned16(dy) && aligned16(dx) && (reinterpret_cast<uintptr_t>(idx) & 3) == 0);
  long long total = (long long)n * (h / 2) * (w_ / 2) * (c / 4);
  if (total == 0) return BPX_OK;
  maxpool_bwd_idx_kernel<<<pool_grid(n * (h / 2)), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const uchar4*>(idx), reinterpret_cast<const float4*>(dy),
      reinterpret_cast<float4*>(dx), n, h, w_, c / 4, dx_amax);
  return launch_status();
}

bpx_status_t bpx_softmax_xent(const float* logits, const int32_t* labels,
                              int b_local, int b_global, int classes,
                              float* loss_out, float* dlogits, void* stream) {
  BPX_CHECK_ARG(b_local >= 0 && b_global >= 1 && classes >= 1 && loss_out);
  cudaStream_t st = as_stream(stream);
  if (b_local == 0) {
    cudaMemsetAsync(loss_out, 0, sizeof(float), st);
    return launch_status();
  }
  BPX_CHECK_ARG(logits && labels && dlogits);
  // per-row losses are parked at loss_out[1 .. b_local]
  xent_rows<<<b_local, 256, 0, st>>>(logits, labels, classes, 1.0f / b_global,
                                     dlogits, loss_out + 1);
  xent_sum<<<1, 32, 0, st>>>(loss_out + 1, b_local, loss_out);
  return launch_status(2);
}

bpx_status_t bpx_sgd_update(float* w, const float* g, size_t n, float lr,
                            void* stream) {
  BPX_CHECK_ARG(w && g);
  if (n == 0) return BPX_OK;
  cudaStream_t st = as_stream(stream);
  int k = 0;
  if (aligned16(w) && aligned16(g)) {
    long long n4 = (long long)(n / 4);
    if (n4) { sgd_kernel<<<ew_grid(n4), 256, 0, st>>>(
        reinterpret_cast<float4*>(w), reinterpret_cast<const float4*>(g), n4, lr); ++k; }
    long long tail = (long long)n - 4 * n4;
    if (tail) { sgd_tail<<<1, 256, 0, st>>>(w + 4 * n4, g + 4 * n4, tail, lr); ++k; }
  } else {
    sgd_tail<<<(int)cdivll((long long)n, 256), 256, 0, st>>>(w, g, (long long)n, lr);
    ++k;
  }
  return launch_status(k);
}

}  // extern "C"
