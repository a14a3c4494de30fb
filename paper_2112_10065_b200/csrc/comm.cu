// Cross-GPU data movement of the burst-parallel step over NVLink peer
// memory (pointers from CUDA IPC / torch symmetric memory, or local
// pointers when peers are simulated on one device in tests).
//
//  * bpx_reshard_pull        -- the modeled `transfer` op
//                               (/root/reference/pkg/src/burstplan/simulator.py:242-253)
//  * bpx_allreduce_sum_prefix -- the modeled `allreduce` op (:264-278)
//  * bpx_signal_barrier      -- ordering between the two sides of a P2P phase
//
// All copies are 16-byte vectorised when every segment is 16-byte aligned
// (activation rows are multiples of 16 bytes for every VGG layer), else
// byte-granular; CTAs stride the segment list so one launch moves all of it.
#include "common.cuh"

namespace bpx {

constexpr int kMaxSeg = 64;
constexpr int kMaxPeers = 16;

struct SegTable {
  const char* src[kMaxSeg];
  char* dst[kMaxSeg];
  unsigned long long bytes[kMaxSeg];
  unsigned long long start[kMaxSeg + 1];   // prefix sums of bytes
  int n;
};

// VEC: every thread moves U = 4 16-byte vectors per round (all four loads
// issued before the stores: four requests in flight per thread, which the
// peer-read latency over NVLink needs as much as HBM does).
template <bool VEC>
__global__ void reshard_kernel(SegTable t) {
  constexpr int U = VEC ? 4 : 1;
  constexpr unsigned long long E = VEC ? 16 : 1;
  const unsigned long long total = t.start[t.n];
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x * E;
  unsigned long long i = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) * E;
  int seg = 0;
  for (; i < total; i += U * stride) {
    int sg[U];
    unsigned long long off[U];
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned long long j = i + u * stride;
      sg[u] = -1;
      if (j < total) {
        while (j >= t.start[seg + 1]) ++seg;      // monotone in j
        sg[u] = seg;
        off[u] = j - t.start[seg];
        if (VEC) v[u] = *reinterpret_cast<const int4*>(t.src[seg] + off[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (sg[u] < 0) continue;
      if (VEC) *reinterpret_cast<int4*>(t.dst[sg[u]] + off[u]) = v[u];
      else t.dst[sg[u]][off[u]] = t.src[sg[u]][off[u]];
    }
  }
}

struct PeerTable {
  const float* p[kMaxPeers];
  int g;
};

__global__ void allreduce_pull_kernel(PeerTable t, float4* __restrict__ out, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 s = reinterpret_cast<const float4*>(t.p[0])[i];
    for (int r = 1; r < t.g; ++r) {            // fixed rank order -> identical on every rank
      float4 v = reinterpret_cast<const float4*>(t.p[r])[i];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    out[i] = s;
  }
}
__global__ void allreduce_pull_scalar(PeerTable t, float* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float s = t.p[0][i];
    for (int r = 1; r < t.g; ++r) s += t.p[r][i];
    out[i] = s;
  }
}

struct PadTable {
  unsigned int* pad[kMaxPeers];
  int g, rank;
  unsigned int epoch;
};

__global__ void signal_barrier_kernel(PadTable t) {
  int tid = threadIdx.x;
  if (tid < t.g) {
    // publish: every write this stream issued before us is visible system-wide
    __threadfence_system();
    volatile unsigned int* slot = t.pad[tid] + t.rank;
    *slot = t.epoch;
    volatile unsigned int* mine = t.pad[t.rank] + tid;
    while ((int)(*mine - t.epoch) < 0) { }
    __threadfence_system();
  }
}

// Graph-replayable variant: the epoch lives in device memory (this rank's
// counter for the group), incremented by the kernel itself, so every replay
// of a captured barrier waits for the NEXT epoch instead of a frozen one.
struct PadTableDev {
  unsigned int* pad[kMaxPeers];
  unsigned int* counter;
  int g, rank;
};

__global__ void signal_barrier_dev_kernel(PadTableDev t) {
  __shared__ unsigned int e;
  if (threadIdx.x == 0) e = ++(*t.counter);
  __syncthreads();
  const int tid = threadIdx.x;
  if (tid < t.g) {
    __threadfence_system();
    volatile unsigned int* slot = t.pad[tid] + t.rank;
    *slot = e;
    volatile unsigned int* mine = t.pad[t.rank] + tid;
    while ((int)(*mine - e) < 0) { }
    __threadfence_system();
  }
}

// Bounded barrier of the P2P backend (comm.PeerComm).  Same epoch protocol
// as signal_barrier_dev_kernel, but a waiter gives up when a peer does not
// arrive within timeout_ns (%globaltimer) or when any participant raised
// its abort word: it then records the reason in this rank's status word,
// raises every participant's abort word (so their barriers fail fast
// instead of spinning forever) and returns.  The host reads the status
// after the step (PeerComm.check) and raises CommError -- a dead or late
// peer can no longer hang the job.
struct BarrierTable {
  unsigned int* pad[kMaxPeers];
  unsigned int* abort_word[kMaxPeers];
  unsigned int* counter;
  unsigned int* status;
  unsigned long long timeout_ns;
  int g, rank;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void peer_barrier_kernel(BarrierTable t) {
  __shared__ unsigned int e;
  __shared__ int fail;
  if (threadIdx.x == 0) {
    e = ++(*t.counter);
    fail = 0;
  }
  __syncthreads();
  const int tid = threadIdx.x;
  if (tid < t.g) {
    __threadfence_system();
    volatile unsigned int* slot = t.pad[tid] + t.rank;
    *slot = e;
    volatile unsigned int* mine = t.pad[t.rank] + tid;
    volatile unsigned int* ab = t.abort_word[t.rank];
    const unsigned long long t0 = global_ns();
    unsigned int spins = 0;
    while ((int)(*mine - e) < 0) {
      if (*ab != 0) { atomicMax(&fail, 2); break; }
      if ((++spins & 255u) == 0 && global_ns() - t0 > t.timeout_ns) { atomicMax(&fail, 1); break; }
    }
    if (*ab != 0) atomicMax(&fail, 2);         // an abort is sticky: later barriers fail too
    __threadfence_system();
  }
  __syncthreads();
  if (fail && tid < t.g) {
    if (tid == 0) atomicMax(t.status, (unsigned int)fail);
    atomicExch(t.abort_word[tid], 1u);
    __threadfence_system();
  }
}

}  // namespace bpx

using namespace bpx;

extern "C" {

bpx_status_t bpx_reshard_pull(const void* const* src_ptrs, const size_t* src_offsets,
                              void* dst, const size_t* dst_offsets, const size_t* nbytes,
                              int n_seg, void* stream) {
  BPX_CHECK_ARG(n_seg >= 0 && n_seg <= kMaxSeg);
  if (n_seg == 0) return BPX_OK;
  BPX_CHECK_ARG(src_ptrs && src_offsets && dst && dst_offsets && nbytes);
  SegTable t{};
  bool vec = true;
  unsigned long long acc = 0;
  int k = 0;
  for (int i = 0; i < n_seg; ++i) {
    if (nbytes[i] == 0) continue;
    BPX_CHECK_ARG(src_ptrs[i] != nullptr);
    t.src[k] = static_cast<const char*>(src_ptrs[i]) + src_offsets[i];
    t.dst[k] = static_cast<char*>(dst) + dst_offsets[i];
    t.bytes[k] = nbytes[i];
    t.start[k] = acc;
    acc += nbytes[i];
    vec = vec && aligned16(t.src[k]) && aligned16(t.dst[k]) && nbytes[i] % 16 == 0;
    ++k;
  }
  t.n = k;
  t.start[k] = acc;
  if (acc == 0) return BPX_OK;
  long long units = vec ? (long long)(acc / 16) : (long long)acc;
  int grid = (int)std::min<long long>(cdivll(units, vec ? 1024 : 256), 4LL * num_sms());
  if (vec) reshard_kernel<true><<<grid, 256, 0, as_stream(stream)>>>(t);
  else reshard_kernel<false><<<grid, 256, 0, as_stream(stream)>>>(t);
  return launch_status();
}

bpx_status_t bpx_allreduce_sum_prefix(const float* const* peers, int g, float* out,
                                      size_t n, void* stream) {
  BPX_CHECK_ARG(peers && out && g >= 1 && g <= kMaxPeers);
  if (n == 0) return BPX_OK;
  PeerTable t{};
  bool vec = aligned16(out) && n % 4 == 0;
  for (int r = 0; r < g; ++r) {
    BPX_CHECK_ARG(peers[r] != nullptr);
    t.p[r] = peers[r];
    vec = vec && aligned16(peers[r]);
  }
  t.g = g;
  cudaStream_t st = as_stream(stream);
  if (vec) {
    long long n4 = (long long)(n / 4);
    int grid = (int)std::min<long long>(cdivll(n4, 256), 4LL * num_sms());
    allreduce_pull_kernel<<<grid, 256, 0, st>>>(t, reinterpret_cast<float4*>(out), n4);
  } else {
    int grid = (int)std::min<long long>(cdivll((long long)n, 256), 4LL * num_sms());
    allreduce_pull_scalar<<<grid, 256, 0, st>>>(t, out, (long long)n);
  }
  return launch_status();
}

bpx_status_t bpx_signal_barrier(uint32_t* const* pads, int rank, int g, uint32_t epoch,
                                void* stream) {
  BPX_CHECK_ARG(pads && g >= 1 && g <= kMaxPeers && rank >= 0 && rank < g);
  PadTable t{};
  for (int r = 0; r < g; ++r) {
    BPX_CHECK_ARG(pads[r] != nullptr);
    t.pad[r] = pads[r];
  }
  t.g = g; t.rank = rank; t.epoch = epoch;
  signal_barrier_kernel<<<1, 32, 0, as_stream(stream)>>>(t);
  return launch_status();
}

bpx_status_t bpx_signal_barrier_dev(uint32_t* const* pads, uint32_t* counter, int rank, int g,
                                    void* stream) {
  BPX_CHECK_ARG(pads && counter && g >= 1 && g <= kMaxPeers && rank >= 0 && rank < g);
  PadTableDev t{};
  for (int r = 0; r < g; ++r) {
    BPX_CHECK_ARG(pads[r] != nullptr);
    t.pad[r] = pads[r];
  }
  t.counter = counter;
  t.g = g; t.rank = rank;
  signal_barrier_dev_kernel<<<1, 32, 0, as_stream(stream)>>>(t);
  return launch_status();
}

bpx_status_t bpx_peer_barrier(uint32_t* const* pads, uint32_t* const* aborts,
                              uint32_t* counter, uint32_t* status, int rank, int g,
                              unsigned long long timeout_ns, void* stream) {
  BPX_CHECK_ARG(pads && aborts && counter && status && g >= 1 && g <= kMaxPeers &&
                rank >= 0 && rank < g && timeout_ns > 0);
  BarrierTable t{};
  for (int r = 0; r < g; ++r) {
    BPX_CHECK_ARG(pads[r] != nullptr && aborts[r] != nullptr);
    t.pad[r] = pads[r];
    t.abort_word[r] = aborts[r];
  }
  t.counter = counter;
  t.status = status;
  t.timeout_ns = timeout_ns;
  t.g = g; t.rank = rank;
  peer_barrier_kernel<<<1, 32, 0, as_stream(stream)>>>(t);
  return launch_status();
}

}  // extern "C"
