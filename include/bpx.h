/*
 * libbpx -- C-ABI of the B200 burst-parallel training runtime.
 *
 * The reference (`burstplan`, /root/reference/pkg) has no FFI: it *models*
 * each per-iteration op as an OpRecord with a priced duration
 * (simulator.py:175-196, compile_timeline :211-298).  Each entry point below
 * is the real sm_100a implementation of one of those modeled ops; the
 * comment on each names the reference construct it replaces.
 *
 * Conventions (all entry points):
 *   - plain device pointers + sizes; no torch / CUDA types in signatures
 *     (`stream` is a cudaStream_t passed as void*; NULL = legacy stream);
 *   - stream-ordered, asynchronous, no host synchronisation, no allocation:
 *     scratch space is caller-provided (query sizes with *_workspace);
 *     every call is CUDA-graph capturable;
 *   - return BPX_OK (0) or a nonzero bpx_status_t, never abort/throw;
 *   - fp32 storage, fp32-accurate arithmetic (tensor-core paths use a
 *     3xTF32 split); activations are NHWC, conv weights OHWI
 *     ([Cout][3][3][Cin]), dense weights [out][in];
 *   - deterministic: fixed-order reductions, bitwise run-to-run stable.
 */
#ifndef BPX_H_
#define BPX_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BPX_API __attribute__((visibility("default")))
#else
#define BPX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int bpx_status_t;

enum {
  BPX_OK = 0,
  BPX_ERR_INVALID_ARGUMENT = 1, /* bad shape / null pointer / alignment   */
  BPX_ERR_LAUNCH = 2,           /* cudaGetLastError after launch != 0     */
  BPX_ERR_UNSUPPORTED = 3,      /* shape outside what the kernels handle  */
  BPX_ERR_WORKSPACE = 4,        /* caller workspace too small             */
  BPX_ERR_ARCH = 5              /* device is not sm_100 (no fallback)     */
};

/* Human-readable name of a status code (static storage). */
BPX_API const char* bpx_status_string(bpx_status_t status);
/* ABI version, bumped on any signature change. */
BPX_API int bpx_abi_version(void);
/* Kernel launches this process issued through libbpx so far (host count;
 * a CUDA-graph replay re-runs the captured launches without counting). */
BPX_API long long bpx_launch_count(void);
/* Engine that served the calling thread's last conv3x3 / linear call:
 * "fdt" (TMA fwd/dgrad), "wgh" (TMA wgrad), "wgt" (conv1_1 wgrad), "c1"
 * (conv1_1 fwd), "dtc"
 * (dense fwd/dgrad), "dwt" (dense wgrad), "dns" (dense FFMA, <= 8 rows or
 * 1000 outputs), "tc" (pixel-batched 1x1 convs); legacy: "simt", "ts",
 * "wg", "small".  Static storage.                                         */
BPX_API const char* bpx_last_engine(void);
/* conv3x3 / linear calls this process sent to a legacy engine.            */
BPX_API long long bpx_legacy_engine_calls(void);
/* SM budget of the calling host thread's later launches (0 = all SMs):
 * persistent grids and split-K factors are sized to at most n SMs, so work
 * launched or graph-captured under a budget keeps the rest of the GPU free
 * for other streams (the background job under multiplexing).  Returns the
 * previous budget.                                                        */
BPX_API int bpx_set_sm_budget(int n);
/* 1 if the current device is sm_100 (the only supported target). */
BPX_API int bpx_device_supported(void);

/* ---- per-layer compute: replaces the modeled `compute` OpRecord ------
 * (simulator.py:254-261; cost = comp(i,g) from graph.py:352-385 at the
 * per-GPU batch ceil(B/g)).  n = that per-GPU batch.                      */

/* y = relu?(conv3x3_pad1(x, w) + bias).  x:[n,h,w,cin] y:[n,h,w,cout]     */
BPX_API bpx_status_t bpx_conv3x3_fwd(const float* x, const float* w, const float* bias,
                             float* y, int n, int h, int w_, int cin, int cout,
                             int relu, void* ws, size_t ws_bytes, void* stream);
BPX_API size_t bpx_conv3x3_fwd_workspace(int n, int h, int w_, int cin, int cout);
/* Same op with its fp16x3 operands prepared by the caller (DESIGN.md,
 * "fp16x3"): w_hi / w_lo / w_amax = the weights split by bpx_f16_split
 * (fp16 [cout][3][3][cin] each, and the split span's max |w| bits), made
 * once per update instead of once per call; x_amax = max |x| as bits
 * (bpx_absmax, or written by the producer of x; the 3-channel first conv
 * (Cin = 3, Cout = 64) reduces x into it itself as it reads x -- atomicMax,
 * a no-op on a word that already holds it -- so a zeroed word will do).
 * Each may be NULL (the call then prepares it in its workspace).  y_amax
 * (nullable): atomicMax'ed
 * with the max |y| bits -- the next conv's x_amax, fused into this
 * producer (zero it first).  bpx_conv3x3_dgrad_presplit likewise, with
 * dz_amax for dz and dx_amax for dx.                                       */
BPX_API bpx_status_t bpx_conv3x3_fwd_presplit(const float* x, const float* w,
                                      const void* w_hi, const void* w_lo,
                                      const unsigned* w_amax, unsigned* x_amax,
                                      unsigned* y_amax, const float* bias, float* y,
                                      int n, int h, int w_, int cin, int cout, int relu,
                                      void* ws, size_t ws_bytes, void* stream);
/* *amax = max |x[i]| as its fp32 bit pattern (x 16-B aligned).           */
BPX_API bpx_status_t bpx_absmax(const float* x, size_t n, unsigned* amax, void* stream);
/* fp16x3 weight split: *amax = max |w|, s = 14 - floor(log2 *amax) (so
 * |w 2^s| < 2^15), hi = fp16(w 2^s), lo = fp16(w 2^s - hi); hi, lo hold n
 * fp16 each (8-B aligned), in w's layout.                                  */
BPX_API bpx_status_t bpx_f16_split(const float* w, size_t n, void* hi, void* lo,
                                   unsigned* amax, void* stream);
/* Batched bpx_f16_split of nseg weight tensors in three graph nodes (a
 * memset of the nwords amax words, one max launch, one split launch): segs
 * is a DEVICE array of records {const float* w; void* hi; void* lo;
 * unsigned* amax; int64 n4; int64 blk0}, n4 = floats / 4 (w 16-B aligned,
 * hi/lo 8-B aligned), blk0 = the segment's first block with
 * bpx_f16_split_batch_chunk() float4 per block; blocks = the total.        */
BPX_API bpx_status_t bpx_f16_split_batch(const void* segs, int nseg, long long blocks,
                                         unsigned* words, size_t nwords, void* stream);
BPX_API int bpx_f16_split_batch_chunk(void);

/* dx = conv3x3_transpose(dz, w) [* (mask_src > 0) if mask_src != NULL].
 * dz:[n,h,w,cout] dx,mask_src:[n,h,w,cin].  mask_src is the layer input
 * when that input is a ReLU output: fuses the previous ReLU's backward.   */
BPX_API bpx_status_t bpx_conv3x3_dgrad(const float* dz, const float* w,
                               const float* mask_src, float* dx, int n, int h,
                               int w_, int cin, int cout, void* ws,
                               size_t ws_bytes, void* stream);
BPX_API size_t bpx_conv3x3_dgrad_workspace(int n, int h, int w_, int cin, int cout);
BPX_API bpx_status_t bpx_conv3x3_dgrad_presplit(const float* dz, const float* w,
                                        const void* w_hi, const void* w_lo,
                                        const unsigned* w_amax, const unsigned* dz_amax,
                                        unsigned* dx_amax, const float* mask_src, float* dx,
                                        int n, int h, int w_, int cin, int cout, void* ws,
                                        size_t ws_bytes, void* stream);

/* dw[cout,3,3,cin] = sum_pixels dz (x) im2col(x);  dbias[cout] = sum dz.  */
BPX_API bpx_status_t bpx_conv3x3_wgrad(const float* x, const float* dz, float* dw,
                               float* dbias, int n, int h, int w_, int cin,
                               int cout, void* ws, size_t ws_bytes,
                               void* stream);
BPX_API size_t bpx_conv3x3_wgrad_workspace(int n, int h, int w_, int cin, int cout);
/* Same op with the operands' max |v| words supplied (bpx_absmax; each
 * nullable): the fp16x3 engine scales x and dz by powers of two from them. */
BPX_API bpx_status_t bpx_conv3x3_wgrad_presplit(const float* x, const float* dz,
                                        const unsigned* x_amax, const unsigned* dz_amax,
                                        float* dw, float* dbias, int n, int h, int w_,
                                        int cin, int cout, void* ws, size_t ws_bytes,
                                        void* stream);

/* y[b,out] = relu?(x[b,in] . w[out,in]^T + bias)                           */
BPX_API bpx_status_t bpx_linear_fwd(const float* x, const float* w, const float* bias,
                            float* y, int b, int in, int out, int relu,
                            void* ws, size_t ws_bytes, void* stream);
BPX_API size_t bpx_linear_fwd_workspace(int b, int in, int out);
/* dx[b,in] = dy[b,out] . w [* (mask_src > 0)]                              */
BPX_API bpx_status_t bpx_linear_dgrad(const float* dy, const float* w,
                              const float* mask_src, float* dx, int b, int in,
                              int out, void* ws, size_t ws_bytes, void* stream);
BPX_API size_t bpx_linear_dgrad_workspace(int b, int in, int out);
/* dw[out,in] = dy^T . x ;  dbias[out] = sum_b dy                           */
BPX_API bpx_status_t bpx_linear_wgrad(const float* x, const float* dy, float* dw,
                              float* dbias, int b, int in, int out, void* ws,
                              size_t ws_bytes, void* stream);
BPX_API size_t bpx_linear_wgrad_workspace(int b, int in, int out);

/* 2x2/stride-2 max pool, NHWC; bwd routes dy to the first max of each
 * window (PyTorch order) recomputed from x.                                */
BPX_API bpx_status_t bpx_maxpool2x2_fwd(const float* x, float* y, int n, int h, int w_,
                                int c, void* stream);
BPX_API bpx_status_t bpx_maxpool2x2_bwd(const float* x, const float* dy, float* dx,
                                int n, int h, int w_, int c, void* stream);
/* Same pool, keeping each window's first-max position (idx: one byte per
 * output element, values 0..3 in (row, col) order) for a backward that
 * reads idx + dy instead of x + dy.  y_amax / dx_amax (nullable):
 * atomicMax'ed with the max |v| bits of the output (the consumer conv's
 * fp16x3 scale word; zero it before the step).                             */
BPX_API bpx_status_t bpx_maxpool2x2_fwd_idx(const float* x, float* y, uint8_t* idx, int n,
                                    int h, int w_, int c, unsigned* y_amax, void* stream);
BPX_API bpx_status_t bpx_maxpool2x2_bwd_idx(const uint8_t* idx, const float* dy, float* dx,
                                    int n, int h, int w_, int c, unsigned* dx_amax,
                                    void* stream);

/* ---- branch/join elements of the residual net behind `wideresnet_like`
 * (synth.py:126-169; the `add` layers of its residual diamonds, the stage
 * transitions where hw halves, and the pool before the classifier).
 * Residual join (post-activation basic block, ResNet "option A" shortcut):
 *   y = relu?(a + P(s)),  a, y: [n][h][w][c],  s: [n][h*f][w*f][cs], cs <= c,
 *   P = stride-f subsample (f = 2 if down) + zero channel padding cs -> c.
 * y_amax (nullable): atomicMax'ed with max |y| bits (zero it first).      */
BPX_API bpx_status_t bpx_residual_add_fwd(const float* a, const float* s, float* y, int n,
                                  int h, int w_, int c, int cs, int down, int relu,
                                  unsigned* y_amax, void* stream);
/* Gradient into the skip source h ([n][h*f][w*f][cs], grad wrt h's
 * pre-activation; mask = h's ReLU output):
 *   dh = (accumulate ? dh : 0) + [sampled pixel] * (dmain + (mask > 0) * dz[.., :cs])
 * dmain (nullable, [n][h][w][cs]) = the already-masked data gradient of a
 * first conv that read the subsampled h; accumulate and dmain are exclusive. */
BPX_API bpx_status_t bpx_residual_skip_bwd(const float* dz, const float* dmain,
                                   const float* mask, float* dh, int n, int h, int w_,
                                   int c, int cs, int down, int accumulate, void* stream);
/* y[n][h][w][c] = x[n][2h][2w][c] (stride-2 subsample of the stage input) */
BPX_API bpx_status_t bpx_subsample2_fwd(const float* x, float* y, int n, int h, int w_,
                                int c, void* stream);
/* dx[n][2h][2w][c] = dy[n][h][w][c] at even (row, col), 0 elsewhere       */
BPX_API bpx_status_t bpx_subsample2_bwd(const float* dy, float* dx, int n, int h, int w_,
                                int c, void* stream);
/* dst += src (n floats, n % 4 == 0): gradient fan-in across layouts        */
BPX_API bpx_status_t bpx_accumulate(float* dst, const float* src, size_t n, void* stream);
/* ---- branch/join elements of the four-tower net behind `inception_like`
 * (synth.py:172-226).  Pool tower: 3x3 / stride-1 / pad-1 max pool over the
 * first cs channels of x [n][h][w][c] -> y, idx [n][h][w][cs] (idx = first
 * max position 0..8, row-major window); bwd writes all c channels of dx
 * (0 beyond cs), gathering each input's gradient in fixed order.           */
BPX_API bpx_status_t bpx_maxpool3x3_fwd_idx(const float* x, float* y, uint8_t* idx, int n,
                                    int h, int w_, int c, int cs, void* stream);
BPX_API bpx_status_t bpx_maxpool3x3_bwd_idx(const uint8_t* idx, const float* dy, float* dx,
                                    int n, int h, int w_, int c, int cs, void* stream);
/* Channel concat of k <= 4 NHWC parts (cs[i] channels each, multiples of 4)
 * over npix pixels; bwd slices dy back into the parts.                     */
BPX_API bpx_status_t bpx_concat_fwd(const float* const* parts, const int* cs, int k, float* y,
                            long long npix, void* stream);
BPX_API bpx_status_t bpx_concat_bwd(const float* dy, float* const* parts, const int* cs, int k,
                            long long npix, void* stream);
/* y[n][i][j][c] = x[n][2i+off][2j+off][c], off in {0, 1} (35 -> 17 keeps the
 * odd pixels); bwd: dx = dy at those pixels, 0 elsewhere.                   */
BPX_API bpx_status_t bpx_subsample_fwd(const float* x, float* y, int n, int hin, int win,
                               int h, int w_, int c, int off, void* stream);
BPX_API bpx_status_t bpx_subsample_bwd(const float* dy, float* dx, int n, int hin, int win,
                               int h, int w_, int c, int off, void* stream);
/* Global average pool [n][h][w][c] -> [n][c]; bwd: dx = dy / (h*w), masked
 * by (mask > 0) when mask (the pooled ReLU output) is given.               */
BPX_API bpx_status_t bpx_global_avgpool_fwd(const float* x, float* y, int n, int h, int w_,
                                    int c, void* stream);
BPX_API bpx_status_t bpx_global_avgpool_bwd(const float* dy, const float* mask, float* dx,
                                    int n, int h, int w_, int c, void* stream);

/* ---- synchronised batch normalisation of the residual nets' convs
 * (the reference has no BN notion).  z, y, g, dz:
 * [npix][c] NHWC (npix = this rank's pixels, ntot = the whole layer
 * group's); gamma_beta = [beta ; gamma] (2c, the layer's "bias" slot).
 * stats / sums are 2c floats of LOCAL per-channel sums that the caller
 * allreduces over the layer's group [0, g) before the apply steps, so every
 * rank normalises with full-batch statistics whatever g is.
 *   stats    = [sum z ; sum z^2]
 *   y        = act(gamma * (z - mu) * rstd + beta),  mu, var from stats / ntot
 *   sums     = [sum g ; sum g * xhat]  (= the local [dbeta ; dgamma])
 *   dz       = gamma * rstd * (g - sums0/ntot - xhat * sums1/ntot)
 * Fixed-order fp64 sums: bitwise reproducible.  c % 4 == 0, c <= 4096.
 * y_amax / dz_amax (nullable): atomicMax'ed with the output's max |v| bits
 * (the fp16x3 scale word of the conv that reads it; zero it first).        */
BPX_API size_t bpx_bn_workspace(long long npix, int c);
BPX_API bpx_status_t bpx_bn_stats(const float* z, long long npix, int c, float* stats,
                          void* ws, size_t ws_bytes, void* stream);
BPX_API bpx_status_t bpx_bn_apply(const float* z, const float* stats, const float* gamma_beta,
                          long long npix, long long ntot, int c, float eps, int relu,
                          float* y, unsigned* y_amax, void* stream);
BPX_API bpx_status_t bpx_bn_bwd_sums(const float* g, const float* z, const float* stats,
                             long long npix, long long ntot, int c, float eps, float* sums,
                             void* ws, size_t ws_bytes, void* stream);
BPX_API bpx_status_t bpx_bn_bwd_apply(const float* g, const float* z, const float* stats,
                              const float* sums, const float* gamma_beta, long long npix,
                              long long ntot, int c, float eps, float* dz,
                              unsigned* dz_amax, void* stream);

/* Mean softmax cross-entropy over the GLOBAL batch: loss_out[0] =
 * sum_{local rows} CE / b_global (fixed order); loss_out must hold
 * b_local + 1 floats ([1..b_local] = per-row terms);
 * dlogits = (softmax - onehot) / b_global.                                 */
BPX_API bpx_status_t bpx_softmax_xent(const float* logits, const int32_t* labels,
                              int b_local, int b_global, int classes,
                              float* loss_out, float* dlogits, void* stream);

/* w -= lr * g  (plain SGD, fp32)                                           */
BPX_API bpx_status_t bpx_sgd_update(float* w, const float* g, size_t n, float lr,
                            void* stream);

/* ---- sample resharding: replaces the modeled `transfer` OpRecord ------
 * (simulator.py:242-253; volume = moved_samples * act bytes, costs.py:85-118).
 * Pull model: this rank copies each segment from a (peer-mapped) source
 * pointer into its own buffer.  src_ptrs / src_offsets / dst_offsets /
 * nbytes are HOST arrays of n_seg (<= 64) entries, one per contiguous run
 * (host-side index map: costs.reshard_segments); they are captured by value
 * into the launch, so the call is CUDA-graph safe.
 * Pointers may be NVLink peer addresses (P2P loads) or local.              */
BPX_API bpx_status_t bpx_reshard_pull(const void* const* src_ptrs,
                              const size_t* src_offsets, void* dst,
                              const size_t* dst_offsets, const size_t* nbytes,
                              int n_seg, void* stream);

/* ---- subset gradient allreduce: replaces the modeled `allreduce` ------
 * (simulator.py:264-278; ring volume 2N(g-1)/g, costs.py:130-140).
 * One-shot pull allreduce over ranks [0,g): out = sum_{r<g} peers[r][0:n]
 * accumulated in rank order (bitwise identical on every rank).  `peers`
 * is a host array of g device pointers (peer-mapped).                      */
BPX_API bpx_status_t bpx_allreduce_sum_prefix(const float* const* peers, int g,
                                      float* out, size_t n, void* stream);

/* Cross-GPU flag barrier for graph-captured P2P phases: write `epoch` into
 * slot `rank` of every peer's signal pad, then spin until all g slots of
 * the local pad reach `epoch`.  pads[r] = rank r's pad (g uint32 slots).   */
BPX_API bpx_status_t bpx_signal_barrier(uint32_t* const* pads, int rank, int g,
                                uint32_t epoch, void* stream);
/* Same barrier for CUDA-graph replay: the epoch is this rank's device
 * counter for the group (*counter), incremented by the kernel, so each
 * replay waits for the next epoch.  Every participant calls it in the same
 * sequence.                                                                */
BPX_API bpx_status_t bpx_signal_barrier_dev(uint32_t* const* pads, uint32_t* counter,
                                    int rank, int g, void* stream);

/* Bounded barrier of the P2P backend: the device-epoch protocol of
 * bpx_signal_barrier_dev over pads[0..g) (pads[r] = rank r's g slots for
 * this group), but a waiter stops after timeout_ns without a peer's arrival
 * or as soon as its own abort word (aborts[rank]) is nonzero; it then
 * writes the reason into *status (1 = timeout, 2 = aborted; atomic max),
 * raises every participant's abort word and returns.  The caller reads
 * *status after the phase and fails the step (no hang on a dead peer).    */
BPX_API bpx_status_t bpx_peer_barrier(uint32_t* const* pads, uint32_t* const* aborts,
                              uint32_t* counter, uint32_t* status, int rank, int g,
                              unsigned long long timeout_ns, void* stream);

/* ---- engine-pinned variants (tests / benchmarks): force the FFMA
 * implicit-GEMM engine regardless of shape, same semantics as above.      */
BPX_API bpx_status_t bpx_simt_conv3x3_fwd(const float* x, const float* w,
                                          const float* bias, float* y, int n,
                                          int h, int w_, int cin, int cout,
                                          int relu, void* stream);
BPX_API bpx_status_t bpx_simt_conv3x3_dgrad(const float* dz, const float* w,
                                            const float* mask_src, float* dx,
                                            int n, int h, int w_, int cin,
                                            int cout, void* stream);
BPX_API bpx_status_t bpx_simt_conv3x3_wgrad(const float* x, const float* dz,
                                            float* dw, float* dbias, int n,
                                            int h, int w_, int cin, int cout,
                                            void* ws, size_t ws_bytes,
                                            void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BPX_H_ */
