// C-ABI entry points of the per-layer compute ops (conv3x3 / dense),
// dispatching each call to the fastest engine that handles the shape.
#include "common.cuh"
#include "simt_api.h"
#include "tc_api.h"

using namespace bpx;

// Which engine served the calling thread's last conv/dense call, and how many
// calls this process sent to a legacy engine (the FFMA implicit GEMM, the
// per-thread-gather TS engine, the SS engine, the old wgrad engine, the
// small-Cin FFMA kernels): tests assert that every VGG-16 op at the
// benchmarked per-GPU batches takes a TMA tensor-core engine, and bench.py
// reports the legacy count of its step.
static thread_local const char* g_engine = "";
static long long g_legacy_calls = 0;
static inline void use(const char* e) { g_engine = e; }
static inline void legacy(const char* e) {
  g_engine = e;
  __atomic_add_fetch(&g_legacy_calls, 1, __ATOMIC_RELAXED);
}

extern "C" {

const char* bpx_last_engine(void) { return g_engine; }
long long bpx_legacy_engine_calls(void) { return __atomic_load_n(&g_legacy_calls, __ATOMIC_RELAXED); }

size_t bpx_conv3x3_fwd_workspace(int n, int h, int w_, int cin, int cout) {
  size_t a = tc_conv_fwd_ws(n, h, w_, cin, cout), b = ts_conv_ws(cin, cout);
  size_t c = fdt_conv_ws(n, h, w_, cin, cout);
  a = a > b ? a : b;
  return a > c ? a : c;
}

bpx_status_t bpx_conv3x3_fwd(const float* x, const float* w, const float* bias, float* y,
                             int n, int h, int w_, int cin, int cout, int relu, void* ws,
                             size_t ws_bytes, void* stream) {
  return bpx_conv3x3_fwd_presplit(x, w, nullptr, nullptr, nullptr, nullptr, nullptr, bias, y, n,
                                  h, w_, cin, cout, relu, ws, ws_bytes, stream);
}

// The fdt / c1 epilogues reduce max |out| into the caller's word; the
// legacy engines do not, so the call does it after them.
static bpx_status_t with_amax(bpx_status_t s, const float* out, size_t n, unsigned* amax,
                              cudaStream_t st) {
  if (s == BPX_OK && amax && n) {
    absmax_into(out, n, amax, st);
    count_launches(1);
  }
  return s;
}

static bool split_args(const void* hi, const void* lo, const unsigned* amax, F16Weights& wt) {
  if (!hi && !lo && !amax) return true;
  if (!hi || !lo || !amax || !aligned16(hi) || !aligned16(lo)) return false;
  wt.hi = hi; wt.lo = lo; wt.amax = amax;
  return true;
}

bpx_status_t bpx_conv3x3_fwd_presplit(const float* x, const float* w, const void* w_hi,
                                      const void* w_lo, const unsigned* w_amax,
                                      unsigned* x_amax, unsigned* y_amax,
                                      const float* bias, float* y, int n, int h, int w_,
                                      int cin, int cout, int relu, void* ws, size_t ws_bytes,
                                      void* stream) {
  BPX_CHECK_ARG(x && w && y && n >= 0 && h > 0 && w_ > 0 && cin > 0 && cout > 0);
  BPX_CHECK_ARG(cout % 4 == 0 && aligned16(y) && aligned16(w));
  F16Weights wt;
  BPX_CHECK_ARG(split_args(w_hi, w_lo, w_amax, wt));
  cudaStream_t st = as_stream(stream);
  if (c1_conv_fwd_ok(cin, cout)) {
    use("c1");
    bpx_status_t s = c1_conv_fwd(x, w, bias, y, n, h, w_, relu, x_amax, y_amax, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
    // the other engines leave x_amax alone: keep the first conv's promise
    if (x_amax && aligned16(x)) {
      absmax_into(x, (size_t)n * h * w_ * cin, x_amax, st);
      count_launches(1);
    }
  }
  const size_t ny = (size_t)n * h * w_ * cout;
  if (small_conv_fwd_ok(cin, cout))
    return legacy("small"),
           with_amax(small_conv_fwd(x, w, bias, y, n, h, w_, cin, cout, relu, st), y, ny, y_amax,
                     st);
  if (fdt_conv_ok(cin, cout, w_) && aligned16(x)) {
    use("fdt");
    bpx_status_t s = fdt_conv_fwd(x, w, wt.hi ? &wt : nullptr, x_amax, y_amax, bias, y, n, h,
                                  w_, cin, cout, relu, ws, ws_bytes, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
  }
  if (ts_conv_ok(cin, cout))
    return legacy("ts"),
           with_amax(ts_conv_fwd(x, w, bias, y, n, h, w_, cin, cout, relu, ws, ws_bytes, st), y,
                     ny, y_amax, st);
  if (tc_conv_fwd_ok(n, h, w_, cin, cout))
    return legacy("tc"),
           with_amax(tc_conv_fwd(x, w, bias, y, n, h, w_, cin, cout, relu, ws, ws_bytes, st), y,
                     ny, y_amax, st);
  return legacy("simt"),
         with_amax(simt_conv_fwd(x, w, bias, y, n, h, w_, cin, cout, relu, st), y, ny, y_amax,
                   st);
}

size_t bpx_conv3x3_dgrad_workspace(int n, int h, int w_, int cin, int cout) {
  size_t a = tc_conv_dgrad_ws(n, h, w_, cin, cout), b = ts_conv_ws(cin, cout);
  size_t c = fdt_conv_ws(n, h, w_, cin, cout);
  a = a > b ? a : b;
  return a > c ? a : c;
}

bpx_status_t bpx_conv3x3_dgrad(const float* dz, const float* w, const float* mask_src,
                               float* dx, int n, int h, int w_, int cin, int cout,
                               void* ws, size_t ws_bytes, void* stream) {
  return bpx_conv3x3_dgrad_presplit(dz, w, nullptr, nullptr, nullptr, nullptr, nullptr, mask_src,
                                    dx, n, h, w_, cin, cout, ws, ws_bytes, stream);
}

bpx_status_t bpx_conv3x3_dgrad_presplit(const float* dz, const float* w, const void* w_hi,
                                        const void* w_lo, const unsigned* w_amax,
                                        const unsigned* dz_amax, unsigned* dx_amax,
                                        const float* mask_src, float* dx, int n, int h, int w_,
                                        int cin, int cout, void* ws, size_t ws_bytes,
                                        void* stream) {
  BPX_CHECK_ARG(dz && w && dx && n >= 0 && h > 0 && w_ > 0 && cin > 0 && cout > 0);
  BPX_CHECK_ARG(cin % 4 == 0 && aligned16(dx) && aligned16(w));
  F16Weights wt;
  BPX_CHECK_ARG(split_args(w_hi, w_lo, w_amax, wt));
  cudaStream_t st = as_stream(stream);
  if (fdt_conv_ok(cin, cout, w_) && aligned16(dz) && (!mask_src || aligned16(mask_src))) {
    use("fdt");
    bpx_status_t s = fdt_conv_dgrad(dz, w, wt.hi ? &wt : nullptr, dz_amax, dx_amax, mask_src, dx,
                                    n, h, w_, cin, cout, ws, ws_bytes, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
  }
  const size_t nx = (size_t)n * h * w_ * cin;
  if (ts_conv_ok(cin, cout))
    return legacy("ts"),
           with_amax(ts_conv_dgrad(dz, w, mask_src, dx, n, h, w_, cin, cout, ws, ws_bytes, st),
                     dx, nx, dx_amax, st);
  if (tc_conv_dgrad_ok(n, h, w_, cin, cout))
    return legacy("tc"),
           with_amax(tc_conv_dgrad(dz, w, mask_src, dx, n, h, w_, cin, cout, ws, ws_bytes, st),
                     dx, nx, dx_amax, st);
  return legacy("simt"),
         with_amax(simt_conv_dgrad(dz, w, mask_src, dx, n, h, w_, cin, cout, st), dx, nx,
                   dx_amax, st);
}

size_t bpx_conv3x3_wgrad_workspace(int n, int h, int w_, int cin, int cout) {
  size_t a = simt_conv_wgrad_ws(n, h, w_, cin, cout);
  size_t b = tc_conv_wgrad_ws(n, h, w_, cin, cout);
  size_t c = wg_conv_ws(n, h, w_, cin, cout);
  size_t d = wgt_conv_ws(n, h, w_, cin, cout);
  size_t g = wgh_conv_ws(n, h, w_, cin, cout);
  d = d > g ? d : g;
  g = wgc_conv_ws(n, h, w_, cin, cout);
  d = d > g ? d : g;
  g = wg1_conv_ws(n, h, w_, cin, cout);
  d = d > g ? d : g;
  size_t e = small_conv_wgrad_ws(n, h, w_, cin, cout);
  size_t f = thin_conv_wgrad_ws(n, h, w_, cin, cout);
  e = e > f ? e : f;
  size_t m = a > b ? a : b;
  m = m > c ? m : c;
  m = m > d ? m : d;
  return m > e ? m : e;
}

bpx_status_t bpx_conv3x3_wgrad(const float* x, const float* dz, float* dw, float* dbias,
                               int n, int h, int w_, int cin, int cout, void* ws,
                               size_t ws_bytes, void* stream) {
  return bpx_conv3x3_wgrad_presplit(x, dz, nullptr, nullptr, dw, dbias, n, h, w_, cin, cout, ws,
                                    ws_bytes, stream);
}

bpx_status_t bpx_conv3x3_wgrad_presplit(const float* x, const float* dz, const unsigned* x_amax,
                                        const unsigned* dz_amax, float* dw, float* dbias, int n,
                                        int h, int w_, int cin, int cout, void* ws,
                                        size_t ws_bytes, void* stream) {
  BPX_CHECK_ARG(x && dz && dw && n >= 0 && h > 0 && w_ > 0 && cin > 0 && cout > 0);
  BPX_CHECK_ARG(ws || ws_bytes == 0);
  cudaStream_t st = as_stream(stream);
  if (wg1_conv_ok(n, h, w_, cin, cout) && aligned16(x) && aligned16(dz) && aligned16(dw) &&
      (!dbias || aligned16(dbias)) && aligned16(ws))
    return use("wg1"), wg1_conv_wgrad(x, dz, x_amax, dz_amax, dw, dbias, n, h, w_, ws, ws_bytes,
                                      st);
  if (wgc_conv_ok(n, h, w_, cin, cout) && aligned16(x) && aligned16(dz) && aligned16(dw) &&
      (!dbias || aligned16(dbias)) && aligned16(ws))
    return use("wgc"), wgc_conv_wgrad(x, dz, x_amax, dz_amax, dw, dbias, n, h, w_, ws, ws_bytes,
                                      st);
  if (wgh_conv_ok(cin, cout) && aligned16(x) && aligned16(dz) && aligned16(dw) &&
      (!dbias || aligned16(dbias)) && aligned16(ws))
    return use("wgh"), wgh_conv_wgrad(x, dz, x_amax, dz_amax, dw, dbias, n, h, w_, cin, cout, ws,
                                      ws_bytes, st);
  if (wgt_conv_ok(cin, cout) && aligned16(x) && aligned16(dz) && aligned16(dw) &&
      (!dbias || aligned16(dbias)))
    return use("wgt"), wgt_conv_wgrad(x, dz, dw, dbias, n, h, w_, cin, cout, ws, ws_bytes, st);
  if (thin_conv_wgrad_ok(cin, cout, w_)) {
    use("thin");
    bpx_status_t s = thin_conv_wgrad(x, dz, dw, dbias, n, h, w_, cin, cout, ws, ws_bytes, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
  }
  if (small_conv_wgrad_ok(cin, cout) && aligned16(dz))
    return legacy("small"), small_conv_wgrad(x, dz, dw, dbias, n, h, w_, cin, cout, ws, ws_bytes, st);
  if (wg_conv_ok(cin, cout))
    return legacy("wg"), wg_conv_wgrad(x, dz, dw, dbias, n, h, w_, cin, cout, ws, ws_bytes, st);
  if (tc_conv_wgrad_ok(n, h, w_, cin, cout))
    return legacy("tc"), tc_conv_wgrad(x, dz, dw, dbias, n, h, w_, cin, cout, ws, ws_bytes, st);
  return legacy("simt"), simt_conv_wgrad(x, dz, dw, dbias, n, h, w_, cin, cout, ws, ws_bytes, st);
}

static size_t max3(size_t a, size_t b, size_t c) {
  size_t m = a > b ? a : b;
  return m > c ? m : c;
}
size_t bpx_linear_fwd_workspace(int b, int in, int out) {
  size_t m = max3(simt_linear_fwd_ws(b, in, out), tc_linear_fwd_ws(b, in, out),
                  dns_linear_ws(b, in, out));
  size_t d = dtc_linear_ws(b, in, out);
  return m > d ? m : d;
}
size_t bpx_linear_dgrad_workspace(int b, int in, int out) {
  size_t m = max3(simt_linear_dgrad_ws(b, in, out), tc_linear_dgrad_ws(b, in, out),
                  dns_linear_ws(b, in, out));
  size_t d = dtc_linear_ws(b, in, out);
  return m > d ? m : d;
}
size_t bpx_linear_wgrad_workspace(int b, int in, int out) {
  size_t m = max3(simt_linear_wgrad_ws(b, in, out), tc_linear_wgrad_ws(b, in, out),
                  dns_linear_ws(b, in, out));
  size_t d = max3(dwt_linear_ws(b, in, out), thin_linear_ws(b, in, out), 0);
  return m > d ? m : d;
}

bpx_status_t bpx_linear_fwd(const float* x, const float* w, const float* bias, float* y,
                            int b, int in, int out, int relu, void* ws, size_t ws_bytes,
                            void* stream) {
  BPX_CHECK_ARG(x && w && y && b >= 0 && in > 0 && out > 0 && aligned16(w));
  cudaStream_t st = as_stream(stream);
  if (dtc_linear_ok(b, in, out)) {
    use("dtc");
    bpx_status_t s = dtc_linear_fwd(x, w, bias, y, b, in, out, relu, ws, ws_bytes, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
  }
  if (dns_linear_ok(b, in, out))
    return use("dns"), dns_linear_fwd(x, w, bias, y, b, in, out, relu, ws, ws_bytes, st);
  // pixel-batched 1x1 convs with 32 outputs (the four-tower net's towers)
  if (thin_linear_ok(b, in, out)) {
    use("thin");
    bpx_status_t s = thin_linear_fwd(x, w, bias, y, b, in, out, relu, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
  }
  // pixel-batched dense ops (the 1x1 convs of the four-tower net: b = pixels)
  // also go to the tensor-core engine: the FFMA fallback's fwd orientation
  // took ~3 ms at b = 39200, in = 128, out = 32
  if (tc_linear_ok(b, in, out) || (b > 256 && b % 4 == 0 && in % 4 == 0 && out % 4 == 0))
    return use("tc"), tc_linear_fwd(x, w, bias, y, b, in, out, relu, ws, ws_bytes, st);
  return legacy("simt"), simt_linear_fwd(x, w, bias, y, b, in, out, relu, ws, ws_bytes, st);
}

bpx_status_t bpx_linear_dgrad(const float* dy, const float* w, const float* mask_src,
                              float* dx, int b, int in, int out, void* ws, size_t ws_bytes,
                              void* stream) {
  BPX_CHECK_ARG(dy && w && dx && b >= 0 && in > 0 && out > 0 && aligned16(w));
  cudaStream_t st = as_stream(stream);
  if (dtc_linear_ok(b, in, out)) {
    use("dtc");
    bpx_status_t s = dtc_linear_dgrad(dy, w, mask_src, dx, b, in, out, ws, ws_bytes, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
  }
  if (dns_linear_ok(b, in, out))
    return use("dns"), dns_linear_dgrad(dy, w, mask_src, dx, b, in, out, ws, ws_bytes, st);
  if (thin_linear_ok(b, in, out)) {
    use("thin");
    bpx_status_t s = thin_linear_dgrad(dy, w, mask_src, dx, b, in, out, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
  }
  if (tc_linear_ok(b, in, out) || (b > 256 && b % 4 == 0 && in % 4 == 0 && out % 4 == 0))
    return use("tc"), tc_linear_dgrad(dy, w, mask_src, dx, b, in, out, ws, ws_bytes, st);
  return legacy("simt"), simt_linear_dgrad(dy, w, mask_src, dx, b, in, out, ws, ws_bytes, st);
}

bpx_status_t bpx_linear_wgrad(const float* x, const float* dy, float* dw, float* dbias,
                              int b, int in, int out, void* ws, size_t ws_bytes,
                              void* stream) {
  BPX_CHECK_ARG(x && dy && dw && b >= 0 && in > 0 && out > 0 && aligned16(dw));
  cudaStream_t st = as_stream(stream);
  // tensor-core engine above 8 rows: both engines are bound by writing dW,
  // but the FFMA outer product's math grows with b (B200, fc1: 189 vs 93 us
  // at b = 32, 118 vs 91 at 16; at b <= 8 the FFMA kernel is ~14 us faster)
  if (b > 8 && dwt_linear_ok(b, in, out)) {
    use("dwt");
    bpx_status_t s = dwt_linear_wgrad(x, dy, dw, dbias, b, in, out, ws, ws_bytes, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
  }
  if (dns_linear_ok(b, in, out))
    return use("dns"), dns_linear_wgrad(x, dy, dw, dbias, b, in, out, ws, ws_bytes, st);
  if (thin_linear_ok(b, in, out)) {
    use("thin");
    bpx_status_t s = thin_linear_wgrad(x, dy, dw, dbias, b, in, out, ws, ws_bytes, st);
    if (s != BPX_ERR_UNSUPPORTED) return s;
  }
  if (tc_linear_ok(b, in, out) || (b > 256 && b % 4 == 0 && in % 4 == 0 && out % 4 == 0))
    return use("tc"), tc_linear_wgrad(x, dy, dw, dbias, b, in, out, ws, ws_bytes, st);
  return legacy("simt"), simt_linear_wgrad(x, dy, dw, dbias, b, in, out, ws, ws_bytes, st);
}

// Engine-pinned variants for tests and benchmarks (same semantics).
bpx_status_t bpx_simt_conv3x3_fwd(const float* x, const float* w, const float* bias,
                                  float* y, int n, int h, int w_, int cin, int cout,
                                  int relu, void* stream) {
  return simt_conv_fwd(x, w, bias, y, n, h, w_, cin, cout, relu, as_stream(stream));
}
bpx_status_t bpx_simt_conv3x3_dgrad(const float* dz, const float* w, const float* mask,
                                    float* dx, int n, int h, int w_, int cin, int cout,
                                    void* stream) {
  return simt_conv_dgrad(dz, w, mask, dx, n, h, w_, cin, cout, as_stream(stream));
}
bpx_status_t bpx_simt_conv3x3_wgrad(const float* x, const float* dz, float* dw,
                                    float* dbias, int n, int h, int w_, int cin, int cout,
                                    void* ws, size_t ws_bytes, void* stream) {
  return simt_conv_wgrad(x, dz, dw, dbias, n, h, w_, cin, cout, ws, ws_bytes,
                         as_stream(stream));
}

}  // extern "C"
