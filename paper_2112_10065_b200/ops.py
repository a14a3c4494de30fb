"""ctypes binding of libbpx (include/bpx.h) for torch CUDA tensors.

Each wrapper checks dtype / device / contiguity, passes raw device pointers
and the *current* torch CUDA stream, and turns a nonzero bpx_status_t into
``KernelError``.  There is deliberately no CPU or PyTorch fallback: if the
library is missing the first call raises ``ExtensionMissingError``.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

from .errors import ExtensionMissingError, KernelError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BPX_LIB", os.path.join(_HERE, "libbpx.so"))  # BPX_LIB: A/B timing of builds

_lib = None

_c_float_p = ctypes.c_void_p
_SIGS = {
    # name: (restype, argtypes)
    "bpx_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "bpx_abi_version": (ctypes.c_int, []),
    "bpx_device_supported": (ctypes.c_int, []),
    "bpx_launch_count": (ctypes.c_longlong, []),
    "bpx_last_engine": (ctypes.c_char_p, []),
    "bpx_legacy_engine_calls": (ctypes.c_longlong, []),
    "bpx_set_sm_budget": (ctypes.c_int, [ctypes.c_int]),
    "bpx_conv3x3_fwd": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 6
                        + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_conv3x3_fwd_workspace": (ctypes.c_size_t, [ctypes.c_int] * 5),
    "bpx_conv3x3_fwd_presplit": (ctypes.c_int, [_c_float_p] * 9 + [ctypes.c_int] * 6
                                 + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_conv3x3_dgrad_presplit": (ctypes.c_int, [_c_float_p] * 9 + [ctypes.c_int] * 5
                                   + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_conv3x3_wgrad_presplit": (ctypes.c_int, [_c_float_p] * 6 + [ctypes.c_int] * 5
                                   + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_f16_split_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong,
                                           ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_f16_split_batch_chunk": (ctypes.c_int, []),
    "bpx_absmax": (ctypes.c_int, [_c_float_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]),
    "bpx_f16_split": (ctypes.c_int, [_c_float_p, ctypes.c_size_t] + [ctypes.c_void_p] * 4),
    "bpx_conv3x3_dgrad": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 5
                          + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_conv3x3_dgrad_workspace": (ctypes.c_size_t, [ctypes.c_int] * 5),
    "bpx_conv3x3_wgrad": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 5
                          + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_conv3x3_wgrad_workspace": (ctypes.c_size_t, [ctypes.c_int] * 5),
    "bpx_linear_fwd": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 4
                       + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_linear_fwd_workspace": (ctypes.c_size_t, [ctypes.c_int] * 3),
    "bpx_linear_dgrad": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 3
                         + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_linear_dgrad_workspace": (ctypes.c_size_t, [ctypes.c_int] * 3),
    "bpx_linear_wgrad": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 3
                         + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_linear_wgrad_workspace": (ctypes.c_size_t, [ctypes.c_int] * 3),
    "bpx_maxpool2x2_fwd": (ctypes.c_int, [_c_float_p] * 2 + [ctypes.c_int] * 4
                           + [ctypes.c_void_p]),
    "bpx_maxpool2x2_bwd": (ctypes.c_int, [_c_float_p] * 3 + [ctypes.c_int] * 4
                           + [ctypes.c_void_p]),
    "bpx_maxpool2x2_fwd_idx": (ctypes.c_int, [_c_float_p] * 3 + [ctypes.c_int] * 4
                               + [ctypes.c_void_p, ctypes.c_void_p]),
    "bpx_maxpool2x2_bwd_idx": (ctypes.c_int, [_c_float_p] * 3 + [ctypes.c_int] * 4
                               + [ctypes.c_void_p, ctypes.c_void_p]),
    "bpx_residual_add_fwd": (ctypes.c_int, [_c_float_p] * 3 + [ctypes.c_int] * 7
                             + [ctypes.c_void_p, ctypes.c_void_p]),
    "bpx_residual_skip_bwd": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 7
                              + [ctypes.c_void_p]),
    "bpx_subsample2_fwd": (ctypes.c_int, [_c_float_p] * 2 + [ctypes.c_int] * 4
                           + [ctypes.c_void_p]),
    "bpx_subsample2_bwd": (ctypes.c_int, [_c_float_p] * 2 + [ctypes.c_int] * 4
                           + [ctypes.c_void_p]),
    "bpx_accumulate": (ctypes.c_int, [_c_float_p] * 2 + [ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_maxpool3x3_fwd_idx": (ctypes.c_int, [_c_float_p] * 3 + [ctypes.c_int] * 5
                               + [ctypes.c_void_p]),
    "bpx_maxpool3x3_bwd_idx": (ctypes.c_int, [_c_float_p] * 3 + [ctypes.c_int] * 5
                               + [ctypes.c_void_p]),
    "bpx_concat_fwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                      _c_float_p, ctypes.c_longlong, ctypes.c_void_p]),
    "bpx_concat_bwd": (ctypes.c_int, [_c_float_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p]),
    "bpx_subsample_fwd": (ctypes.c_int, [_c_float_p] * 2 + [ctypes.c_int] * 7
                          + [ctypes.c_void_p]),
    "bpx_subsample_bwd": (ctypes.c_int, [_c_float_p] * 2 + [ctypes.c_int] * 7
                          + [ctypes.c_void_p]),
    "bpx_global_avgpool_fwd": (ctypes.c_int, [_c_float_p] * 2 + [ctypes.c_int] * 4
                               + [ctypes.c_void_p]),
    "bpx_global_avgpool_bwd": (ctypes.c_int, [_c_float_p] * 3 + [ctypes.c_int] * 4
                               + [ctypes.c_void_p]),
    "bpx_softmax_xent": (ctypes.c_int, [_c_float_p, ctypes.c_void_p]
                         + [ctypes.c_int] * 3 + [_c_float_p, _c_float_p, ctypes.c_void_p]),
    "bpx_bn_workspace": (ctypes.c_size_t, [ctypes.c_longlong, ctypes.c_int]),
    "bpx_bn_stats": (ctypes.c_int, [_c_float_p, ctypes.c_longlong, ctypes.c_int, _c_float_p,
                                    ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_bn_apply": (ctypes.c_int, [_c_float_p] * 3 + [ctypes.c_longlong] * 2
                     + [ctypes.c_int, ctypes.c_float, ctypes.c_int, _c_float_p,
                        ctypes.c_void_p, ctypes.c_void_p]),
    "bpx_bn_bwd_sums": (ctypes.c_int, [_c_float_p] * 3 + [ctypes.c_longlong] * 2
                        + [ctypes.c_int, ctypes.c_float, _c_float_p, ctypes.c_void_p,
                           ctypes.c_size_t, ctypes.c_void_p]),
    "bpx_bn_bwd_apply": (ctypes.c_int, [_c_float_p] * 5 + [ctypes.c_longlong] * 2
                         + [ctypes.c_int, ctypes.c_float, _c_float_p, ctypes.c_void_p,
                            ctypes.c_void_p]),
    "bpx_sgd_update": (ctypes.c_int, [_c_float_p, _c_float_p, ctypes.c_size_t,
                                      ctypes.c_float, ctypes.c_void_p]),
    "bpx_reshard_pull": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_void_p]),
    "bpx_allreduce_sum_prefix": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int,
                                                ctypes.c_void_p, ctypes.c_size_t,
                                                ctypes.c_void_p]),
    "bpx_signal_barrier_dev": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_void_p]),
    "bpx_peer_barrier": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_ulonglong, ctypes.c_void_p]),
    "bpx_signal_barrier": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_uint32,
                                          ctypes.c_void_p]),
    "bpx_simt_conv3x3_fwd": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 6
                             + [ctypes.c_void_p]),
    "bpx_simt_conv3x3_dgrad": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 5
                               + [ctypes.c_void_p]),
    "bpx_simt_conv3x3_wgrad": (ctypes.c_int, [_c_float_p] * 4 + [ctypes.c_int] * 5
                               + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def load_library(path: str = LIB_PATH):
    """Load (once) and type the C-ABI; raises ExtensionMissingError."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ExtensionMissingError(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    try:
        lib = ctypes.CDLL(path)
    except OSError as exc:
        raise ExtensionMissingError(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def launch_count() -> int:
    """Kernel launches issued through libbpx by this process so far."""
    return int(load_library().bpx_launch_count())


def last_engine() -> str:
    """Engine that served this thread's last conv3x3 / linear call
    (fdt, wgt, c1, dtc, dwt, dns, tc; legacy: simt, ts, wg, small)."""
    return load_library().bpx_last_engine().decode()


def set_sm_budget(n: int) -> int:
    """SM budget (0 = all) for this thread's later libbpx launches; returns
    the previous one (bpx_set_sm_budget)."""
    return int(load_library().bpx_set_sm_budget(int(n)))


class sm_budget:
    """Context manager: launches (and graph captures) inside use <= n SMs."""

    def __init__(self, n: int):
        self.n = n

    def __enter__(self):
        self.prev = set_sm_budget(self.n)
        return self

    def __exit__(self, *exc):
        set_sm_budget(self.prev)


def legacy_engine_calls() -> int:
    """conv / dense calls this process sent to a legacy engine."""
    return int(load_library().bpx_legacy_engine_calls())


def _check(status: int, what: str) -> None:
    if status != 0:
        name = _lib.bpx_status_string(status).decode()
        raise KernelError(f"{what} failed: {name}", status)


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise KernelError("libbpx takes CUDA tensors only (no CPU fallback)")
    if not t.is_contiguous():
        raise KernelError("libbpx takes contiguous tensors")
    return t.data_ptr()


def _f32(*ts):
    for t in ts:
        if t is not None and t.dtype != torch.float32:
            raise KernelError(f"expected float32, got {t.dtype}")


def _stream():
    return torch.cuda.current_stream().cuda_stream


class Workspace:
    """Grow-only scratch buffer shared by consecutive calls on one stream."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.buf = torch.empty(0, dtype=torch.uint8, device=self.device)

    def get(self, nbytes: int) -> tuple[int, int]:
        if nbytes > self.buf.numel():
            self.buf = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        return (self.buf.data_ptr() if self.buf.numel() else None), self.buf.numel()

    def reserve(self, nbytes: int) -> None:
        self.get(nbytes)


def _ws(ws: Optional[Workspace], nbytes: int, device):
    if nbytes == 0:
        return None, 0
    if ws is None:
        ws = Workspace(device)
    return ws.get(nbytes)


# ---------------------------------------------------------------- layers

class F16Split:
    """A weight tensor in fp16x3 form (bpx_f16_split): fp16 hi and lo arrays
    in the weights' layout and the max |w| word that sets their power-of-two
    scale.  ``refresh(w)`` re-splits after an update."""

    def __init__(self, w: torch.Tensor):
        n = w.numel()
        self.n = n
        self.hi = torch.empty(n, dtype=torch.float16, device=w.device)
        self.lo = torch.empty(n, dtype=torch.float16, device=w.device)
        self.amax = torch.zeros(4, dtype=torch.int32, device=w.device)

    def refresh(self, w: torch.Tensor) -> "F16Split":
        f16_split(w, self)
        return self

    def dequant(self) -> torch.Tensor:
        """(hi + lo) / 2^s in fp64: what the tensor core multiplies (tests)."""
        s = f16_scale_exp(int(self.amax[0].item()) & 0xFFFFFFFF)
        return (self.hi.double() + self.lo.double()) * 2.0 ** (-s)


class F16SplitBatch:
    """fp16x3 splits of several weight tensors refreshed together (three
    graph nodes per update, bpx_f16_split_batch): ``splits[k]`` is the
    F16Split view of ``ws[k]``.  The tensors must keep their storage.
    ``extra`` = ``extra_words`` int32 words of the caller's, zeroed by every
    refresh's memset."""

    def __init__(self, ws: list, extra_words: int = 0):
        lib = load_library()
        dev = ws[0].device
        offs, tot = [], 0
        for w in ws:
            _f32(w)
            if w.numel() % 4 or not w.is_contiguous():
                raise KernelError("F16SplitBatch: contiguous tensors of 4k floats")
            offs.append(tot)
            tot += (w.numel() + 7) // 8 * 8            # 16-B aligned fp16 slices
        self.hi = torch.empty(tot, dtype=torch.float16, device=dev)
        self.lo = torch.empty(tot, dtype=torch.float16, device=dev)
        self.words = torch.zeros(4 * len(ws) + extra_words, dtype=torch.int32, device=dev)
        # caller-owned words zeroed by the same memset on every refresh
        self.extra = self.words[4 * len(ws):]
        chunk = lib.bpx_f16_split_batch_chunk()
        rows, blk = [], 0
        self.splits = []
        for k, (w, o) in enumerate(zip(ws, offs)):
            n = w.numel()
            sp = F16Split.__new__(F16Split)
            sp.n, sp.hi, sp.lo = n, self.hi[o:o + n], self.lo[o:o + n]
            sp.amax = self.words[4 * k:4 * k + 4]
            self.splits.append(sp)
            rows.append([w.data_ptr(), sp.hi.data_ptr(), sp.lo.data_ptr(), sp.amax.data_ptr(),
                         n // 4, blk])
            blk += -(-(n // 4) // chunk)
        self.blocks = blk
        self.table = torch.tensor(rows, dtype=torch.int64).to(dev)
        self.ws = ws

    def refresh(self) -> "F16SplitBatch":
        lib = load_library()
        _check(lib.bpx_f16_split_batch(_ptr(self.table), len(self.ws), self.blocks,
                                       _ptr(self.words), self.words.numel(), _stream()),
               "bpx_f16_split_batch")
        return self


def f16_scale_exp(amax_bits: int) -> int:
    """Scale exponent s of a tensor whose max |v| has fp32 bits ``amax_bits``:
    max |v| 2^s < 2^15 (tc_ptx.cuh f16_scale_exp)."""
    e = (amax_bits >> 23) & 0xFF
    if amax_bits == 0 or e == 255:
        return 0
    return max(-126, min(126, 141 - e))


def f16_split(w, sp: F16Split):
    lib = load_library()
    _f32(w)
    if w.numel() != sp.n:
        raise KernelError("f16_split: size mismatch")
    _check(lib.bpx_f16_split(_ptr(w), w.numel(), _ptr(sp.hi), _ptr(sp.lo), _ptr(sp.amax),
                             _stream()), "bpx_f16_split")
    return sp


def absmax(x, out):
    """out[0] (int32 tensor) = max |x| as fp32 bits."""
    lib = load_library()
    _f32(x)
    _check(lib.bpx_absmax(_ptr(x), x.numel(), _ptr(out), _stream()), "bpx_absmax")
    return out


def _split_ptrs(wsplit):
    if wsplit is None:
        return None, None, None
    return _ptr(wsplit.hi), _ptr(wsplit.lo), _ptr(wsplit.amax)


def conv3x3_fwd(x, w, bias, y, relu=True, ws: Optional[Workspace] = None, wsplit=None,
                x_amax=None, y_amax=None):
    """``wsplit`` (optional F16Split of w) and ``x_amax`` (optional int32 word
    with max |x|, from ``absmax``) are the fp16x3 operand forms the call
    otherwise prepares itself; ``y_amax`` (optional, zeroed int32 word)
    receives max |y| for the next conv."""
    lib = load_library()
    _f32(x, w, bias, y)
    n, h, wd, cin = x.shape
    cout = w.shape[0]
    need = lib.bpx_conv3x3_fwd_workspace(n, h, wd, cin, cout)
    wp, wb = _ws(ws, need, x.device)
    _check(lib.bpx_conv3x3_fwd_presplit(_ptr(x), _ptr(w), *_split_ptrs(wsplit), _ptr(x_amax),
                                        _ptr(y_amax), _ptr(bias), _ptr(y), n, h, wd, cin, cout, int(relu),
                                        wp, wb, _stream()),
           "bpx_conv3x3_fwd")
    return y


def conv3x3_dgrad(dz, w, mask_src, dx, ws: Optional[Workspace] = None, wsplit=None,
                  dz_amax=None, dx_amax=None):
    lib = load_library()
    _f32(dz, w, mask_src, dx)
    n, h, wd, cout = dz.shape
    cin = w.shape[3]
    need = lib.bpx_conv3x3_dgrad_workspace(n, h, wd, cin, cout)
    wp, wb = _ws(ws, need, dz.device)
    _check(lib.bpx_conv3x3_dgrad_presplit(_ptr(dz), _ptr(w), *_split_ptrs(wsplit),
                                          _ptr(dz_amax), _ptr(dx_amax), _ptr(mask_src), _ptr(dx),
                                          n, h, wd,
                                          cin, cout, wp, wb, _stream()),
           "bpx_conv3x3_dgrad")
    return dx


def conv3x3_wgrad(x, dz, dw, dbias, ws: Optional[Workspace] = None, x_amax=None,
                  dz_amax=None):
    lib = load_library()
    _f32(x, dz, dw, dbias)
    n, h, wd, cin = x.shape
    cout = dz.shape[3]
    need = lib.bpx_conv3x3_wgrad_workspace(n, h, wd, cin, cout)
    wp, wb = _ws(ws, need, x.device)
    _check(lib.bpx_conv3x3_wgrad_presplit(_ptr(x), _ptr(dz), _ptr(x_amax), _ptr(dz_amax),
                                          _ptr(dw), _ptr(dbias), n, h, wd, cin, cout, wp, wb,
                                          _stream()),
           "bpx_conv3x3_wgrad")
    return dw


def conv_workspace_bytes(n, h, w, cin, cout) -> int:
    lib = load_library()
    return max(lib.bpx_conv3x3_fwd_workspace(n, h, w, cin, cout),
               lib.bpx_conv3x3_dgrad_workspace(n, h, w, cin, cout),
               lib.bpx_conv3x3_wgrad_workspace(n, h, w, cin, cout))


def linear_fwd(x, w, bias, y, relu, ws: Optional[Workspace] = None):
    lib = load_library()
    _f32(x, w, bias, y)
    b, fin = x.shape
    fout = w.shape[0]
    need = lib.bpx_linear_fwd_workspace(b, fin, fout)
    wp, wb = _ws(ws, need, x.device)
    _check(lib.bpx_linear_fwd(_ptr(x), _ptr(w), _ptr(bias), _ptr(y), b, fin, fout,
                              int(relu), wp, wb, _stream()), "bpx_linear_fwd")
    return y


def linear_dgrad(dy, w, mask_src, dx, ws: Optional[Workspace] = None):
    lib = load_library()
    _f32(dy, w, mask_src, dx)
    b, fout = dy.shape
    fin = w.shape[1]
    need = lib.bpx_linear_dgrad_workspace(b, fin, fout)
    wp, wb = _ws(ws, need, dy.device)
    _check(lib.bpx_linear_dgrad(_ptr(dy), _ptr(w), _ptr(mask_src), _ptr(dx), b,
                                fin, fout, wp, wb, _stream()), "bpx_linear_dgrad")
    return dx


def linear_wgrad(x, dy, dw, dbias, ws: Optional[Workspace] = None):
    lib = load_library()
    _f32(x, dy, dw, dbias)
    b, fin = x.shape
    fout = dy.shape[1]
    need = lib.bpx_linear_wgrad_workspace(b, fin, fout)
    wp, wb = _ws(ws, need, x.device)
    _check(lib.bpx_linear_wgrad(_ptr(x), _ptr(dy), _ptr(dw), _ptr(dbias), b, fin,
                                fout, wp, wb, _stream()), "bpx_linear_wgrad")
    return dw


def linear_workspace_bytes(b, fin, fout) -> int:
    lib = load_library()
    return max(lib.bpx_linear_fwd_workspace(b, fin, fout),
               lib.bpx_linear_dgrad_workspace(b, fin, fout),
               lib.bpx_linear_wgrad_workspace(b, fin, fout))


def maxpool2x2_fwd(x, y):
    lib = load_library()
    _f32(x, y)
    n, h, w, c = x.shape
    _check(lib.bpx_maxpool2x2_fwd(_ptr(x), _ptr(y), n, h, w, c, _stream()),
           "bpx_maxpool2x2_fwd")
    return y


def maxpool2x2_bwd(x, dy, dx):
    lib = load_library()
    _f32(x, dy, dx)
    n, h, w, c = x.shape
    _check(lib.bpx_maxpool2x2_bwd(_ptr(x), _ptr(dy), _ptr(dx), n, h, w, c,
                                  _stream()), "bpx_maxpool2x2_bwd")
    return dx


def residual_add_fwd(a, s, y, relu=True, y_amax=None):
    """y = relu(a + P(s)): the join of a residual diamond; ``s`` may have
    fewer channels (zero-padded) and twice the spatial size (subsampled).
    ``y_amax`` (int32 word, optional): atomicMax'ed with max |y| bits."""
    lib = load_library()
    _f32(a, s, y)
    n, h, w, c = a.shape
    cs = s.shape[3]
    down = 1 if s.shape[1] == 2 * h and h > 0 else 0
    _check(lib.bpx_residual_add_fwd(_ptr(a), _ptr(s), _ptr(y), n, h, w, c, cs, down,
                                    int(relu), _ptr(y_amax), _stream()),
           "bpx_residual_add_fwd")
    return y


def residual_skip_bwd(dz, mask, dh, dmain=None, accumulate=True):
    """Gradient of the join into its skip source (see include/bpx.h)."""
    lib = load_library()
    _f32(dz, mask, dh)
    n, h, w, c = dz.shape
    cs = dh.shape[3]
    down = 1 if dh.shape[1] == 2 * h and h > 0 else 0
    _check(lib.bpx_residual_skip_bwd(_ptr(dz), _ptr(dmain) if dmain is not None else None,
                                     _ptr(mask), _ptr(dh), n, h, w, c, cs, down,
                                     int(accumulate), _stream()), "bpx_residual_skip_bwd")
    return dh


def subsample2_fwd(x, y):
    lib = load_library()
    _f32(x, y)
    n, h, w, c = y.shape
    _check(lib.bpx_subsample2_fwd(_ptr(x), _ptr(y), n, h, w, c, _stream()),
           "bpx_subsample2_fwd")
    return y


def subsample2_bwd(dy, dx):
    lib = load_library()
    _f32(dy, dx)
    n, h, w, c = dy.shape
    _check(lib.bpx_subsample2_bwd(_ptr(dy), _ptr(dx), n, h, w, c, _stream()),
           "bpx_subsample2_bwd")
    return dx


def accumulate(dst, src):
    """dst += src (same number of floats)."""
    lib = load_library()
    _f32(dst, src)
    if dst.numel() != src.numel():
        raise KernelError("accumulate: size mismatch")
    _check(lib.bpx_accumulate(_ptr(dst), _ptr(src), dst.numel(), _stream()), "bpx_accumulate")
    return dst


def maxpool3x3_fwd_idx(x, y, idx):
    """3x3 / stride-1 / pad-1 max pool over the first y.shape[3] channels of x."""
    lib = load_library()
    _f32(x, y)
    n, h, w, c = x.shape
    _check(lib.bpx_maxpool3x3_fwd_idx(_ptr(x), _ptr(y), _ptr(idx), n, h, w, c, y.shape[3],
                                      _stream()), "bpx_maxpool3x3_fwd_idx")
    return y


def maxpool3x3_bwd_idx(idx, dy, dx):
    lib = load_library()
    _f32(dy, dx)
    n, h, w, c = dx.shape
    _check(lib.bpx_maxpool3x3_bwd_idx(_ptr(idx), _ptr(dy), _ptr(dx), n, h, w, c, dy.shape[3],
                                      _stream()), "bpx_maxpool3x3_bwd_idx")
    return dx


def _part_arrays(parts):
    k = len(parts)
    ptrs = (ctypes.c_void_p * 4)(*[_ptr(t) for t in parts] + [None] * (4 - k))
    cs = (ctypes.c_int * 4)(*[t.shape[-1] for t in parts] + [0] * (4 - k))
    return ptrs, cs, k


def concat_fwd(parts, y):
    """y[..., :] = cat(parts, channel dim) (NHWC, same pixel count)."""
    lib = load_library()
    _f32(y, *parts)
    ptrs, cs, k = _part_arrays(parts)
    npix = y.numel() // y.shape[-1]
    _check(lib.bpx_concat_fwd(ptrs, cs, k, _ptr(y), npix, _stream()), "bpx_concat_fwd")
    return y


def concat_bwd(dy, parts):
    lib = load_library()
    _f32(dy, *parts)
    ptrs, cs, k = _part_arrays(parts)
    npix = dy.numel() // dy.shape[-1]
    _check(lib.bpx_concat_bwd(_ptr(dy), ptrs, cs, k, npix, _stream()), "bpx_concat_bwd")
    return parts


def subsample_fwd(x, y, off):
    """y[:, i, j] = x[:, 2i+off, 2j+off]."""
    lib = load_library()
    _f32(x, y)
    n, hin, win, c = x.shape
    _check(lib.bpx_subsample_fwd(_ptr(x), _ptr(y), n, hin, win, y.shape[1], y.shape[2], c, off,
                                 _stream()), "bpx_subsample_fwd")
    return y


def subsample_bwd(dy, dx, off):
    lib = load_library()
    _f32(dy, dx)
    n, hin, win, c = dx.shape
    _check(lib.bpx_subsample_bwd(_ptr(dy), _ptr(dx), n, hin, win, dy.shape[1], dy.shape[2], c,
                                 off, _stream()), "bpx_subsample_bwd")
    return dx


def global_avgpool_fwd(x, y):
    lib = load_library()
    _f32(x, y)
    n, h, w, c = x.shape
    _check(lib.bpx_global_avgpool_fwd(_ptr(x), _ptr(y), n, h, w, c, _stream()),
           "bpx_global_avgpool_fwd")
    return y


def global_avgpool_bwd(dy, mask, dx):
    lib = load_library()
    _f32(dy, dx)
    n, h, w, c = dx.shape
    _check(lib.bpx_global_avgpool_bwd(_ptr(dy), _ptr(mask) if mask is not None else None,
                                      _ptr(dx), n, h, w, c, _stream()),
           "bpx_global_avgpool_bwd")
    return dx


def maxpool2x2_fwd_idx(x, y, idx, y_amax=None):
    """Pool forward that also records each window's first-max position
    (``idx``: uint8, same shape as ``y``)."""
    lib = load_library()
    _f32(x, y)
    n, h, w, c = x.shape
    _check(lib.bpx_maxpool2x2_fwd_idx(_ptr(x), _ptr(y), _ptr(idx), n, h, w, c, _ptr(y_amax),
                                      _stream()),
           "bpx_maxpool2x2_fwd_idx")
    return y


def maxpool2x2_bwd_idx(idx, dy, dx, dx_amax=None):
    lib = load_library()
    _f32(dy, dx)
    n, h, w, c = dx.shape
    _check(lib.bpx_maxpool2x2_bwd_idx(_ptr(idx), _ptr(dy), _ptr(dx), n, h, w, c, _ptr(dx_amax),
                                      _stream()),
           "bpx_maxpool2x2_bwd_idx")
    return dx


def softmax_xent(logits, labels, b_global, loss_out, dlogits):
    lib = load_library()
    _f32(logits, loss_out, dlogits)
    if labels.dtype != torch.int32:
        raise KernelError("labels must be int32")
    b, classes = logits.shape
    if loss_out.numel() < b + 1:
        raise KernelError("loss_out needs b_local + 1 floats")
    _check(lib.bpx_softmax_xent(_ptr(logits), _ptr(labels), b, b_global, classes,
                                _ptr(loss_out), _ptr(dlogits), _stream()),
           "bpx_softmax_xent")
    return loss_out


BN_EPS = 1e-5


def _npc(t):
    """(pixels, channels) of an NHWC activation (or [rows][c])."""
    return t.numel() // t.shape[-1], t.shape[-1]


def bn_stats(z, stats, ws: Optional[Workspace] = None):
    """stats[0:c] = sum z, stats[c:2c] = sum z^2 over this rank's pixels."""
    lib = load_library()
    _f32(z, stats)
    npix, c = _npc(z)
    wp, wb = _ws(ws, lib.bpx_bn_workspace(npix, c), z.device)
    _check(lib.bpx_bn_stats(_ptr(z), npix, c, _ptr(stats), wp, wb, _stream()), "bpx_bn_stats")


def bn_apply(z, stats, gamma_beta, ntot, y, relu, eps=BN_EPS, y_amax=None):
    """y_amax (int32 word, optional): atomicMax'ed with max |y| bits."""
    lib = load_library()
    _f32(z, stats, gamma_beta, y)
    npix, c = _npc(z)
    _check(lib.bpx_bn_apply(_ptr(z), _ptr(stats), _ptr(gamma_beta), npix, int(ntot), c,
                            float(eps), int(relu), _ptr(y), _ptr(y_amax), _stream()),
           "bpx_bn_apply")


def bn_bwd_sums(g, z, stats, ntot, sums, ws: Optional[Workspace] = None, eps=BN_EPS):
    lib = load_library()
    _f32(g, z, stats, sums)
    npix, c = _npc(z)
    wp, wb = _ws(ws, lib.bpx_bn_workspace(npix, c), z.device)
    _check(lib.bpx_bn_bwd_sums(_ptr(g), _ptr(z), _ptr(stats), npix, int(ntot), c, float(eps),
                               _ptr(sums), wp, wb, _stream()), "bpx_bn_bwd_sums")


def bn_bwd_apply(g, z, stats, sums, gamma_beta, ntot, dz, eps=BN_EPS, dz_amax=None):
    """dz_amax (int32 word, optional): atomicMax'ed with max |dz| bits."""
    lib = load_library()
    _f32(g, z, stats, sums, gamma_beta, dz)
    npix, c = _npc(z)
    _check(lib.bpx_bn_bwd_apply(_ptr(g), _ptr(z), _ptr(stats), _ptr(sums), _ptr(gamma_beta),
                                npix, int(ntot), c, float(eps), _ptr(dz), _ptr(dz_amax),
                                _stream()),
           "bpx_bn_bwd_apply")


def bn_workspace_bytes(npix, c) -> int:
    return int(load_library().bpx_bn_workspace(int(npix), int(c)))


def sgd_update(w, g, lr):
    lib = load_library()
    _f32(w, g)
    _check(lib.bpx_sgd_update(_ptr(w), _ptr(g), w.numel(), float(lr), _stream()),
           "bpx_sgd_update")


# ---------------------------------------------------------------- comm

def reshard_pull(srcs: Sequence[int], src_offsets: Sequence[int], dst: torch.Tensor,
                 dst_offsets: Sequence[int], nbytes: Sequence[int]):
    """Copy n_seg byte runs from (peer) device addresses into ``dst``."""
    lib = load_library()
    n = len(nbytes)
    arr = lambda T, v: (T * max(n, 1))(*v)
    _check(lib.bpx_reshard_pull(ctypes.cast(arr(ctypes.c_void_p, srcs), ctypes.c_void_p),
                                ctypes.cast(arr(ctypes.c_size_t, src_offsets), ctypes.c_void_p),
                                _ptr(dst),
                                ctypes.cast(arr(ctypes.c_size_t, dst_offsets), ctypes.c_void_p),
                                ctypes.cast(arr(ctypes.c_size_t, nbytes), ctypes.c_void_p),
                                n, _stream()), "bpx_reshard_pull")


def allreduce_sum_prefix(peer_ptrs: Sequence[int], out: torch.Tensor, n: int):
    lib = load_library()
    arr = (ctypes.c_void_p * len(peer_ptrs))(*peer_ptrs)
    _check(lib.bpx_allreduce_sum_prefix(ctypes.cast(arr, ctypes.c_void_p),
                                        len(peer_ptrs), _ptr(out), int(n), _stream()),
           "bpx_allreduce_sum_prefix")


def peer_barrier(pad_ptrs: Sequence[int], abort_ptrs: Sequence[int], counter: int,
                 status: int, rank: int, timeout_ns: int):
    """Bounded device barrier over len(pad_ptrs) ranks (bpx_peer_barrier)."""
    lib = load_library()
    g = len(pad_ptrs)
    pads = (ctypes.c_void_p * g)(*pad_ptrs)
    aborts = (ctypes.c_void_p * g)(*abort_ptrs)
    _check(lib.bpx_peer_barrier(ctypes.cast(pads, ctypes.c_void_p),
                                ctypes.cast(aborts, ctypes.c_void_p), counter, status,
                                rank, g, int(timeout_ns), _stream()), "bpx_peer_barrier")


def signal_barrier(pad_ptrs: Sequence[int], rank: int, epoch: int):
    lib = load_library()
    arr = (ctypes.c_void_p * len(pad_ptrs))(*pad_ptrs)
    _check(lib.bpx_signal_barrier(ctypes.cast(arr, ctypes.c_void_p), rank,
                                  len(pad_ptrs), epoch & 0xFFFFFFFF, _stream()),
           "bpx_signal_barrier")


# ---------------------------------------------------------------- pinned engine

def simt_conv3x3_fwd(x, w, bias, y, relu=True):
    lib = load_library()
    n, h, wd, cin = x.shape
    _check(lib.bpx_simt_conv3x3_fwd(_ptr(x), _ptr(w), _ptr(bias), _ptr(y), n, h, wd,
                                    cin, w.shape[0], int(relu), _stream()),
           "bpx_simt_conv3x3_fwd")
    return y


def simt_conv3x3_dgrad(dz, w, mask_src, dx):
    lib = load_library()
    n, h, wd, cout = dz.shape
    _check(lib.bpx_simt_conv3x3_dgrad(_ptr(dz), _ptr(w), _ptr(mask_src), _ptr(dx), n,
                                      h, wd, w.shape[3], cout, _stream()),
           "bpx_simt_conv3x3_dgrad")
    return dx


def simt_conv3x3_wgrad(x, dz, dw, dbias, ws: Optional[Workspace] = None):
    lib = load_library()
    n, h, wd, cin = x.shape
    cout = dz.shape[3]
    need = lib.bpx_conv3x3_wgrad_workspace(n, h, wd, cin, cout)
    wp, wb = _ws(ws, need, x.device)
    _check(lib.bpx_simt_conv3x3_wgrad(_ptr(x), _ptr(dz), _ptr(dw), _ptr(dbias), n, h,
                                      wd, cin, cout, wp, wb, _stream()),
           "bpx_simt_conv3x3_wgrad")
    return dw


def signal_barrier_dev(pad_ptrs: Sequence[int], counter_ptr: int, rank: int):
    """Graph-replayable cross-GPU barrier (device-resident epoch counter)."""
    lib = load_library()
    arr = (ctypes.c_void_p * len(pad_ptrs))(*pad_ptrs)
    _check(lib.bpx_signal_barrier_dev(ctypes.cast(arr, ctypes.c_void_p), counter_ptr, rank,
                                      len(pad_ptrs), _stream()), "bpx_signal_barrier_dev")
