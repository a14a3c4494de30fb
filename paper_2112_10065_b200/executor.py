"""B200 executor of a burst-parallel plan: the real counterpart of the
reference's simulated execution model.

The reference expands a plan into an op program (`compile_timeline`,
/root/reference/pkg/src/burstplan/simulator.py:211-298) and *simulates* it
(`simulate` :451-819).  ``BurstStep`` runs that program on the GPU(s):

* layer i runs on ranks [0, g_i), each with the contiguous ceil-split
  sample block ``shard_range(B, g_i, rank)`` (costs.py:85-104);
* a g change between consecutive layers is a reshard of activations
  (forward) and of their gradients (backward) -- the `transfer` op;
* after the backward pass, weight gradients of every layer with g > 1 are
  summed over ranks [0, g) -- the `allreduce` op -- bucketed per g (the
  plan and the reference's serial, non-overlapped charging are unchanged);
* plain SGD updates every replica identically.

Every FLOP runs in libbpx (ops.py); torch provides device memory, streams,
CUDA graphs and torch.distributed.  ``run`` / ``run_two_phase`` mirror the
reference's ``simulate`` / ``run_two_phase`` signatures and return the same
``(SimTrace, SimMetrics)`` types, filled from CUDA-event timestamps.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Iterable, Optional

import torch

from . import ops
from .comm import LocalComm, TorchComm
from .costs import shard_range
from .errors import GraphCaptureError, GraphFormatError, UnsupportedTopologyError
from .graph import CompGraph, ceil_div
from .network import LayerSpec, NetSpec, init_params, net_for_graph, synthetic_batch
from .planner import TrainingPlan
from .timeline import (FG_TASK, SimConfig, SimMetrics, SimTrace, compile_timeline,
                       feedback_update, metrics_from_trace, us_to_ticks)


@dataclass
class _Layer:
    spec: LayerSpec
    g: int
    s0: int              # first global sample of this rank's shard
    b: int               # local batch (0 if the ceil split ran out)
    active: bool         # rank < g
    x: Optional[torch.Tensor] = None       # input (g layout)
    y: Optional[torch.Tensor] = None       # output
    dy: Optional[torch.Tensor] = None      # grad wrt output (pre-ReLU for ReLU layers)
    dx: Optional[torch.Tensor] = None      # grad wrt input (masked by the input's ReLU)
    w: Optional[torch.Tensor] = None
    bias: Optional[torch.Tensor] = None
    dw: Optional[torch.Tensor] = None
    dbias: Optional[torch.Tensor] = None
    wsplit: Optional[object] = None        # conv: fp16x3 split of w (ops.F16Split), per update
    amax: Optional[torch.Tensor] = None    # conv: [0] max |x| bits, [4] max |dz| bits
    x_fused: bool = False                  # amax[0] written by the producer of x
    dz_fused: bool = False                 # amax[4] written by the writer of dy
    y_amax: Optional[torch.Tensor] = None  # word this layer's fwd kernel max-reduces y into
    bn_y_amax: Optional[torch.Tensor] = None  # BN conv: word its normalise pass reduces y into
    dx_amax: Optional[torch.Tensor] = None  # word this layer's bwd kernel reduces dx into
    src_i: int = -1                        # input layer (-1: the network input / concat)
    srcs_i: tuple = ()                     # concat: joined layers
    dx_acc: bool = False                   # dx is private: accumulate into the source's dy
    cat_dst: tuple = ()                    # concat bwd targets (source dy or private)
    cat_acc: tuple = ()                    # concat: (source index, private buffer) pairs
    cat_in: tuple = ()                     # concat fwd parts (source y, or a resharded copy)
    xedges: tuple = ()                     # input edges (src, part) crossing a GPU-count change
    xdy: dict = field(default_factory=dict)    # source side: (consumer, part) -> landing buffer
    idx: Optional[torch.Tensor] = None     # pool: first-max position per output
    reshard_in: bool = False               # input arrives through a reshard
    xs: Optional[torch.Tensor] = None      # down conv: stride-2 subsample of x
    dxs: Optional[torch.Tensor] = None     # down conv: data gradient at the low resolution
    s: Optional[torch.Tensor] = None       # add: shortcut input (skip source's y, add layout)
    skip_i: int = -1                       # add: index of the skip source layer
    join: str = ""                         # add: shortcut-gradient path (fused|direct|reshard)
    dskip: Optional[torch.Tensor] = None   # add: shortcut gradient in the add's layout
    dskip_src: Optional[torch.Tensor] = None   # add: ... resharded to the source's layout
    z: Optional[torch.Tensor] = None       # bn: the conv output before normalisation
    dz: Optional[torch.Tensor] = None      # bn: gradient wrt z
    bnf: Optional[torch.Tensor] = None     # bn: [sum z ; sum z^2], allreduced over [0, g)
    bnb: Optional[torch.Tensor] = None     # bn: [sum g ; sum g*xhat], allreduced over [0, g)


class BurstStep:
    """One rank's share of a burst-parallel training step on one device."""

    def __init__(self, plan: TrainingPlan, graph: CompGraph, *, device=None,
                 comm=None, seed: int = 0, lr: float = 0.01,
                 params: Optional[dict] = None, net: Optional[NetSpec] = None,
                 kernels=None):
        self.net = net or net_for_graph(graph)
        self.B = plan.global_batch
        self.comm = comm or LocalComm()
        self.rank = self.comm.rank
        # `kernels` exists only so tests can drive the multi-rank
        # orchestration on CPU (gloo) with an oracle op set; the product
        # always runs libbpx and fails loudly if it is missing.
        self.k = kernels or ops
        if kernels is None:
            ops.load_library()
            self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        else:
            self.device = torch.device(device or "cpu")
        self.lr = lr
        gs = [g for lid, g in plan.assignments if not graph.layer(lid).is_virtual]
        if len(gs) != len(self.net.layers):
            raise GraphFormatError("plan does not cover every executable layer")
        if max(gs) > self.comm.world:
            raise GraphFormatError(f"plan uses {max(gs)} GPUs, world is {self.comm.world}")
        params = params if params is not None else init_params(self.net, seed)
        dev = self.device
        self.layers: list[_Layer] = []
        for spec, g in zip(self.net.layers, gs):
            s0, s1 = shard_range(self.B, g, self.rank)
            self.layers.append(_Layer(spec, g, s0, s1 - s0, self.rank < g))

        # ---- buckets of gradients per g (one flat buffer per g) ----------
        self.buckets: dict[int, torch.Tensor] = {}
        sizes: dict[int, int] = {}
        for L in self.layers:
            if L.active and L.spec.param_shapes():
                sizes[L.g] = sizes.get(L.g, 0) + _pad4(L.spec.n_params())
        # parameters live in flat buffers with the same layout as the gradient
        # buckets, so the SGD update is one launch per bucket
        self.pbuckets: dict[int, torch.Tensor] = {}
        cursor = {g: 0 for g in sizes}

        names = {L.spec.name: i for i, L in enumerate(self.layers)}
        # residual joins (branch/join diamonds: skip source S -> conv1 ->
        # conv2 -> add, plus the shortcut S -> add).  The shortcut gradient
        # reaches S.dy after conv1's data gradient (and its reshard) wrote it:
        #   fused   S, conv1 (a stride-2 transition) and add share g: one
        #           kernel writes S.dy = P^T(conv1's low-res dx) + shortcut;
        #   direct  S and add share g: the shortcut term is accumulated in place;
        #   reshard otherwise: the shortcut input is resharded S -> add layout
        #           in the forward, its gradient add -> S layout in the
        #           backward and accumulated into S.dy (the reference's
        #           `transfer` of a branch edge, simulator.py:242-253).
        self.join_after: dict[int, int] = {}       # conv1 index -> add index
        for i, L in enumerate(self.layers):
            if L.spec.kind != "add":
                continue
            L.skip_i = names[L.spec.skip]
            c1 = L.skip_i + 1
            if c1 >= i or self.layers[c1].spec.kind not in ("conv", "conv1x1"):
                raise GraphFormatError(f"{L.spec.name}: shortcut does not span a conv chain")
            S, C1 = self.layers[L.skip_i], self.layers[c1]
            if S.g != L.g:
                L.join = "reshard"
            elif C1.spec.down and C1.spec.kind == "conv" and C1.g == S.g:
                L.join = "fused"
            else:
                L.join = "direct"
            self.join_after[c1] = i

        # input edges: the previous layer (a chain edge), a named earlier
        # layer (a branch edge), or several (concat).  Any edge may cross a
        # GPU-count change: its source's output is resharded into the
        # consumer's layout before the consumer runs, and the consumer's
        # input gradient is resharded back (the reference's `transfer`,
        # simulator.py:242-253).  A layer feeding several consumers gets its
        # gradient from all of them: the consumer whose backward runs first
        # (the highest index) writes the source's dy -- through the backward
        # transfer when the edge crosses g -- the others land in private
        # buffers (in the source's layout) that are accumulated into it.
        consumers = branch_topology([L.spec for L in self.layers], [L.g for L in self.layers])
        for i, L in enumerate(self.layers):
            sp = L.spec
            if sp.kind == "concat":
                L.srcs_i = tuple(names[n] for n in sp.srcs)
                L.xedges = tuple((j, k) for k, j in enumerate(L.srcs_i)
                                 if self.layers[j].g != L.g)
            else:
                L.src_i = names[sp.src] if sp.src is not None else i - 1
                if L.src_i >= 0 and self.layers[L.src_i].g != L.g:
                    L.xedges = ((L.src_i, -1),)
        self.consumers = consumers

        # P2P backend: every buffer a peer reads lives in a symmetric heap
        # (PeerComm.make_heap, collective): the producer side of each
        # reshard and the gradient buckets of g > 1
        self.heap = None
        sym = self._peer_visible(sizes) if hasattr(self.comm, "make_heap") else {}
        if hasattr(self.comm, "make_heap"):
            self.heap = self.comm.make_heap(sym)
        for g, n in sizes.items():
            if ("bucket", g) in sym:
                self.buckets[g] = self.heap.view(("bucket", g), (n,))
            else:
                self.buckets[g] = torch.zeros(n, dtype=torch.float32, device=dev)
            self.pbuckets[g] = torch.zeros(n, dtype=torch.float32, device=dev)

        def _buf(key, shape):
            if key in sym:
                return self.heap.view(key, shape)
            return torch.empty(shape, dtype=torch.float32, device=dev)

        ws_need = 0
        for i, L in enumerate(self.layers):
            sp = L.spec
            if not L.active:
                continue
            src = self.layers[L.src_i] if L.src_i >= 0 else None
            prev = src
            L.reshard_in = src is not None and src.g != L.g
            if sp.kind == "concat":
                L.x = None
            elif src is None or L.reshard_in:
                L.x = torch.empty(sp.in_shape(L.b), dtype=torch.float32, device=dev)
            else:
                L.x = src.y.view(sp.in_shape(L.b))
            L.y = _buf(("y", i), sp.out_shape(L.b))
            if sp.kind == "pool" and hasattr(self.k, "maxpool2x2_fwd_idx"):
                L.idx = torch.empty(sp.out_shape(L.b), dtype=torch.uint8, device=dev)
            if sp.kind == "pool3":
                L.idx = torch.empty(sp.out_shape(L.b), dtype=torch.uint8, device=dev)
            if sp.kind == "add" and L.reshard_in:
                # the join passes its gradient on unchanged (L.dx is L.dy
                # below), so the backward transfer's source is L.dy itself
                L.dy = _buf(("dx", i), sp.out_shape(L.b))
            else:
                L.dy = torch.empty(sp.out_shape(L.b), dtype=torch.float32, device=dev)
            if src is not None:
                last = consumers[L.src_i][-1] == i
                if L.reshard_in or not last:
                    L.dx = _buf(("dx", i), sp.in_shape(L.b))
                    L.dx_acc = not L.reshard_in
                else:
                    L.dx = src.dy.view(sp.in_shape(L.b))
            if sp.kind == "concat":
                dst, acc, cin = [], [], []
                for k, j in enumerate(L.srcs_i):
                    S = self.layers[j]
                    pshape = (L.b,) + tuple(S.spec.out_shape(1)[1:])
                    if S.g != L.g:            # part arrives / leaves by reshard
                        cin.append(torch.empty(pshape, dtype=torch.float32, device=dev))
                        dst.append(_buf(("cdy", i, k), pshape))
                    elif consumers[j][-1] == i:
                        cin.append(S.y)
                        dst.append(S.dy)
                    else:
                        cin.append(S.y)
                        buf = torch.empty_like(S.dy)
                        dst.append(buf)
                        acc.append((j, buf))
                L.cat_dst, L.cat_acc, L.cat_in = tuple(dst), tuple(acc), tuple(cin)
            if sp.down:
                low = (L.b, sp.hw, sp.hw, sp.cin)
                L.xs = torch.empty(low, dtype=torch.float32, device=dev)
                L.dxs = torch.empty(low, dtype=torch.float32, device=dev)
            if sp.kind == "add":
                # the join passes its (pre-ReLU) gradient to conv2 unchanged:
                # conv2's output gradient IS the add's (same layout), or its
                # backward transfer when conv2 runs on another GPU count
                L.dx = L.dy
                if not L.reshard_in:
                    prev.dy = L.dy
                S = self.layers[L.skip_i]
                sshape = (L.b,) + tuple(S.spec.out_shape(1)[1:])
                if L.join == "reshard":
                    L.s = torch.empty(sshape, dtype=torch.float32, device=dev)
                else:
                    L.s = S.y
                if L.join != "fused" and L.join != "direct":
                    L.dskip = _buf(("dskip", i), sshape)
            if sp.bn:
                L.z = torch.empty(sp.out_shape(L.b), dtype=torch.float32, device=dev)
                L.dz = torch.empty(sp.out_shape(L.b), dtype=torch.float32, device=dev)
                L.bnf = _buf(("bnf", i), (2 * sp.cout,))
                L.bnb = _buf(("bnb", i), (2 * sp.cout,)) if L.g > 1 else None
                ws_need = max(ws_need, self.k.bn_workspace_bytes(
                    L.b * sp.hw * sp.hw, sp.cout))
            ps = sp.param_shapes()
            if ps:
                w, b = params[sp.name]
                flat, pflat = self.buckets[L.g], self.pbuckets[L.g]
                c = cursor[L.g]
                nw, nb = w.numel(), b.numel()
                L.w = pflat[c:c + nw].view(ps[0])
                L.w.copy_(w.reshape(ps[0]))
                L.bias = pflat[c + nw:c + nw + nb]
                L.bias.copy_(b.reshape(-1))
                L.dw = flat[c:c + nw].view(ps[0])
                L.dbias = flat[c + nw:c + nw + nb]
                cursor[L.g] = c + _pad4(nw + nb)
                if sp.kind == "conv":
                    ws_need = max(ws_need, self.k.conv_workspace_bytes(
                        L.b, sp.hw, sp.hw, sp.cin, sp.cout))
                elif sp.kind == "conv1x1":
                    ws_need = max(ws_need, self.k.linear_workspace_bytes(
                        L.b * sp.hw * sp.hw, sp.cin, sp.cout))
                else:
                    ws_need = max(ws_need, self.k.linear_workspace_bytes(L.b, sp.cin, sp.cout))
        # cross-g edges, source side: the backward transfer lands in the
        # source's dy when this consumer writes it first, else in a private
        # buffer (source layout) accumulated into dy afterwards
        for i, L in enumerate(self.layers):
            for j, k in L.xedges:
                S = self.layers[j]
                if S.active and consumers[j][-1] != i:
                    S.xdy[(i, k)] = torch.empty_like(S.dy)
        # conv weights in fp16x3 form (fp16 hi/lo + scale word): split once
        # per update (after SGD), then fwd and dgrad load them by TMA
        # and one max |v| word per conv operand (x for fwd + wgrad, dz for
        # dgrad + wgrad), reduced once per step and shared by the engines
        self.wbatch = None
        self._words_zeroed = False
        self.amax_words = None
        if hasattr(self.k, "F16Split"):
            convs = [L for L in self.layers if L.active and L.spec.kind == "conv"]
            if convs:       # the operand words ride on the weight split's memset
                self.wbatch = self.k.F16SplitBatch([L.w for L in convs],
                                                   extra_words=8 * len(convs))
                words = self.wbatch.extra
            else:
                words = torch.zeros(8, dtype=torch.int32, device=dev)
            for j, L in enumerate(convs):
                L.wsplit = self.wbatch.splits[j]
                # the fp16x3 engines' shapes (fdt / wgh / wgc / wg1): Cout % 64
                # and Cin % 32 or the 3-channel first conv; the 32-wide towers
                # of the four-tower net run the FFMA / TS engines without words
                if L.spec.cout % 64 == 0 and (L.spec.cin % 32 == 0 or L.spec.cin == 3):
                    L.amax = words[8 * j:8 * j + 8]
            self._split_w()
            self.amax_words = words
            self._fuse_amax(consumers)
        for L in self.layers:
            if L.join == "reshard":
                S = self.layers[L.skip_i]
                if S.active:
                    L.dskip_src = torch.empty_like(S.y)
        self.ws = self.k.Workspace(dev)
        self.ws.reserve(ws_need)
        last = self.layers[-1]
        self.loss_buf = torch.zeros(max(last.b, 0) + 1, dtype=torch.float32, device=dev)
        self.labels = torch.zeros(max(last.b, 1), dtype=torch.int32, device=dev)
        self.graph: Optional[torch.cuda.CUDAGraph] = None
        self.op_events: Optional[list] = None

    def _peer_visible(self, bucket_sizes: dict) -> dict:
        """{heap key: nbytes} of this rank's buffers that peers read: the
        output of a layer whose consumer runs on another GPU count (forward
        reshard source), the data gradient of such a consumer (backward
        reshard source), a resharded shortcut's source output and gradient,
        the gradient buckets of g > 1, and the loss partial."""
        out = {}
        for i, L in enumerate(self.layers):
            for j, k in L.xedges:
                P = self.layers[j]
                if P.active:
                    out[("y", j)] = 4 * P.spec.out_elems() * P.b
                if L.active:
                    key = ("cdy", i, k) if k >= 0 else ("dx", i)
                    out[key] = 4 * P.spec.out_elems() * L.b
            if L.join == "reshard":
                S = self.layers[L.skip_i]
                if S.active:
                    out[("y", L.skip_i)] = 4 * S.spec.out_elems() * S.b
                if L.active:
                    out[("dskip", i)] = 4 * S.spec.out_elems() * L.b
            if L.spec.bn and L.active and L.g > 1:       # SyncBN sums over [0, g)
                out[("bnf", i)] = out[("bnb", i)] = 8 * L.spec.cout
        for g, n in bucket_sizes.items():
            if g > 1:
                out[("bucket", g)] = 4 * n
        out[("loss",)] = 16
        return out

    # ------------------------------------------------------------ data
    @property
    def input(self) -> Optional[torch.Tensor]:
        L0 = self.layers[0]
        return L0.x if L0.active else None

    def input_range(self) -> tuple[int, int]:
        L0 = self.layers[0]
        return L0.s0, L0.s0 + L0.b

    def label_range(self) -> tuple[int, int]:
        L = self.layers[-1]
        return L.s0, L.s0 + L.b

    def input_pairs(self, x_global: torch.Tensor, labels_global: torch.Tensor) -> list:
        """[(device destination, host source)] of this rank's input shards
        (x: NHWC [B,...], labels [B])."""
        pairs = []
        a, b = self.input_range()
        if self.layers[0].active and b > a:
            x0 = self.layers[0].x
            pairs.append((x0, x_global[a:b].reshape(x0.shape)))
        a, b = self.label_range()
        if self.layers[-1].active and b > a:
            pairs.append((self.labels[:b - a], labels_global[a:b]))
        return pairs

    def load(self, x_global: torch.Tensor, labels_global: torch.Tensor) -> None:
        """Copy this rank's shards to the device; async when the sources
        are pinned host tensors."""
        for dst, src in self.input_pairs(x_global, labels_global):
            dst.copy_(src, non_blocking=True)

    # ------------------------------------------------------------ step
    def _bn_ntot(self, L) -> int:
        """Pixels of the whole layer group (the global batch)."""
        return self.B * L.spec.hw * L.spec.hw

    def _bn_allreduce(self, i: int, key: str, t: torch.Tensor) -> None:
        L = self.layers[i]
        if L.g <= 1:
            return
        if self.heap is not None:
            self.heap.allreduce((key, i), t, L.g)
        else:
            self.comm.allreduce(t, L.g)

    def _bn_fwd(self, i: int) -> None:
        """z -> y: local sums, allreduce over [0, g), normalise (+ReLU)."""
        L = self.layers[i]
        self.k.bn_stats(L.z, L.bnf, ws=self.ws)
        self._bn_allreduce(i, "bnf", L.bnf)
        kw = {"y_amax": L.bn_y_amax} if L.bn_y_amax is not None else {}
        self.k.bn_apply(L.z, L.bnf, L.bias, self._bn_ntot(L), L.y, L.spec.relu, **kw)

    def _bn_bwd(self, i: int) -> torch.Tensor:
        """dy -> dz.  The local sums are the layer's [dbeta ; dgamma] (summed
        over [0, g) later by the gradient-bucket allreduce); a copy is
        allreduced now for the data gradient."""
        L = self.layers[i]
        self.k.bn_bwd_sums(L.dy, L.z, L.bnf, self._bn_ntot(L), L.dbias, ws=self.ws)
        sums = L.dbias
        if L.g > 1:
            L.bnb.copy_(L.dbias)
            self._bn_allreduce(i, "bnb", L.bnb)
            sums = L.bnb
        kw = {"dz_amax": L.amax[4:5]} if L.amax is not None and L.dz_fused else {}
        self.k.bn_bwd_apply(L.dy, L.z, L.bnf, sums, L.bias, self._bn_ntot(L), L.dz, **kw)
        return L.dz

    def _fuse_amax(self, consumers) -> None:
        """Fuse each conv's fp16x3 scale words into the kernels that write its
        operands where that kernel writes the operand buffer itself: x from
        a conv forward (fdt / c1 epilogue) or a 2x2 max pool on the same g
        (a chain edge, no reshard), a residual join or a BN conv's normalise
        pass, dz from the dgrad of its only consumer (a conv or a pool) on
        the same g or, for a BN conv, from its own BN backward.  Every other
        operand gets one
        bpx_absmax launch.  The words are zeroed with the weights' split after
        each update (one memset), or by the first active layer's forward when
        no update preceded it."""
        self.first_active = min((i for i, L in enumerate(self.layers) if L.active), default=-1)
        if os.environ.get("BPX_FUSE_AMAX", "1") == "0":
            return
        for i, L in enumerate(self.layers):
            sp = L.spec
            if L.amax is None or sp.down:
                continue
            if sp.bn:
                L.dz_fused = True     # its own BN backward (bn_bwd_apply) writes dz
            if L.src_i < 0 and sp.kind == "conv" and sp.cin == 3 and sp.cout == 64:
                L.x_fused = True      # the first-conv engine (c1) reduces x as it reads it
            if L.src_i >= 0 and not L.reshard_in and self.layers[L.src_i].g == L.g:
                S = self.layers[L.src_i]
                if S.spec.kind == "conv" and S.spec.bn and S.active:
                    S.bn_y_amax = L.amax[0:1]      # the BN normalise pass writes x
                    L.x_fused = True
                elif ((S.spec.kind == "conv" and not S.spec.bn) or S.spec.kind == "add" or
                        (S.spec.kind == "pool" and S.idx is not None)):
                    S.y_amax = L.amax[0:1]
                    L.x_fused = True
            if sp.bn:
                continue              # consumers' data gradients are not its dz
            cons = consumers[i]
            if len(cons) == 1:
                C = self.layers[cons[0]]
                # (an inactive consumer's flags are never set: compare g)
                if (C.active and C.g == L.g and not C.reshard_in and not C.dx_acc and
                        not C.spec.bn and
                        ((C.spec.kind == "conv" and not C.spec.down) or
                         (C.spec.kind == "pool" and C.idx is not None))):
                    C.dx_amax = L.amax[4:5]
                    L.dz_fused = True

    def _ya(self, L) -> dict:
        return {"y_amax": L.y_amax} if L.y_amax is not None else {}

    def _xa(self, L, x) -> dict:
        """fp16x3: max |x| word of conv L's input, reduced here (one launch)
        and reused by the layer's weight gradient."""
        if L.amax is None:
            return {}
        if not L.x_fused:
            self.k.absmax(x, L.amax[0:1])
        return {"x_amax": L.amax[0:1]}

    def _dza(self, L, dz) -> tuple:
        """fp16x3 keyword arguments of conv L's wgrad and dgrad: the stored
        max |x| word and max |dz| reduced here."""
        if L.amax is None:      # no words of its own; it may still feed one
            return {}, ({"dx_amax": L.dx_amax} if L.dx_amax is not None else {})
        if not L.dz_fused:
            self.k.absmax(dz, L.amax[4:5])
        da = {"wsplit": L.wsplit, "dz_amax": L.amax[4:5]}
        if L.dx_amax is not None:
            da["dx_amax"] = L.dx_amax
        wa = {"x_amax": L.amax[0:1], "dz_amax": L.amax[4:5]}
        return wa, da

    def _fwd(self, i: int) -> None:
        L = self.layers[i]
        sp = L.spec
        if i == getattr(self, "first_active", None) and self.amax_words is not None:
            # fused producers atomicMax into the words: zeroed by the weight
            # split after the last update, else here
            if not self._words_zeroed:
                self.amax_words.zero_()
            self._words_zeroed = False
        lo = {"wsplit": L.wsplit} if L.wsplit is not None else {}
        if sp.bn:
            # conv without bias / activation into z, then the synchronised BN
            x = L.x
            if sp.down:
                x = self._sub_fwd(L)
            if sp.kind == "conv":
                self.k.conv3x3_fwd(x, L.w, None, L.z, relu=False, ws=self.ws, **lo,
                                   **self._xa(L, x))
            else:
                P = L.b * sp.hw * sp.hw
                self.k.linear_fwd(x.reshape(P, sp.cin), L.w.view(sp.cout, sp.cin), None,
                                  L.z.view(P, sp.cout), False, ws=self.ws)
            self._bn_fwd(i)
            return
        if sp.kind == "conv" and sp.down:
            self._sub_fwd(L)
            self.k.conv3x3_fwd(L.xs, L.w, L.bias, L.y, relu=sp.relu, ws=self.ws, **lo,
                               **self._xa(L, L.xs), **self._ya(L))
        elif sp.kind == "conv1x1":
            x = self._sub_fwd(L) if sp.down else L.x
            P = L.b * sp.hw * sp.hw
            self.k.linear_fwd(x.reshape(P, sp.cin), L.w.view(sp.cout, sp.cin), L.bias,
                              L.y.view(P, sp.cout), sp.relu, ws=self.ws)
        elif sp.kind == "pool3":
            self.k.maxpool3x3_fwd_idx(self._sub_fwd(L) if sp.down else L.x, L.y, L.idx)
        elif sp.kind == "concat":
            self.k.concat_fwd(list(L.cat_in), L.y)
        elif sp.kind == "conv":
            self.k.conv3x3_fwd(L.x, L.w, L.bias, L.y, relu=sp.relu, ws=self.ws, **lo,
                               **self._xa(L, L.x), **self._ya(L))
        elif sp.kind == "add":
            self.k.residual_add_fwd(L.x, L.s, L.y, relu=sp.relu, **self._ya(L))
        elif sp.kind == "gap":
            self.k.global_avgpool_fwd(L.x, L.y)
        elif sp.kind == "pool":
            if L.idx is not None:
                self.k.maxpool2x2_fwd_idx(L.x, L.y, L.idx, **self._ya(L))
            else:
                self.k.maxpool2x2_fwd(L.x, L.y)
        else:
            self.k.linear_fwd(L.x.view(L.b, sp.cin), L.w, L.bias, L.y, sp.relu, ws=self.ws)

    def _join_bwd(self, i: int) -> None:
        """Shortcut gradient of the join at ``i`` (add-active ranks): runs
        after the block's first conv has written (fused: produced the
        low-resolution part of) the source's gradient."""
        L = self.layers[i]
        src, c1 = self.layers[L.skip_i], self.layers[L.skip_i + 1]
        if L.join == "fused":
            self.k.residual_skip_bwd(L.dy, L.s, src.dy, dmain=c1.dxs, accumulate=False)
        elif L.join == "direct":
            self.k.residual_skip_bwd(L.dy, L.s, src.dy, accumulate=True)
        else:
            self.k.residual_skip_bwd(L.dy, L.s, L.dskip, accumulate=False)

    def _skip_reshard(self, i: int, backward: bool) -> None:
        L = self.layers[i]
        S = self.layers[L.skip_i]
        bps = 4 * S.spec.out_elems()
        if self.heap is not None:
            if not backward:
                self.heap.reshard(("y", L.skip_i), S.g, L.s if L.active else None, L.g,
                                  self.B, bps)
            else:
                self.heap.reshard(("dskip", i), L.g, L.dskip_src if S.active else None, S.g,
                                  self.B, bps)
        elif not backward:
            self.comm.reshard(S.y if S.active else None, S.g,
                              L.s if L.active else None, L.g, self.B, bps)
        else:
            self.comm.reshard(L.dskip if L.active else None, L.g,
                              L.dskip_src if S.active else None, S.g, self.B, bps)

    def _skip_accumulate(self, i: int) -> None:
        L = self.layers[i]
        self.k.accumulate(self.layers[L.skip_i].dy, L.dskip_src)

    def _sub_fwd(self, L) -> torch.Tensor:
        """Stride-2 subsample of a down layer's input into L.xs."""
        off = L.spec.sub_off
        if off == 0 and hasattr(self.k, "subsample2_fwd"):
            self.k.subsample2_fwd(L.x, L.xs)
        else:
            self.k.subsample_fwd(L.x, L.xs, off)
        return L.xs

    def _sub_bwd(self, L) -> None:
        off = L.spec.sub_off
        if off == 0 and hasattr(self.k, "subsample2_bwd"):
            self.k.subsample2_bwd(L.dxs, L.dx)
        else:
            self.k.subsample_bwd(L.dxs, L.dx, off)

    def _fanin(self, i: int) -> None:
        """Accumulate this consumer's private input gradient(s) into the
        source's dy (a fan-out source's non-first consumers)."""
        L = self.layers[i]
        if L.dx_acc:
            self.k.accumulate(self.layers[L.src_i].dy, L.dx)
        for j, buf in L.cat_acc:
            self.k.accumulate(self.layers[j].dy, buf)

    def _chain_transfer(self, i: int) -> bool:
        L = self.layers[i]
        return i > 0 and L.src_i == i - 1 and self.layers[i - 1].g != L.g

    def _fused_down(self, i: int) -> bool:
        """conv ``i`` is a transition conv whose low-res data gradient the
        join folds into the source's gradient (no separate upsample)."""
        j = self.join_after.get(i)
        return j is not None and self.layers[j].join == "fused"

    def _bwd(self, i: int) -> None:
        L = self.layers[i]
        sp = L.spec
        mask = L.x if sp.in_relu else None
        if sp.kind == "add":
            return                      # main path: identity (conv2.dy is L.dy)
        if sp.kind == "concat":
            self.k.concat_bwd(L.dy, list(L.cat_dst))
            return
        dy = self._bn_bwd(i) if sp.bn else L.dy
        dbias = None if sp.bn else L.dbias      # bn: [dbeta ; dgamma] came from _bn_bwd
        if sp.kind == "conv1x1":
            P = L.b * sp.hw * sp.hw
            x2 = (L.xs if sp.down else L.x).reshape(P, sp.cin)
            dy2, w2 = dy.view(P, sp.cout), L.w.view(sp.cout, sp.cin)
            self.k.linear_wgrad(x2, dy2, L.dw.view(sp.cout, sp.cin), dbias, ws=self.ws)
            if L.src_i >= 0:
                dxt = L.dxs if sp.down else L.dx
                self.k.linear_dgrad(dy2, w2, x2 if sp.in_relu else None, dxt.view(P, sp.cin),
                                    ws=self.ws)
                if sp.down:
                    self._sub_bwd(L)
            return
        if sp.kind == "pool3":
            self.k.maxpool3x3_bwd_idx(L.idx, L.dy, L.dxs if sp.down else L.dx)
            if sp.down:
                self._sub_bwd(L)
            return
        if sp.kind == "gap":
            self.k.global_avgpool_bwd(L.dy, mask, L.dx)
        elif sp.kind == "conv" and sp.down:
            wa, da = self._dza(L, dy)
            self.k.conv3x3_wgrad(L.xs, dy, L.dw, dbias, ws=self.ws, **wa)
            self.k.conv3x3_dgrad(dy, L.w, L.xs if sp.in_relu else None, L.dxs, ws=self.ws, **da)
            if not self._fused_down(i):
                self._sub_bwd(L)
        elif sp.kind == "conv":
            wa, da = self._dza(L, dy)
            self.k.conv3x3_wgrad(L.x, dy, L.dw, dbias, ws=self.ws, **wa)
            if i > 0:
                self.k.conv3x3_dgrad(dy, L.w, mask, L.dx, ws=self.ws, **da)
        elif sp.kind == "pool":
            if L.idx is not None:
                self.k.maxpool2x2_bwd_idx(L.idx, L.dy, L.dx,
                                          **({"dx_amax": L.dx_amax} if L.dx_amax is not None
                                             else {}))
            else:
                self.k.maxpool2x2_bwd(L.x, L.dy, L.dx)
        else:
            x2 = L.x.view(L.b, sp.cin)
            self.k.linear_wgrad(x2, L.dy, L.dw, L.dbias, ws=self.ws)
            if i > 0:
                self.k.linear_dgrad(L.dy, L.w, None if mask is None else x2,
                                 L.dx.view(L.b, sp.cin), ws=self.ws)

    def _edge_reshard(self, i: int, j: int, k: int, backward: bool) -> None:
        """The transfer of input edge j -> i (part k of a concat, -1
        otherwise): forward j.y (g_j layout) -> i's input (g_i layout);
        backward i's input gradient -> j.dy, or j's landing buffer."""
        L, S = self.layers[i], self.layers[j]
        bps = 4 * S.spec.out_elems()
        if not backward:
            dst = (L.cat_in[k] if k >= 0 else L.x) if L.active else None
            if self.heap is not None:
                self.heap.reshard(("y", j), S.g, dst, L.g, self.B, bps)
            else:
                self.comm.reshard(S.y if S.active else None, S.g, dst, L.g, self.B, bps)
            return
        dst = None
        if S.active:
            dst = S.xdy.get((i, k), S.dy)
        if self.heap is not None:
            key = ("cdy", i, k) if k >= 0 else ("dx", i)
            self.heap.reshard(key, L.g, dst, S.g, self.B, bps)
        else:
            src = (L.cat_dst[k] if k >= 0 else L.dx) if L.active else None
            self.comm.reshard(src, L.g, dst, S.g, self.B, bps)

    def _edge_accumulate(self, i: int, j: int, k: int) -> None:
        S = self.layers[j]
        self.k.accumulate(S.dy, S.xdy[(i, k)])

    def _mark(self, tag):
        if self.op_events is not None and self.device.type == "cuda":
            # external=True: a real event-record node when captured in a graph
            ev = torch.cuda.Event(enable_timing=True, external=True)
            ev.record()
            self.op_events.append((tag, ev))

    # ------------------------------------------------------------ program
    def program(self) -> list:
        """This rank's per-iteration op list in issue order: (key, fn) with
        key = (kind, index, phase).  Kinds are the reference's OpRecord
        kinds (compute / transfer / allreduce, simulator.py:175-196) plus
        the loss and the SGD update; a layer's `compute` is split into its
        fwd and bwd halves, which run at different times for real."""
        prog = []
        n = len(self.layers)
        for i in range(n):
            for j, k in self.layers[i].xedges:
                prog.append((("transfer", i, "fwd" if k < 0 else f"fwd{k}"),
                             lambda i=i, j=j, k=k: self._edge_reshard(i, j, k, False)))
            if self.layers[i].join == "reshard":
                prog.append((("transfer", i, "skip_fwd"),
                             lambda i=i: self._skip_reshard(i, False)))
            if self.layers[i].active:
                prog.append((("compute", i, "fwd"), lambda i=i: self._fwd(i)))
        if self.layers[-1].active:
            prog.append((("loss", n - 1, "fwd"), self._loss))
        for i in reversed(range(n)):
            if self.layers[i].active and self.layers[i].spec.kind != "add":
                prog.append((("compute", i, "bwd"), lambda i=i: self._bwd(i)))
                if self.layers[i].dx_acc or self.layers[i].cat_acc:
                    prog.append((("compute", i, "fanin"), lambda i=i: self._fanin(i)))
            for j, k in self.layers[i].xedges:
                prog.append((("transfer", i, "bwd" if k < 0 else f"bwd{k}"),
                             lambda i=i, j=j, k=k: self._edge_reshard(i, j, k, True)))
                if self.layers[j].active and (i, k) in self.layers[j].xdy:
                    prog.append((("compute", i, "xacc" if k < 0 else f"xacc{k}"),
                                 lambda i=i, j=j, k=k: self._edge_accumulate(i, j, k)))
            if i in self.join_after:
                # the join's backward = its shortcut gradient, after conv1's
                # data gradient (and its transfer) wrote the source's dy
                j = self.join_after[i]
                J = self.layers[j]
                if J.active:
                    prog.append((("compute", j, "bwd"), lambda j=j: self._join_bwd(j)))
                if J.join == "reshard":
                    prog.append((("transfer", j, "skip_bwd"),
                                 lambda j=j: self._skip_reshard(j, True)))
                    if self.layers[J.skip_i].active:
                        prog.append((("compute", j, "skip_acc"),
                                     lambda j=j: self._skip_accumulate(j)))
        for g in sorted(self.buckets, reverse=True):
            if g > 1:
                prog.append((("allreduce", g, "sync"), lambda g=g: self._allreduce(g)))
        prog.append((("sgd", 0, "update"), self._sgd))
        return prog

    def _allreduce(self, g: int) -> None:
        if self.heap is not None:
            self.heap.allreduce(("bucket", g), self.buckets[g], g)
        else:
            self.comm.allreduce(self.buckets[g], g)

    def _loss(self) -> None:
        last = self.layers[-1]
        self.k.softmax_xent(last.y, self.labels[:last.b], self.B, self.loss_buf, last.dy)

    def _sgd(self) -> None:
        for g in sorted(self.buckets):
            self.k.sgd_update(self.pbuckets[g], self.buckets[g], self.lr)
        self._split_w()

    def _split_w(self) -> None:
        if self.wbatch is not None:
            self.wbatch.refresh()
            self._words_zeroed = True

    def run_ops(self, prog) -> None:
        for key, fn in prog:
            self._mark((key, "start"))
            fn()
            self._mark((key, "end"))

    def forward_backward(self) -> None:
        prog = self.program()
        self.run_ops([op for op in prog if op[0][0] not in ("allreduce", "sgd")])

    def sync_and_update(self) -> None:
        prog = self.program()
        self.run_ops([op for op in prog if op[0][0] in ("allreduce", "sgd")])

    def step(self) -> None:
        if self.graph is not None:
            self.graph.replay()
            return
        self.run_ops(self.program())

    def _warm(self, prog, warmup: int) -> None:
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.run_ops(prog)
        torch.cuda.current_stream().wait_stream(s)

    def capture(self, warmup: int = 2) -> None:
        """Capture the whole step (kernels + NCCL) as one CUDA graph; the
        warm-up runs on a side stream as torch requires."""
        record = self.op_events is not None
        self.op_events = None
        prog = self.program()
        self._warm(prog, warmup)
        if record:          # external events become record nodes in the graph
            self.op_events = []
        self.graph = self._graph_or_eager(prog, None)

    def capture_segments(self, cut: set, warmup: int = 1, pool=None) -> list:
        """Capture the step as consecutive graphs, starting a new graph at
        every program index in ``cut`` (used to isolate feedback-flagged
        ops so background work can be held off around them).  Returns
        [(first_index, keys, graph)]."""
        prog = self.program()
        # the eager warm-up must not leave its own op events behind: per-op
        # timing would add the warm-up's durations to every replay's
        record, self.op_events = self.op_events, None
        self._warm(prog, warmup)
        self.op_events = record
        bounds = sorted({0, len(prog)} | {c for c in cut if 0 < c < len(prog)})
        segs = []
        for a, b in zip(bounds, bounds[1:]):
            segs.append((a, [k for k, _ in prog[a:b]], self._graph_or_eager(prog[a:b], pool)))
        return segs

    def _graph_or_eager(self, ops, pool):
        """A CUDA graph of ``ops``.  A failed capture is fatal
        (GraphCaptureError): replaying eagerly would silently change what
        is measured.  ``BPX_ALLOW_EAGER_REPLAY=1`` opts into the eager
        replay (same results, more launch overhead) for debugging."""
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g, pool=pool):
                self.run_ops(ops)
            return g
        except Exception as exc:                      # pragma: no cover (GPU only)
            import sys
            torch.cuda.synchronize()
            if self.op_events is not None:
                self.op_events.clear()
            if os.environ.get("BPX_ALLOW_EAGER_REPLAY", "") != "1":
                raise GraphCaptureError(
                    f"CUDA-graph capture of the step failed ({type(exc).__name__}: {exc})"
                ) from exc
            print(f"[bpx] CUDA-graph capture failed ({type(exc).__name__}: {exc}); "
                  "replaying the op program eagerly (BPX_ALLOW_EAGER_REPLAY=1)",
                  file=sys.stderr)
            return _EagerReplay(self, ops)

    def loss(self) -> float:
        """Global mean loss (sum of shard partials over the last layer's g)."""
        last = self.layers[-1]
        if self.heap is not None:
            part = self.heap.view(("loss",), (1,))
            if last.active:
                part.copy_(self.loss_buf[:1])
            self.heap.allreduce(("loss",), part, last.g)
            val = float(part.item())
            self.comm.check()
            return val
        part = self.loss_buf[:1].clone() if last.active else torch.zeros(1, device=self.device)
        if last.g > 1:
            self.comm.allreduce(part, last.g)
        return float(part.item())

    def grads(self) -> dict:
        return {L.spec.name: (L.dw, L.dbias) for L in self.layers
                if L.active and L.w is not None}

    def params(self) -> dict:
        return {L.spec.name: (L.w, L.bias) for L in self.layers
                if L.active and L.w is not None}


class _EagerReplay:
    """Stands in for a captured CUDA graph: replay() runs the ops."""

    def __init__(self, step: "BurstStep", ops):
        self.step, self.ops = step, list(ops)

    def replay(self) -> None:
        self.step.run_ops(self.ops)


def branch_topology(specs, gs) -> dict:
    """Input edges of every layer -> {source index: [consumer indices]}, in
    consumer order.  Every edge may cross a GPU-count change (a reshard);
    raises UnsupportedTopologyError for an input that is not an earlier
    layer."""
    names = {sp.name: i for i, sp in enumerate(specs)}
    consumers: dict[int, list] = {}
    for i, sp in enumerate(specs):
        if sp.kind == "concat":
            edges = tuple(names[n] for n in sp.srcs)
        else:
            j = names[sp.src] if sp.src is not None else i - 1
            edges = (j,) if j >= 0 else ()
        for j in edges:
            if j >= i:
                raise UnsupportedTopologyError(f"{sp.name}: input {specs[j].name} is not earlier")
            consumers.setdefault(j, []).append(i)
    return consumers


def _pad4(n: int) -> int:
    return (n + 3) // 4 * 4


# ---------------------------------------------------------------------------
# reference-shaped entry points


_COMMS: dict = {}


def _dist_comm(plan_gs=()):
    """The process's communicator for the default torch.distributed world:
    NCCL/gloo collectives by default, ``BPX_COMM=peer`` selects the P2P
    backend (comm.PeerComm: libbpx kernels over IPC-mapped peer memory,
    needs CUDA_MODULE_LOADING=EAGER).  One instance per (backend, world),
    created collectively with every prefix group [0, g), g = 2..world, and
    reused by every run / sweep point (no per-call groups or arenas)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return LocalComm()
    world, rank = dist.get_world_size(), dist.get_rank()
    peer = os.environ.get("BPX_COMM", "").lower() == "peer"
    key = ("peer" if peer else "torch", world, id(dist.group.WORLD))
    comm = _COMMS.get(key)
    if comm is None:
        if peer:
            from .comm import PeerComm
            comm = PeerComm(rank, world, range(2, world + 1))
        else:
            comm = TorchComm(rank, world, range(2, world + 1))
        _COMMS[key] = comm
    return comm


def run(plan: TrainingPlan, graph: CompGraph, n_gpus: int,
        bg_graph: Optional[CompGraph] = None, config: Optional[SimConfig] = None,
        iterations: int = 4, sensitive: Iterable[str] = (),
        baseline_fg_iteration_us: Optional[float] = None, *,
        inputs=None, seed: int = 0, lr: float = 0.01,
        step: Optional[BurstStep] = None, bg=None, measure_ops: bool = False,
        bg_sm_budget: Optional[int] = None, fg_sm_budget: int = 0):
    """Execute ``iterations`` training steps of ``plan`` on real GPUs.

    Same call shape and return types as the reference's
    ``simulate(compile_timeline(plan, graph, n_gpus, bg_graph, config), ...)``
    (simulator.py:451-456): ``(SimTrace, SimMetrics)`` with ticks of 0.1 us
    taken from CUDA events (iteration ends are the max over ranks).  Launch
    one process per GPU (torchrun) for n_gpus > 1.  ``inputs`` = (x NHWC
    [B,...], labels [B]) host tensors (pinned); every iteration copies its
    input shard in, end to end.  With ``bg_graph`` every GPU also trains a
    single-GPU background job on a low-priority stream (multiplex.py),
    its kernels sized to ``bg_sm_budget`` SMs (default: $BPX_BG_SM_BUDGET,
    0 = the whole GPU), the foreground's to ``fg_sm_budget`` (0 = all);
    ``sensitive`` names foreground ops (``multiplex.op_name``) that must
    not overlap background work.  bg samples/s is summed over GPUs.
    """
    from .multiplex import BgJob, Multiplexer, op_name
    config = config or SimConfig()
    tl = compile_timeline(plan, graph, n_gpus, bg_graph, config)
    comm = step.comm if step is not None else _dist_comm({g for _, g in plan.assignments})
    if comm.world != n_gpus:
        raise GraphFormatError(f"n_gpus={n_gpus} but world size is {comm.world}")
    st = step or BurstStep(plan, graph, comm=comm, seed=seed, lr=lr)
    if inputs is None:
        x, y = synthetic_batch(st.net, plan.global_batch, seed)
        inputs = (x.pin_memory(), y.pin_memory())
    if bg is None and bg_graph is not None:
        bg = BgJob(bg_graph, config, seed=seed + 1, sm_budget=bg_sm_budget)
    mux = Multiplexer(st, bg, config, sensitive, measure_ops=measure_ops,
                      fg_sm_budget=fg_sm_budget)
    trace = SimTrace()
    try:
        trace = mux.run(iterations, inputs, trace, rank=comm.rank,
                        comm=comm if comm.world > 1 else None)
        comm.check()
    except BaseException:
        if hasattr(comm, "abort"):
            comm.abort()             # peers' barriers fail fast instead of spinning
        raise
    base = baseline_fg_iteration_us or tl.predicted_fg_iteration_us
    metrics = metrics_from_trace(trace, n_gpus, tl.global_batch, tl.bg_batch, config,
                                 iterations, base)
    if comm.world > 1 and bg is not None:
        tot = comm.sum_scalar(metrics.bg_throughput_samples_per_s, st.device)
        metrics = SimMetrics(metrics.fg_iteration_time_us_mean,
                             metrics.fg_iteration_time_us_p99,
                             metrics.fg_throughput_samples_per_s, tot,
                             metrics.fg_throughput_samples_per_s + tot,
                             metrics.per_gpu_utilization, metrics.qos_degradation)
    trace.bg_job = bg
    return trace, metrics


def run_two_phase(plan: TrainingPlan, graph: CompGraph, n_gpus: int,
                  bg_graph: Optional[CompGraph] = None,
                  config: Optional[SimConfig] = None, iterations: int = 4,
                  feedback_rounds: int = 1,
                  baseline_fg_iteration_us: Optional[float] = None, **kw):
    """Measured counterpart of the reference's run_two_phase
    (simulator.py:959-977): time every foreground op alone, then collocated
    with the background; flag ops slowed beyond ``slowdown_ban_threshold``
    (feedback_update, :896-911) and re-run with them protected.  Returns
    ``(trace, metrics, flags)``."""
    config = config or SimConfig()
    st = kw.pop("step", None)
    if st is None:
        comm = _dist_comm({g for _, g in plan.assignments})
        st = BurstStep(plan, graph, comm=comm, seed=kw.get("seed", 0),
                       lr=kw.get("lr", 0.01))
    iso, _ = run(plan, graph, n_gpus, None, config, iterations, (),
                 baseline_fg_iteration_us, step=st, measure_ops=True, **kw)
    isolated = {k: sum(v) / len(v) for k, v in iso.op_durations.items() if v}
    flags: frozenset = frozenset()
    bg = None
    trace, metrics = None, None
    comm = st.comm
    for _ in range(feedback_rounds):
        trace, metrics = run(plan, graph, n_gpus, bg_graph, config, iterations, flags,
                             baseline_fg_iteration_us, step=st, bg=bg, measure_ops=True,
                             **kw)
        bg = trace.bg_job
        trace.op_isolated.update(isolated)
        # every rank flags from its own op durations; the union is the one
        # global flag set the reference computes (feedback_update over all
        # ops), so every rank protects the same ops and leaves the loop at
        # the same round (same number of collective run() calls)
        mine = feedback_update(trace, config, flags)
        new = frozenset().union(*comm.allgather_object(sorted(mine)))
        if new == flags:
            break
        flags = new
    trace, metrics = run(plan, graph, n_gpus, bg_graph, config, iterations, flags,
                         baseline_fg_iteration_us, step=st, bg=bg, **kw)
    trace.op_isolated.update(isolated)
    return trace, metrics, flags
