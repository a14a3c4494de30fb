"""Executable networks behind the planner's synthetic graphs.

The reference's graphs carry only costs (`synth.py:86-123` for VGG-16);
the executor needs the real layers.  ``NetSpec`` binds each graph layer
name to a concrete op with shapes, in the same order, so a plan's
``(layer_id, g)`` list maps 1:1 onto executable layers.

VGG-16 here is the real network (conv bias, fc1 25088->4096, 138,357,544
parameters) without dropout.  Layouts: activations NHWC,
conv weights OHWI ([Cout][3][3][Cin]), dense weights [out][in] with fc1's
input in NHWC-flatten order (h, w, c).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import torch

from .errors import GraphFormatError
from .graph import CompGraph


@dataclass(frozen=True)
class LayerSpec:
    name: str
    kind: str            # conv | conv1x1 | pool | pool3 | dense | add | gap | concat
    cin: int             # channels (conv/pool/add/gap) or input features (dense)
    cout: int
    hw: int              # spatial size the layer computes at (pool: input); 0 for dense
    relu: bool           # output passes through ReLU
    in_relu: bool        # input is a ReLU output (dgrad fuses its mask)
    down: bool = False   # conv: input is 2hw x 2hw, subsampled by 2 first
    skip: Optional[str] = None   # add: the skip (shortcut) source layer
    skip_c: int = 0      # add: channels of the skip source (<= cin, zero-padded)
    skip_down: bool = False      # add: skip source is 2hw x 2hw (subsampled)
    src: Optional[str] = None    # input layer (None: the previous layer)
    srcs: tuple = ()             # concat: the joined layers, in channel order
    ihw: int = 0                 # down: input size when not 2*hw (2*hw+1: odd pixels kept)
    bn: bool = False             # conv: synchronised BatchNorm over [0, g) after the conv
                                 # (no conv bias; the "bias" slot holds [beta ; gamma])

    @property
    def out_hw(self) -> int:
        return self.hw // 2 if self.kind == "pool" else self.hw

    @property
    def in_hw(self) -> int:
        if not self.down:
            return self.hw
        return self.ihw or 2 * self.hw

    @property
    def sub_off(self) -> int:
        """Offset of the stride-2 subsample of a down layer (0 or 1)."""
        return self.in_hw - 2 * self.hw

    def in_elems(self) -> int:
        """Input floats per sample."""
        return self.in_hw * self.in_hw * self.cin if self.kind != "dense" else self.cin

    def out_elems(self) -> int:
        if self.kind in ("dense", "gap"):
            return self.cout
        return self.out_hw * self.out_hw * self.cout

    def in_shape(self, b: int) -> tuple[int, ...]:
        if self.kind == "dense":
            return (b, self.cin)
        return (b, self.in_hw, self.in_hw, self.cin)

    def out_shape(self, b: int) -> tuple[int, ...]:
        if self.kind in ("dense", "gap"):
            return (b, self.cout)
        return (b, self.out_hw, self.out_hw, self.cout)

    def param_shapes(self) -> Optional[tuple[tuple[int, ...], tuple[int, ...]]]:
        nb = 2 * self.cout if self.bn else self.cout
        if self.kind == "conv":
            return (self.cout, 3, 3, self.cin), (nb,)
        if self.kind == "conv1x1":
            return (self.cout, 1, 1, self.cin), (nb,)
        if self.kind == "dense":
            return (self.cout, self.cin), (self.cout,)
        return None

    def n_params(self) -> int:
        ps = self.param_shapes()
        return 0 if ps is None else math.prod(ps[0]) + math.prod(ps[1])

    def fwd_flops(self) -> int:
        """Algorithmic fwd FLOPs per sample (2 per MAC; bias/ReLU excluded)."""
        if self.kind == "conv":
            return 2 * 9 * self.cin * self.cout * self.hw * self.hw
        if self.kind == "conv1x1":
            return 2 * self.cin * self.cout * self.hw * self.hw
        if self.kind == "dense":
            return 2 * self.cin * self.cout
        return 0


@dataclass(frozen=True)
class NetSpec:
    name: str
    input_hw: int
    input_c: int
    classes: int
    layers: tuple[LayerSpec, ...]

    def by_name(self) -> dict[str, LayerSpec]:
        return {l.name: l for l in self.layers}

    def n_params(self) -> int:
        return sum(l.n_params() for l in self.layers)

    def train_flops_per_sample(self) -> int:
        """fwd + dgrad + wgrad, minus the first layer's dgrad (its input is
        the image): the roofline's algorithmic work."""
        f = sum(l.fwd_flops() for l in self.layers)
        return 3 * f - self.layers[0].fwd_flops()


def vgg16() -> NetSpec:
    layers = []
    hw, cin = 224, 3
    first = True
    for stage, (cout, n) in enumerate(((64, 2), (128, 2), (256, 3), (512, 3), (512, 3)),
                                      start=1):
        for j in range(1, n + 1):
            layers.append(LayerSpec(f"conv{stage}_{j}", "conv", cin, cout, hw, True,
                                    not first))
            first = False
            cin = cout
        layers.append(LayerSpec(f"pool{stage}", "pool", cout, cout, hw, False, True))
        hw //= 2
    feats = hw * hw * cin
    for k, (fout, relu) in enumerate(((4096, True), (4096, True), (1000, False)), start=1):
        layers.append(LayerSpec(f"fc{k}", "dense", feats, fout, 0, relu, True))
        feats = fout
    return NetSpec("vgg16", 224, 3, 1000, tuple(layers))


def mlp_for_chain(graph: CompGraph) -> NetSpec:
    """Executable stand-in for the reference's ``custom`` chain family
    (synth.py:229-244; small_bg_model, the default background job): one
    dense layer per graph layer with width ~sqrt(params) rounded to 16, so
    each layer carries about the graph's parameter count (2 M for
    small_bg_model -> 1408 x 1408) and runs the short kernels the family
    models.  ReLU everywhere but the classifier."""
    real = [l for l in graph.layers if not l.is_virtual]
    width = max(16, int(math.isqrt(max(real[0].params_bytes // 4, 1))) // 16 * 16)
    layers = tuple(LayerSpec(l.name, "dense", width, width, 0, i + 1 < len(real), i > 0)
                   for i, l in enumerate(real))
    return NetSpec(f"mlp{width}x{len(real)}", 1, width, width, layers)


def wideresnet_net(graph: CompGraph, bn: bool = True) -> NetSpec:
    """Executable residual net behind the reference's ``wideresnet_like``
    family (synth.py:126-169), shapes read off the graph itself: channels
    from each conv's 9*cin*cout parameters, spatial size from its activation
    bytes.  Builder decisions (the reference family only prices layers,
    SURVEY.md §8d C3):

    * stem: 3x3 conv 3 -> 64 at the stem's resolution (100x100; the graph's
      nominal input is 3x400x400 -- the executable net takes the stem's
      100x100 input directly);
    * each diamond is a post-activation basic block: conv1 + ReLU, conv2,
      ``add`` = ReLU(conv2 + shortcut); at a stage transition (hw halves)
      conv1 reads a stride-2 subsample of its input, and the shortcut is
      ResNet "option A": stride-2 subsample + zero channel padding (the
      graph has no projection layer, so the shortcut has no parameters);
    * ``pool`` = global average pool; ``fc`` = dense (channels -> 1000).
      The graph gives fc the rest of a 127 M parameter budget; the
      executable classifier is the real 512 x 1000 layer;
    * every conv is followed by batch normalisation (``bn=True``; the
      reference has no BN notion), synchronised over the
      layer's GPU group [0, g): statistics of the whole global batch, so
      the numerics do not depend on the plan (``bn=False`` builds the
      normalisation-free variant with the Fixup-style init).
    """
    real = [l for l in graph.layers if not l.is_virtual]
    ids = {l.id for l in real}
    by_id = {l.id: l for l in real}
    out_c: dict[int, int] = {}
    out_hw: dict[int, int] = {}
    relu_out: dict[int, bool] = {}
    specs = []
    input_hw = 0
    for l in real:
        preds = [p for p in l.predecessors if p in ids]
        succs = [by_id[s] for s in l.successors if s in ids]
        if l.kind == "conv":
            k = 1 if l.name.endswith("_1x1") else 9      # bottleneck 1x1 convs (resnet50_like)
            cin = out_c[preds[0]] if preds else 3
            cout = l.params_bytes // 4 // (k * cin)
            hw = math.isqrt(l.activation_bytes_per_sample // (4 * cout))
            if k * cin * cout * 4 != l.params_bytes or cout * hw * hw * 4 != \
                    l.activation_bytes_per_sample:
                raise GraphFormatError(f"{l.name}: not a {'1x1' if k == 1 else '3x3'} conv shape")
            if not preds:
                input_hw = hw
            ihw = out_hw[preds[0]] if preds else hw
            if ihw not in (hw, 2 * hw):
                raise GraphFormatError(f"{l.name}: input {ihw} -> {hw} is not 1x or /2")
            # a conv feeding only a join is the block's second conv: no ReLU
            relu = not (len(succs) == 1 and succs[0].kind == "add")
            if k == 1 and ihw != hw:
                raise GraphFormatError(f"{l.name}: strided 1x1 convs are not built")
            specs.append(LayerSpec(l.name, "conv" if k == 9 else "conv1x1", cin, cout, hw, relu,
                                   bool(preds) and relu_out[preds[0]], down=ihw == 2 * hw,
                                   bn=bn))
            out_c[l.id], out_hw[l.id], relu_out[l.id] = cout, hw, relu
        elif l.kind == "add":
            main = [p for p in preds if by_id[p].kind == "conv"
                    and len([s for s in by_id[p].successors if s in ids]) == 1
                    and p != preds[-1]]
            if len(preds) != 2 or len(main) != 1:
                raise GraphFormatError(f"{l.name}: expected (conv2, shortcut) inputs")
            m = main[0]
            sk = preds[0] if preds[1] == m else preds[1]
            c, hw = out_c[m], out_hw[m]
            if out_hw[sk] not in (hw, 2 * hw) or out_c[sk] > c:
                raise GraphFormatError(f"{l.name}: shortcut shape does not fit")
            specs.append(LayerSpec(l.name, "add", c, c, hw, True, False,
                                   skip=by_id[sk].name, skip_c=out_c[sk],
                                   skip_down=out_hw[sk] == 2 * hw))
            out_c[l.id], out_hw[l.id], relu_out[l.id] = c, hw, True
        elif l.kind == "pool":
            p = preds[0]
            specs.append(LayerSpec(l.name, "gap", out_c[p], out_c[p], out_hw[p], False,
                                   relu_out[p]))
            out_c[l.id], out_hw[l.id], relu_out[l.id] = out_c[p], 1, False
        elif l.kind == "dense":
            p = preds[0]
            fout = l.activation_bytes_per_sample // 4
            specs.append(LayerSpec(l.name, "dense", out_c[p], fout, 0, False, relu_out[p]))
            out_c[l.id], out_hw[l.id], relu_out[l.id] = fout, 1, False
        else:
            raise GraphFormatError(f"{l.name}: kind {l.kind!r} not executable")
    return NetSpec("wrn", input_hw, 3, specs[-1].cout, tuple(specs))


INCEPTION_CH, INCEPTION_HALF = 64, 32     # synth.py:172-226: stem / tower widths


def inception_net(graph: CompGraph) -> NetSpec:
    """Executable four-tower net behind the reference's ``inception_like``
    family (synth.py:172-226).  The family rescales conv parameters to a
    24 M budget, so channels come from its own constants (stem 64, towers
    32, concat 4 x 32) and resolutions from the activation bytes (35 -> 17
    -> 8).  Builder decisions: 3x3 convs and the ``_1x1`` convs (run as
    pixel-batched dense ops) carry a ReLU; ``stem_pool`` and each module's
    ``pool_proj`` are 3x3 / stride-1 max pools, the latter over the first 32
    channels of the module input (a parameter-free projection); where the
    resolution drops, each tower's first layer reads a stride-2 subsample
    of the module input keeping the odd pixels (35 -> 17 -> 8); the
    classifier is dense on the NHWC-flattened last concat (8*8*128 -> 1000)."""
    real = [l for l in graph.layers if not l.is_virtual]
    ids = {l.id for l in real}
    by_id = {l.id: l for l in real}
    c_of: dict[int, int] = {}
    hw_of: dict[int, int] = {}
    specs = []
    input_hw = 0
    for l in real:
        preds = [p for p in l.predecessors if p in ids]
        src = by_id[preds[0]] if preds else None
        tower = l.name.startswith("m")
        if l.kind in ("conv", "pool"):
            cout = INCEPTION_HALF if tower else (INCEPTION_CH if l.kind == "conv" or src is None
                                                  else c_of[src.id])
            hw = math.isqrt(l.activation_bytes_per_sample // (4 * cout))
            if cout * hw * hw * 4 != l.activation_bytes_per_sample:
                raise GraphFormatError(f"{l.name}: activation bytes do not fit {cout} channels")
            cin = c_of[src.id] if src else 3
            ihw = hw_of[src.id] if src else hw
            if not src:
                input_hw = hw
            if ihw not in (hw, 2 * hw, 2 * hw + 1):
                raise GraphFormatError(f"{l.name}: input {ihw} -> {hw} is not 1x or /2")
            down = ihw != hw
            if l.kind == "conv":
                kind = "conv1x1" if l.name.endswith("_1x1") else "conv"
                specs.append(LayerSpec(l.name, kind, cin, cout, hw, True, src is not None,
                                       down=down, src=src.name if src else None,
                                       ihw=ihw if down else 0))
            else:
                if cout > cin:
                    raise GraphFormatError(f"{l.name}: pool projects {cin} -> {cout}")
                specs.append(LayerSpec(l.name, "pool3", cin, cout, hw, False, False, down=down,
                                       src=src.name, ihw=ihw if down else 0))
        elif l.kind == "concat":
            hws = {hw_of[p] for p in preds}
            if len(hws) != 1 or not 1 <= len(preds) <= 4:
                raise GraphFormatError(f"{l.name}: concat inputs differ in size")
            cout = sum(c_of[p] for p in preds)
            hw = hws.pop()
            specs.append(LayerSpec(l.name, "concat", cout, cout, hw, False, False,
                                   srcs=tuple(by_id[p].name for p in preds)))
        elif l.kind == "dense":
            cin = c_of[src.id] * hw_of[src.id] ** 2
            cout = l.activation_bytes_per_sample // 4
            specs.append(LayerSpec(l.name, "dense", cin, cout, 0, False, True, src=src.name))
            hw = 1
        else:
            raise GraphFormatError(f"{l.name}: kind {l.kind!r} not executable")
        c_of[l.id], hw_of[l.id] = cout, hw
    return NetSpec("inception", input_hw, 3, specs[-1].cout, tuple(specs))


_REGISTRY = {"vgg_like": lambda g: vgg16(), "custom": mlp_for_chain,
             "wideresnet_like": wideresnet_net, "inception_like": inception_net,
             "resnet50_like": wideresnet_net}


def net_for_graph(graph: CompGraph) -> NetSpec:
    """The executable network behind a planner graph; layer names must
    match the graph's non-virtual layers one for one, in order."""
    fn = _REGISTRY.get(graph.name)
    if fn is None:
        raise GraphFormatError(f"no executable network registered for graph {graph.name!r}")
    net = fn(graph)
    names = [l.name for l in graph.layers if not l.is_virtual]
    if names != [l.name for l in net.layers]:
        raise GraphFormatError(f"graph {graph.name!r} layers do not match {net.name}")
    return net


def init_params(net: NetSpec, seed: int = 0) -> dict[str, tuple[torch.Tensor, torch.Tensor]]:
    """torchvision-style init on CPU (kaiming_normal fan_out/relu for convs --
    fan_in for the four-tower net -- N(0, 0.01) for dense, zero bias),
    deterministic in ``seed``."""
    gen = torch.Generator().manual_seed(seed)
    out = {}
    # residual nets have no normalisation layers: the last conv of each
    # residual branch (no ReLU of its own) starts scaled by 1/sqrt(blocks),
    # so the post-activation sum stays O(1) over all diamonds (Fixup-style;
    # unscaled, 34 diamonds overflow fp32 in the forward pass)
    blocks = sum(1 for l in net.layers if l.kind == "add")
    # four-tower nets narrow 128 -> 32 channels in their 1x1 towers: fan-out
    # init would grow the forward variance ~4x per module (fp32 logits in
    # the thousands after 14 modules), so they use fan-in (the forward-
    # preserving Kaiming mode)
    fan_in = any(l.kind == "concat" for l in net.layers)
    for l in net.layers:
        ps = l.param_shapes()
        if ps is None:
            continue
        if l.kind in ("conv", "conv1x1"):
            k = 9 if l.kind == "conv" else 1
            std = math.sqrt(2.0 / ((l.cin if fan_in else l.cout) * k))
            if blocks and not l.relu and not l.bn:
                std /= math.sqrt(blocks)
        else:
            std = 0.01
        w = torch.randn(ps[0], generator=gen, dtype=torch.float32) * std
        b = torch.zeros(ps[1], dtype=torch.float32)
        if l.bn:                          # [beta ; gamma] = [0 ; 1]
            b[l.cout:] = 1.0
        out[l.name] = (w, b)
    return out


def synthetic_batch(net: NetSpec, batch: int, seed: int = 0):
    """x ~ N(0, 1) NHWC and uniform labels, on CPU."""
    gen = torch.Generator().manual_seed(seed)
    x = torch.randn((batch, net.input_hw, net.input_hw, net.input_c), generator=gen,
                    dtype=torch.float32)
    y = torch.randint(0, net.classes, (batch,), generator=gen, dtype=torch.int64)
    return x, y.to(torch.int32)
