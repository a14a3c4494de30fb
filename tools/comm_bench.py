"""HBM-side speed of the P2P data-path kernels on one B200 (peers simulated
as separate buffers on the same device, so every byte is an HBM read or
write; across GPUs the same kernels read over NVLink instead).

* reshard_pull: the C1 plan's transfers (plan(vgg_like B=32, 8, 2.0):
  8->4 and 4->1, forward and backward) as pulled by the busiest
  destination rank, plus a 1 GiB gather for the kernel's peak;
* allreduce two-shot phases of SymHeap.allreduce: reduce-scatter
  (bpx_allreduce_sum_prefix over g chunk pointers) and all-gather
  (bpx_reshard_pull of g-1 chunks) for the C1 buckets and the DP@8 bucket.

Prints one JSON line per case: bytes read+written per launch, us, GB/s and
the fraction of MEASURED_PEAKS hbm_gbs.  ``--case NAME`` runs one case
(for ncu)."""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_10065_b200 import ops, synth                   # noqa: E402
from paper_2112_10065_b200.costs import reshard_segments        # noqa: E402
from paper_2112_10065_b200.graph import ceil_div                # noqa: E402
from paper_2112_10065_b200.network import vgg16                 # noqa: E402
from paper_2112_10065_b200.planner import plan                  # noqa: E402


def peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / iters


def reshard_case(B, g, h, bps, dst_rank):
    cg, ch = ceil_div(B, g), ceil_div(B, h)
    srcs = [torch.randn(cg * bps // 4, device="cuda") for _ in range(g)]
    dst = torch.empty(ch * bps // 4, device="cuda")
    segs = [sg for sg in reshard_segments(B, g, h) if sg[1] == dst_rank]
    args = ([srcs[p].data_ptr() for p, *_ in segs],
            [(s - p * cg) * bps for p, _, s, _ in segs], dst,
            [(s - q * ch) * bps for _, q, s, _ in segs], [n * bps for *_, n in segs])
    moved = sum(n * bps for *_, n in segs)
    return (lambda: ops.reshard_pull(*args)), 2 * moved


def cases():
    net = vgg16()
    g = synth.vgg_like(seed=0, global_batch=32)
    p = plan(g, 8, 2.0)
    gs = [gi for lid, gi in p.assignments if not g.layer(lid).is_virtual]
    out = {}
    for i in range(1, len(gs)):
        if gs[i] != gs[i - 1]:
            bps = 4 * net.layers[i].in_elems()
            a, b = gs[i - 1], gs[i]
            out[f"reshard_fwd_{net.layers[i].name}_{a}to{b}"] = lambda a=a, b=b, bps=bps: \
                reshard_case(32, a, b, bps, 0)
            out[f"reshard_bwd_{net.layers[i].name}_{b}to{a}"] = lambda a=a, b=b, bps=bps: \
                reshard_case(32, b, a, bps, 0)
    # kernel peak: 1 GiB gathered from 8 sources
    out["reshard_1GiB_8to1"] = lambda: reshard_case(64, 8, 1, (1 << 30) // 64, 0)
    # two-shot allreduce phases: bucket sizes of the C1 plan and of DP@8
    sizes = {}
    for L, gi in zip(net.layers, gs):
        if L.param_shapes():
            sizes[gi] = sizes.get(gi, 0) + L.n_params()
    sizes = {k: v for k, v in sizes.items() if k > 1}
    sizes["dp8"] = sum(L.n_params() for L in net.layers if L.param_shapes())
    for key, n in sizes.items():
        gg = 8 if key == "dp8" else key
        c = ceil_div(ceil_div(n, gg), 4) * 4

        def rs(n=n, gg=gg, c=c):
            bufs = [torch.randn(n, device="cuda") for _ in range(gg)]
            ptrs = [b.data_ptr() for b in bufs]
            out_ = bufs[0][:c]
            return (lambda: ops.allreduce_sum_prefix(ptrs, out_, c)), 4 * c * (gg + 1)

        def ag(n=n, gg=gg, c=c):
            bufs = [torch.randn(n, device="cuda") for _ in range(gg)]
            segs = [(p * c, min(n, (p + 1) * c)) for p in range(1, gg)]
            args = ([bufs[p].data_ptr() for p in range(1, gg)], [4 * a for a, _ in segs],
                    bufs[0], [4 * a for a, _ in segs], [4 * (b - a) for a, b in segs])
            return (lambda: ops.reshard_pull(*args)), 2 * sum(4 * (b - a) for a, b in segs)

        out[f"allreduce_rs_g{gg}_{key}_{4 * n / 1e6:.0f}MB"] = rs
        out[f"allreduce_ag_g{gg}_{key}_{4 * n / 1e6:.0f}MB"] = ag
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default=None)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    pk = peak()
    for name, mk in cases().items():
        if a.case and a.case not in name:
            continue
        fn, nbytes = mk()
        us = timed(fn, a.iters)
        print(json.dumps({"case": name, "bytes_rw": nbytes, "us": us,
                          "gbs": nbytes / us / 1e3, "frac_hbm": nbytes / us / 1e3 / pk}),
              flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
