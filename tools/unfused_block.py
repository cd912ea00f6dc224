"""Whole-block comparison: fused CODA launches vs the unfused cuBLAS + torch sequence.

Same synthetic C4 (or C3) workload as bench.py.  Times one fwd+bwd step of each
path with CUDA events, checks the fused gradients against the unfused ones, and
prints one JSON line.  `--ncu fused|unfused` runs a single step of one path for
an ncu dram-bytes capture.

    python tools/unfused_block.py [--config c4] [--steps 5] [--ncu fused|unfused]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import unfused  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=tuple(bench.CONFIGS))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--ncu", choices=("fused", "unfused"))
    args = ap.parse_args()
    d, inter, m, label = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    P = cd.PrecisionMode.SIMBF16
    cfg = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=P)
    weights, acts, cos, sin = bench.make_workload(cd, d, inter, m, 0, dev)
    W = {k: getattr(weights, k).tensor for k in ("w_out", "w_gate_up", "w_down", "w_qkv")}
    W.update(gamma_ffn=weights.gamma_ffn.tensor.float(), gamma_qkv=weights.gamma_qkv.tensor.float())
    T = {k: v.tensor for k, v in acts.items()}

    def fused_step():
        return bench.run_step(cd, cfg, weights, acts, cos, sin)[1]

    def unfused_step():
        f = unfused.layer_forward(T["x"], T["z"], W, cos.tensor, sin.tensor, cfg.eps)
        return unfused.layer_backward(T["grad_qkv"], T["grad_residual"], f, T["x"], W, cos.tensor, sin.tensor)

    if args.ncu:
        fn = fused_step if args.ncu == "fused" else unfused_step
        fn()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("measure")   # ncu --nvtx --nvtx-include "measure/"
        fn()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        return

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps

    gf = fused_step()
    gu = unfused_step()
    rel = {}
    for k in ("x", "z", "w_out", "w_gate_up", "w_down", "w_qkv", "gamma_ffn", "gamma_qkv"):
        a = getattr(gf, k).tensor.float()
        b = gu[k].float()
        rel[k] = float((a - b).norm() / b.norm())
    tf = timed(fused_step)
    tu = timed(unfused_step)
    flops = bench.flops_per_token(d, inter) * m
    print(json.dumps({"workload": label, "fused_ms": tf, "unfused_ms": tu, "speedup": tu / tf,
                      "fused_tflops": flops / tf / 1e9, "unfused_tflops": flops / tu / 1e9,
                      "fused_tokens_per_s": m / tf * 1e3, "unfused_tokens_per_s": m / tu * 1e3,
                      "rel_err_fused_vs_unfused": rel}), flush=True)


if __name__ == "__main__":
    main()
