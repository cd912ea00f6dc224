"""BASELINE config 2: single fused GEMM + epilogue primitive at 4096^3 bf16, 1 GPU.

For each primitive (plain, scale, row-reduce, SwiGLU, RoPE, residual) times the
fused CODA launch against the unfused sequence (cuBLAS GEMM via torch.matmul +
one torch elementwise op), checks the two agree, and prints one JSON line per
primitive plus a summary.  `--ncu` runs each variant once (for an ncu
dram-bytes capture) without timing.

    python tools/primitive_sweep.py [--size 4096] [--reps 20] [--ncu]
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import unfused  # noqa: E402


def timeit(fn, reps, warmup=5, inner=10):
    """Median device time of one call: `inner` calls captured in a CUDA graph and
    replayed, so host launch latency (Python) is excluded for both variants."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(inner):
            fn()
    g.replay()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / inner)
    return statistics.median(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ncu", action="store_true")
    args = ap.parse_args()
    n = args.size
    dev = torch.device("cuda", 0)
    P = cd.PrecisionMode.SIMBF16
    g = torch.Generator(device=dev).manual_seed(0)
    A = (torch.randn((n, n), generator=g, device=dev) / n ** 0.5).to(torch.bfloat16)
    B = (torch.randn((n, n), generator=g, device=dev) / n ** 0.5).to(torch.bfloat16)
    C = torch.randn((n, n), generator=g, device=dev).to(torch.bfloat16)
    r = (0.5 + torch.rand(n, generator=g, device=dev)).float()
    a, b, c = (cd.DenseMatrix.from_tensor(t, P) for t in (A, B, C))
    rv = cd.Vector.from_tensor(r, cd.PrecisionMode.SIM32)
    cos, sin = cd.rope_tables(n, n, precision=P)
    kw = dict(precision=P)
    prob = cd.GemmProblem(m=n, n=n, k=n, precision=P)

    def rowreduce_unfused():
        y = A @ B
        return (y.float() ** 2).view(n, n // 128, 128).sum(-1), y

    variants = {
        "plain": (lambda: cd.run_gemm(prob, a, b).main.tensor, lambda: A @ B),
        "scale": (lambda: cd.gemm_row_scale(a, b, rv, **kw).main.tensor,
                  lambda: ((A @ B).float() * r[:, None]).to(torch.bfloat16)),
        "row_reduce": (lambda: cd.run_gemm(prob, a, b, cd.EpilogueProgram([cd.PartialSumSq("s")])).aux["s"].tensor,
                       lambda: rowreduce_unfused()[0]),
        "swiglu": (lambda: cd.gemm_swiglu(a, b, **kw).main.tensor, lambda: unfused.swiglu(A @ B)),
        "rope": (lambda: cd.gemm_rope(a, b, cos, sin, **kw).main.tensor,
                 lambda: unfused.rope(A @ B, cos.tensor, sin.tensor)),
        "residual": (lambda: cd.run_gemm(prob, a, b, cd.EpilogueProgram([cd.ResidualAdd("c")]), {"c": c}).main.tensor,
                     lambda: A @ B + C),
    }
    if args.ncu:
        for name, (fused, unf) in variants.items():
            fused()
            unf()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("measure")   # ncu --nvtx --nvtx-include "measure/"
        for name, (fused, unf) in variants.items():
            torch.cuda.nvtx.range_push(name)
            fused()
            unf()
            torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        return
    flops = 2.0 * n ** 3
    rows = []
    for name, (fused, unf) in variants.items():
        yf, yu = fused().float(), unf().float()
        rel = float((yf - yu).norm() / yu.norm())
        tf = timeit(fused, args.reps)
        tu = timeit(unf, args.reps)
        row = {"primitive": name, "size": n, "fused_ms": tf, "unfused_ms": tu, "speedup": tu / tf,
               "fused_tflops": flops / tf / 1e9, "unfused_tflops": flops / tu / 1e9, "rel_err_vs_unfused": rel}
        rows.append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps({"summary": "c2 primitive sweep", "geomean_speedup":
                      statistics.geometric_mean(r["speedup"] for r in rows)}), flush=True)


if __name__ == "__main__":
    main()
