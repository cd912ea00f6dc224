"""Single-GEMM micro-benchmark with engine options A/B'd in-process (CUDA-graph timed).

    python tools/gemm_bench.py --shape 4096,4096,4096 --variant split=1 --variant split=0
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import os  # noqa: E402

os.environ.setdefault("CODA_LIB", "exp")   # measurement knobs live in the experiment build
from paper_2605_19269_b200 import _build  # noqa: E402

_build.build(experiments=True)

import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", action="append", required=True, help="m,n,k[,ta,tb]")
    ap.add_argument("--variant", action="append", required=True)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--inner", type=int, default=10, help="launches per captured graph (one timed replay)")
    ap.add_argument("--pad", type=int, default=0, help="extra elements per row of A and B (row-pitch experiment)")
    args = ap.parse_args()
    P = cd.PrecisionMode.SIMBF16
    for spec in args.shape:
        parts = [int(x) for x in spec.split(",")]
        m, n, k = parts[:3]
        ta, tb = (bool(parts[3]), bool(parts[4])) if len(parts) == 5 else (False, False)
        def mk(r, c):
            t = torch.randn((r, c + args.pad), device="cuda").to(torch.bfloat16)
            return t[:, :c] if args.pad else t

        A = mk(*((k, m) if ta else (m, k)))
        B = mk(*((n, k) if tb else (k, n)))
        a, b = cd.DenseMatrix.from_tensor(A, P), cd.DenseMatrix.from_tensor(B, P)
        prob = cd.GemmProblem(m=m, n=n, k=k, trans_a=ta, trans_b=tb, precision=P)
        graphs = []
        for v in args.variant:
            opts = {kk: int(x) for kk, x in (kv.split("=") for kv in v.split(","))}
            for kk, x in opts.items():
                _native.set_option(kk, x)
            for _ in range(3):
                cd.run_gemm(prob, a, b)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            _native.prepare_stream_workspace(torch.device("cuda", 0), cap)   # split-K tail inside the graph
            with torch.cuda.graph(g, stream=cap):
                for _ in range(args.inner):
                    cd.run_gemm(prob, a, b)
            graphs.append((v, g))
        times = {v: [] for v, _ in graphs}
        for rep in range(args.reps):
            # rotate the variant order every rep: no variant always runs first after the sync
            for v, g in graphs[rep % len(graphs):] + graphs[:rep % len(graphs)]:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                times[v].append(e0.elapsed_time(e1) / args.inner)
        res = {v: statistics.median(t) for v, t in times.items()}
        print(json.dumps({"shape": spec, **{v: {"ms": t, "tflops": 2 * m * n * k / t / 1e9} for v, t in res.items()}}),
              flush=True)


if __name__ == "__main__":
    main()
