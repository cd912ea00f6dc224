"""Epilogue overhead of every fused C4 launch: fused launch vs a plain GEMM of the same
shape and operand majorness, timed back to back in the same process (rounds interleave).

    python tools/epi_overhead.py [--rounds 5]
"""
from __future__ import annotations

import argparse
import re
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import os  # noqa: E402

os.environ.setdefault("CODA_LIB", "exp")   # measurement knobs live in the experiment build
from paper_2605_19269_b200 import _build  # noqa: E402

_build.build(experiments=True)

import bench  # noqa: E402
import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import _native  # noqa: E402

SHAPE = re.compile(r"(\d+)x(\d+)x(\d+)( TN| NT)?")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--option", action="append", default=[], help="engine option name=value for the fused runs")
    args = ap.parse_args()
    d, inter, m, _ = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    P = cd.PrecisionMode.SIMBF16
    cfg = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=P)
    weights, acts, cos, sin = bench.make_workload(cd, d, inter, m, 0, dev)
    step = lambda: bench.run_step(cd, cfg, weights, acts, cos, sin)  # noqa: E731
    step()
    prof = _native.profile_launches(step, reps=1)
    plains = {}
    for tag in prof:
        mt = SHAPE.search(tag)
        if not mt:
            continue
        mm, nn, kk = (int(x) for x in mt.groups()[:3])
        ta, tb = mt.group(4) == " TN", mt.group(4) == " NT"
        A = (torch.randn((kk, mm) if ta else (mm, kk), device=dev) * 0.05).to(torch.bfloat16)
        B = (torch.randn((nn, kk) if tb else (kk, nn), device=dev) * 0.05).to(torch.bfloat16)
        plains[tag] = (cd.GemmProblem(m=mm, n=nn, k=kk, trans_a=ta, trans_b=tb, precision=P),
                       cd.DenseMatrix.from_tensor(A, P), cd.DenseMatrix.from_tensor(B, P))
    fused = {t: [] for t in plains}
    plain = {t: [] for t in plains}

    def run_plains():
        for t, (pr, a, b) in plains.items():
            cd.run_gemm(pr, a, b, kernel_name="plain:" + t)

    opts = [(kv.split("=")[0], int(kv.split("=")[1])) for kv in args.option]
    for kk, vv in opts:
        _native.set_option(kk, vv)
    for _ in range(args.rounds):
        step()
        pf = _native.profile_launches(step, reps=1)
        run_plains()
        pp = _native.profile_launches(run_plains, reps=1)
        for t in plains:
            fused[t].append(pf[t]["avg_ms"])
            key = next(k for k in pp if k.startswith("plain:" + t.split(" ")[0]) and t.split(" ", 1)[1] in k)
            plain[t].append(pp[key]["avg_ms"])
    tf, tp = 0.0, 0.0
    for t in plains:
        f, p = statistics.median(fused[t]), statistics.median(plain[t])
        tf += f
        tp += p
        print(f"{t[:52]:52s} fused {f:7.3f} ms  plain {p:7.3f} ms  overhead {100 * (f / p - 1):+6.1f}%")
    print(f"{'GEMM total':52s} fused {tf:7.3f} ms  plain {tp:7.3f} ms  overhead {100 * (tf / tp - 1):+6.1f}%")


if __name__ == "__main__":
    main()
