"""Persistent-GEMM robustness when some SMs are busy with another kernel (a stand-in
for an NCCL collective on a side stream): a long, narrow CODA GEMM is launched on a
side stream first and occupies `--busy` SM pairs; the measured GEMM is launched right
after on the main stream.  Static round-robin scheduling must wait for the busy SMs;
the dynamic scheduler hands their tiles to the free ones.

    python tools/interfere.py --busy 8
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
from paper_2605_19269_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--busy", type=int, default=8, help="CTA pairs occupied by the side-stream kernel")
    ap.add_argument("--busy-k", type=int, default=65536)
    ap.add_argument("--shape", default="16384,28672,4096")
    ap.add_argument("--reps", type=int, default=8)
    args = ap.parse_args()
    P = cd.PrecisionMode.SIMBF16
    m, n, k = (int(x) for x in args.shape.split(","))
    mk = lambda r, c: cd.DenseMatrix.from_tensor((torch.randn((r, c), device="cuda") * 0.05).to(torch.bfloat16), P)  # noqa: E731
    a, b = mk(m, k), mk(k, n)
    prob = cd.GemmProblem(m=m, n=n, k=k, precision=P)
    bk = args.busy_k
    ia, ib = mk(256, bk), mk(bk, 256 * args.busy)
    iprob = cd.GemmProblem(m=256, n=256 * args.busy, k=bk, precision=P)
    side = torch.cuda.Stream()
    main_s = torch.cuda.current_stream()
    times = {}
    for r in range(args.reps + 2):          # variants interleaved rep by rep (same power state)
        for sched in (0, 1):
            _native.set_option("sched", sched)
            for mode in ("alone", "with_busy"):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if mode == "with_busy":
                    _native.set_option("split", 0)     # keep the side kernel on its `busy` pairs
                    with torch.cuda.stream(side):
                        cd.run_gemm(iprob, ia, ib)
                    _native.set_option("split", 1)
                    torch.cuda._sleep(20000)   # let the side kernel take its SMs first
                e0.record(main_s)
                cd.run_gemm(prob, a, b)
                e1.record(main_s)
                torch.cuda.synchronize()
                if r >= 2:
                    times.setdefault(f"sched={sched} {mode}", []).append(e0.elapsed_time(e1))
    res = {key: round(statistics.median(v), 4) for key, v in times.items()}
    # the side kernel alone, for reference
    _native.set_option("split", 0)
    cd.run_gemm(iprob, ia, ib)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cd.run_gemm(iprob, ia, ib)
    e1.record()
    torch.cuda.synchronize()
    _native.set_option("split", 1)
    res["side kernel alone"] = round(e0.elapsed_time(e1), 4)
    print(json.dumps({"shape": args.shape, "busy_pairs": args.busy, "ms": res}))


if __name__ == "__main__":
    main()
