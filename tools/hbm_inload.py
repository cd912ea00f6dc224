"""HBM-bound launches in the block's power state: rope_backward_stat at C4 and a plain
device copy of the same byte count, each timed with CUDA events (a) queued back to back
on an otherwise idle GPU and (b) right behind three K7-shaped GEMMs (the step's
condition: the rope follows K7), with NVML SM / memory clocks and power sampled over
each phase.  Every measured launch sits behind queued device work, so no host time is
inside its events.

    python tools/hbm_inload.py [--iters 40]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19269_b200 as cd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=40)
    args = ap.parse_args()
    P = cd.PrecisionMode.SIMBF16
    dev = torch.device("cuda", 0)
    m, d = 16384, 4096
    q = 3 * d
    cos, sin = cd.qkv_rope_tables(m, d, precision=P)
    g = cd.DenseMatrix.from_tensor(torch.randn(m, q, device=dev).to(torch.bfloat16), P)
    r = cd.DenseMatrix.from_tensor(torch.randn(m, q, device=dev).to(torch.bfloat16), P)
    a = cd.DenseMatrix.from_tensor((torch.randn(m, d, device=dev) * 0.05).to(torch.bfloat16), P)
    b = cd.DenseMatrix.from_tensor((torch.randn(d, q, device=dev) * 0.05).to(torch.bfloat16), P)
    prob = cd.GemmProblem(m, q, d, precision=P)
    byts = 2 * m * q * 2 + 2 * m * (d // 2) * 2 + m * q * 2 + m * (q // 128) * 4
    src = torch.empty(byts // 2, dtype=torch.uint8, device=dev)      # copy: reads + writes = byts
    dst = torch.empty_like(src)
    peak = bench.peaks()["hbm_gbs"]

    def rope():
        cd.rope_backward_stat(g, r, cos, sin, precision=P)

    def copy():
        dst.copy_(src)

    ops = {"rope_backward_stat": (rope, byts), "copy": (copy, 2 * src.numel())}
    out = {}
    for mode in ("queued", "after_gemm"):
        for name, (fn, nbytes) in ops.items():
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            evs = []
            with bench.clock_sampler(0) as clocks:
                for it in range(args.iters):
                    if mode == "after_gemm":
                        for _ in range(3):
                            cd.run_gemm(prob, a, b)
                    else:
                        fn()       # keeps the queue ahead of the measured launch
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    fn()
                    e1.record()
                    evs.append((e0, e1))
                torch.cuda.synchronize()
            ts = [x.elapsed_time(y) for x, y in evs][5:]
            ms = statistics.median(ts)
            gbs = nbytes / ms / 1e6
            out[f"{name}:{mode}"] = {"ms": round(ms, 4), "GB/s": round(gbs, 1), "frac_of_peak": round(gbs / peak, 3),
                                     "bytes": nbytes, "clocks": clocks.summary()}
            print(name, mode, out[f"{name}:{mode}"], flush=True)
    for mode in ("queued", "after_gemm"):
        out[f"rope_vs_copy:{mode}"] = round(out[f"rope_backward_stat:{mode}"]["GB/s"] / out[f"copy:{mode}"]["GB/s"], 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
