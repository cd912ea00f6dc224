"""Sustained (power-capped) GEMM throughput and energy: CODA plain GEMM vs cuBLAS.

For each shape, alternates a CUDA graph of back-to-back CODA launches and a graph
of back-to-back torch.matmul (cuBLAS) launches, each run ~1.5 s so the 1 kW power
cap is in its steady state.  Reports TFLOP/s, NVML SM clock (median of 10 ms
samples) and energy per PFLOP from the NVML total-energy counter.

    python tools/vs_cublas.py [--rounds 2] [--seconds 1.5]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import pynvml  # noqa: E402
import torch  # noqa: E402

import os  # noqa: E402

if "--persist" in sys.argv or "--wave-sync" in sys.argv or "--backoff" in sys.argv:
    os.environ.setdefault("CODA_LIB", "exp")   # the persist option lives in the experiment build
    from paper_2605_19269_b200 import _build  # noqa: E402

    _build.build(experiments=True)
import paper_2605_19269_b200 as cd  # noqa: E402

SHAPES = {  # name: (m, n, k, trans_a, trans_b) — C4 launch shapes + a square one
    "K6 16384x28672x4096 NN": (16384, 28672, 4096, False, False),
    "K9a 16384x4096x28672 NT": (16384, 4096, 28672, False, True),
    "wgrad_gu 4096x28672x16384 TN": (4096, 28672, 16384, True, False),
    "square 8192^3 NN": (8192, 8192, 8192, False, False),
    "K10 16384x14336x4096 NT": (16384, 14336, 4096, False, True),
    "K4a 16384x4096x4096 NN": (16384, 4096, 4096, False, False),
    "wgrad_down 14336x4096x16384 TN": (14336, 4096, 16384, True, False),
}


class Sampler:
    def __init__(self, h):
        self.h, self.clk, self.pw, self.reasons = h, [], [], 0
        self._stop = threading.Event()

    def __enter__(self):
        def run():
            while not self._stop.is_set():
                try:
                    self.clk.append(pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM))
                    self.pw.append(pynvml.nvmlDeviceGetPowerUsage(self.h) / 1e3)
                    self.reasons |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    pass
                self._stop.wait(0.01)

        self.e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(self.h)
        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self.t.join()
        self.joules = (pynvml.nvmlDeviceGetTotalEnergyConsumption(self.h) - self.e0) / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--seconds", type=float, default=1.5)
    ap.add_argument("--shape", action="append", help="subset of SHAPES keys (prefix match)")
    ap.add_argument("--raster", type=int, action="append", help="also run CODA with these raster groups")
    ap.add_argument("--persist", action="store_true", help="also run CODA non-persistent (experiment build)")
    ap.add_argument("--wave-sync", type=int, action="append", help="also run CODA with this soft wave barrier %%")
    ap.add_argument("--backoff", type=int, action="append", help="also run CODA with this epilogue wait sleep (ns)")
    args = ap.parse_args()
    from paper_2605_19269_b200 import _native
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    P = cd.PrecisionMode.SIMBF16
    for name, (m, n, k, ta, tb) in SHAPES.items():
        if args.shape and not any(name.startswith(s) for s in args.shape):
            continue
        A = (torch.randn((k, m) if ta else (m, k), device="cuda") * k ** -0.25).to(torch.bfloat16)
        B = (torch.randn((n, k) if tb else (k, n), device="cuda") * k ** -0.25).to(torch.bfloat16)
        a, b = cd.DenseMatrix.from_tensor(A, P), cd.DenseMatrix.from_tensor(B, P)
        prob = cd.GemmProblem(m=m, n=n, k=k, trans_a=ta, trans_b=tb, precision=P)
        At = A.t() if ta else A
        Bt = B.t() if tb else B
        out = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
        flops = 2.0 * m * n * k

        def coda():
            cd.run_gemm(prob, a, b)

        def cublas():
            torch.matmul(At, Bt, out=out)

        per = {}
        graphs = {}
        def coda_np():
            _native.set_option("persist", 0)
            cd.run_gemm(prob, a, b)
            _native.set_option("persist", 1)

        def coda_ws(pct):
            def fn():
                _native.set_option("wave_sync", pct)
                cd.run_gemm(prob, a, b)
                _native.set_option("wave_sync", 0)
            return fn

        def coda_bo(ns):
            def fn():
                _native.set_option("backoff", ns)
                cd.run_gemm(prob, a, b)
                _native.set_option("backoff", 0)
            return fn

        variants = [(f"coda_bo{n}", coda_bo(n), 8) for n in (args.backoff or [])] + \
                   [("coda", coda, 8)] + [(f"coda_r{g}", coda, g) for g in (args.raster or [])] + \
                   ([("coda_nonpersist", coda_np, 8)] if args.persist else []) + \
                   [(f"coda_ws{p}", coda_ws(p), 8) for p in (args.wave_sync or [])] + [("cublas", cublas, None)]
        cap = torch.cuda.Stream()
        _native.prepare_stream_workspace(torch.device("cuda", torch.cuda.current_device()), cap)
        for label, fn, raster in variants:
            if raster is not None:
                _native.set_option("raster", raster)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            reps = max(4, int(args.seconds * 1e3 / max(e0.elapsed_time(e1), 1e-3)))
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):     # own split-K workspace inside the graph
                for _ in range(reps):
                    fn()
            graphs[label] = (g, reps)
            per[label] = []
        _native.set_option("raster", 8)
        for _ in range(args.rounds):
            for label, (g, reps) in graphs.items():
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with Sampler(h) as s:
                    e0.record()
                    g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                per[label].append({"tflops": flops / ms / 1e9, "ms": ms,
                                   "sm_mhz": statistics.median(s.clk) if s.clk else None,
                                   "watts": statistics.median(s.pw) if s.pw else None,
                                   "j_per_pflop": s.joules / (flops * reps / 1e15),
                                   "reasons": hex(s.reasons)})
        res = {"shape": name}
        for label, runs in per.items():
            best = max(runs, key=lambda r: r["tflops"])
            res[label] = {kk: round(v, 3) if isinstance(v, float) else v for kk, v in best.items()}
        for label in per:
            if label.startswith("coda"):
                res[f"{label}/cublas"] = round(res[label]["tflops"] / res["cublas"]["tflops"], 4)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
