"""Interleaved in-process A/B of pipeline variants of the C4 (or other) block step.

Variants (comma-separated in one --variant):
  plain            the reference schedule (default)
  fold             gains folded into W (PipelineConfig.fold_gamma), fold launches inside the step
  fold_cached      gains folded once outside the step (what an optimizer writing W' would give)
  cap=N            backward GEMMs limited to N SMs (room for a concurrent all-reduce)
  tokens=M         token count (per-rank shape proxies)

    python tools/ab_pipeline.py --config c4 --rounds 12 --variant plain --variant fold --variant cap=132
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import _native  # noqa: E402


def parse(v: str) -> dict:
    out = {}
    for kv in v.split(","):
        if "=" in kv:
            k, x = kv.split("=")
            out[k] = int(x)
        else:
            out[kv] = True
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=tuple(bench.CONFIGS))
    ap.add_argument("--rounds", type=int, default=12)
    ap.add_argument("--variant", action="append", required=True)
    ap.add_argument("--breakdown", action="store_true", help="also per-launch times (2 profiled steps per variant)")
    args = ap.parse_args()
    d, inter, m0, label = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    variants = [parse(v) for v in args.variant]
    work = {}
    for v in variants:
        m = v.get("tokens", m0)
        if m not in work:
            work[m] = bench.make_workload(cd, d, inter, m, 0, dev, blocks=bench.BLOCKS.get(args.config, 1))
    times = {i: [] for i in range(len(variants))}
    cached = {}

    def run(i):
        v = variants[i]
        m = v.get("tokens", m0)
        weights, acts, cos, sin = work[m]
        fold = bool(v.get("fold") or v.get("fold_cached"))
        cfg = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=cd.PrecisionMode.SIMBF16, fold_gamma=fold)
        if v.get("fold_cached"):
            if m not in cached:
                cached[m] = cd.fold_gains(weights)
            fwd = cd.layer_forward(acts["x"], acts["z"], weights, cos, sin, config=cfg, folded=cached[m])
            with _native.limit_sms(v.get("cap", 0)):
                cd.layer_backward(acts["grad_qkv"], fwd.tape, weights, grad_residual=acts["grad_residual"],
                                  config=cfg)
            return
        bench.run_step(cd, cfg, weights, acts, cos, sin, bwd_sms=v.get("cap", 0))

    for i in range(len(variants)):
        for _ in range(3):
            run(i)
    torch.cuda.synchronize()
    for _ in range(args.rounds):
        for i in range(len(variants)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(i)
            e1.record()
            torch.cuda.synchronize()
            times[i].append(e0.elapsed_time(e1))
    out = []
    for i, v in enumerate(variants):
        med = statistics.median(times[i])
        m = v.get("tokens", m0)
        row = {"variant": args.variant[i], "tokens": m, "median_ms": med, "min_ms": min(times[i]),
               "tokens_per_s": m / med * 1e3,
               "block_tflops": bench.flops_per_token(d, inter) * m / (med / 1e3) / 1e12}
        if args.breakdown:
            prof = _native.profile_launches(lambda: run(i), reps=2)
            row["launch_ms"] = {k: round(r["avg_ms"], 4) for k, r in prof.items()}
        out.append(row)
    print(json.dumps({"workload": label, "rounds": args.rounds, "results": out}), flush=True)


if __name__ == "__main__":
    main()
