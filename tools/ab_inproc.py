"""Interleaved in-process A/B of engine options on one benchmark workload.

Alternates the variants step by step (same GPU, same thermal / power state) and
reports the median device time per variant:

    python tools/ab_inproc.py --config c4 --rounds 12 --variant cg=2 --variant cg=1
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

import bench  # noqa: E402
import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import _native  # noqa: E402


def parse(v: str) -> dict:
    return {k: int(x) for k, x in (kv.split("=") for kv in v.split(","))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=tuple(bench.CONFIGS))
    ap.add_argument("--rounds", type=int, default=12)
    ap.add_argument("--variant", action="append", required=True, help="e.g. cg=2,pdl=1")
    ap.add_argument("--tokens", type=int, default=0, help="override the config's token count (per-rank shape proxies)")
    args = ap.parse_args()
    d, inter, m, label = bench.CONFIGS[args.config]
    if args.tokens:
        m, label = args.tokens, f"{label} at {args.tokens} tokens"
    dev = torch.device("cuda", 0)
    cfg = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=cd.PrecisionMode.SIMBF16)
    weights, acts, cos, sin = bench.make_workload(cd, d, inter, m, 0, dev, blocks=bench.BLOCKS.get(args.config, 1))
    variants = [parse(v) for v in args.variant]
    times = {i: [] for i in range(len(variants))}

    def run(i):
        for k, v in variants[i].items():
            _native.set_option(k, v)
        bench.run_step(cd, cfg, weights, acts, cos, sin)

    for i in range(len(variants)):   # warm every variant (kernel attributes, caches)
        for _ in range(3):
            run(i)
    torch.cuda.synchronize()
    nv = len(variants)
    for rnd in range(args.rounds):
        for i in [(rnd + j) % nv for j in range(nv)]:     # rotated order
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            run(i)          # untimed lead step: the timed one starts behind queued device work
            e0.record()
            run(i)
            e1.record()
            torch.cuda.synchronize()
            times[i].append(e0.elapsed_time(e1))
    out = []
    for i, v in enumerate(variants):
        med = statistics.median(times[i])
        out.append({"variant": v, "median_ms": med, "tokens_per_s": m / med * 1e3, "min_ms": min(times[i])})
    print(json.dumps({"workload": label, "rounds": args.rounds, "results": out}), flush=True)


if __name__ == "__main__":
    main()
