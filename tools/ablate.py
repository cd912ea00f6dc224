"""Per-launch device time of the C4 step under engine-option variants, interleaved.

    python tools/ablate.py --variant ablate=0 --variant ablate=1 --variant ablate=2 --variant ablate=3
(ablate: 1 = skip epilogue side-operand TMA loads, 2 = skip epilogue TMA stores — results
invalid, timing only).
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--variant", action="append", required=True)
    args = ap.parse_args()
    d, inter, m, _ = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    cfg = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=cd.PrecisionMode.SIMBF16)
    weights, acts, cos, sin = bench.make_workload(cd, d, inter, m, 0, dev)
    variants = [{k: int(x) for k, x in (kv.split("=") for kv in v.split(","))} for v in args.variant]
    per = [dict() for _ in variants]

    def setv(i):
        for k, v in variants[i].items():
            _native.set_option(k, v)

    for i in range(len(variants)):
        setv(i)
        for _ in range(2):
            bench.run_step(cd, cfg, weights, acts, cos, sin)
    torch.cuda.synchronize()
    for _ in range(args.rounds):
        for i in range(len(variants)):
            setv(i)
            bench.run_step(cd, cfg, weights, acts, cos, sin)   # settle
            prof = _native.profile_launches(lambda: bench.run_step(cd, cfg, weights, acts, cos, sin), reps=1)
            for tag, r in prof.items():
                per[i].setdefault(tag, []).append(r["avg_ms"])
    tags = list(per[0])
    print(json.dumps({"variants": args.variant}))
    for t in tags:
        print(f"{t[:48]:48s} " + " ".join(f"{statistics.median(per[i][t]):8.3f}" for i in range(len(variants))))
    print(f"{'TOTAL':48s} " + " ".join(f"{sum(statistics.median(v) for v in per[i].values()):8.3f}"
                                         for i in range(len(variants))))


if __name__ == "__main__":
    main()
