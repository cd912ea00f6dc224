"""Host-side cost of the data-parallel step (world-1 NCCL group on one GPU).

Runs the C4 block step with each wgrad hook and reports, per step, the host time
spent enqueueing and a cProfile of where it goes (collective calls, stream/event
bookkeeping, kernel launches).  A step whose host enqueue exceeds its device time
starves the GPU, which is what a multi-GPU strong-scaled step (2.2 ms of device work
per rank at P = 8) cannot afford.

    python tools/dist_host_probe.py [--hook rsag|allreduce|none] [--steps 10]
"""

import argparse
import cProfile
import io
import os
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hook", default="rsag", choices=("rsag", "allreduce", "none"))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--reserve", type=int, default=8)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import paper_2605_19269_b200 as cd
    from paper_2605_19269_b200 import parallel

    device = torch.device("cuda", 0)
    torch.cuda.set_device(device)
    hook = None
    if args.hook != "none":
        os.environ.setdefault("NCCL_MAX_CTAS", str(max(1, args.reserve)))
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", device_id=device, rank=0, world_size=1)
        cls = parallel.WgradReduceScatter if args.hook == "rsag" else parallel.WgradAllReduce
        hook = cls(dist, device, reserve_sms=args.reserve)
    d, inter, _, _ = bench.CONFIGS["c4"]
    cfg = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=cd.PrecisionMode.SIMBF16)
    weights, acts, cos, sin = bench.make_workload(cd, d, inter, args.tokens, 0, device)

    def step():
        bench.run_step(cd, cfg, weights, acts, cos, sin, hook)
        if hook is not None:
            hook.wait()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per = []
    e0.record(s)
    prof = cProfile.Profile()
    for _ in range(args.steps):
        t = time.perf_counter()
        prof.enable()
        step()
        prof.disable()
        per.append((time.perf_counter() - t) * 1e3)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"hook={args.hook} tokens={args.tokens}: device {e0.elapsed_time(e1) / args.steps:.2f} ms/step, "
          f"host enqueue per step {['%.2f' % x for x in per]} ms")
    out = io.StringIO()
    pstats.Stats(prof, stream=out).sort_stats("tottime").print_stats(18)
    print(out.getvalue())
    if hook is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
