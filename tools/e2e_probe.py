"""Why is e2e slower than the device step?  Times, alternately:
  device   — the C4 step on device-resident inputs;
  h2d_bg   — the same step with an independent 805 MB H2D copy per step running beside it;
  d2h_bg   — the same step with an independent 134 MB D2H copy per step beside it.
"""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19269_b200 as cd  # noqa: E402


def main():
    d, inter, m, _ = bench.CONFIGS["c4"]
    dev = torch.device("cuda", 0)
    cfg = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=cd.PrecisionMode.SIMBF16)
    weights, acts, cos, sin = bench.make_workload(cd, d, inter, m, 0, dev)
    nbytes = sum(v.tensor.numel() * v.tensor.element_size() for v in acts.values())
    hsrc = torch.empty(nbytes // 2, dtype=torch.bfloat16).pin_memory()
    ddst = torch.empty(nbytes // 2, dtype=torch.bfloat16, device=dev)
    dsrc = torch.empty(m * d, dtype=torch.bfloat16, device=dev)
    hdst = torch.empty(m * d, dtype=torch.bfloat16).pin_memory()
    side = torch.cuda.Stream(dev)
    stream = torch.cuda.current_stream()
    steps = 10

    def run(kind):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            if kind == "h2d_bg":
                with torch.cuda.stream(side):
                    ddst.copy_(hsrc, non_blocking=True)
            elif kind == "d2h_bg":
                with torch.cuda.stream(side):
                    hdst.copy_(dsrc, non_blocking=True)
            bench.run_step(cd, cfg, weights, acts, cos, sin)
        e1.record(stream)
        stream.wait_stream(side)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    # the bench's e2e loop, with a timeline of events per step
    host = [{k: (v.tensor * (1.0 + 0.01 * j)).to(v.tensor.dtype).cpu().pin_memory() for k, v in acts.items()}
            for j in range(2)]
    dev_in = [{k: torch.empty_like(v.tensor) for k, v in acts.items()} for _ in range(2)]
    h2d_stream, d2h_stream = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    out_host = [torch.empty((m, d), dtype=torch.bfloat16).pin_memory() for _ in range(2)]

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def e2e(nsteps):
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        marks = []

        def issue_copy(s):
            b = s % 2
            with torch.cuda.stream(h2d_stream):
                if s >= 2:
                    h2d_stream.wait_event(consumed[b])
                c0 = ev()
                c0.record(h2d_stream)
                for k in host[b]:
                    dev_in[b][k].copy_(host[b][k], non_blocking=True)
                c1 = ev()
                c1.record(h2d_stream)
                copied[b].record(h2d_stream)
                marks.append(("copy", s, c0, c1))

        t0 = ev()
        t0.record(stream)
        h2d_stream.wait_stream(stream)
        issue_copy(0)
        for s in range(nsteps):
            b = s % 2
            if s + 1 < nsteps:
                issue_copy(s + 1)
            stream.wait_event(copied[b])
            s0 = ev()
            s0.record(stream)
            a = {k: cd.DenseMatrix.from_tensor(dev_in[b][k], cd.PrecisionMode.SIMBF16) for k in dev_in[b]}
            _, bwd = bench.run_step(cd, cfg, weights, a, cos, sin)
            s1 = ev()
            s1.record(stream)
            consumed[b].record(stream)
            marks.append(("step", s, s0, s1))
            with torch.cuda.stream(d2h_stream):
                d2h_stream.wait_event(consumed[b])
                out_host[b].copy_(bwd.x.tensor, non_blocking=True)
                bwd.x.tensor.record_stream(d2h_stream)
        stream.wait_stream(d2h_stream)
        stream.wait_stream(h2d_stream)
        t1 = ev()
        t1.record(stream)
        torch.cuda.synchronize()
        print("e2e total ms/step", round(t0.elapsed_time(t1) / nsteps, 3))
        for kind, s, a0, a1 in sorted(marks, key=lambda x: t0.elapsed_time(x[2])):
            print(f"  {kind:5s} {s:2d}  {t0.elapsed_time(a0):8.2f} -> {t0.elapsed_time(a1):8.2f}")

    e2e(2)
    e2e(8)

    kinds = ("device", "h2d_bg", "d2h_bg")
    for k in kinds:
        run(k)
    res = {k: [] for k in kinds}
    for _ in range(3):
        for k in kinds:
            res[k].append(run(k))
    print(json.dumps({k: round(statistics.median(v), 3) for k, v in res.items()}))


if __name__ == "__main__":
    main()
