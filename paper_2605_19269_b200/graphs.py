"""Whole-step CUDA graphs for the fused block (B200 extension; the reference has no device).

An eager block step is 15 kernel launches enqueued from Python through the C-ABI
(~1.3 ms of host time per step), plus ~0.2 ms per torch.distributed call when a
weight-gradient hook reduces across ranks.  At the per-rank shapes of a strong-scaled
job (2048 tokens of LLaMA-3-8B per GPU: ~2.3 ms of device work) the host would be
the bottleneck.  `StepGraph` captures one call of a step function — its launches,
the hook's collectives on their side stream and the join — and replays it with one
host call.

Static-buffer contract (the usual CUDA-graph one): the captured launches read and
write the exact tensors they saw at capture.  Refill the input tensors in place
(`tensor.copy_(...)`) between replays; the outputs returned by the captured call are
overwritten by every replay.  The split-K workspace of the capture stream is
allocated before capture (`_native.prepare_stream_workspace`), so the graph never
shares split counters with eager launches on other streams.
"""

from __future__ import annotations

from typing import Any, Callable

from . import _native


class StepGraph:
    """Capture `fn()` once as a CUDA graph; `replay()` re-runs all of its device work.

    `warmup` eager calls run first (on the capture stream) so lazy initialisation —
    NCCL communicators, allocator pools, tensor maps — happens outside capture.
    """

    def __init__(self, fn: Callable[[], Any], device=None, warmup: int = 1):
        import torch

        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.stream = torch.cuda.Stream(self.device)
        _native.prepare_stream_workspace(self.device, self.stream)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        torch.cuda.synchronize(self.device)
        self.graph = torch.cuda.CUDAGraph()
        c0 = _native.launch_count()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self.outputs = fn()
        # CODA kernels per replay (collectives and copies of the step not counted)
        self.launches = _native.launch_count() - c0

    def replay(self) -> Any:
        """Enqueue the captured step on the current stream; returns the captured outputs."""
        self.graph.replay()
        return self.outputs


def capture_step(fn: Callable[[], Any], device=None, warmup: int = 1) -> StepGraph:
    """StepGraph(fn, device, warmup)."""
    return StepGraph(fn, device=device, warmup=warmup)


__all__ = ["StepGraph", "capture_step"]
