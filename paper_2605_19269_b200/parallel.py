"""Token-sharded data parallelism for the fused block.

Every epilogue statistic of the block is per token (row): sum-of-squares ->
inverse RMS, relocated row dots -> s, RoPE angles by absolute position.  So
rows shard across ranks with NO communication in the forward and in the
row-local backward; the only cross-token sums are the weight gradients and
the two gain gradients (reference kernels.py:936-1001, 946, 980), which are
all-reduced (sum) once per block.  Rank p owns rows [start, stop) and builds
its RoPE tables with `start` as the position offset (kernels.py:161, 175).

Parity choice: weight gradients are produced unrounded in float32
(`layer_backward(..., wgrad_hook=...)` -> out_f32), reduced, and rounded to
bf16 once afterwards — the same single rounding as the reference's store
(engine.py:443-447).
"""

from __future__ import annotations

from dataclasses import dataclass

# gradients summed over token shards; everything else is row-local
REDUCED = ("w_qkv", "gamma_qkv", "w_down", "w_gate_up", "gamma_ffn", "w_out")
ROW_LOCAL = ("x", "z")


@dataclass(frozen=True)
class TokenShard:
    rank: int
    world: int
    start: int
    stop: int

    @property
    def rows(self) -> int:
        return self.stop - self.start


def shard(tokens: int, rank: int, world: int, scaling: str = "strong") -> TokenShard:
    """Rows owned by `rank`.

    strong: `tokens` is the global count, split contiguously (remainder to the
    low ranks); weak: every rank owns `tokens` rows of a world*tokens job.
    """
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    if scaling == "weak":
        return TokenShard(rank, world, rank * tokens, (rank + 1) * tokens)
    base, rem = divmod(tokens, world)
    start = rank * base + min(rank, rem)
    return TokenShard(rank, world, start, start + base + (1 if rank < rem else 0))


class WgradAllReduce:
    """`wgrad_hook` for layer_backward: all-reduce(sum) each gradient as soon as it exists.

    On CUDA tensors the collective runs on a side stream that waits for the
    producing launch, so NCCL over NVLink overlaps the remaining backward
    GEMMs; `wait()` joins it back before the step's results are used.  On CPU
    tensors (gloo, tests) it is a plain synchronous all_reduce.
    """

    def __init__(self, dist, device=None, f32: bool = True, reserve_sms: int = 0):
        self.dist = dist
        # while a reduction is in flight the persistent GEMMs this thread enqueues use
        # num_sms - reserve_sms SMs, so the collective on the side stream has SMs of its own
        # (the first weight gradient arrives a quarter into the backward: the launches before
        # it, and the next step's forward after wait(), run on every SM)
        self.reserve_sms = int(reserve_sms)
        self._capped = None
        # f32: layer_backward hands over unrounded float32 weight gradients and rounds the
        # reduced sums once (the reference's single rounding); False: bf16 gradients are
        # reduced as stored (half the bytes on the wire, one rounding per partial)
        self.f32 = f32
        self.side = None
        if device is not None and getattr(device, "type", None) == "cuda":
            import torch

            self.side = torch.cuda.Stream(device)
        self.names: list[str] = []

    def __call__(self, name: str, tensor) -> None:
        self.names.append(name)
        if self.side is None:
            self.dist.all_reduce(tensor)
            return
        import torch

        self._cap()

        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(tensor.device))
        with torch.cuda.stream(self.side):
            self.side.wait_event(ev)
            self.dist.all_reduce(tensor)
        tensor.record_stream(self.side)

    def _cap(self) -> None:
        """First reduction in flight: cap this thread's GEMM launches until wait()."""
        from . import _native

        if self.reserve_sms > 0 and self._capped is None:
            self._capped = _native.limit_sms(max(1, _native.num_sms() - self.reserve_sms))
            self._capped.__enter__()

    def wait(self) -> None:
        if self.side is not None:
            import torch

            torch.cuda.current_stream(self.side.device).wait_stream(self.side)
        if self._capped is not None:
            self._capped.__exit__(None, None, None)
            self._capped = None
