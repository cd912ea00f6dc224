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
        # names reduced in the current (or, after wait(), the last) step, in order
        self.names: list[str] = []
        self._joined = False

    def _note(self, name: str) -> None:
        if self._joined:           # a new step: keep only this step's names (bounded)
            self.names.clear()
            self._joined = False
        self.names.append(name)

    def __call__(self, name: str, tensor) -> None:
        self._note(name)
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
        self._joined = True
        if self.side is not None:
            import torch

            torch.cuda.current_stream(self.side.device).wait_stream(self.side)
        if self._capped is not None:
            self._capped.__exit__(None, None, None)
            self._capped = None


class WgradReduceScatter(WgradAllReduce):
    """`wgrad_hook` that reduce-scatters the f32 weight gradients and all-gathers bf16.

    The reference rounds a weight gradient once, after the f32 sum
    (engine.py:443-447).  An f32 all-reduce followed by that rounding moves
    2 (P-1)/P x 4 bytes per element through every rank; here each rank sums only
    its 1/P slice in f32 (NCCL reduce-scatter), rounds that slice to bf16 once
    (coda_convert_f32_bf16 on the side stream) and the rounded slices are
    all-gathered: (P-1)/P x (4 + 2) bytes per element, 25 % fewer on the wire, with
    the same single rounding of the same f32 sum.

    Protocol with layer_backward: an unrounded f32 weight gradient of the SIMBF16 path
    is handed over with `reduce_unrounded(name, t)` and its bf16 sum taken back with
    `reduced(name)` after `wait()`.  Everything else — gain vectors, gradients already
    in storage precision (SIM32), shapes whose element count the world size does not
    divide — goes through `hook(name, t)`, which leaves the f32 sum in place (NCCL
    all-reduce on CUDA; on CPU tensors, the gloo tests, a synchronous reduce-scatter +
    all-gather pair).
    """

    def __init__(self, dist, device=None, reserve_sms: int = 0):
        super().__init__(dist, device, f32=True, reserve_sms=reserve_sms)
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self._out: dict = {}

    def _splits(self, tensor) -> bool:
        return (tensor.dim() == 2 and tensor.is_contiguous() and tensor.numel() % self.world == 0
                and tensor.numel() > 0)

    def __call__(self, name: str, tensor) -> None:
        """Sum over ranks in place."""
        import torch

        if self.side is not None or not self._splits(tensor):
            return super().__call__(name, tensor)
        self._note(name)
        flat = tensor.view(-1)
        shard = torch.empty(flat.numel() // self.world, dtype=tensor.dtype)
        self.dist.reduce_scatter_tensor(shard, flat)
        self.dist.all_gather_into_tensor(flat, shard)

    def reduce_unrounded(self, name: str, tensor) -> None:
        """Sum the unrounded f32 gradient over ranks and round it to bf16 once; the result
        is `reduced(name)` after wait() (or, when the slice path does not apply, the sum
        is left in place and `reduced(name)` is None)."""
        import torch

        if self.side is None or tensor.dtype != torch.float32 or not self._splits(tensor):
            return self(name, tensor)
        import ctypes

        from . import _native as nat

        self._note(name)
        self._cap()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(tensor.device))
        rows, cols = tensor.shape
        n = tensor.numel() // self.world
        # the slice as a matrix when whole rows split evenly (vectorised rounding kernel)
        shape = (rows // self.world, cols) if rows % self.world == 0 else (1, n)
        with torch.cuda.stream(self.side):
            self.side.wait_event(ev)
            shard = torch.empty(shape, dtype=torch.float32, device=tensor.device)
            self.dist.reduce_scatter_tensor(shard.view(-1), tensor.view(-1))
            half = torch.empty(shape, dtype=torch.bfloat16, device=tensor.device)
            nat.call("coda_convert_f32_bf16", ctypes.byref(nat.tensor_desc(shard)),
                     ctypes.byref(nat.tensor_desc(half, nat.BF16)), self.side.cuda_stream)
            out = torch.empty((rows, cols), dtype=torch.bfloat16, device=tensor.device)
            self.dist.all_gather_into_tensor(out.view(-1), half.view(-1))
        tensor.record_stream(self.side)
        # `out` belongs to the side stream's pool; the caller's stream reads it after wait()
        out.record_stream(torch.cuda.current_stream(tensor.device))
        self._out[name] = out

    def reduced(self, name: str):
        """The bf16 sum handed over by reduce_unrounded(name), once (None if it was summed in place)."""
        return self._out.pop(name, None)


class PeerWgradReduce(WgradAllReduce):
    """`wgrad_hook` whose weight-gradient GEMMs sum across ranks inside their epilogue.

    Instead of "GEMM, then all-reduce", every rank's launch of a weight gradient
    (coda_gemm_peer_reduce) writes each f32 output tile into the landing buffer of the
    tile's owner rank through peer memory (CUDA IPC, NVLink P2P between GPUs); the last
    rank to deliver a tile sums the partials in rank order, rounds to bf16 once and
    stores the tile into every rank's result — the reduce-scatter and the all-gather ride
    on the GEMM's own epilogue, tile by tile, while the mainloop computes the next tile.
    Bytes per rank on the wire: (P-1)/P of the f32 partial out, (P-1)/P of the bf16 sum
    in, against 2 (P-1)/P of the f32 gradient for a ring all-reduce.

    Gain gradients (vectors) and the folded-gain weight gradients keep the NCCL path of
    WgradAllReduce.  `wait()` ends the step with a cross-rank barrier (an NCCL all-reduce
    of one element, or a host barrier on gloo), after which every rank's results are
    complete and the landing buffers may be reused.  The returned gradients live in
    buffers owned by the hook and are overwritten by its next step.
    """

    def __init__(self, dist, device, reserve_sms: int = 0):
        super().__init__(dist, device, f32=True, reserve_sms=reserve_sms)
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.device = device
        if self.world > 8:
            raise ValueError(f"peer reduction supports up to 8 ranks, got {self.world}")
        self._regions: dict = {}
        self._pending = False

    def _region(self, name: str, m: int, n: int):
        """Landing / counter / result buffers of one weight gradient, mapped on every rank."""
        import torch
        from torch.multiprocessing.reductions import reduce_tensor

        from . import _native as nat
        from .tensors import alloc_matrix

        key = (name, m, n)
        reg = self._regions.get(key)
        if reg is not None:
            return reg
        slot_bytes, ctr_bytes = nat.peer_reduce_sizes(m, n, self.world)
        slots = torch.empty(slot_bytes // 4, dtype=torch.float32, device=self.device)
        ctr = torch.zeros(ctr_bytes // 4, dtype=torch.int32, device=self.device)
        out = alloc_matrix(m, n, torch.bfloat16, self.device)
        torch.cuda.synchronize(self.device)            # zeroed counters before any peer arrives
        mine = [reduce_tensor(t) for t in (slots, ctr, out)]
        gathered = [None] * self.world
        self.dist.all_gather_object(gathered, mine)
        peers = []
        for r, objs in enumerate(gathered):
            peers.append([slots, ctr, out] if r == self.rank else [fn(*args) for fn, args in objs])
        desc = nat.PeerReduce()
        desc.world, desc.rank = self.world, self.rank
        for r, (s, c, o) in enumerate(peers):
            desc.slots[r], desc.counters[r], desc.out[r] = s.data_ptr(), c.data_ptr(), o.data_ptr()
        desc.ld_out = out.stride(0)
        desc.slot_bytes, desc.counter_bytes = slot_bytes, ctr_bytes
        reg = {"desc": desc, "out": out, "keep": peers}
        self._regions[key] = reg
        return reg

    def gemm(self, name: str, a, b, *, precision):
        """dW = a^T b of this rank's token shard, summed over ranks (bf16, complete after wait())."""
        import ctypes

        import torch

        from . import _native as nat
        from .tensors import DenseMatrix

        k, m = a.tensor.shape
        n = b.tensor.shape[1]
        reg = self._region(name, m, n)
        prob = nat.Problem(m, n, k, 1, 0, nat.BF16, nat.BF16, 0, nat.sm_limit(), None, 0)
        stream = torch.cuda.current_stream(a.tensor.device).cuda_stream
        nat.call("coda_gemm_peer_reduce", ctypes.byref(prob), ctypes.byref(nat.tensor_desc(a.tensor)),
                 ctypes.byref(nat.tensor_desc(b.tensor)), ctypes.byref(reg["desc"]), stream,
                 tag=f"gemm_peer_reduce {m}x{n}x{k} TN", flops=2.0 * m * n * k)
        self._note(name)
        self._pending = True
        return DenseMatrix._wrap(reg["out"], precision)

    def wait(self) -> None:
        super().wait()
        if not self._pending:
            return
        import torch

        # every rank's peer-reduce launches have finished -> all results are complete
        if self.dist.get_backend() == "nccl":
            t = torch.zeros(1, device=self.device)
            self.dist.all_reduce(t)
        else:
            torch.cuda.current_stream(self.device).synchronize()
            self.dist.barrier()
        self._pending = False
