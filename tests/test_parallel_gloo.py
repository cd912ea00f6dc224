"""World-size-2 gloo test of the token-sharded data-parallel decomposition.

Each rank runs the block on its row shard (RoPE tables offset by the shard's
first position), all-reduces the weight/gain gradients with the same
`WgradAllReduce` hook object the GPU path uses, and must reproduce the
single-process full-batch gradients.  The per-rank compute here is the CPU
oracle (the GPU box runs the same decomposition with CUDA kernels + NCCL).
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    from oracle import coda_oracle as O

    m, d, ffn = 64, 32, 96
    rng = np.random.default_rng(7)
    mode = O.SIM32
    w = O.random_layer(rng, d, ffn, mode)
    x, z = (O.q(rng.standard_normal((m, d)), mode) for _ in range(2))
    gq = O.q(rng.standard_normal((m, 3 * d)), mode)
    gr = O.q(rng.standard_normal((m, d)), mode)
    return m, d, w, x, z, gq, gr, mode


def _worker(rank, world, port, out_dir, scaling, kind="allreduce"):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    from oracle import coda_oracle as O
    from paper_2605_19269_b200 import parallel

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, d, w, x, z, gq, gr, mode = _problem()
    tokens = m if scaling == "strong" else m // world
    sh = parallel.shard(tokens, rank, world, scaling)
    sl = slice(sh.start, sh.stop)
    cos, sin = O.qkv_rope_tables(sh.rows, d, O.EXACT64, start=sh.start)
    fwd = O.layer_ref_forward(x[sl], z[sl], w, cos, sin)
    bwd = O.layer_ref_backward(gq[sl], gr[sl], fwd, x[sl], w, cos, sin)
    hook = parallel.WgradReduceScatter(dist) if kind == "rsag" else parallel.WgradAllReduce(dist)
    for name in parallel.REDUCED:
        t = torch.from_numpy(np.ascontiguousarray(bwd[name]))
        hook(name, t)
        bwd[name] = t.numpy()
    hook.wait()
    np.savez(Path(out_dir) / f"rank{rank}.npz", start=sh.start, stop=sh.stop, **bwd, qkv=fwd["qkv"])
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling,kind", [("strong", "allreduce"), ("weak", "allreduce"), ("strong", "rsag")])
def test_token_sharded_grads_match_full_batch(tmp_path, scaling, kind):
    """kind "rsag": WgradReduceScatter — reduce-scatter + all-gather in place of the all-reduce."""
    import torch.multiprocessing as mp

    from oracle import coda_oracle as O
    from paper_2605_19269_b200 import parallel

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), scaling, kind), nprocs=world, join=True,
                       start_method="spawn")
    m, d, w, x, z, gq, gr, mode = _problem()
    cos, sin = O.qkv_rope_tables(m, d, O.EXACT64)
    fwd = O.layer_ref_forward(x, z, w, cos, sin)
    full = O.layer_ref_backward(gq, gr, fwd, x, w, cos, sin)
    shards = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    assert [int(s["start"]) for s in shards] == [0, m // 2]
    for name in parallel.REDUCED:
        for s in shards:
            assert O.rel_error(s[name], full[name]) < 1e-12, name
    for name in parallel.ROW_LOCAL:
        got = np.concatenate([s[name] for s in shards], axis=0)
        assert O.rel_error(got, full[name]) < 1e-12, name
    qkv = np.concatenate([s["qkv"] for s in shards], axis=0)
    assert O.rel_error(qkv, fwd["qkv"]) < 1e-12


def test_shard_bounds():
    from paper_2605_19269_b200 import parallel

    assert [(s.start, s.stop) for s in (parallel.shard(10, r, 3) for r in range(3))] == [(0, 4), (4, 7), (7, 10)]
    assert parallel.shard(16384, 3, 8).rows == 2048
    assert parallel.shard(8192, 2, 8, "weak").start == 16384


def test_layer_backward_waits_for_async_reduction_before_rounding():
    """layer_backward must call hook.wait() before rounding the reduced f32 wgrads (no stream race)."""
    import inspect

    from paper_2605_19269_b200 import kernels

    src = inspect.getsource(kernels.layer_backward)
    assert src.index("wait()") < src.index("to_storage(g, prec)")


def test_hook_caps_sms_only_while_reductions_are_in_flight():
    """WgradAllReduce(reserve_sms=k): from the first reduction until wait(), this thread's GEMM
    launches are capped at num_sms - k (room for the NCCL kernels on the side stream); before
    the first weight gradient and after wait() they use every SM.  Exercised with a stand-in
    side stream and collective (no GPU)."""
    sys.path.insert(0, str(ROOT))
    from paper_2605_19269_b200 import _native, parallel

    class FakeDist:
        def __init__(self):
            self.calls = []

        def all_reduce(self, t):
            self.calls.append(t)

    hook = parallel.WgradAllReduce(FakeDist(), None, reserve_sms=8)
    orig_num_sms = _native.num_sms
    try:
        _native.num_sms = lambda: 148
        assert _native.sm_limit() == 0
        hook._cap()                     # what the first reduction does on the CUDA path
        assert _native.sm_limit() == 140
        hook._cap()                     # later reductions keep the same cap
        assert _native.sm_limit() == 140
        hook.wait()
        assert _native.sm_limit() == 0 and hook._capped is None
        none = parallel.WgradAllReduce(FakeDist(), None)
        none._cap()
        assert _native.sm_limit() == 0
    finally:
        _native.num_sms = orig_num_sms


def test_reduce_scatter_hook_protocol():
    """WgradReduceScatter: `hook(name, t)` always leaves the sum in place (gains, SIM32
    storage-precision gradients); `reduce_unrounded` is the only entry that may hand the
    result back through `reduced()` instead, and without a CUDA side stream it also sums in
    place (reduced() is None).  layer_backward uses reduce_unrounded only for the unrounded
    f32 partials of the SIMBF16 path."""
    import inspect

    import torch

    sys.path.insert(0, str(ROOT))
    from paper_2605_19269_b200 import kernels, parallel

    class OneRank:
        def get_world_size(self):
            return 1

        def get_rank(self):
            return 0

        def reduce_scatter_tensor(self, out, inp):
            out.copy_(inp * 2)           # stand-in "sum" of two identical ranks

        def all_gather_into_tensor(self, out, inp):
            out.copy_(inp)

        def all_reduce(self, t):
            t.mul_(2)

    hook = parallel.WgradReduceScatter(OneRank())
    t = torch.ones(4, 6)
    hook("w_out", t)
    assert torch.equal(t, torch.full((4, 6), 2.0)) and hook.reduced("w_out") is None
    v = torch.ones(5)
    hook("gamma_ffn", v)                 # vectors: all-reduce in place
    assert torch.equal(v, torch.full((5,), 2.0))
    u = torch.ones(4, 6)
    hook.reduce_unrounded("w_qkv", u)    # no side stream: in place
    assert torch.equal(u, torch.full((4, 6), 2.0)) and hook.reduced("w_qkv") is None
    src = inspect.getsource(kernels.layer_backward)
    assert 'getattr(wgrad_hook, "reduce_unrounded", None) if f32 else None' in src


def test_hook_names_are_per_step():
    """A long run must not grow the hook's name list: after wait() the next reduction
    starts a new step's list."""
    import torch

    sys.path.insert(0, str(ROOT))
    from paper_2605_19269_b200 import parallel

    class FakeDist:
        def all_reduce(self, t):
            pass

    hook = parallel.WgradAllReduce(FakeDist())
    for step in range(3):
        for name in parallel.REDUCED:
            hook(name, torch.zeros(2))
        hook.wait()
        assert hook.names == list(parallel.REDUCED), step
