"""GPU test of the token-sharded data-parallel backward (parallel.WgradAllReduce).

Two processes share cuda:0 and a gloo process group (NCCL needs one GPU per
rank; the box running the tests has one).  Each rank runs the fused CUDA block
on its half of the tokens with `layer_backward(wgrad_hook=WgradAllReduce)`:
f32 weight gradients are all-reduced on a side stream as soon as they exist and
rounded to bf16 once.  The reduced gradients must match the single-process
full-batch run (same CUDA kernels) and the float64 oracle.
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(prec="SIMBF16"):
    sys.path.insert(0, str(ROOT))
    from oracle import coda_oracle as O

    m, d, ffn = 256, 128, 512
    rng = np.random.default_rng(21)
    mode = getattr(O, prec)
    w = O.random_layer(rng, d, ffn, mode, scale=0.1)
    x, z = (O.q(rng.standard_normal((m, d)), mode) for _ in range(2))
    gq = O.q(rng.standard_normal((m, 3 * d)), mode)
    gr = O.q(rng.standard_normal((m, d)), mode)
    return m, d, ffn, w, x, z, gq, gr


def _run(rank, world, sl, hook=None, fold=False, prec="SIMBF16"):
    import paper_2605_19269_b200 as cd

    m, d, ffn, w, x, z, gq, gr = _inputs(prec)
    P = getattr(cd.PrecisionMode, prec)
    M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
    weights = cd.LayerWeights(w_out=M(w["w_out"]), gamma_ffn=cd.Vector.from_array(w["gamma_ffn"], P),
                              w_gate_up=M(w["w_gate_up"]), w_down=M(w["w_down"]),
                              gamma_qkv=cd.Vector.from_array(w["gamma_qkv"], P), w_qkv=M(w["w_qkv"]))
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, precision=P, fold_gamma=fold)
    rows = sl.stop - sl.start
    cos, sin = cd.qkv_rope_tables(rows, d, start=sl.start, precision=P)
    fwd = cd.layer_forward(M(x[sl]), M(z[sl]), weights, cos, sin, config=cfg)
    bwd = cd.layer_backward(M(gq[sl]), fwd.tape, weights, grad_residual=M(gr[sl]), config=cfg, wgrad_hook=hook)
    if hook is not None:
        hook.wait()
    import torch

    torch.cuda.synchronize()
    return {k: getattr(bwd, k).data for k in ("x", "z", "w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv",
                                              "w_qkv")}


def _worker(rank, world, port, out_dir, reserve=0, fold=False, kind="allreduce", prec="SIMBF16"):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    from paper_2605_19269_b200 import parallel

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = _inputs()[0]
    sh = parallel.shard(m, rank, world)
    dev = torch.device("cuda", 0)
    hook = (parallel.WgradReduceScatter(dist, dev, reserve_sms=reserve) if kind == "rsag"
            else parallel.WgradAllReduce(dist, dev, reserve_sms=reserve))
    grads = _run(rank, world, slice(sh.start, sh.stop), hook, fold=fold, prec=prec)
    from paper_2605_19269_b200 import _native

    assert _native.sm_limit() == 0                   # the cap ends with wait()
    assert set(hook.names) == set(parallel.REDUCED)
    if kind == "rsag" and prec == "SIMBF16":
        # the same f32 sums rounded once: bit-identical to the all-reduce path (P = 2 sums commute)
        ar = _run(rank, world, slice(sh.start, sh.stop), parallel.WgradAllReduce(dist, dev), fold=fold)
        grads.update({"ar_" + k: v for k, v in ar.items()})
    np.savez(Path(out_dir) / f"rank{rank}.npz", **grads)
    dist.destroy_process_group()


@pytest.mark.parametrize("reserve,fold,kind", [(0, False, "allreduce"), (8, False, "allreduce"), (8, True, "allreduce"),
                                               (8, False, "rsag"), (0, True, "rsag")])
def test_sharded_fused_backward_matches_full_batch(cuda_ready, tmp_path, reserve, fold, kind):
    """reserve > 0: the hook caps the GEMMs' SMs while the all-reduce is in flight; fold: the
    gain-folded block, whose gain gradients come from the weight-gradient epilogue and are
    all-reduced like the weights; kind "rsag": WgradReduceScatter (f32 reduce-scatter, bf16
    rounding of each rank's slice, bf16 all-gather)."""
    import torch.multiprocessing as mp

    from oracle import coda_oracle as O
    from paper_2605_19269_b200 import parallel

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), reserve, fold, kind), nprocs=world,
                       join=True,
                       start_method="spawn")
    m = _inputs()[0]
    full = _run(0, 1, slice(0, m), fold=fold)
    shards = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    for name in parallel.REDUCED:
        for s in shards:
            err = O.rel_error(s[name], full[name])
            assert err < 1e-2, (name, err)        # bf16 rounding of two half sums vs one full sum
    for name in parallel.ROW_LOCAL:
        got = np.concatenate([s[name] for s in shards], axis=0)
        assert O.rel_error(got, full[name]) < 1e-2, name
    if kind == "rsag":
        for name in parallel.REDUCED:
            for s in shards:
                assert np.array_equal(s[name], s["ar_" + name]), name


def test_reduce_scatter_hook_sim32(cuda_ready, tmp_path):
    """SIM32 (f32 storage): the weight gradients reach WgradReduceScatter in storage
    precision, so they are summed in place (never rounded to bf16)."""
    import torch.multiprocessing as mp

    from oracle import coda_oracle as O
    from paper_2605_19269_b200 import parallel

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), 0, False, "rsag", "SIM32"), nprocs=world,
                       join=True, start_method="spawn")
    m = _inputs("SIM32")[0]
    full = _run(0, 1, slice(0, m), prec="SIM32")
    shards = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    for name in parallel.REDUCED:
        for s in shards:
            err = O.rel_error(s[name], full[name])
            assert err < 1e-5, (name, err)       # f32 sums of two halves vs one full sum
