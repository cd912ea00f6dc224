"""GPU tests of the weight-gradient GEMM with its cross-rank sum fused into the epilogue
(coda_gemm_peer_reduce, parallel.PeerWgradReduce).

World 1 runs in-process against the plain GEMM.  World 2 runs two processes that share
cuda:0 (the test box has one GPU): the landing, counter and result buffers are mapped
into the other process with CUDA IPC, exactly as between two GPUs over NVLink, and the
result must equal bf16(P0 + P1) of the two ranks' f32 partials bit for bit.
"""

import ctypes
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


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns, round to nearest even (the device's cvt.rn)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _tensor_bits(t) -> np.ndarray:
    import torch

    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _local_desc(m, n, world=1, rank=0):
    import torch

    from paper_2605_19269_b200 import _native as nat
    from paper_2605_19269_b200.tensors import alloc_matrix

    sb, cb = nat.peer_reduce_sizes(m, n, world)
    slots = torch.empty(sb // 4, dtype=torch.float32, device="cuda")
    ctr = torch.zeros(cb // 4, dtype=torch.int32, device="cuda")
    out = alloc_matrix(m, n, torch.bfloat16, torch.device("cuda", 0))
    d = nat.PeerReduce()
    d.world, d.rank = world, rank
    d.slots[0], d.counters[0], d.out[0] = slots.data_ptr(), ctr.data_ptr(), out.data_ptr()
    d.ld_out, d.slot_bytes, d.counter_bytes = out.stride(0), sb, cb
    return d, (slots, ctr, out)


def _launch(desc, a, b):
    import torch

    from paper_2605_19269_b200 import _native as nat

    k, m = a.shape
    n = b.shape[1]
    prob = nat.Problem(m, n, k, 1, 0, nat.BF16, nat.BF16, 0, 0, None, 0)
    nat.call("coda_gemm_peer_reduce", ctypes.byref(prob), ctypes.byref(nat.tensor_desc(a)),
             ctypes.byref(nat.tensor_desc(b)), ctypes.byref(desc), torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("shape", [(512, 768, 1024), (300, 520, 200), (1024, 4096, 256)])
def test_world1_equals_plain_gemm(cuda_ready, shape):
    """One rank: the epilogue's dump / arrive / fold / store path gives exactly the plain
    bf16 GEMM (0 + P rounds like P), twice in a row (counters are left zero)."""
    import torch

    import paper_2605_19269_b200 as cd

    m, n, k = shape
    g = torch.Generator(device="cuda").manual_seed(3)
    a = (torch.randn(k, m, device="cuda", generator=g) / 8).to(torch.bfloat16)
    b = (torch.randn(k, n, device="cuda", generator=g) / 8).to(torch.bfloat16)
    P = cd.PrecisionMode.SIMBF16
    A, B = cd.DenseMatrix.from_tensor(a, P), cd.DenseMatrix.from_tensor(b, P)    # 16-B padded rows
    ref = cd.run_gemm(cd.GemmProblem(m=m, n=n, k=k, trans_a=True, precision=P), A, B).main.tensor
    a, b = A.tensor, B.tensor
    desc, (slots, ctr, out) = _local_desc(m, n)
    for _ in range(2):
        out.fill_(0)
        _launch(desc, a, b)
        torch.cuda.synchronize()
        assert np.array_equal(_tensor_bits(out), _tensor_bits(ref))
        assert int(ctr.abs().sum()) == 0


def test_peer_reduce_validation(cuda_ready):
    """Bad descriptors fail before any launch, with the reference error classes."""
    import torch

    import paper_2605_19269_b200 as cd

    m, n, k = 256, 256, 64
    a = torch.zeros(k, m, dtype=torch.bfloat16, device="cuda")
    b = torch.zeros(k, n, dtype=torch.bfloat16, device="cuda")
    desc, keep = _local_desc(m, n)
    desc.world = 2                       # rank 1's buffers are missing
    with pytest.raises(cd.BindingError):
        _launch(desc, a, b)
    desc.world, desc.rank = 1, 1
    with pytest.raises(cd.ConfigError):
        _launch(desc, a, b)
    desc.rank, desc.slot_bytes = 0, 16
    with pytest.raises(cd.BindingError, match="too small"):
        _launch(desc, a, b)


def _worker(rank, world, port, out_dir, shape):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    import paper_2605_19269_b200 as cd
    from paper_2605_19269_b200 import parallel

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, k = shape
    P = cd.PrecisionMode.SIMBF16
    g = torch.Generator(device="cuda").manual_seed(100 + rank)      # this rank's token shard
    a = cd.DenseMatrix.from_tensor((torch.randn(k, m, device="cuda", generator=g) / 8).to(torch.bfloat16), P)
    b = cd.DenseMatrix.from_tensor((torch.randn(k, n, device="cuda", generator=g) / 8).to(torch.bfloat16), P)
    part = cd.run_gemm(cd.GemmProblem(m=m, n=n, k=k, trans_a=True, precision=P), a, b, out_f32=True).main.tensor
    hook = parallel.PeerWgradReduce(dist, torch.device("cuda", 0))
    outs = []
    for step in range(2):                # the second step reuses the landing buffers and counters
        res = hook.gemm("w", a, b, precision=P)
        hook.wait()
        outs.append(res.tensor.clone())
    torch.cuda.synchronize()
    np.savez(Path(out_dir) / f"rank{rank}.npz", part=part.cpu().numpy(),
             out0=outs[0].view(torch.int16).cpu().numpy(), out1=outs[1].view(torch.int16).cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shape", [(512, 1024, 384), (300, 520, 200)])
def test_two_ranks_sum_bitwise(cuda_ready, tmp_path, shape):
    """Two processes on one GPU, buffers shared through CUDA IPC: every rank's result is
    bf16(P0 + P1) of the f32 partials, bit for bit, on both steps and both ranks."""
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), shape), nprocs=world, join=True,
                       start_method="spawn")
    r = [dict(np.load(tmp_path / f"rank{i}.npz")) for i in range(world)]
    want = _bf16_bits(r[0]["part"] + r[1]["part"])       # rank order: (0 + P0) + P1
    for i in range(world):
        for key in ("out0", "out1"):
            got = r[i][key].view(np.uint16)
            assert np.array_equal(got, want), (i, key, int((got != want).sum()))


def _layer_worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    from paper_2605_19269_b200 import parallel

    sys.path.insert(0, str(ROOT / "tests"))
    import test_gpu_parallel as T

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = T._inputs()[0]
    sh = parallel.shard(m, rank, world)
    hook = parallel.PeerWgradReduce(dist, torch.device("cuda", 0))
    grads = T._run(rank, world, slice(sh.start, sh.stop), hook)
    assert set(hook.names) == set(parallel.REDUCED)
    np.savez(Path(out_dir) / f"rank{rank}.npz", **grads)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_block_with_peer_reduce(cuda_ready, tmp_path):
    """The token-sharded block backward with PeerWgradReduce as its wgrad hook equals the
    single-process full batch (same CUDA kernels), and both ranks hold identical weight
    gradients."""
    import torch.multiprocessing as mp

    sys.path.insert(0, str(ROOT / "tests"))
    import test_gpu_parallel as T

    from oracle import coda_oracle as O
    from paper_2605_19269_b200 import parallel

    world = 2
    mp.start_processes(_layer_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    m = T._inputs()[0]
    full = T._run(0, 1, slice(0, m))
    shards = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    for name in parallel.REDUCED:
        assert np.array_equal(shards[0][name], shards[1][name]), name
        err = O.rel_error(shards[0][name], full[name])
        assert err < 1e-2, (name, err)
    for name in parallel.ROW_LOCAL:
        got = np.concatenate([s[name] for s in shards], axis=0)
        assert O.rel_error(got, full[name]) < 1e-2, name
