"""bench.py's JSON contract on the GPU: one line with every key the driver reads, for the fp32
parity config (fast) and a reduced-token C4 run (the default workload's code path)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline", "cpu_baseline")


def _bench(*args):
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True, timeout=600,
                       cwd=str(ROOT))
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_c1(cuda_ready):
    out = _bench("--config", "c1", "--steps", "3", "--warmup", "3", "--cpu-sample", "128")
    for k in REQUIRED:
        assert k in out, k
    assert out["n_gpus"] == 1 and out["steps"] == 3 and out["warmup"] == 3
    assert out["dtype"] == "f32" and out["higher_is_better"] is True
    assert out["gpu_launches"] > 0 and out["value"] > 0
    assert out["e2e"]["h2d_bytes_per_step"] > 0 and out["e2e"]["d2h_bytes_per_step"] > 0
    assert out["cpu_baseline"]["kind"] == "port" and out["cpu_baseline"]["cores"] >= 1
    assert out["parity"]["rel_err_max"] <= 1e-5


def test_bench_line_c4_reduced(cuda_ready):
    out = _bench("--tokens", "2048", "--steps", "3", "--warmup", "3", "--no-cpu", "--ab-rounds", "2")
    for k in REQUIRED:
        assert k in out, k
    assert out["dtype"] == "bf16" and out["config"]["tokens_per_gpu"] == 2048
    assert out["roofline"]["bound"] == "tensor" and 0 < out["roofline"]["frac"] < 1.5
    assert out["gpu_launches"] == 3 * 15          # 15 kernels per block step (deferred finalizers)
    ab = out["fold_gamma_ab"]
    assert ab["ms_reference_schedule"] > 0 and ab["ms_gamma_folded"] > 0


def test_bench_line_graph_with_collectives(cuda_ready):
    """The N > 1 defaults on one GPU: a one-rank NCCL group, the reduce-scatter / all-gather
    weight-gradient hook and every loop (device-timed and e2e) replayed as CUDA graphs; the
    host enqueue is the graph launch only."""
    out = _bench("--tokens", "2048", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-parity", "--ab-rounds", "0",
                 "--force-dist", "--graph")
    for k in REQUIRED:
        assert k in out, k
    assert out["cuda_graph"] is True and out["e2e"]["cuda_graph"] is True
    assert out["wgrad_reduce"] == "WgradReduceScatter"
    assert out["host_enqueue_ms_per_step"] < 0.5
    assert out["gpu_launches"] > 3 * 15            # the block's kernels plus the slice roundings
    assert out["value"] > 0 and out["e2e"]["value"] > 0
    assert out["weak_scaling"]["cuda_graph"] is True and out["weak_scaling"]["value"] > 0


def test_bench_two_ranks_share_one_gpu(cuda_ready):
    """The multi-rank bench path on a one-GPU box: --gpus 2 spawns two ranks (torchrun,
    127.0.0.1 rendezvous), both on cuda:0 over gloo, token-sharded C4 with the weight-
    gradient hook, max-over-ranks timing, the weak-scaling extra and the e2e loop; rank 0
    prints one line with n_gpus 2 (a functional check, not a measurement)."""
    out = _bench("--gpus", "2", "--share-gpu", "--tokens", "2048", "--steps", "3", "--warmup", "3", "--no-cpu",
                 "--no-parity", "--ab-rounds", "0")
    assert out["n_gpus"] == 2 and out["share_gpu"] is True and out["scaling"] == "strong"
    assert out["config"]["tokens_per_gpu"] == 1024 and out["config"]["global_tokens"] == 2048
    assert out["wgrad_reduce"] == "WgradAllReduce" and out["cuda_graph"] is False
    assert out["value"] > 0 and out["e2e"]["value"] > 0
    assert out["weak_scaling"]["global_tokens"] == 4096 and out["weak_scaling"]["value"] > 0


def test_bench_two_ranks_full_size_dp_parity(cuda_ready):
    """Two token-sharded ranks on one GPU (gloo) run the full C4 fixture batch, 8192 tokens
    each; after the weight-gradient reduction the six reduced gradients match the
    single-GPU full-size oracle fixture (bf16 bar 2e-2)."""
    out = _bench("--gpus", "2", "--share-gpu", "--steps", "3", "--warmup", "3", "--no-cpu", "--ab-rounds", "0")
    pf = out["parity_fullsize"]
    assert pf is not None and pf["outputs"] == 6 and pf["pass"] is True, pf
    assert pf["rel_err_max"] <= 2e-2


def test_bench_force_dist_full_size_parity(cuda_ready):
    """A one-rank NCCL group with the default N > 1 hook (f32 reduce-scatter, bf16 rounding,
    bf16 all-gather): the reduced full-size C4 weight and gain gradients match the oracle
    fixture exactly as well as the plain single-GPU path does."""
    out = _bench("--force-dist", "--steps", "3", "--warmup", "3", "--no-cpu", "--ab-rounds", "0")
    pf = out["parity_fullsize"]
    assert out["wgrad_reduce"] == "WgradReduceScatter"
    assert pf["outputs"] == 6 and pf["pass"] is True and pf["rel_err_max"] <= 3.5e-3, pf
