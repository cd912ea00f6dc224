"""bench.py contract pieces that need no GPU: the algorithmic flop counts behind
roofline.achieved / block_tflops and the token sharding used by
the multi-GPU launch."""

import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2605_19269_b200 import parallel  # noqa: E402


@pytest.mark.parametrize("cfg,mflops", [("c1", 6.29), ("c3", 402.65), ("c4", 1459.6), ("c5", 1459.6)])
def test_flops_per_token_matches_baseline(cfg, mflops):
    d, inter, _, _ = bench.CONFIGS[cfg]
    assert bench.flops_per_token(d, inter) / 1e6 == pytest.approx(mflops, rel=2e-3)


def test_c4_block_total_flops():
    d, inter, m, _ = bench.CONFIGS["c4"]
    assert bench.flops_per_token(d, inter) * m / 1e12 == pytest.approx(23.914, rel=1e-3)


def test_gqa_flops_use_the_packed_width():
    d, inter = 4096, 14336
    full, gqa = bench.flops_per_token(d, inter), bench.flops_per_token(d, inter, kv=1024)
    # only the qkv projection shrinks: Q = d + 2 kv instead of 3d
    assert full - gqa == pytest.approx(3 * 2 * d * (3 * d - (d + 2 * 1024)))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_strong_and_weak_sharding_cover_the_job(world):
    tokens = 16384
    strong = [parallel.shard(tokens, r, world, "strong") for r in range(world)]
    assert strong[0].start == 0 and strong[-1].stop == tokens
    assert all(a.stop == b.start for a, b in zip(strong, strong[1:]))
    weak = [parallel.shard(tokens, r, world, "weak") for r in range(world)]
    assert all(s.rows == tokens for s in weak) and weak[-1].stop == world * tokens


def _run_bench(*args, timeout=240):
    import subprocess

    root = Path(__file__).resolve().parents[1]
    return subprocess.run([sys.executable, str(root / "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=str(root))


def test_launcher_spawns_ranks_gloo():
    """`bench.py --gpus 2` without a torchrun environment launches 2 ranks itself (gloo on CPU
    here): one JSON line from rank 0 with n_gpus 2, strong sharding of the config's tokens, and
    the block's weight gradients all-reduced in production order."""
    import json

    p = _run_bench("--gpus", "2", "--launcher-check", "--config", "c1", "--steps", "2", "--warmup", "3")
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["launcher_check"] is True
    assert out["scaling"] == "strong"
    assert out["config"]["global_tokens"] == 128 and out["config"]["tokens_per_rank"] == 64
    assert out["names"] == ["w_qkv", "gamma_qkv", "w_down", "w_gate_up", "gamma_ffn", "w_out"]
    d, inter = 256, 1024
    assert out["allreduce_bytes_per_step"] == 4 * (d * 3 * d + d + inter * d + d * 2 * inter + d + d * d)


def test_launcher_fails_loudly_without_enough_gpus():
    import torch

    if torch.cuda.device_count() >= 8:
        pytest.skip("enough GPUs for --gpus 8")
    p = _run_bench("--gpus", "8", "--steps", "2", "--warmup", "3", timeout=120)
    assert p.returncode == 2
    assert "CUDA device" in p.stderr
