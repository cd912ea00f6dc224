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
