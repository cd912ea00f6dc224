"""Finalizers on the GPU, mirroring the reference's tests/test_reductions.py behaviours:
direct formulas, blocking invariance across the reference's tile contexts, the eps
floor, empty-coverage / wrong-kind / bad-width rejections, LSE shift stability and
empty-block handling, column-sum reduction, CE length and unvisited-row errors.
SIM32 values: identity GEMMs make the epilogue see the inputs exactly."""

import math

import numpy as np
import pytest

from paper_2605_19269_b200.epilogue import StoreKind

pytestmark = pytest.mark.gpu


def _cd():
    import paper_2605_19269_b200 as cd

    return cd


def _slot(values, prim, tile=(4, 4), rtn=4, **bind):
    cd = _cd()
    P = cd.PrecisionMode.SIM32
    m, n = values.shape
    a = cd.DenseMatrix.from_array(values, P)
    b = cd.DenseMatrix.from_array(np.eye(n), P)
    p = cd.GemmProblem(m=m, n=n, k=n, tile_shape=cd.TileShape(*tile), reduction_tile_n=rtn, precision=P)
    return cd.run_gemm(p, a, b, cd.EpilogueProgram(prim), bind, store_main=False)


def _lse_ref(x):
    mx = x.max(axis=1, keepdims=True)
    return (mx + np.log(np.exp(x - mx).sum(axis=1, keepdims=True)))[:, 0]


def test_finalize_rms_formula_blocking_and_eps(cuda_ready):
    cd = _cd()
    rng = np.random.default_rng(0)
    x = rng.standard_normal((6, 10)).astype(np.float32).astype(np.float64)
    r = cd.finalize_rms(_slot(x, [cd.PartialSumSq()]).aux["sumsq"], eps=1e-6)
    assert np.allclose(r.data, 1.0 / np.sqrt(np.mean(x * x, axis=1) + 1e-6), rtol=1e-6)
    x = rng.standard_normal((5, 24)).astype(np.float32).astype(np.float64)
    outs = [cd.finalize_rms(_slot(x, [cd.PartialSumSq()], tile=t, rtn=q).aux["sumsq"]).data
            for t, q in (((4, 4), 4), ((4, 24), 24), ((4, 8), 3), ((4, 5), 2))]
    for o in outs[1:]:
        assert np.allclose(o, outs[0], rtol=1e-6)
    z = cd.finalize_rms(_slot(np.zeros((3, 8)), [cd.PartialSumSq()]).aux["sumsq"], eps=1e-6)
    assert np.allclose(z.data, 1.0 / math.sqrt(1e-6), rtol=1e-6)


def test_finalize_rejections(cuda_ready):
    import torch

    cd = _cd()
    P = cd.PrecisionMode.SIM32
    empty = cd.PartialSlot(StoreKind.ROW_SUM, torch.zeros((2, 1), device="cuda"), np.array([0]), P)
    with pytest.raises(cd.DegenerateError):
        cd.finalize_rms(empty)
    lse = _slot(np.zeros((2, 4)), [cd.OnlineLse()]).aux["lse"]
    with pytest.raises(cd.ConfigError):
        cd.finalize_rms(lse)
    with pytest.raises(cd.ConfigError):
        cd.finalize_rowdot(_slot(np.ones((2, 4)), [cd.PartialSumSq()]).aux["sumsq"], d=0)
    with pytest.raises(cd.ConfigError):
        cd.reduce_row_partials(_slot(np.ones((2, 4)), [cd.PartialSumSq()]).aux["sumsq"])


def test_finalize_rowdot_divides_by_declared_width(cuda_ready):
    import torch

    cd = _cd()
    rng = np.random.default_rng(3)
    x, w = rng.standard_normal((4, 10)), rng.standard_normal((4, 10))
    data = torch.tensor((x * w).reshape(4, 5, 2).sum(axis=2), dtype=torch.float32, device="cuda")
    slot = cd.PartialSlot(StoreKind.ROW_SUM, data, np.full(5, 2), cd.PrecisionMode.SIM32)
    s = cd.finalize_rowdot(slot, d=16)
    assert np.allclose(s.data, np.sum(x * w, axis=1) / 16, rtol=1e-5)


def test_combine_lse_formula_blocking_shifts(cuda_ready):
    cd = _cd()
    rng = np.random.default_rng(4)
    x = (rng.standard_normal((6, 13)) * 3).astype(np.float32).astype(np.float64)
    got = cd.combine_lse(_slot(x, [cd.OnlineLse()], rtn=3).aux["lse"])
    assert np.allclose(got.data, _lse_ref(x), rtol=1e-6)
    x = rng.standard_normal((4, 32)).astype(np.float32).astype(np.float64)
    base = cd.combine_lse(_slot(x, [cd.OnlineLse()], tile=(4, 32), rtn=32).aux["lse"]).data
    for t, q in (((4, 4), 4), ((4, 16), 5), ((4, 32), 1)):
        assert np.allclose(cd.combine_lse(_slot(x, [cd.OnlineLse()], tile=t, rtn=q).aux["lse"]).data, base,
                           rtol=1e-6)
    x = np.array([[1000.0, -1000.0, 999.0, 998.0]])
    got = cd.combine_lse(_slot(x, [cd.OnlineLse()], rtn=1).aux["lse"])
    assert np.all(np.isfinite(got.data)) and np.allclose(got.data, _lse_ref(x), rtol=1e-6)


def test_combine_lse_empty_blocks_and_rows(cuda_ready):
    import torch

    cd = _cd()
    P = cd.PrecisionMode.SIM32
    data = np.full((2, 3, 2), -np.inf)
    data[..., 1] = 0.0
    data[:, 1, 0] = [2.0, 5.0]        # one real block, two never-written ones
    data[:, 1, 1] = 1.0
    slot = cd.PartialSlot(StoreKind.ROW_PAIR, torch.tensor(data, dtype=torch.float32, device="cuda"),
                          np.array([4, 4, 4]), P)
    assert np.allclose(cd.combine_lse(slot).data, [2.0, 5.0], atol=1e-6)
    data = np.full((2, 2, 2), -np.inf)
    data[..., 1] = 0.0
    data[0, 0, 0], data[0, 0, 1] = 1.0, 1.0
    slot = cd.PartialSlot(StoreKind.ROW_PAIR, torch.tensor(data, dtype=torch.float32, device="cuda"),
                          np.array([2, 2]), P)
    with pytest.raises(cd.DegenerateError):
        cd.combine_lse(slot)


def test_reduce_row_partials_sums_tile_rows(cuda_ready):
    cd = _cd()
    rng = np.random.default_rng(6)
    x = rng.standard_normal((10, 6)).astype(np.float32).astype(np.float64)
    out = cd.reduce_row_partials(_slot(x, [cd.PartialColSum()]).aux["colsum"])
    assert np.allclose(out.data, x.sum(axis=0), atol=1e-5)


def test_cross_entropy_finalize_matches_and_rejects(cuda_ready):
    import torch

    cd = _cd()
    rng = np.random.default_rng(7)
    logits = (rng.standard_normal((5, 12)) * 2).astype(np.float32).astype(np.float64)
    labels = rng.integers(0, 12, size=5)
    res = _slot(logits, [cd.OnlineLse(), cd.TargetGather()], labels=labels)
    losses, mean = cd.cross_entropy_finalize(res.aux["target"], cd.combine_lse(res.aux["lse"]))
    want = _lse_ref(logits) - logits[np.arange(5), labels]
    assert np.allclose(losses.data, want, rtol=1e-5, atol=1e-6)
    assert mean == pytest.approx(float(want.mean()), rel=1e-5)
    S = cd.PrecisionMode.SIM32
    with pytest.raises(cd.DimensionError):
        cd.cross_entropy_finalize(cd.Vector.from_tensor(torch.ones(2, device="cuda"), S),
                                  cd.Vector.from_tensor(torch.ones(1, device="cuda"), S))
