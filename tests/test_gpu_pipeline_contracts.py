"""Pipeline contracts on the GPU, mirroring the reference's tests/test_kernels.py:
the K4 contract (gains in main, scale deferred), the deferred scale completing the
norm through K5, validation errors (rope_backward_stat shapes, weights, tape), the
backward without a residual gradient, and outputs on the storage grid."""

import dataclasses

import numpy as np
import pytest

from oracle import coda_oracle as O

pytestmark = pytest.mark.gpu


def _cd():
    import paper_2605_19269_b200 as cd

    return cd




def _mk(cd, rng, r, c, P):
    return cd.DenseMatrix.from_array(rng.standard_normal((r, c)), P)


def test_residual_partial_rms_contract_and_deferred_scale(cuda_ready):
    cd = _cd()
    P = cd.PrecisionMode.SIM32
    rng = np.random.default_rng(1)
    a, b, z = _mk(cd, rng, 6, 4, P), _mk(cd, rng, 4, 10, P), _mk(cd, rng, 6, 10, P)
    gamma = cd.Vector.from_array(1 + 0.1 * rng.standard_normal(10), P)
    k4 = cd.gemm_residual_partial_rms(a, b, z, gamma, precision=P)
    pre = a.data @ b.data + z.data
    assert O.rel_error(k4.main.data, pre * gamma.data) <= 1e-6          # main carries the gains
    assert O.rel_error(k4.aux["pre_norm"].data, pre) <= 1e-6
    assert np.allclose(k4.aux["sumsq"].data.sum(axis=1), np.sum(pre * pre, axis=1), rtol=1e-5)
    w1 = _mk(cd, rng, 10, 5, P)
    r = cd.finalize_rms(k4.aux["sumsq"], 1e-6)
    k5 = cd.gemm_row_scale(k4.main, w1, r, precision=P)
    normed = pre / np.sqrt(np.mean(pre * pre, axis=1, keepdims=True) + 1e-6) * gamma.data
    assert O.rel_error(k5.main.data, normed @ w1.data) <= 1e-5       # the scale completes the norm


def test_rope_backward_stat_validates_shapes(cuda_ready):
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(2)
    grad = _mk(cd, rng, 4, 6, P)
    cos, sin = cd.rope_tables(4, 6, precision=P)
    with pytest.raises(cd.DimensionError):
        cd.rope_backward_stat(grad, _mk(cd, rng, 4, 8, P), cos, sin, precision=P)


def _build(cd, seed, P):
    rng = np.random.default_rng(seed)
    cfg = cd.PipelineConfig(hidden=8, ffn=16, precision=P)
    w = cd.LayerWeights.random(rng, cfg)
    x, z = _mk(cd, rng, 6, 8, P), _mk(cd, rng, 6, 8, P)
    cos, sin = cd.qkv_rope_tables(6, 8, precision=P)
    return rng, cfg, w, x, z, cos, sin


def test_weights_and_tape_are_validated(cuda_ready):
    cd = _cd()
    P = cd.PrecisionMode.SIM32
    rng, c, w, x, z, cos, sin = _build(cd, 5, P)
    with pytest.raises(cd.DimensionError):
        cd.layer_forward(x, z, dataclasses.replace(w, w_down=w.w_gate_up), cos, sin, config=c)
    fwd = cd.layer_forward(x, z, w, cos, sin, config=c)
    gq = _mk(cd, rng, 6, 24, P)
    with pytest.raises(cd.TapeError):
        cd.layer_backward(gq, dataclasses.replace(fwd.tape, preact=fwd.tape.pre_norm_a), w, config=c)


def test_backward_without_residual_grad(cuda_ready):
    cd = _cd()
    P = cd.PrecisionMode.SIM32
    rng, c, w, x, z, cos, sin = _build(cd, 2, P)
    fwd = cd.layer_forward(x, z, w, cos, sin, config=c)
    gq = _mk(cd, rng, 6, 24, P)
    bwd = cd.layer_backward(gq, fwd.tape, w, config=c)
    wd = {k: getattr(w, k).data for k in ("w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv", "w_qkv")}
    ref = O.layer_ref_forward(x.data, z.data, wd, cos.data, sin.data)
    want = O.layer_ref_backward(gq.data, None, ref, x.data, wd, cos.data, sin.data)
    for k in O.GRAD_KEYS:
        assert O.rel_error(getattr(bwd, k).data, want[k]) <= 1e-5, k
    assert bwd.ledger.launches == 13


def test_reduced_precision_outputs_live_on_grid(cuda_ready):
    cd = _cd()
    for P, om in ((cd.PrecisionMode.SIM32, O.SIM32), (cd.PrecisionMode.SIMBF16, O.SIMBF16)):
        _, c, w, x, z, cos, sin = _build(cd, 7, P)
        got = cd.layer_forward(x, z, w, cos, sin, config=c)
        assert got.qkv.precision is P
        assert np.array_equal(O.q(got.qkv.data, om), got.qkv.data)
