"""GPU acceptance gate modelled on the reference's own (tests/test_acceptance.py of tilefuse).

  1. every fused launch vs the oracle on seeded ragged shapes, cycling the
     reference's four tile contexts (its TILES list), both precisions;
  2. traffic records equal the reference ledger byte for byte;
  3. the row-statistic relocation identity <grad, rope(z)> = <rope^T(grad), z>;
  4. blocked LSE: uniform logits give loss = ln V exactly (V = 32768).
"""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import coda_oracle as O

pytestmark = pytest.mark.gpu

# (tile shape, reduction_tile_n) contexts of the reference acceptance test (test_acceptance.py:64-69)
TILES = [((16, 24), 10), ((32, 32), 32), ((8, 24), 4), ((128, 128), 128)]
TOL = {"sim32": 1e-5, "simbf16": 2e-2}


def _cd():
    import paper_2605_19269_b200 as cd

    return cd


@pytest.mark.parametrize("mode", ["sim32", "simbf16"])
@pytest.mark.parametrize("case", range(8))
def test_kernels_random_ragged_vs_oracle(cuda_ready, mode, case):
    cd = _cd()
    rng = np.random.default_rng([7, case, 0 if mode == "sim32" else 1])
    (tm, tn), rtn = TILES[case % len(TILES)]
    m, k = int(rng.integers(4, 300)), int(rng.integers(4, 300))
    n = 2 * int(rng.integers(2, 150))
    P = cd.PrecisionMode.SIM32 if mode == "sim32" else cd.PrecisionMode.SIMBF16
    kw = dict(tile_shape=cd.TileShape(tm, tn), reduction_tile_n=rtn, precision=P)
    q = lambda *s, sc=1.0: O.q(rng.standard_normal(s) * sc, mode)  # noqa: E731
    a, b, bt, z = q(m, k), q(k, n, sc=k ** -0.5), q(n, k, sc=k ** -0.5), q(m, n)
    pre, gin, pre2 = q(m, n), q(m, n), q(m, 2 * n)
    gamma = O.q(1 + 0.1 * rng.standard_normal(n), mode)
    r = O.stat_q(0.5 + rng.random(m), mode)
    s = O.stat_q(0.1 * rng.standard_normal(m), mode)
    cos, sin = (t[:, :n] for t in O.qkv_rope_tables(m, n, mode))
    labels = rng.integers(0, n, m).astype(np.int64)
    M = lambda x: cd.DenseMatrix.from_array(x, P)  # noqa: E731
    V = lambda x, p=P: cd.Vector.from_array(x, p)  # noqa: E731
    S = cd.stat_mode(P)
    tol = TOL[mode]
    errs = {}

    def chk(name, got, want):
        errs[name] = O.rel_error(got, want) if np.linalg.norm(want) else float(np.max(np.abs(got)))

    k1 = cd.gemm_rope(M(a), M(b), M(cos), M(sin), **kw)
    chk("k1", k1.main.data, O.k_rope(a, b, cos, sin, mode)["main"])
    k2 = cd.gemm_swiglu(M(a), M(b), save_preact=True, **kw)
    o2 = O.k_swiglu(a, b, mode, save_preact=True)
    chk("k2", k2.main.data, o2["main"])
    chk("k2_pre", k2.aux["preact"].data, o2["preact"])
    k4 = cd.gemm_residual_partial_rms(M(a), M(b), M(z), V(gamma), **kw)
    o4 = O.k_residual_partial_rms(a, b, z, gamma, mode, tn, rtn)
    chk("k4", k4.main.data, o4["main"])
    chk("k4_sumsq", k4.aux["sumsq"].data, o4["sumsq"][0])
    assert np.array_equal(k4.aux["sumsq"].counts, o4["sumsq"][1])
    chk("k4_r", cd.finalize_rms(k4.aux["sumsq"]).data, O.finalize_rms(o4["sumsq"], 1e-6, mode))
    chk("k6", cd.gemm_rms_swiglu(M(a), M(b), V(r, S), **kw).main.data, O.k_rms_swiglu(a, b, r, mode)["main"])
    chk("k7", cd.gemm_rms_rope(M(a), M(b), V(r, S), M(cos), M(sin), **kw).main.data,
        O.k_rms_rope(a, b, r, cos, sin, mode)["main"])
    k8 = cd.gemm_rms_partial_xent(M(a), M(b), V(r, S), labels, **kw)
    o8 = O.k_partial_xent(a, b, labels, mode, tn, rtn, scale=r)
    chk("k8_target", k8.aux["target"].data, o8["target"])
    chk("k8_lse", cd.combine_lse(k8.aux["lse"]).data, O.combine_lse(o8["lse"], mode))
    k9 = cd.gemm_rmsnorm_backward(M(a), M(bt), M(pre), V(r, S), V(gamma), V(s, S), grad_in=M(gin), trans_b=True,
                                  **kw)
    o9 = O.k_rmsnorm_backward(a, bt, pre, r, gamma, s, mode, grad_in=gin, tile_m=tm, trans_b=True)
    chk("k9", k9.main.data, o9["main"])
    chk("k9_normed", k9.aux["normed"].data, o9["normed"])
    chk("k9_gg", k9.aux["gamma_grad"].data, o9["gamma_grad"][0])
    k10 = cd.gemm_swiglu_backward(M(a), M(bt), M(pre2), trans_b=True, **kw)
    o10 = O.k_swiglu_backward(a, bt, pre2, mode, tn, rtn, trans_b=True)
    chk("k10", k10.main.data, o10["main"])
    chk("k10_rowdot", k10.aux["rowdot"].data, o10["rowdot"][0])
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, (m, k, n, (tm, tn), rtn, bad)


@pytest.mark.parametrize("tag,mode", [("ragged", "sim32"), ("ragged", "simbf16"), ("default", "sim32"),
                                      ("default", "simbf16")])
def test_traffic_records_equal_reference_ledger(cuda_ready, tag, mode):
    cd = _cd()
    g = load_golden(f"kernels_{tag}_{mode}")
    m, k, n, tm, tn, rtn = (int(v) for v in g["meta"])
    P = cd.PrecisionMode.SIM32 if mode == "sim32" else cd.PrecisionMode.SIMBF16
    kw = dict(tile_shape=cd.TileShape(tm, tn), reduction_tile_n=rtn, precision=P)
    M = lambda key: cd.DenseMatrix.from_array(g[key], P)  # noqa: E731
    a, b, bt, z, cos, sin, pre, gin, pre2 = (M(x) for x in ("a", "b", "bt", "z", "cos", "sin", "pre", "gin",
                                                           "preact2"))
    gamma = cd.Vector.from_array(g["gamma"], P)
    r = cd.Vector.from_array(g["r"], cd.stat_mode(P))
    s = cd.Vector.from_array(g["s"], cd.stat_mode(P))
    lab = g["labels"].astype(np.int64)
    recs = [cd.gemm_rope(a, b, cos, sin, **kw).record, cd.gemm_swiglu(a, b, save_preact=True, **kw).record,
            cd.gemm_partial_xent(a, b, lab, store_logits=True, **kw).record,
            cd.gemm_residual_partial_rms(a, b, z, gamma, **kw).record, cd.gemm_row_scale(a, b, r, **kw).record,
            cd.gemm_rms_swiglu(a, b, r, **kw).record, cd.gemm_rms_rope(a, b, r, cos, sin, **kw).record,
            cd.gemm_rms_partial_xent(a, b, r, lab, **kw).record,
            cd.gemm_rmsnorm_backward(a, bt, pre, r, gamma, s, grad_in=gin, trans_b=True, **kw).record,
            cd.gemm_swiglu_backward(a, bt, pre2, trans_b=True, **kw).record]
    got = np.array([[x.read_bytes, x.write_bytes] for x in recs], dtype=np.int64)
    assert np.array_equal(got, g["records"]), (got, g["records"])


def test_statistic_relocation_identity(cuda_ready):
    """rope preserves row dots: rowdot(grad, rope(z)) == rowdot(rope^T(grad), z) (acceptance #3)."""
    cd = _cd()
    rng = np.random.default_rng(3)
    m, n = 96, 384
    P = cd.PrecisionMode.SIM32
    z = O.q(rng.standard_normal((m, n)), O.SIM32)
    grad = O.q(rng.standard_normal((m, n)), O.SIM32)
    cos, sin = (t[:, :n] for t in O.qkv_rope_tables(m, n, O.SIM32))
    rotated = O.q(O.rope(z, cos, sin), O.SIM32)
    M = lambda x: cd.DenseMatrix.from_array(x, P)  # noqa: E731
    gz, rd = cd.rope_backward_stat(M(grad), M(rotated), M(cos), M(sin), precision=P)
    s = cd.finalize_rowdot(rd, n).data
    direct = np.sum(gz.data * z, axis=1) / n
    assert O.rel_error(s, direct) < 1e-5


def test_uniform_logits_give_ln_vocab(cuda_ready):
    """All-zero vocabulary weights: every logit is 0, loss = ln V exactly (acceptance #6, V = 32768)."""
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    m, d, v = 64, 64, 32768
    rng = np.random.default_rng(0)
    a = cd.DenseMatrix.from_array(rng.standard_normal((m, d)), P)
    b = cd.DenseMatrix.from_array(rng.standard_normal((d, d)) * 0.1, P)
    z = cd.DenseMatrix.from_array(rng.standard_normal((m, d)), P)
    gamma = cd.Vector.from_array(np.ones(d), P)
    wv = cd.DenseMatrix.from_array(np.zeros((d, v)), P)
    labels = rng.integers(0, v, m).astype(np.int64)
    res = cd.lm_head_forward(a, b, z, gamma, wv, labels, config=cd.PipelineConfig(hidden=d, precision=P))
    assert abs(res.mean_loss - math.log(v)) / math.log(v) < 1e-6
    assert np.allclose(res.lse.data, np.float32(math.log(v)), rtol=1e-6)


def test_xent_error_paths(cuda_ready):
    """The reference's CE errors survive the single host read: a NaN (unvisited) target
    raises MissingGatherError, a row with no LSE values raises DegenerateError, in the
    reference's order (reductions.py:101-168)."""
    import torch

    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    S = cd.stat_mode(P)
    m = 6
    lse = cd.Vector.from_tensor(torch.zeros(m, device="cuda"), S)
    tgt = torch.zeros(m, device="cuda")
    tgt[3] = float("nan")
    with pytest.raises(cd.MissingGatherError):
        cd.cross_entropy_finalize(cd.Vector.from_tensor(tgt, S), lse)
    bad_lse = torch.zeros(m, device="cuda")
    bad_lse[1] = float("nan")
    with pytest.raises(cd.DegenerateError):
        cd.cross_entropy_finalize(cd.Vector.from_tensor(tgt, S), cd.Vector.from_tensor(bad_lse, S), check_lse=True)
    losses, mean = cd.cross_entropy_finalize(cd.Vector.from_tensor(torch.full((m,), 0.5, device="cuda"), S),
                                             cd.Vector.from_tensor(torch.full((m,), 2.0, device="cuda"), S))
    assert mean == pytest.approx(1.5) and np.allclose(losses.data, 1.5)
