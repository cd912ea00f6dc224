"""GPU tests of the pipelines and B200 extensions added in round 2.

* pipeline_grrg_forward / pipeline_grrg_canonical (reference kernels.py:635-713,
  tests/test_kernels.py:298-325): oracle parity, fused == canonical, three launches;
* interleave_gate_up / split_gate_up (kernels.py:209-236);
* gamma folded into W (north_star): fold_gains, the wgrad gain epilogue, the folded
  layer forward/backward against the unfolded fused-order oracle;
* SM-limited launches (room for a concurrent collective) are bit-identical;
* split-K inside CUDA-graph capture: a stream without its own workspace runs unsplit,
  a prepared capture stream reproduces the eager split bits;
* the wave-tail split completes with far fewer SMs than clusters (no co-residency).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import coda_oracle as O

pytestmark = pytest.mark.gpu

WKEYS = ("w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv", "w_qkv")


def _cd():
    import paper_2605_19269_b200 as cd

    return cd


def _mode(P):
    cd = _cd()
    return O.SIM32 if P is cd.PrecisionMode.SIM32 else O.SIMBF16


# ----------------------------------------------------------------------------- GRRG


def _grrg_inputs(P, seed, m=300, k=200, d=384, n=260):
    cd = _cd()
    rng = np.random.default_rng(seed)
    M = lambda *s: cd.DenseMatrix.from_array(rng.standard_normal(s) * 0.3, P)  # noqa: E731
    x, w0, z = M(m, k), M(k, d), M(m, d)
    gamma = cd.Vector.from_array(1 + 0.1 * rng.standard_normal(d), P)
    w1 = M(d, n)
    return x, w0, z, gamma, w1, cd.PipelineConfig(hidden=d, precision=P)


@pytest.mark.parametrize("prec", ["SIMBF16", "SIM32"])
def test_grrg_forward_matches_oracle_in_three_launches(cuda_ready, prec):
    import torch

    cd = _cd()
    from paper_2605_19269_b200 import _native

    P = getattr(cd.PrecisionMode, prec)
    x, w0, z, gamma, w1, cfg = _grrg_inputs(P, 0)
    c0 = _native.launch_count()
    got = cd.pipeline_grrg_forward(x, w0, z, gamma, w1, config=cfg)
    launches = _native.launch_count() - c0
    torch.cuda.synchronize()
    mode = _mode(P)
    ref = O.grrg_forward(x.data, w0.data, z.data, gamma.data, w1.data, mode)
    tol = 1e-5 if P is cd.PrecisionMode.SIM32 else 2e-2
    for key, g, r in (("y", got.y.data, ref["y"]), ("pre_norm", got.pre_norm.data, ref["pre_norm"]),
                      ("normed", got.normed.data, ref["normed"]), ("inv_rms", got.inv_rms.data, ref["inv_rms"])):
        assert O.rel_error(g, r) <= tol, (key, O.rel_error(g, r))
    # the reference pins three launches (tests/test_kernels.py:322-325): the ledger keeps that
    # logical count; on the device the finalize runs inside K5's epilogue, so SIMBF16 enqueues
    # two kernels (SIM32 adds operand splits and K-chunk passes)
    assert got.ledger.launches == 3
    if P is cd.PrecisionMode.SIMBF16:
        assert launches == 2


@pytest.mark.parametrize("prec", ["SIMBF16", "SIM32"])
def test_grrg_fused_matches_canonical(cuda_ready, prec):
    cd = _cd()
    P = getattr(cd.PrecisionMode, prec)
    x, w0, z, gamma, w1, cfg = _grrg_inputs(P, 1)
    fused = cd.pipeline_grrg_forward(x, w0, z, gamma, w1, config=cfg)
    canon, ledger = cd.pipeline_grrg_canonical(x, w0, z, gamma, w1, config=cfg)
    tol = 1e-5 if P is cd.PrecisionMode.SIM32 else 2e-2
    assert O.rel_error(fused.y.data, canon.data) <= tol
    assert ledger.launches == 4          # GEMM, residual add, rmsnorm, GEMM
    assert fused.ledger.total_bytes < ledger.total_bytes


# ----------------------------------------------------------------------------- gate/up layout


def test_interleave_and_split_gate_up(cuda_ready):
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(2)
    g, u = (cd.DenseMatrix.from_array(rng.standard_normal((96, 40)), P) for _ in range(2))
    w = cd.interleave_gate_up(g, u)
    assert w.shape == (96, 80)
    ref = np.empty((96, 80))
    ref[:, 0::2], ref[:, 1::2] = g.data, u.data
    assert np.array_equal(w.data, ref)
    g2, u2 = cd.split_gate_up(w)
    assert np.array_equal(g2.data, g.data) and np.array_equal(u2.data, u.data)
    with pytest.raises(cd.DimensionError):
        cd.interleave_gate_up(g, cd.DenseMatrix.from_array(rng.standard_normal((96, 42)), P))
    with pytest.raises(cd.DimensionError):
        cd.split_gate_up(cd.DenseMatrix.from_array(rng.standard_normal((8, 7)), P))
    # SwiGLU over the interleaved weight == silu(x g) * (x u)
    x = cd.DenseMatrix.from_array(rng.standard_normal((128, 96)) * 0.2, P)
    act = cd.gemm_swiglu(x, w, precision=P).main.data
    gx, ux = O.gemm(x.data, g.data, O.SIMBF16), O.gemm(x.data, u.data, O.SIMBF16)
    assert O.rel_error(act, gx * O.sigmoid(gx) * ux) <= 2e-2


# ----------------------------------------------------------------------------- gamma folding


def test_scale_rows_bit_exact(cuda_ready):
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(4)
    for shape in ((256, 1024), (130, 264), (3, 17)):
        w = cd.DenseMatrix.from_array(rng.standard_normal(shape), P)
        g = cd.Vector.from_array(1 + 0.1 * rng.standard_normal(shape[0]), P)
        got = cd.scale_rows(w, g).data
        want = O.bf16_round((g.data[:, None] * w.data).astype(np.float32))
        assert np.array_equal(got, want), shape


def test_wgrad_gain_epilogue_vs_oracle(cuda_ready):
    """dW = diag(gain) a^T b and dgain = rowsum(W * a^T b), one launch (+ finalize)."""
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(6)
    k, d, n = 640, 256, 768
    M = lambda *s: cd.DenseMatrix.from_array(rng.standard_normal(s) * 0.3, P)  # noqa: E731
    a, b, w = M(k, d), M(k, n), M(d, n)
    gain = cd.Vector.from_array(1 + 0.1 * rng.standard_normal(d), P)
    res = cd.gemm_wgrad_gain(a, b, w, gain, precision=P)
    dgain = cd.finalize_rowdot(res.aux["gain_dot"], 1)
    t = O.gemm(a.data, b.data, O.SIMBF16, trans_a=True)
    assert O.rel_error(res.main.data, O.q(t * gain.data[:, None], O.SIMBF16)) <= 1e-3   # bf16 1-ulp flips
    assert O.rel_error(dgain.data, (t.astype(np.float64) * w.data).sum(axis=1)) <= 1e-5


def _layer_case(P, m=384, d=256, ffn=1024, seed=8):
    cd = _cd()
    rng = np.random.default_rng(seed)
    mode = _mode(P)
    w = O.random_layer(rng, d, ffn, mode)
    x, z = (O.q(rng.standard_normal((m, d)), mode) for _ in range(2))
    cos, sin = O.qkv_rope_tables(m, d, mode)
    gq = O.q(rng.standard_normal((m, 3 * d)), mode)
    gr = O.q(rng.standard_normal((m, d)), mode)
    Mx = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
    Vx = lambda a: cd.Vector.from_array(a, P)  # noqa: E731
    weights = cd.LayerWeights(w_out=Mx(w["w_out"]), gamma_ffn=Vx(w["gamma_ffn"]), w_gate_up=Mx(w["w_gate_up"]),
                              w_down=Mx(w["w_down"]), gamma_qkv=Vx(w["gamma_qkv"]), w_qkv=Mx(w["w_qkv"]))
    of = O.layer_forward(x, z, w, cos, sin, mode)
    ob = O.layer_backward(gq, of, w, mode, grad_residual=gr)
    return dict(w=weights, x=Mx(x), z=Mx(z), cos=cd.qkv_rope_tables(m, d, precision=P)[0], gq=Mx(gq), gr=Mx(gr),
                of=of, ob=ob, d=d, ffn=ffn, m=m)


def _run_layer(case, cfg, hook=None):
    cd = _cd()
    cos, sin = cd.qkv_rope_tables(case["m"], case["d"], precision=cfg.precision)
    fwd = cd.layer_forward(case["x"], case["z"], case["w"], cos, sin, config=cfg)
    bwd = cd.layer_backward(case["gq"], fwd.tape, case["w"], grad_residual=case["gr"], config=cfg, wgrad_hook=hook)
    return fwd, bwd


@pytest.mark.parametrize("shape", [(384, 256, 1024), (300, 192, 640)])
def test_folded_layer_vs_oracle(cuda_ready, shape):
    """The gain-folded block (K4 without RowVecMul / gained store, folded K6/K7/K9, wgrad gain
    epilogue) matches the reference's unfolded fused-order algorithm within the bf16 bar
    (aligned shape: specialised kernels; ragged shape: generic interpreter for the gain epilogue)."""
    import torch

    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    m, d, ffn = shape
    case = _layer_case(P, m=m, d=d, ffn=ffn)
    cfg = cd.PipelineConfig(hidden=case["d"], ffn=case["ffn"], precision=P, fold_gamma=True)
    fwd, bwd = _run_layer(case, cfg)
    torch.cuda.synchronize()
    errs = {"qkv": O.rel_error(fwd.qkv.data, case["of"]["qkv"]),
            "residual": O.rel_error(fwd.residual.data, case["of"]["residual"])}
    errs.update({k: O.rel_error(getattr(bwd, k).data, case["ob"][k]) for k in O.GRAD_KEYS})
    print("folded vs oracle:", {k: f"{v:.2e}" for k, v in errs.items()})
    assert max(errs.values()) <= 2e-2, errs
    # the folded forward stores no gained copy: the K4 launches keep pre_norm only
    assert fwd.tape.folded is not None
    assert fwd.ledger.write_bytes < _run_layer(case, cd.PipelineConfig(hidden=case["d"], ffn=case["ffn"],
                                                                        precision=P))[0].ledger.write_bytes


def test_folded_backward_needs_folded_tape(cuda_ready):
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    case = _layer_case(P, m=128)
    plain = cd.PipelineConfig(hidden=case["d"], ffn=case["ffn"], precision=P)
    folded = cd.PipelineConfig(hidden=case["d"], ffn=case["ffn"], precision=P, fold_gamma=True)
    cos, sin = cd.qkv_rope_tables(case["m"], case["d"], precision=P)
    fwd = cd.layer_forward(case["x"], case["z"], case["w"], cos, sin, config=plain)
    with pytest.raises(cd.TapeError):
        cd.layer_backward(case["gq"], fwd.tape, case["w"], config=folded)


# ----------------------------------------------------------------------------- SM limit / split-K


def test_sm_limited_launches_bit_identical(cuda_ready):
    """Capping the persistent grid (SMs left for a concurrent collective) changes the schedule,
    never the bits of an unsplit launch (K below the wave-tail split threshold).  Split-K
    launches may split differently under a cap, which changes only the f32 accumulation order:
    they are compared within tolerance."""
    import torch

    cd = _cd()
    from paper_2605_19269_b200 import _native

    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(9)
    M = lambda *s: cd.DenseMatrix.from_array(rng.standard_normal(s) / 64, P)  # noqa: E731
    a, b = M(4096, 1024), M(4096, 2304)        # wgrad-shaped: (1024 x 2304) tiles, K = 4096
    prob = cd.GemmProblem(m=1024, n=2304, k=4096, trans_a=True, precision=P)
    a2, b2 = M(8192, 1024), M(8192, 2304)      # K = 8192: split tail when uncapped
    prob2 = cd.GemmProblem(m=1024, n=2304, k=8192, trans_a=True, precision=P)
    ref2 = cd.run_gemm(prob2, a2, b2).main.data
    for cap in (132, 64, 8):
        with _native.limit_sms(cap):
            got2 = cd.run_gemm(prob2, a2, b2).main.data
        assert O.rel_error(got2, ref2) <= 1e-2, cap
    case = _layer_case(P, m=512)
    cfg = cd.PipelineConfig(hidden=case["d"], ffn=case["ffn"], precision=P)

    def run():
        out = [cd.run_gemm(prob, a, b).main.data]
        fwd, bwd = _run_layer(case, cfg)
        out += [fwd.qkv.data] + [getattr(bwd, k).data for k in O.GRAD_KEYS]
        torch.cuda.synchronize()
        return out

    ref = run()
    for cap in (132, 64, 8):
        with _native.limit_sms(cap):
            got = run()
        for i, (x, y) in enumerate(zip(ref, got)):
            assert np.array_equal(x, y), (cap, i)


def test_split_tail_without_coresidency(cuda_ready):
    """A split tail whose pieces outnumber the SMs of the launch still completes: pieces never
    wait for one another (the last arrival folds), so a 2-SM grid finishes a 9-wave launch."""
    import torch

    cd = _cd()
    from paper_2605_19269_b200 import _native

    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(10)
    a = cd.DenseMatrix.from_array(rng.standard_normal((1280, 8192)) / 64, P)
    b = cd.DenseMatrix.from_array(rng.standard_normal((8192, 512)) / 64, P)
    prob = cd.GemmProblem(m=1280, n=512, k=8192, precision=P)
    ref = O.q(O.gemm(a.data, b.data, O.SIMBF16), O.SIMBF16)
    for cap in (2, 6, 10):
        with _native.limit_sms(cap):
            got = cd.run_gemm(prob, a, b).main
        torch.cuda.synchronize()
        assert O.rel_error(got.data, ref) <= 1e-2, cap


def test_graph_capture_workspace(cuda_ready):
    """Capturing on a stream without its own workspace runs unsplit (never borrows another
    stream's counters); a prepared capture stream reproduces the eager split bits."""
    import torch

    cd = _cd()
    from paper_2605_19269_b200 import _native

    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(11)
    a = cd.DenseMatrix.from_array(rng.standard_normal((8192, 1024)) / 64, P)
    b = cd.DenseMatrix.from_array(rng.standard_normal((8192, 2304)) / 64, P)
    prob = cd.GemmProblem(m=1024, n=2304, k=8192, trans_a=True, precision=P)
    eager = cd.run_gemm(prob, a, b).main.data
    dev = torch.device("cuda", 0)
    for prepared in (False, True):
        s = torch.cuda.Stream(dev)
        if prepared:
            _native.prepare_stream_workspace(dev, s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            out = cd.run_gemm(prob, a, b)
        for _ in range(3):
            g.replay()
            cd.run_gemm(prob, a, b)     # eager launches on the default stream in between
        torch.cuda.synchronize()
        got = out.main.data
        if prepared:
            assert np.array_equal(got, eager)
        else:
            assert O.rel_error(got, eager) <= 1e-2


# ----------------------------------------------------------------------------- deferred finalizers


@pytest.mark.parametrize("shape", [(384, 256, 1024), (300, 192, 640)])
@pytest.mark.parametrize("prec", ["SIMBF16", "SIM32"])
def test_deferred_finalizers_bit_identical(cuda_ready, prec, shape):
    """finalize_rms / finalize_rowdot folded into the consuming GEMM epilogues (VERDICT r01
    next #6) give the same bits as their standalone kernels, including the tape's r vectors,
    and the SIMBF16 block runs in 15 launches instead of 19."""
    import torch

    cd = _cd()
    from paper_2605_19269_b200 import _native, reductions

    P = getattr(cd.PrecisionMode, prec)
    m, d, ffn = shape
    case = _layer_case(P, m=m, d=d, ffn=ffn)
    cfg = cd.PipelineConfig(hidden=case["d"], ffn=case["ffn"], precision=P)

    def run():
        c0 = _native.launch_count()
        fwd, bwd = _run_layer(case, cfg)
        n = _native.launch_count() - c0
        torch.cuda.synchronize()
        out = [fwd.qkv.data, fwd.residual.data, fwd.tape.inv_rms_a.data, fwd.tape.inv_rms_b.data]
        return out + [getattr(bwd, k).data for k in O.GRAD_KEYS], n

    deferred, n_def = run()
    with reductions.eager_finalizers():
        eager, n_eager = run()
    for i, (x, y) in enumerate(zip(deferred, eager)):
        assert np.array_equal(x, y), i
    assert n_eager - n_def == 4
    if P is cd.PrecisionMode.SIMBF16 and shape == (384, 256, 1024):
        assert (n_eager, n_def) == (19, 15)


def test_pending_finalizer_materializes_on_read(cuda_ready):
    """A finalizer result read before (or without) any consuming launch runs its own kernel."""
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(12)
    a = cd.DenseMatrix.from_array(rng.standard_normal((200, 96)), P)
    b = cd.DenseMatrix.from_array(rng.standard_normal((96, 300)) * 0.1, P)
    z = cd.DenseMatrix.from_array(rng.standard_normal((200, 300)), P)
    g = cd.Vector.from_array(np.ones(300), P)
    k4 = cd.gemm_residual_partial_rms(a, b, z, g, precision=P)
    r = cd.finalize_rms(k4.aux["sumsq"])
    assert r._pending is not None
    want = O.finalize_rms((k4.aux["sumsq"].data, k4.aux["sumsq"].counts), 1e-6, O.SIMBF16)
    assert np.array_equal(r.data, want)
    assert r._pending is None
    # consumed by a RowScale launch: the launch writes the vector, no standalone kernel
    r2 = cd.finalize_rms(k4.aux["sumsq"])
    y = cd.gemm_row_scale(k4.main, cd.DenseMatrix.from_array(rng.standard_normal((300, 64)), P), r2, precision=P)
    assert r2._pending is None
    assert np.array_equal(r2.data, want)
    assert y.main.shape == (200, 64)


def test_rope_backward_stat_deep_path(cuda_ready):
    """The deep-load boundary kernel (compact tables, n % 6144 == 0) matches the oracle and is
    bit-identical to the full-table kernel on the same values."""
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    m, d = 301, 2048
    rng = np.random.default_rng(13)
    cos_c, sin_c = cd.qkv_rope_tables(m, d, start=5, precision=P)
    assert cd.kernels.rope_compact_of(cos_c, sin_c) is not None
    cos_f, sin_f = cd.DenseMatrix.from_tensor(cos_c.tensor, P), cd.DenseMatrix.from_tensor(sin_c.tensor, P)
    g = cd.DenseMatrix.from_array(rng.standard_normal((m, 3 * d)), P)
    r = cd.DenseMatrix.from_array(rng.standard_normal((m, 3 * d)), P)
    gz_b, rd_b = cd.rope_backward_stat(g, r, cos_c, sin_c, precision=P)
    gz_f, rd_f = cd.rope_backward_stat(g, r, cos_f, sin_f, precision=P)
    assert np.array_equal(gz_b.data, gz_f.data)
    assert np.array_equal(rd_b.data, rd_f.data)
    ogz, (ord_, cnt) = O.rope_backward_stat(g.data, r.data, cos_f.data, sin_f.data, O.SIMBF16)
    assert O.rel_error(gz_b.data, ogz) <= 1e-3
    assert O.rel_error(rd_b.data, ord_) <= 1e-5
    assert list(rd_b.counts) == list(cnt)


@pytest.mark.parametrize("fold", [False, True])
def test_step_leaves_no_deferred_work(cuda_ready, fold):
    """Every statistic a layer step returns has been computed inside the step: no pending
    finalizer survives in the tape or the gradients (a deferred finalizer nobody consumes would
    otherwise run outside a timed region, or never)."""
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    case = _layer_case(P, m=256)
    cfg = cd.PipelineConfig(hidden=case["d"], ffn=case["ffn"], precision=P, fold_gamma=fold)
    fwd, bwd = _run_layer(case, cfg)
    vecs = [fwd.tape.inv_rms_a, fwd.tape.inv_rms_b, bwd.gamma_ffn, bwd.gamma_qkv]
    assert all(getattr(v, "_pending", None) is None for v in vecs)
