"""GPU parity of the fused layer forward + backward (§8 rows a29-a31).

  * golden: reference engine outputs (tilefuse, SIM32 / SIMBF16) on stored inputs;
  * C1 tiny fp32 config (M=128, d=256, I=1024): every gradient vs the float64
    canonical oracle at <= 1e-5 relative, and vs the fused-order oracle;
  * bf16 at a mid size vs the fused-order oracle at <= 2e-2.
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import coda_oracle as O

pytestmark = pytest.mark.gpu

WKEYS = ("w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv", "w_qkv")


def _cd():
    import paper_2605_19269_b200 as cd

    return cd


def _run_layer(cd, P, cfg, x, z, w, cos, sin, gq, gr):
    M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
    weights = cd.LayerWeights(w_out=M(w["w_out"]), gamma_ffn=cd.Vector.from_array(w["gamma_ffn"], P),
                              w_gate_up=M(w["w_gate_up"]), w_down=M(w["w_down"]),
                              gamma_qkv=cd.Vector.from_array(w["gamma_qkv"], P), w_qkv=M(w["w_qkv"]))
    fwd = cd.layer_forward(M(x), M(z), weights, M(cos), M(sin), config=cfg)
    bwd = cd.layer_backward(M(gq), fwd.tape, weights, grad_residual=M(gr), config=cfg)
    return fwd, bwd


@pytest.mark.parametrize("tag", ["tiny", "ragged"])
@pytest.mark.parametrize("mode", ["sim32", "simbf16"])
def test_layer_vs_reference_golden(cuda_ready, tag, mode):
    cd = _cd()
    g = load_golden(f"layer_{tag}_{mode}")
    m, d, ffn, tm, tn, rtn = (int(v) for v in g["meta"])
    P = {"sim32": cd.PrecisionMode.SIM32, "simbf16": cd.PrecisionMode.SIMBF16}[mode]
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, tile_m=tm, tile_n=tn, reduction_tile_n=rtn, precision=P)
    w = {k: g[k] for k in WKEYS}
    fwd, bwd = _run_layer(cd, P, cfg, g["x"], g["z"], w, g["cos"], g["sin"], g["grad_qkv"], g["grad_residual"])
    tol = 1e-5 if mode == "sim32" else 2e-2
    errs = {"qkv": O.rel_error(fwd.qkv.data, g["qkv"]), "residual": O.rel_error(fwd.residual.data, g["residual"])}
    for key in O.GRAD_KEYS:
        errs[key] = O.rel_error(getattr(bwd, key).data, g[f"g_{key}"])
    print(f"\n[{tag}/{mode}] vs reference engine: " + ", ".join(f"{k}={v:.2e}" for k, v in errs.items()))
    assert max(errs.values()) <= tol, errs
    # and vs the float64 canonical chain
    ref = {"qkv": O.rel_error(fwd.qkv.data, g["ref_qkv"])}
    for key in O.GRAD_KEYS:
        ref[key] = O.rel_error(getattr(bwd, key).data, g[f"ref_g_{key}"])
    assert max(ref.values()) <= tol, ref


def test_c1_tiny_fp32_vs_float64_oracle(cuda_ready):
    """BASELINE config 0: d=256, ffn(I)=1024 (F=2048), 128 tokens, fp32 path <= 1e-5."""
    cd = _cd()
    m, d, ffn = 128, 256, 2048
    rng = np.random.default_rng(0)
    w = O.random_layer(rng, d, ffn, O.SIM32)
    x = O.q(rng.standard_normal((m, d)), O.SIM32)
    z = O.q(rng.standard_normal((m, d)), O.SIM32)
    cos, sin = O.qkv_rope_tables(m, d, O.SIM32)
    gq = O.q(rng.standard_normal((m, 3 * d)), O.SIM32)
    gr = O.q(rng.standard_normal((m, d)), O.SIM32)
    P = cd.PrecisionMode.SIM32
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, precision=P)
    fwd, bwd = _run_layer(cd, P, cfg, x, z, w, cos, sin, gq, gr)
    ref = O.layer_ref_forward(x, z, w, cos, sin)
    refb = O.layer_ref_backward(gq, gr, ref, x, w, cos, sin)
    errs = {"qkv": O.rel_error(fwd.qkv.data, ref["qkv"]), "residual": O.rel_error(fwd.residual.data, ref["h1b"])}
    mx = {"qkv": float(np.max(np.abs(fwd.qkv.data - ref["qkv"])))}
    for key in O.GRAD_KEYS:
        got = getattr(bwd, key).data
        errs[key] = O.rel_error(got, refb[key])
        mx[key] = float(np.max(np.abs(got - refb[key])))
    print("\n[C1 fp32] rel vs f64: " + ", ".join(f"{k}={v:.2e}" for k, v in errs.items()))
    print("[C1 fp32] max abs:    " + ", ".join(f"{k}={v:.2e}" for k, v in mx.items()))
    assert max(errs.values()) <= 1e-5, errs
    # fused-order oracle (same precision model) agrees too
    of = O.layer_forward(x, z, w, cos, sin, O.SIM32)
    ob = O.layer_backward(gq, of, w, O.SIM32, grad_residual=gr)
    for key in O.GRAD_KEYS:
        assert O.rel_error(getattr(bwd, key).data, ob[key]) <= 1e-5, key


def test_bf16_mid_layer_vs_fused_oracle(cuda_ready):
    """bf16 path at a shape with several GPU tiles in every dimension."""
    cd = _cd()
    m, d, ffn = 512, 512, 2816
    rng = np.random.default_rng(1)
    mode = O.SIMBF16
    w = O.random_layer(rng, d, ffn, mode, scale=0.05)
    x = O.q(rng.standard_normal((m, d)), mode)
    z = O.q(rng.standard_normal((m, d)), mode)
    cos, sin = O.qkv_rope_tables(m, d, mode)
    gq = O.q(rng.standard_normal((m, 3 * d)), mode)
    gr = O.q(rng.standard_normal((m, d)), mode)
    P = cd.PrecisionMode.SIMBF16
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, precision=P)
    fwd, bwd = _run_layer(cd, P, cfg, x, z, w, cos, sin, gq, gr)
    of = O.layer_forward(x, z, w, cos, sin, mode)
    ob = O.layer_backward(gq, of, w, mode, grad_residual=gr)
    errs = {"qkv": O.rel_error(fwd.qkv.data, of["qkv"])}
    for key in O.GRAD_KEYS:
        errs[key] = O.rel_error(getattr(bwd, key).data, ob[key])
    print("\n[bf16 512x512x2816] rel vs fused oracle: " + ", ".join(f"{k}={v:.2e}" for k, v in errs.items()))
    assert max(errs.values()) <= 2e-2, errs


def test_eps_path_all_zero_input(cuda_ready):
    """reference tests/test_kernels.py:385-393: zero x, z -> r = 1/sqrt(eps), qkv = 0."""
    cd = _cd()
    P = cd.PrecisionMode.SIM32
    d, ffn, m = 16, 32, 8
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, precision=P)
    rng = np.random.default_rng(0)
    w = cd.LayerWeights.random(rng, cfg)
    zero = cd.DenseMatrix.from_array(np.zeros((m, d)), P)
    cos, sin = cd.qkv_rope_tables(m, d, precision=P)
    fwd = cd.layer_forward(zero, zero, w, cos, sin, config=cfg)
    assert np.all(fwd.qkv.data == 0.0)
    np.testing.assert_allclose(fwd.tape.inv_rms_a.data, np.float32(1.0 / np.sqrt(np.float32(1e-6))), rtol=1e-6)


@pytest.mark.parametrize("mode_name", ["sim32", "simbf16"])
def test_block_stack_vs_chained_oracle(cuda_ready, mode_name):
    """3-block stack (x_{l+1} = V span of qkv_l, z_{l+1} = residual_l) vs the oracle chained the same way."""
    cd = _cd()
    from paper_2605_19269_b200 import stack

    m, d, ffn, L = 192, 128, 512, 3
    mode = O.SIM32 if mode_name == "sim32" else O.SIMBF16
    P = cd.PrecisionMode.SIM32 if mode_name == "sim32" else cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(4)
    ws = [O.random_layer(rng, d, ffn, mode, scale=0.1) for _ in range(L)]
    x = O.q(rng.standard_normal((m, d)), mode)
    z = O.q(rng.standard_normal((m, d)), mode)
    cos, sin = O.qkv_rope_tables(m, d, mode)
    gq = O.q(rng.standard_normal((m, 3 * d)), mode)
    gr = O.q(rng.standard_normal((m, d)), mode)
    # oracle chain
    fw, xi, zi = [], x, z
    for w in ws:
        f = O.layer_forward(xi, zi, w, cos, sin, mode)
        fw.append(f)
        xi, zi = f["qkv"][:, 2 * d:], f["residual"]
    ref_grads = [None] * L
    g_q, g_r = gq, gr
    for l in range(L - 1, -1, -1):
        b = O.layer_backward(g_q, fw[l], ws[l], mode, grad_residual=g_r)
        ref_grads[l] = b
        g_q = np.concatenate([np.zeros((m, 2 * d)), b["x"]], axis=1)
        g_r = b["z"]
    # device stack
    M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
    dws = [cd.LayerWeights(w_out=M(w["w_out"]), gamma_ffn=cd.Vector.from_array(w["gamma_ffn"], P),
                           w_gate_up=M(w["w_gate_up"]), w_down=M(w["w_down"]),
                           gamma_qkv=cd.Vector.from_array(w["gamma_qkv"], P), w_qkv=M(w["w_qkv"])) for w in ws]
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, precision=P)
    res = stack.stack_forward(M(x), M(z), dws, M(cos), M(sin), config=cfg)
    grads = stack.stack_backward(M(gq), M(gr), res, dws, config=cfg)
    tol = 1e-5 if mode_name == "sim32" else 2e-2
    assert O.rel_error(res.qkv.data, fw[-1]["qkv"]) <= tol
    worst = 0.0
    for l in range(L):
        for key in O.GRAD_KEYS:
            worst = max(worst, O.rel_error(getattr(grads[l], key).data, ref_grads[l][key]))
    print(f"\n[stack {mode_name}] worst grad rel err {worst:.2e}")
    assert worst <= tol


@pytest.mark.parametrize("mode_name", ["sim32", "simbf16"])
def test_gqa_kv_width_layer(cuda_ready, mode_name):
    """GQA extension: packed projection q (d) + k (kv) + v (kv).

    The CUDA path vs the fused-order oracle and the float64 canonical chain at the
    same kv width (no reference counterpart; kv_width=None is the reference layout)."""
    cd = _cd()
    m, d, ffn, kv = 256, 256, 1024, 64
    mode = O.SIM32 if mode_name == "sim32" else O.SIMBF16
    P = cd.PrecisionMode.SIM32 if mode_name == "sim32" else cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(11)
    w = O.random_layer(rng, d, ffn, mode, scale=0.1, kv_width=kv)
    x, z = (O.q(rng.standard_normal((m, d)), mode) for _ in range(2))
    cos, sin = O.qkv_rope_tables(m, d, mode, kv_width=kv)
    gq = O.q(rng.standard_normal((m, d + 2 * kv)), mode)
    gr = O.q(rng.standard_normal((m, d)), mode)
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, precision=P, kv_width=kv)
    c2, s2 = cd.qkv_rope_tables(m, d, precision=P, kv_width=kv)
    assert np.array_equal(c2.data, cos) and np.array_equal(s2.data, sin)
    fwd, bwd = _run_layer(cd, P, cfg, x, z, w, cos, sin, gq, gr)
    assert fwd.qkv.shape == (m, d + 2 * kv)
    tol = 1e-5 if mode_name == "sim32" else 2e-2
    of = O.layer_forward(x, z, w, cos, sin, mode)
    ob = O.layer_backward(gq, of, w, mode, grad_residual=gr)
    errs = {"qkv": O.rel_error(fwd.qkv.data, of["qkv"])}
    errs.update({k: O.rel_error(getattr(bwd, k).data, ob[k]) for k in O.GRAD_KEYS})
    print(f"\n[GQA kv={kv} {mode_name}] rel vs fused oracle: " + ", ".join(f"{k}={v:.2e}" for k, v in errs.items()))
    assert max(errs.values()) <= tol, errs
    if mode_name == "sim32":
        ref = O.layer_ref_forward(x, z, w, cos, sin)
        refb = O.layer_ref_backward(gq, gr, ref, x, w, cos, sin)
        e64 = {k: O.rel_error(getattr(bwd, k).data, refb[k]) for k in O.GRAD_KEYS}
        e64["qkv"] = O.rel_error(fwd.qkv.data, ref["qkv"])
        assert max(e64.values()) <= 1e-5, e64


def test_compact_rope_tables_bit_identical(cuda_ready):
    """qkv_rope_tables attaches a compact (m, d/2) form that K7 and rope_backward_stat load
    instead of the full (m, 3d) tables; results must be bit-identical to the full tables."""
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    m, d, ffn = 640, 256, 1024
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, precision=P)
    rng = np.random.default_rng(13)
    w = cd.LayerWeights.random(rng, cfg, scale=0.05)
    M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
    x, z = M(rng.standard_normal((m, d))), M(rng.standard_normal((m, d)))
    gq, gr = M(rng.standard_normal((m, 3 * d))), M(rng.standard_normal((m, d)))
    cos_c, sin_c = cd.qkv_rope_tables(m, d, start=7, precision=P)
    assert cos_c._rope is not None and cos_c._rope[0] is sin_c._rope[0]
    assert (cos_c._rope[1], sin_c._rope[1]) == ("cos", "sin")
    assert cos_c._rope[0].cos.shape == (m, d // 2)
    # the same values without the compact form (full-table path)
    cos_f, sin_f = cd.DenseMatrix.from_tensor(cos_c.tensor, P), cd.DenseMatrix.from_tensor(sin_c.tensor, P)
    assert cos_f._rope is None
    outs = []
    for c, s in ((cos_c, sin_c), (cos_f, sin_f)):
        fwd = cd.layer_forward(x, z, w, c, s, config=cfg)
        bwd = cd.layer_backward(gq, fwd.tape, w, grad_residual=gr, config=cfg)
        gz, rd = cd.rope_backward_stat(gq, fwd.qkv, c, s, precision=P)
        outs.append([fwd.qkv.data, gz.data, rd.data] + [getattr(bwd, k).data for k in O.GRAD_KEYS])
    for i, (a, b) in enumerate(zip(*outs)):
        assert np.array_equal(a, b), f"output {i} differs between compact and full RoPE tables"
    # and the compact path agrees with the fused-order oracle
    of = O.layer_forward(x.data, z.data, {k: getattr(w, k).data for k in WKEYS}, cos_f.data, sin_f.data, O.SIMBF16)
    assert O.rel_error(outs[0][0], of["qkv"]) <= 2e-2


def test_compact_rope_roles_respected(cuda_ready):
    """Swapped (sin, cos) or duplicated (cos, cos) bindings of compact-capable tables must
    compute exactly what was bound, like the generic path and the reference."""
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    m, d = 256, 256
    rng = np.random.default_rng(5)
    cos_c, sin_c = cd.qkv_rope_tables(m, d, precision=P)
    assert cd.kernels.rope_compact_of(cos_c, sin_c) is not None
    assert cd.kernels.rope_compact_of(sin_c, cos_c) is None
    assert cd.kernels.rope_compact_of(cos_c, cos_c) is None
    a = cd.DenseMatrix.from_array(rng.standard_normal((m, d)), P)
    b = cd.DenseMatrix.from_array(rng.standard_normal((d, 3 * d)) * 0.1, P)
    for c, s in ((sin_c, cos_c), (cos_c, cos_c)):
        got = cd.gemm_rope(a, b, c, s, precision=P).main.data
        want = O.k_rope(a.data, b.data, c.data, s.data, O.SIMBF16)["main"]
        assert O.rel_error(got, want) <= 1e-3          # bf16 stores: isolated 1-ulp flips only
        gq = cd.DenseMatrix.from_array(rng.standard_normal((m, 3 * d)), P)
        gz, _ = cd.rope_backward_stat(gq, gq, c, s, precision=P)
        ogz, _ = O.rope_backward_stat(gq.data, gq.data, c.data, s.data, O.SIMBF16)
        assert O.rel_error(gz.data, ogz) <= 1e-3


@pytest.mark.parametrize("m,n", [(300, 512), (256, 96), (128, 4096)])
@pytest.mark.parametrize("backward", [False, True])
def test_plain_rope_tables_compact_bit_identical(cuda_ready, m, n, backward):
    """rope_tables(m, width) attaches a compact (m, width/2) form (hidden = width); the
    fused GEMM + PairwiseRope (K1, forward and backward rotation) loads it instead of
    the full tables with bit-identical results, and rope_backward_stat, which keeps the
    full tables for this layout, still runs."""
    cd = _cd()
    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(m + n)
    a = cd.DenseMatrix.from_array(rng.standard_normal((m, 192)) / 8, P)
    b = cd.DenseMatrix.from_array(rng.standard_normal((192, n)) / 8, P)
    cos_c, sin_c = cd.rope_tables(m, n, start=3, precision=P)
    spec = cd.kernels.rope_compact_of(cos_c, sin_c)
    assert spec is not None and spec.hidden == n and spec.cos.shape == (m, n // 2)
    cos_f, sin_f = cd.DenseMatrix.from_tensor(cos_c.tensor, P), cd.DenseMatrix.from_tensor(sin_c.tensor, P)
    got = cd.gemm_rope(a, b, cos_c, sin_c, backward=backward, precision=P).main.data
    want = cd.gemm_rope(a, b, cos_f, sin_f, backward=backward, precision=P).main.data
    assert np.array_equal(got, want)
    ref = O.k_rope(a.data, b.data, cos_f.data, sin_f.data, O.SIMBF16, backward=backward)["main"]
    assert O.rel_error(got, ref) <= 2e-2
    if not backward:
        g = cd.DenseMatrix.from_array(rng.standard_normal((m, n)), P)
        gz1, rd1 = cd.rope_backward_stat(g, cd.DenseMatrix.from_array(got, P), cos_c, sin_c, precision=P)
        gz2, rd2 = cd.rope_backward_stat(g, cd.DenseMatrix.from_array(got, P), cos_f, sin_f, precision=P)
        assert np.array_equal(gz1.data, gz2.data) and np.array_equal(rd1.data, rd2.data)
