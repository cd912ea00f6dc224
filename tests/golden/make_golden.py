"""Generate golden vectors from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package `tilefuse` read-only from
/root/reference/pkg/src, runs its own kernels / pipelines on seeded inputs and
stores inputs + outputs as compressed .npz fixtures next to this script.  The
fixtures pin the CPU oracle (oracle/coda_oracle.py) and, on the GPU box, the
CUDA path; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import tilefuse as tf  # noqa: E402
from tilefuse import oracles  # noqa: E402

OUT = Path(__file__).resolve().parent
MODES = {"sim32": tf.PrecisionMode.SIM32, "simbf16": tf.PrecisionMode.SIMBF16, "exact64": tf.PrecisionMode.EXACT64}


def mat(rng, shape, mode, scale=1.0):
    return tf.DenseMatrix.from_array(rng.standard_normal(shape) * scale, mode)


def save(name, **arrays):
    """Store float payloads as float32 in the simulated modes (lossless: every
    stored value lies on the f32 grid); float64 canonical references stay f64."""
    f32 = not name.endswith("exact64") and name != "kat"
    out = {}
    for k, v in arrays.items():
        v = np.asarray(v)
        if f32 and v.dtype == np.float64 and not k.startswith("ref_"):
            assert np.array_equal(v.astype(np.float32).astype(np.float64), v), (name, k)
            v = v.astype(np.float32)
        out[k] = v
    np.savez_compressed(OUT / f"{name}.npz", **out)


def slot(s):
    return np.asarray(s.data), np.asarray(s.counts)


def kernels_case(tag, mode_name, m, k, n, tile, rtn, seed):
    """Every single-launch kernel at one ragged shape and tile context."""
    mode = MODES[mode_name]
    rng = np.random.default_rng(seed)
    ts = tf.TileShape(*tile)
    kw = dict(tile_shape=ts, reduction_tile_n=rtn, precision=mode)
    a = mat(rng, (m, k), mode)
    b = mat(rng, (k, n), mode, 1.0 / np.sqrt(k))
    bt = mat(rng, (n, k), mode, 1.0 / np.sqrt(k))
    z = mat(rng, (m, n), mode)
    gamma = tf.Vector.from_array(1.0 + 0.1 * rng.standard_normal(n), mode)
    r = tf.Vector.from_array(0.5 + rng.random(m), tf.stat_mode(mode))
    s = tf.Vector.from_array(0.1 * rng.standard_normal(m), tf.stat_mode(mode))
    cos, sin = tf.rope_tables(m, n, start=3, precision=mode)
    pre = mat(rng, (m, n), mode)
    gin = mat(rng, (m, n), mode)
    preact2 = mat(rng, (m, 2 * n), mode)
    labels = rng.integers(0, n, size=m)
    out = dict(a=a.data, b=b.data, bt=bt.data, z=z.data, gamma=gamma.data, r=r.data, s=s.data, cos=cos.data,
               sin=sin.data, pre=pre.data, gin=gin.data, preact2=preact2.data, labels=labels,
               meta=np.array([m, k, n, tile[0], tile[1], rtn]))
    out["k1"] = tf.gemm_rope(a, b, cos, sin, **kw).main.data
    out["k1_bwd"] = tf.gemm_rope(a, b, cos, sin, backward=True, **kw).main.data
    k2 = tf.gemm_swiglu(a, b, save_preact=True, **kw)
    out["k2"], out["k2_preact"] = k2.main.data, k2.aux["preact"].data
    k3 = tf.gemm_partial_xent(a, b, labels, store_logits=True, **kw)
    out["k3"], out["k3_target"] = k3.main.data, k3.aux["target"].data
    out["k3_lse_data"], out["k3_lse_counts"] = slot(k3.aux["lse"])
    out["k3_lse"] = tf.combine_lse(k3.aux["lse"]).data
    k4 = tf.gemm_residual_partial_rms(a, b, z, gamma, **kw)
    out["k4"], out["k4_pre_norm"] = k4.main.data, k4.aux["pre_norm"].data
    out["k4_sumsq_data"], out["k4_sumsq_counts"] = slot(k4.aux["sumsq"])
    out["k4_r"] = tf.finalize_rms(k4.aux["sumsq"], 1e-6).data
    out["k5"] = tf.gemm_row_scale(a, b, r, **kw).main.data
    k6 = tf.gemm_rms_swiglu(a, b, r, **kw)
    out["k6"], out["k6_preact"] = k6.main.data, k6.aux["preact"].data
    out["k7"] = tf.gemm_rms_rope(a, b, r, cos, sin, **kw).main.data
    k8 = tf.gemm_rms_partial_xent(a, b, r, labels, **kw)
    out["k8_target"] = k8.aux["target"].data
    out["k8_lse"] = tf.combine_lse(k8.aux["lse"]).data
    k9 = tf.gemm_rmsnorm_backward(a, bt, pre, r, gamma, s, grad_in=gin, trans_b=True, **kw)
    out["k9"], out["k9_normed"] = k9.main.data, k9.aux["normed"].data
    out["k9_gg_data"], out["k9_gg_counts"] = slot(k9.aux["gamma_grad"])
    out["k9_dgamma"] = tf.reduce_row_partials(k9.aux["gamma_grad"]).data
    k10 = tf.gemm_swiglu_backward(a, bt, preact2, trans_b=True, **kw)
    out["k10"], out["k10_recompute"] = k10.main.data, k10.aux["recompute"].data
    out["k10_rowdot_data"], out["k10_rowdot_counts"] = slot(k10.aux["rowdot"])
    out["k10_s"] = tf.finalize_rowdot(k10.aux["rowdot"], 7).data
    gz, rd = tf.rope_backward_stat(z, pre, cos, sin, tile_n=tile[1], reduction_tile_n=rtn, precision=mode)
    out["rbs_gz"] = gz.data
    out["rbs_data"], out["rbs_counts"] = slot(rd)
    # transposed-A (wgrad layout) plain GEMM
    at = mat(rng, (k, m), mode)
    out["at"] = at.data
    out["wgrad"] = tf.run_gemm(tf.GemmProblem(m=m, n=n, k=k, trans_a=True, precision=mode, tile_shape=ts,
                                              reduction_tile_n=rtn), at, b).main.data
    # reference traffic ledger records (read, write bytes) of each launch above
    out["records"] = np.array([[r.read_bytes, r.write_bytes] for r in (
        tf.gemm_rope(a, b, cos, sin, **kw).record, k2.record, k3.record, k4.record,
        tf.gemm_row_scale(a, b, r, **kw).record, k6.record, tf.gemm_rms_rope(a, b, r, cos, sin, **kw).record,
        k8.record, k9.record, k10.record)], dtype=np.int64)
    save(f"kernels_{tag}_{mode_name}", **out)


def layer_case(tag, mode_name, m, d, ffn, tile, rtn, seed, scale=0.2):
    mode = MODES[mode_name]
    rng = np.random.default_rng(seed)
    cfg = tf.PipelineConfig(hidden=d, ffn=ffn, tile_m=tile[0], tile_n=tile[1], reduction_tile_n=rtn,
                            precision=mode)
    w = tf.LayerWeights.random(rng, cfg, scale=scale)
    x = mat(rng, (m, d), mode)
    z = mat(rng, (m, d), mode)
    cos, sin = tf.qkv_rope_tables(m, d, start=0, precision=mode)
    gq = mat(rng, (m, 3 * d), mode)
    gr = mat(rng, (m, d), mode)
    fwd = tf.layer_forward(x, z, w, cos, sin, config=cfg)
    bwd = tf.layer_backward(gq, fwd.tape, w, grad_residual=gr, config=cfg)
    ref = oracles.layer_ref_forward(x.data, z.data, w.w_out.data, w.gamma_ffn.data, w.w_gate_up.data,
                                    w.w_down.data, w.gamma_qkv.data, w.w_qkv.data, cos.data, sin.data)
    refb = oracles.layer_ref_backward(gq.data, gr.data, ref, x.data, w.w_out.data, w.gamma_ffn.data,
                                      w.w_gate_up.data, w.w_down.data, w.gamma_qkv.data, w.w_qkv.data, cos.data,
                                      sin.data)
    out = dict(meta=np.array([m, d, ffn, tile[0], tile[1], rtn]), x=x.data, z=z.data, cos=cos.data, sin=sin.data,
               grad_qkv=gq.data, grad_residual=gr.data,
               w_out=w.w_out.data, gamma_ffn=w.gamma_ffn.data, w_gate_up=w.w_gate_up.data, w_down=w.w_down.data,
               gamma_qkv=w.gamma_qkv.data, w_qkv=w.w_qkv.data,
               qkv=fwd.qkv.data, residual=fwd.residual.data, pre_norm_a=fwd.tape.pre_norm_a.data,
               inv_rms_a=fwd.tape.inv_rms_a.data, preact=fwd.tape.preact.data, inv_rms_b=fwd.tape.inv_rms_b.data,
               ref_qkv=ref["qkv"], ref_h1b=ref["h1b"])
    for key in ("x", "z", "w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv", "w_qkv"):
        out[f"g_{key}"] = getattr(bwd, key).data
        out[f"ref_g_{key}"] = refb[key]
    save(f"layer_{tag}_{mode_name}", **out)


def kat_case():
    """Known-answer values frozen by the reference's own tests."""
    vals = np.array([1.0, 1.00390625, 1.005859375, 1.0078125, -2.5e-3, 3.14159265, 65504.0, 1e-30, -7.77e7],
                    dtype=np.float64)
    save("kat", bf16_in=vals, bf16_out=tf.quantize(vals, tf.PrecisionMode.SIMBF16),
         sigmoid1=np.array(oracles.sigmoid_ref(np.array([1.0]))),
         swiglu12=np.array(oracles.swiglu_ref(np.array([[1.0, 2.0]]))),
         layout=np.array([b.width for b in tf.row_block_layout(10, 4, 3)]))


def codt_case():
    """Containers written by the reference's codt.write_tensor, plus their values."""
    from tilefuse.codt import write_tensor

    rng = np.random.default_rng(9)
    vals = {}
    for tag, mode in MODES.items():
        m = tf.DenseMatrix.from_array(rng.standard_normal((5, 9)), mode)
        write_tensor(OUT / f"ref_{tag}_matrix.codt", m)
        vals[f"{tag}_matrix"] = m.data
        v = tf.Vector.from_array(np.linspace(-3, 3, 11), mode)
        write_tensor(OUT / f"ref_{tag}_vector.codt", v)
        vals[f"{tag}_vector"] = v.data
    np.savez_compressed(OUT / "codt_values.npz", **vals)


if __name__ == "__main__":
    codt_case()
    kat_case()
    for mode in ("sim32", "simbf16", "exact64"):
        kernels_case("ragged", mode, m=37, k=45, n=50, tile=(16, 24), rtn=10, seed=11)
        if mode != "exact64":
            kernels_case("default", mode, m=130, k=96, n=264, tile=(128, 128), rtn=128, seed=12)
        layer_case("tiny", mode, m=48, d=64, ffn=256, tile=(128, 128), rtn=128, seed=5)
        layer_case("ragged", mode, m=40, d=32, ffn=96, tile=(16, 24), rtn=10, seed=6)
    print("golden fixtures written to", OUT)
