"""CPU ORACLE — test infrastructure only.

A numpy restatement of the reference algorithm for the hot path (the
`tilefuse` engine semantics of run_gemm + epilogue primitives and the layer
pipelines), written whole-matrix instead of tile-by-tile.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / reference arm may
import it, and only as the checker; the product path never touches it.

Pinning: tests/test_oracle_golden.py checks every function here against
golden vectors produced by the reference package itself
(tests/golden/make_golden.py imports /root/reference/pkg/src/tilefuse in the
build container and commits the outputs), and against the reference's own
frozen known-answer values (tests/test_oracles.py of the reference).

Numerics mirror the reference's precision model (tensors.py:1-15 of the
reference): values are float64 arrays on the storage grid; GEMMs and
epilogue math run at the accumulator dtype (float32 in SIM32/SIMBF16,
float64 in EXACT64); rounding to storage happens only where the reference
stores (engine.py:332-338, 443-447).  Every function cites the reference
file:line it restates (paths relative to pkg/src/tilefuse/).
"""

from __future__ import annotations

import numpy as np

EXACT64, SIM32, SIMBF16 = "exact64", "sim32", "simbf16"


# ----------------------------------------------------------------------------- precision model


def acc_dtype(mode: str):
    """Accumulator dtype (tensors.py:46-49)."""
    return np.float64 if mode == EXACT64 else np.float32


def bf16_round(x) -> np.ndarray:
    """bf16 round-to-nearest-even on the f32 bit pattern (tensors.py:64-79)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    # uint32 wrap-around only happens for NaN payloads, which the mask restores
    r = ((u + np.uint32(0x7FFF) + lsb) & np.uint32(0xFFFF0000)).view(np.float32)
    return np.where(np.isfinite(f), r, f)


def q(x, mode: str) -> np.ndarray:
    """Quantize-on-store to the storage grid, float64 result (tensors.py:82-97)."""
    a = np.asarray(x, dtype=np.float64)
    if mode == EXACT64:
        return a.copy()
    if mode == SIM32:
        return a.astype(np.float32).astype(np.float64)
    return bf16_round(a.astype(np.float32)).astype(np.float64)


def stat_q(x, mode: str) -> np.ndarray:
    """Row statistics live at SIM32 in simulated modes (tensors.py:227-235)."""
    return q(x, EXACT64 if mode == EXACT64 else SIM32)


def rel_error(a, b) -> float:
    """Frobenius relative error in float64 (tensors.py:244-257)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# ----------------------------------------------------------------------------- layouts


def row_blocks(n: int, tile_n: int, rtn: int, scale: int = 1) -> list[tuple[int, int]]:
    """Reduction blocks of a row-directed partial at integer width scale.

    Each tile column [c0, c0+w) of the unscaled grid becomes [c0*s, (c0+w)*s)
    and is sub-blocked into runs of at most rtn (epilogue.py:109-130,
    engine.py:244-269).
    """
    out = []
    for c0 in range(0, n, tile_n):
        lo, hi = c0 * scale, min(c0 + tile_n, n) * scale
        for s in range(lo, hi, rtn):
            out.append((s, min(s + rtn, hi)))
    return out


def row_partials(x: np.ndarray, blocks) -> np.ndarray:
    """(m, nb) block sums of x over columns at x's dtype."""
    return np.stack([x[:, a:b].sum(axis=1) for a, b in blocks], axis=1)


def col_partials(x: np.ndarray, tile_m: int) -> np.ndarray:
    """(Tm, n) sums over each run of tile_m rows (engine.py:293-305, epilogue.py:330-333)."""
    return np.stack([x[r:r + tile_m].sum(axis=0) for r in range(0, x.shape[0], tile_m)], axis=0)


def counts_of(blocks) -> np.ndarray:
    return np.array([b - a for a, b in blocks], dtype=np.int64)


# ----------------------------------------------------------------------------- epilogue math


def gemm(a, b, mode: str, trans_a: bool = False, trans_b: bool = False) -> np.ndarray:
    """Accumulator-precision product of storage-grid operands (engine.py:415-438)."""
    dt = acc_dtype(mode)
    A = np.asarray(a, dtype=dt)
    B = np.asarray(b, dtype=dt)
    return (A.T if trans_a else A) @ (B.T if trans_b else B)


def sigmoid(x: np.ndarray) -> np.ndarray:
    """Overflow-free logistic via exp(-|x|) (epilogue.py:596-599)."""
    e = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e)).astype(x.dtype, copy=False)


def rope(x: np.ndarray, cos: np.ndarray, sin: np.ndarray, backward: bool = False) -> np.ndarray:
    """Adjacent-pair rotation with duplicated tables (epilogue.py:424-440)."""
    if backward:
        sin = -sin
    out = np.empty_like(x)
    x0, x1 = x[:, 0::2], x[:, 1::2]
    out[:, 0::2] = x0 * cos[:, 0::2] - x1 * sin[:, 0::2]
    out[:, 1::2] = x0 * sin[:, 1::2] + x1 * cos[:, 1::2]
    return out


def swiglu(x: np.ndarray) -> np.ndarray:
    """silu(even) * odd, width halves (epilogue.py:460-463)."""
    g, u = x[:, 0::2], x[:, 1::2]
    return g * sigmoid(g) * u


def swiglu_backward(dout: np.ndarray, z: np.ndarray):
    """(interleaved grad, recompute, <z, grad> terms) (epilogue.py:493-515)."""
    g, u = z[:, 0::2], z[:, 1::2]
    sg = sigmoid(g)
    sl = g * sg
    rec = sl * u
    out = np.empty_like(z)
    out[:, 0::2] = dout * u * (sg + sl * (1.0 - sg))
    out[:, 1::2] = dout * sl
    return out, rec, z * out


# ----------------------------------------------------------------------------- fused launches
# Each returns {"main": ..., aux names...} with tiles quantized like the engine stores them,
# partials as (data, counts) at the accumulator dtype.


def _cast(x, mode):
    return np.asarray(x, dtype=acc_dtype(mode))


def k_rope(a, b, cos, sin, mode, backward=False, trans_b=False):
    """K1 gemm_rope (kernels.py:243-266)."""
    t = gemm(a, b, mode, trans_b=trans_b)
    return {"main": q(rope(t, _cast(cos, mode), _cast(sin, mode), backward), mode)}


def k_swiglu(a, b, mode, save_preact=False, trans_b=False):
    """K2 gemm_swiglu (kernels.py:269-294)."""
    t = gemm(a, b, mode, trans_b=trans_b)
    out = {"main": q(swiglu(t), mode)}
    if save_preact:
        out["preact"] = q(t, mode)
    return out


def k_residual_partial_rms(a, b, residual, gamma, mode, tile_n=128, rtn=128, trans_b=False):
    """K4 gemm_residual_partial_rms (kernels.py:325-360): [+C, store, sumsq, *gamma]."""
    t = gemm(a, b, mode, trans_b=trans_b) + _cast(residual, mode)
    blocks = row_blocks(t.shape[1], tile_n, rtn)
    return {
        "main": q(t * _cast(gamma, mode)[None, :], mode),
        "pre_norm": q(t, mode),
        "sumsq": (row_partials(t * t, blocks), counts_of(blocks)),
    }


def k_row_scale(a, b, scale, mode, trans_b=False):
    """K5 gemm_row_scale (kernels.py:363-384)."""
    return {"main": q(gemm(a, b, mode, trans_b=trans_b) * _cast(scale, mode)[:, None], mode)}


def k_rms_swiglu(a, b, scale, mode, trans_b=False):
    """K6 gemm_rms_swiglu (kernels.py:387-410)."""
    t = gemm(a, b, mode, trans_b=trans_b) * _cast(scale, mode)[:, None]
    return {"main": q(swiglu(t), mode), "preact": q(t, mode)}


def k_rms_rope(a, b, scale, cos, sin, mode, trans_b=False):
    """K7 gemm_rms_rope (kernels.py:413-438)."""
    t = gemm(a, b, mode, trans_b=trans_b) * _cast(scale, mode)[:, None]
    return {"main": q(rope(t, _cast(cos, mode), _cast(sin, mode)), mode)}


def k_rmsnorm_backward(a, b, pre_norm, inv_rms, gamma, stat, mode, grad_in=None, tile_m=128,
                       trans_a=False, trans_b=False):
    """K9 gemm_rmsnorm_backward (kernels.py:474-525; primitive epilogue.py:575-586)."""
    D = gemm(a, b, mode, trans_a=trans_a, trans_b=trans_b)
    c = _cast(pre_norm, mode)
    r = _cast(inv_rms, mode)[:, None]
    g = _cast(gamma, mode)[None, :]
    s = _cast(stat, mode)[:, None]
    cn = c * r
    out = (D * g - cn * s) * r
    if grad_in is not None:
        out = out + _cast(grad_in, mode)
    gg = col_partials(D * cn, tile_m)
    counts = np.array([min(tile_m, D.shape[0] - r0) for r0 in range(0, D.shape[0], tile_m)], dtype=np.int64)
    return {"main": q(out, mode), "normed": q(cn * g, mode), "gamma_grad": (gg, counts)}


def k_swiglu_backward(a, b, preact, mode, tile_n=128, rtn=128, trans_b=False):
    """K10 gemm_swiglu_backward (kernels.py:528-557; primitive epilogue.py:493-515)."""
    D = gemm(a, b, mode, trans_b=trans_b)
    out, rec, terms = swiglu_backward(D, _cast(preact, mode))
    blocks = row_blocks(D.shape[1], tile_n, rtn, scale=2)
    return {"main": q(out, mode), "recompute": q(rec, mode),
            "rowdot": (row_partials(terms, blocks), counts_of(blocks))}


def k_partial_xent(a, b, labels, mode, tile_n=128, rtn=128, scale=None, trans_b=False):
    """K3 / K8 (kernels.py:297-322, 441-471): gathered targets + blocked (max, sum) pairs."""
    t = gemm(a, b, mode, trans_b=trans_b)
    if scale is not None:
        t = t * _cast(scale, mode)[:, None]
    labels = np.asarray(labels, dtype=np.int64)
    target = t[np.arange(t.shape[0]), labels].astype(np.float64)
    blocks = row_blocks(t.shape[1], tile_n, rtn)
    pairs = np.empty((t.shape[0], len(blocks), 2), dtype=t.dtype)
    for j, (lo, hi) in enumerate(blocks):
        piece = t[:, lo:hi]
        mx = piece.max(axis=1)
        pairs[:, j, 0] = mx
        pairs[:, j, 1] = np.exp(piece - mx[:, None]).sum(axis=1)
    return {"main": q(t, mode), "target": target, "lse": (pairs, counts_of(blocks))}


def rope_backward_stat(grad, rotated, cos, sin, mode, tile_n=128, rtn=128):
    """Boundary counter-rotation + <grad, rotated> partials (kernels.py:560-617)."""
    g = _cast(grad, mode)
    gz = rope(g, _cast(cos, mode), _cast(sin, mode), backward=True)
    blocks = row_blocks(g.shape[1], tile_n, rtn)
    return q(gz, mode), (row_partials(g * _cast(rotated, mode), blocks), counts_of(blocks))


# ----------------------------------------------------------------------------- finalizers


def finalize_rms(partials, eps: float, mode: str) -> np.ndarray:
    """r = 1/sqrt(sum/d + eps) with sequential ascending block sum (reductions.py:64-80)."""
    data, counts = partials
    dt = acc_dtype(mode)
    x = np.asarray(data, dtype=dt)
    tot = np.zeros(x.shape[0], dtype=dt)
    for j in range(x.shape[1]):
        tot = tot + x[:, j]
    d = dt(int(np.sum(counts)))
    return stat_q(1.0 / np.sqrt(tot / d + dt(eps)), mode)


def finalize_rowdot(partials, d: int, mode: str) -> np.ndarray:
    """s = sum/d with d the normalized width (reductions.py:83-98)."""
    data, _ = partials
    dt = acc_dtype(mode)
    x = np.asarray(data, dtype=dt)
    tot = np.zeros(x.shape[0], dtype=dt)
    for j in range(x.shape[1]):
        tot = tot + x[:, j]
    return stat_q(tot / dt(d), mode)


def reduce_row_partials(partials, mode: str) -> np.ndarray:
    """Column totals of per-tile-row partials (reductions.py:134-145)."""
    data, _ = partials
    dt = acc_dtype(mode)
    x = np.asarray(data, dtype=dt)
    tot = np.zeros(x.shape[1], dtype=dt)
    for i in range(x.shape[0]):
        tot = tot + x[i]
    return stat_q(tot, mode)


def combine_lse(partials, mode: str) -> np.ndarray:
    """Merge (max, scaled-sum) pairs in block order (reductions.py:101-131)."""
    data, _ = partials
    dt = acc_dtype(mode)
    x = np.asarray(data, dtype=dt)
    m = np.full(x.shape[0], -np.inf, dtype=dt)
    s = np.zeros(x.shape[0], dtype=dt)
    with np.errstate(invalid="ignore", over="ignore"):
        for j in range(x.shape[1]):
            mb, sb = x[:, j, 0], x[:, j, 1]
            mn = np.maximum(m, mb)
            so = np.where(np.isneginf(m), dt(0), np.exp(m - mn))
            sn = np.where(np.isneginf(mb), dt(0), np.exp(mb - mn))
            s = s * so + sb * sn
            m = mn
    return stat_q(m + np.log(s), mode)


# ----------------------------------------------------------------------------- pipelines


def qkv_rope_tables(m: int, hidden: int, mode: str, base: float = 10000.0, start: int = 0, kv_width=None):
    """(m, h + 2kv) cos/sin: q and k rotate, v identity (kernels.py:156-206).

    kv_width None (= hidden) is the reference's packed 3h layout, where q and k share
    angles.  The GQA extension (no reference counterpart) rotates the k span with the
    reference's rule applied to its own width (pair p of a width-w span turns by
    t * base^(-2p/w)).
    """
    kv = hidden if kv_width is None else kv_width

    def span(w):
        inv = base ** (-2.0 * np.arange(w // 2, dtype=np.float64) / w)
        ang = (start + np.arange(m, dtype=np.float64))[:, None] * inv[None, :]
        return np.repeat(np.cos(ang), 2, axis=1), np.repeat(np.sin(ang), 2, axis=1)

    cq, sq = span(hidden)
    ck, sk = span(kv)
    cos = np.concatenate([cq, ck, np.ones((m, kv))], axis=1)
    sin = np.concatenate([sq, sk, np.zeros((m, kv))], axis=1)
    return q(cos, mode), q(sin, mode)


def random_layer(rng: np.random.Generator, d: int, ffn: int, mode: str, scale: float = 0.2, kv_width=None) -> dict:
    """Weights in the reference draw order (kernels.py:750-767); w_qkv is (d, d + 2 kv)."""
    mk = lambda *s: q(rng.standard_normal(s) * scale, mode)  # noqa: E731
    w = {}
    w["w_out"] = mk(d, d)
    w["gamma_ffn"] = q(1.0 + 0.1 * rng.standard_normal(d), mode)
    w["w_gate_up"] = mk(d, ffn)
    w["w_down"] = mk(ffn // 2, d)
    w["gamma_qkv"] = q(1.0 + 0.1 * rng.standard_normal(d), mode)
    w["w_qkv"] = mk(d, d + 2 * (d if kv_width is None else kv_width))
    return w


def grrg_forward(x, w0, z, gamma, w1, mode, eps=1e-6, tile_n=128, rtn=128) -> dict:
    """K4 -> finalize -> K5 (kernels.py:635-674)."""
    k4 = k_residual_partial_rms(x, w0, z, gamma, mode, tile_n, rtn)
    r = finalize_rms(k4["sumsq"], eps, mode)
    y = k_row_scale(k4["main"], w1, r, mode)["main"]
    return {"y": y, "pre_norm": k4["pre_norm"], "normed": k4["main"], "inv_rms": r}


def layer_forward(x, z, w: dict, cos, sin, mode, eps=1e-6, tile_n=128, rtn=128) -> dict:
    """Six-launch fused forward (kernels.py:810-869)."""
    k4a = k_residual_partial_rms(x, w["w_out"], z, w["gamma_ffn"], mode, tile_n, rtn)
    ra = finalize_rms(k4a["sumsq"], eps, mode)
    k6 = k_rms_swiglu(k4a["main"], w["w_gate_up"], ra, mode)
    k4b = k_residual_partial_rms(k6["main"], w["w_down"], k4a["pre_norm"], w["gamma_qkv"], mode, tile_n, rtn)
    rb = finalize_rms(k4b["sumsq"], eps, mode)
    qkv = k_rms_rope(k4b["main"], w["w_qkv"], rb, cos, sin, mode)["main"]
    return {"qkv": qkv, "residual": k4b["pre_norm"], "x": x, "pre_norm_a": k4a["pre_norm"], "inv_rms_a": ra,
            "preact": k6["preact"], "pre_norm_b": k4b["pre_norm"], "inv_rms_b": rb, "cos": cos, "sin": sin}


def layer_backward(grad_qkv, tape: dict, w: dict, mode, grad_residual=None, tile_m=128, tile_n=128,
                   rtn=128) -> dict:
    """Thirteen-launch fused backward (kernels.py:885-1013)."""
    d = w["w_out"].shape[0]
    gzb, rd_b = rope_backward_stat(grad_qkv, tape["qkv"], tape["cos"], tape["sin"], mode, tile_n, rtn)
    s_b = finalize_rowdot(rd_b, d, mode)
    k9b = k_rmsnorm_backward(gzb, w["w_qkv"], tape["pre_norm_b"], tape["inv_rms_b"], w["gamma_qkv"], s_b, mode,
                             grad_in=grad_residual, tile_m=tile_m, trans_b=True)
    gh1b = k9b["main"]
    g_wqkv = q(gemm(k9b["normed"], gzb, mode, trans_a=True), mode)
    g_gqkv = reduce_row_partials(k9b["gamma_grad"], mode)
    k10 = k_swiglu_backward(gh1b, w["w_down"], tape["preact"], mode, tile_n, rtn, trans_b=True)
    gza = k10["main"]
    s_a = finalize_rowdot(k10["rowdot"], d, mode)
    g_wdown = q(gemm(k10["recompute"], gh1b, mode, trans_a=True), mode)
    k9a = k_rmsnorm_backward(gza, w["w_gate_up"], tape["pre_norm_a"], tape["inv_rms_a"], w["gamma_ffn"], s_a,
                             mode, grad_in=gh1b, tile_m=tile_m, trans_b=True)
    gh1a = k9a["main"]
    g_wgu = q(gemm(k9a["normed"], gza, mode, trans_a=True), mode)
    g_gffn = reduce_row_partials(k9a["gamma_grad"], mode)
    g_x = q(gemm(gh1a, w["w_out"], mode, trans_b=True), mode)
    g_wout = q(gemm(tape["x"], gh1a, mode, trans_a=True), mode)
    return {"x": g_x, "z": gh1a, "w_out": g_wout, "gamma_ffn": g_gffn, "w_gate_up": g_wgu, "w_down": g_wdown,
            "gamma_qkv": g_gqkv, "w_qkv": g_wqkv,
            # intermediates used by size-independent checks
            "grad_zb": gzb, "grad_h1b": gh1b, "grad_za": gza, "s_a": s_a, "s_b": s_b}


# ----------------------------------------------------------------------------- float64 canonical reference


def _rms64(x, gamma, eps):
    r = 1.0 / np.sqrt(np.mean(x * x, axis=1) + eps)
    return x * r[:, None] * gamma[None, :], r


def _rms64_backward(gout, x, gamma, eps):
    r = 1.0 / np.sqrt(np.mean(x * x, axis=1) + eps)
    n = x * r[:, None]
    s = np.mean(gout * n * gamma[None, :], axis=1)
    return r[:, None] * (gout * gamma[None, :] - n * s[:, None]), np.sum(gout * n, axis=0)


def layer_ref_forward(x, z, w: dict, cos, sin, eps: float = 1e-6) -> dict:
    """Unfused canonical forward in float64 BLAS (oracles.py:178-205)."""
    f = lambda a: np.asarray(a, dtype=np.float64)  # noqa: E731
    h1a = f(x) @ f(w["w_out"]) + f(z)
    na, ra = _rms64(h1a, f(w["gamma_ffn"]), eps)
    za = na @ f(w["w_gate_up"])
    oa = swiglu(za)
    h1b = oa @ f(w["w_down"]) + h1a
    nb, rb = _rms64(h1b, f(w["gamma_qkv"]), eps)
    zb = nb @ f(w["w_qkv"])
    return {"h1a": h1a, "na": na, "ra": ra, "za": za, "oa": oa, "h1b": h1b, "nb": nb, "rb": rb, "zb": zb,
            "qkv": rope(zb, f(cos), f(sin))}


def layer_ref_backward(grad_qkv, grad_residual, fwd: dict, x, w: dict, cos, sin, eps: float = 1e-6) -> dict:
    """Analytic float64 backward of layer_ref_forward (oracles.py:208-229)."""
    f = lambda a: np.asarray(a, dtype=np.float64)  # noqa: E731
    g = f(grad_qkv)
    gzb = np.empty_like(g)
    c, s = f(cos), f(sin)
    gzb[:, 0::2] = g[:, 0::2] * c[:, 0::2] + g[:, 1::2] * s[:, 1::2]
    gzb[:, 1::2] = -g[:, 0::2] * s[:, 0::2] + g[:, 1::2] * c[:, 1::2]
    gnb = gzb @ f(w["w_qkv"]).T
    g_wqkv = fwd["nb"].T @ gzb
    gh1b, g_gqkv = _rms64_backward(gnb, fwd["h1b"], f(w["gamma_qkv"]), eps)
    if grad_residual is not None:
        gh1b = gh1b + f(grad_residual)
    goa = gh1b @ f(w["w_down"]).T
    g_wdown = fwd["oa"].T @ gh1b
    gza, _, _ = swiglu_backward(goa, fwd["za"])
    gna = gza @ f(w["w_gate_up"]).T
    g_wgu = fwd["na"].T @ gza
    gh1a, g_gffn = _rms64_backward(gna, fwd["h1a"], f(w["gamma_ffn"]), eps)
    gh1a = gh1a + gh1b
    return {"x": gh1a @ f(w["w_out"]).T, "z": gh1a.copy(), "w_out": f(x).T @ gh1a, "gamma_ffn": g_gffn,
            "w_gate_up": g_wgu, "w_down": g_wdown, "gamma_qkv": g_gqkv, "w_qkv": g_wqkv}


GRAD_KEYS = ("x", "z", "w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv", "w_qkv")


# ----------------------------------------------------------------------------- LM head (forward pinned, backward derived)


def lm_head_forward(a, b, z, gamma, w_vocab, labels, mode, eps=1e-6, tile_n=128, rtn=128) -> dict:
    """K4 -> finalize -> K8 -> combine_lse -> CE finalize (kernels.py:1032-1076)."""
    k4 = k_residual_partial_rms(a, b, z, gamma, mode, tile_n, rtn)
    r = finalize_rms(k4["sumsq"], eps, mode)
    k8 = k_partial_xent(k4["main"], w_vocab, labels, mode, tile_n, rtn, scale=r)
    lse = combine_lse(k8["lse"], mode)
    losses = stat_q(lse - k8["target"], mode)
    return {"losses": losses, "mean": float(np.mean(losses)), "lse": lse, "normed": k4["main"],
            "pre_norm": k4["pre_norm"], "inv_rms": r, "logits": k8["main"]}


def lm_head_backward(fwd: dict, a, b, gamma, w_vocab, labels, mode, grad_loss=1.0, tile_m=128, tile_n=128,
                     rtn=128) -> dict:
    """Backward of the mean cross entropy through the LM head, in the fused order of the GPU
    extension (no reference counterpart; SPEC.md:415 ends at the loss).  The pieces follow the
    reference's own backward patterns: the logit gradient is softmax - onehot; the RMSNorm
    statistic is relocated to <logits, d logits> exactly as rope_backward_stat relocates it to
    <qkv, d qkv> (kernels.py:560-617), then k_rmsnorm_backward (kernels.py:474-525) and the
    weight gradients as in layer_backward (kernels.py:885-1013).  Pinned by finite differences
    of the f64 forward (tests/test_oracle_golden.py)."""
    dt = acc_dtype(mode)
    m = fwd["normed"].shape[0]
    t = gemm(fwd["normed"], w_vocab, mode) * _cast(fwd["inv_rms"], mode)[:, None]
    p = np.exp(t - _cast(fwd["lse"], mode)[:, None])
    p[np.arange(m), np.asarray(labels, dtype=np.int64)] -= dt(1.0)
    g = p * dt(grad_loss / m)
    blocks = row_blocks(t.shape[1], tile_n, rtn)
    s = finalize_rowdot((row_partials(t * g, blocks), counts_of(blocks)), fwd["normed"].shape[1], mode)
    glog = q(g, mode)
    k9 = k_rmsnorm_backward(glog, w_vocab, fwd["pre_norm"], fwd["inv_rms"], gamma, s, mode, tile_m=tile_m,
                            trans_b=True)
    gh = k9["main"]
    return {"a": q(gemm(gh, b, mode, trans_b=True), mode), "b": q(gemm(a, gh, mode, trans_a=True), mode),
            "z": gh, "gamma": reduce_row_partials(k9["gamma_grad"], mode),
            "w_vocab": q(gemm(k9["normed"], glog, mode, trans_a=True), mode), "d_logits": glog, "s": s}


def lm_head_loss64(a, b, z, gamma, w_vocab, labels, eps=1e-6) -> float:
    """Canonical float64 mean cross entropy of the LM head (oracles.py restated): RMSNorm with
    gain, vocabulary projection, log-softmax at the label."""
    f = lambda x: np.asarray(x, dtype=np.float64)  # noqa: E731
    h = f(a) @ f(b) + f(z)
    r = 1.0 / np.sqrt(np.mean(h * h, axis=1) + eps)
    logits = (h * r[:, None] * f(gamma)[None, :]) @ f(w_vocab)
    mx = logits.max(axis=1)
    lse = mx + np.log(np.exp(logits - mx[:, None]).sum(axis=1))
    return float(np.mean(lse - logits[np.arange(len(labels)), np.asarray(labels, dtype=np.int64)]))
