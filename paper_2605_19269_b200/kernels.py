"""Fused transformer launches and the layer pipelines, B200 edition.

Every `gemm_*` function is ONE persistent sm_100a kernel launch whose
epilogue program is the reference's (tilefuse/kernels.py:243-557); the
pipelines chain them on the current CUDA stream with no host
synchronisation (tilefuse/kernels.py:635-1076).  The normalization gain is
folded into the producing launch (RowVecMul) and the inverse RMS into the
consuming one (RowScale), so the normalized activations never take an extra
HBM round trip.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _native as nat
from . import traffic
from .engine import GemmProblem, KernelResult, block_starts, run_gemm
from .epilogue import (
    AuxTileStore,
    CrossEntropyBackward,
    PartialRowDot,
    EpilogueProgram,
    OnlineLse,
    PairwiseRope,
    PairwiseSwiglu,
    PairwiseSwigluBackward,
    PartialSlot,
    PartialSumSq,
    ResidualAdd,
    RmsNormBackwardLocal,
    RowScale,
    RowVecMul,
    StoreKind,
    TargetGather,
)
from .errors import ConfigError, DimensionError, TapeError
from .reductions import (
    combine_lse,
    cross_entropy_finalize,
    finalize_rms,
    finalize_rowdot,
    reduce_row_partials,
)
from .tensors import (
    DenseMatrix,
    PrecisionMode,
    TileShape,
    Vector,
    alloc_matrix,
    default_device,
    quantize,
)
from .traffic import LaunchRecord, TrafficLedger


def ffn_width(hidden: int) -> int:
    """floor(8*hidden/3) rounded up to a multiple of 256 (kernels.py:64-73)."""
    if hidden <= 0:
        raise ConfigError(f"hidden size must be positive, got {hidden}")
    return -(-((8 * hidden) // 3) // 256) * 256


@dataclass(frozen=True)
class PipelineConfig:
    """Shape, tiling and precision shared by a pipeline (kernels.py:76-121)."""

    hidden: int
    ffn: Optional[int] = None
    tile_m: int = 128
    tile_n: int = 128
    reduction_tile_n: int = 128
    precision: PrecisionMode = PrecisionMode.EXACT64
    eps: float = 1e-6
    rope_base: float = 10000.0
    # GQA extension (no reference counterpart): width of each of the k and v spans of the
    # packed projection.  None = hidden, the reference's packed (q, k, v) of width 3*hidden.
    kv_width: Optional[int] = None
    # B200 extension (north_star "gamma folded into W"): the RMSNorm gains are folded into
    # the consuming weights (W' = diag(gamma) W, formed once per weight update by
    # fold_gains), so the producing K4 launches store only pre_norm; the backward recovers
    # dW = diag(gamma) dW' and dgamma = rowsum(W * dW') in the weight-gradient epilogue.
    fold_gamma: bool = False

    def __post_init__(self):
        if self.hidden <= 0:
            raise ConfigError(f"hidden size must be positive, got {self.hidden}")
        if self.hidden % 2:
            raise ConfigError("hidden size must be even (rotary pairs)")
        if self.ffn is not None and (self.ffn <= 0 or self.ffn % 2):
            raise ConfigError(f"ffn width must be positive and even, got {self.ffn}")
        if min(self.tile_m, self.tile_n, self.reduction_tile_n) <= 0:
            raise ConfigError("tile parameters must be positive")
        if self.eps <= 0:
            raise ConfigError("eps must be positive")
        if self.kv_width is not None and (self.kv_width <= 0 or self.kv_width % 2):
            raise ConfigError(f"kv width must be positive and even, got {self.kv_width}")

    @property
    def ffn_resolved(self) -> int:
        return self.ffn if self.ffn is not None else ffn_width(self.hidden)

    @property
    def kv_resolved(self) -> int:
        return self.hidden if self.kv_width is None else self.kv_width

    @property
    def qkv_width(self) -> int:
        """Packed projection width: q (hidden) + k + v (kv each); 3*hidden by default."""
        return self.hidden + 2 * self.kv_resolved

    @property
    def tile_shape(self) -> TileShape:
        return TileShape(self.tile_m, self.tile_n)

    def launch_kw(self, ledger=None) -> dict:
        return dict(tile_shape=self.tile_shape, reduction_tile_n=self.reduction_tile_n,
                    precision=self.precision, ledger=ledger)


def _problem(a: DenseMatrix, b: DenseMatrix, *, trans_a=False, trans_b=False, tile_shape=TileShape(128, 128),
             reduction_tile_n=128, precision=PrecisionMode.EXACT64) -> GemmProblem:
    m, k = (a.shape[1], a.shape[0]) if trans_a else a.shape
    n, kb = (b.shape[0], b.shape[1]) if trans_b else (b.shape[1], b.shape[0])
    if k != kb:
        raise DimensionError(f"contraction dims differ: a gives {k}, b gives {kb}")
    return GemmProblem(m=m, n=n, k=k, trans_a=trans_a, trans_b=trans_b, tile_shape=tile_shape,
                       reduction_tile_n=reduction_tile_n, precision=precision)


_programs: dict = {}


def _program(prims) -> EpilogueProgram:
    """Validated programs are immutable: build each distinct primitive sequence once."""
    key = tuple(repr(p) for p in prims)
    prog = _programs.get(key)
    if prog is None:
        prog = _programs[key] = EpilogueProgram(prims)
    return prog


def _launch(name, a, b, prims, bindings, *, trans_a=False, trans_b=False, tile_shape=TileShape(128, 128),
            reduction_tile_n=128, precision=PrecisionMode.EXACT64, ledger=None, tile_order=None,
            store_main=True, out_f32=False) -> KernelResult:
    prob = _problem(a, b, trans_a=trans_a, trans_b=trans_b, tile_shape=tile_shape,
                    reduction_tile_n=reduction_tile_n, precision=precision)
    return run_gemm(prob, a, b, _program(prims), bindings, kernel_name=name, ledger=ledger,
                    tile_order=tile_order, store_main=store_main, out_f32=out_f32)


# ---------------------------------------------------------------------------
# rotary tables (kernels.py:156-206)


def _angles(m: int, width: int, base: float, start: int) -> np.ndarray:
    inv_freq = base ** (-2.0 * np.arange(width // 2, dtype=np.float64) / width)
    return (start + np.arange(m, dtype=np.float64))[:, None] * inv_freq[None, :]


def rope_tables(m: int, width: int, *, base: float = 10000.0, start: int = 0,
                precision: PrecisionMode = PrecisionMode.EXACT64) -> tuple[DenseMatrix, DenseMatrix]:
    """cos/sin tables of angle (start+t) * base^(-2p/width), duplicated per pair."""
    import torch

    if width <= 0 or width % 2:
        raise DimensionError(f"rotary width must be positive and even, got {width}")
    if m <= 0:
        raise DimensionError(f"table rows must be positive, got {m}")
    ang = _angles(m, width, base, start)
    dev = default_device()
    out, halves = [], []
    for fn in (np.cos, np.sin):
        half = torch.from_numpy(quantize(fn(ang), precision)).to(dev, dtype=precision.torch_dtype)
        full = alloc_matrix(m, width, precision.torch_dtype, dev)
        full[:, 0::2] = half
        full[:, 1::2] = half
        out.append(DenseMatrix._wrap(full, precision))
        halves.append(half.contiguous())
    if precision is PrecisionMode.SIMBF16 and width % 32 == 0:
        # compact form (one angle per pair, half the bytes) for a rotation over exactly
        # `width` columns: the RopeCompact rule with hidden = width maps column c < width
        # to angle c // 2 (the fused forward epilogue; rope_backward_stat keeps the full
        # tables for it)
        spec = RopeCompact(cos=halves[0], sin=halves[1], hidden=width)
        out[0]._rope = (spec, "cos")
        out[1]._rope = (spec, "sin")
    return out[0], out[1]


def qkv_rope_tables(m: int, hidden: int, *, base: float = 10000.0, start: int = 0,
                    precision: PrecisionMode = PrecisionMode.EXACT64,
                    kv_width: Optional[int] = None) -> tuple[DenseMatrix, DenseMatrix]:
    """Tables for packed (q, k, v): q and k rotate, v is identity (kernels.py:184-206).

    kv_width None (= hidden) is the reference layout, q and k sharing angles.  With a GQA
    kv_width the k span rotates by the reference rule applied to its own width.
    """
    kv = hidden if kv_width is None else kv_width
    c_h, s_h = rope_tables(m, hidden, base=base, start=start, precision=precision)
    c_k, s_k = (c_h, s_h) if kv == hidden else rope_tables(m, kv, base=base, start=start, precision=precision)
    dev = c_h.tensor.device
    out = []
    for src, srck, fill in ((c_h, c_k, 1.0), (s_h, s_k, 0.0)):
        full = alloc_matrix(m, hidden + 2 * kv, precision.torch_dtype, dev)
        full[:, :hidden] = src.tensor
        full[:, hidden:hidden + kv] = srck.tensor
        full[:, hidden + kv:] = fill
        out.append(DenseMatrix._wrap(full, precision))
    if precision is PrecisionMode.SIMBF16 and kv == hidden and hidden % 32 == 0:
        # compact form for the kernels: one angle per pair of the q span (the k span
        # repeats it, the v span is the identity) -- the same bf16 values, 1/6 the bytes
        spec = RopeCompact(cos=c_h.tensor[:, 0::2].contiguous(), sin=s_h.tensor[:, 0::2].contiguous(),
                           hidden=hidden)
        out[0]._rope = (spec, "cos")
        out[1]._rope = (spec, "sin")
    return out[0], out[1]


@dataclass(frozen=True)
class RopeCompact:
    """Compact packed-qkv RoPE tables: (m, hidden/2) bf16 cos/sin, one value per pair.

    Columns [0, 2*hidden) of the full table hold cos[:, (col % hidden) // 2] (q and k
    spans share angles, kernels.py:184-206); columns >= 2*hidden are cos 1 / sin 0.
    A plain `rope_tables(m, width)` pair is the case hidden = width = the table width."""

    cos: object
    sin: object
    hidden: int


def rope_compact_of(cos: DenseMatrix, sin: DenseMatrix) -> Optional[RopeCompact]:
    """The compact form shared by a (cos, sin) pair built together by qkv_rope_tables.

    Each table carries its role; the compact path is taken only when `cos` is that
    pair's cos table and `sin` its sin table (swapped or duplicated tables run the
    full-table path, which reads exactly what was bound)."""
    c, s = getattr(cos, "_rope", None), getattr(sin, "_rope", None)
    if c is None or s is None or c[0] is not s[0] or c[1] != "cos" or s[1] != "sin":
        return None
    spec = c[0]
    if cos.precision is not PrecisionMode.SIMBF16 or cos.rows != spec.cos.shape[0]:
        return None
    return spec


def interleave_gate_up(gate: DenseMatrix, up: DenseMatrix) -> DenseMatrix:
    """Split (gate, up) weights -> interleaved columns (kernels.py:209-226)."""
    if gate.shape != up.shape:
        raise DimensionError(f"gate and up shapes differ: {gate.shape} vs {up.shape}")
    if gate.precision is not up.precision:
        raise ConfigError("gate and up precisions differ")
    out = alloc_matrix(gate.rows, 2 * gate.cols, gate.tensor.dtype, gate.tensor.device)
    out[:, 0::2] = gate.tensor
    out[:, 1::2] = up.tensor
    return DenseMatrix._wrap(out, gate.precision)


def split_gate_up(w: DenseMatrix) -> tuple[DenseMatrix, DenseMatrix]:
    """Inverse of interleave_gate_up (kernels.py:229-236)."""
    if w.cols % 2:
        raise DimensionError(f"interleaved width must be even, got {w.cols}")
    g = alloc_matrix(w.rows, w.cols // 2, w.tensor.dtype, w.tensor.device)
    u = alloc_matrix(w.rows, w.cols // 2, w.tensor.dtype, w.tensor.device)
    g.copy_(w.tensor[:, 0::2])
    u.copy_(w.tensor[:, 1::2])
    return DenseMatrix._wrap(g, w.precision), DenseMatrix._wrap(u, w.precision)


def scale_rows(w: DenseMatrix, gain: Vector) -> DenseMatrix:
    """bf16(diag(gain) W): one HBM-bound launch (csrc coda_scale_rows)."""
    import ctypes
    import torch

    if w.precision is not PrecisionMode.SIMBF16:
        raise ConfigError("gain folding is implemented for the bf16 (SIMBF16) path")
    if len(gain) != w.rows:
        raise DimensionError(f"gain has length {len(gain)}, expected {w.rows}")
    t = w.tensor
    out = alloc_matrix(t.shape[0], t.shape[1], torch.bfloat16, t.device)
    g = gain.tensor if gain.tensor.dtype == torch.float32 else gain.tensor.float()
    nat.call("coda_scale_rows", ctypes.byref(nat.tensor_desc(t)), g.contiguous().data_ptr(),
             ctypes.byref(nat.tensor_desc(out)), torch.cuda.current_stream(t.device).cuda_stream,
             tag="fold_gain")
    return DenseMatrix._wrap(out, w.precision)


@dataclass(frozen=True)
class FoldedGains:
    """Gain-folded consumer weights: w_gate_up' = diag(gamma_ffn) w_gate_up and
    w_qkv' = diag(gamma_qkv) w_qkv (bf16), valid for one set of weights."""

    w_gate_up: DenseMatrix
    w_qkv: DenseMatrix


def fold_gains(weights: "LayerWeights") -> FoldedGains:
    """Form the folded weights once per weight update (two HBM-bound launches)."""
    return FoldedGains(w_gate_up=scale_rows(weights.w_gate_up, weights.gamma_ffn),
                       w_qkv=scale_rows(weights.w_qkv, weights.gamma_qkv))


_ones_cache: dict = {}


def _ones(n: int, precision: PrecisionMode, device) -> Vector:
    import torch

    key = (n, precision, str(device))
    v = _ones_cache.get(key)
    if v is None:
        v = _ones_cache[key] = Vector._wrap(torch.ones(n, dtype=precision.vector_torch_dtype, device=device),
                                            precision)
    return v


def gemm_wgrad_gain(a, b, weight, gain, *, precision=PrecisionMode.EXACT64, tile_shape=TileShape(128, 128),
                    reduction_tile_n=128, ledger=None, out_f32=False):
    """Weight gradient of a gain-folded weight: with dW' = a^T b (trans_a), returns
    main = diag(gain) dW' and aux "gain_dot" = per-row block partials of sum(W * dW'),
    i.e. [PartialRowDot(W), RowScale(gain)] on the wgrad tile (both linear in dW', so
    they commute with the data-parallel all-reduce)."""
    return _launch(traffic.K_GEMM, a, b, [PartialRowDot("weight", "gain_dot"), RowScale("gain")],
                   {"weight": weight, "gain": gain}, trans_a=True, tile_shape=tile_shape,
                   reduction_tile_n=reduction_tile_n, precision=precision, ledger=ledger, out_f32=out_f32)


# ---------------------------------------------------------------------------
# single-launch kernels (kernels.py:243-557)

def gemm_rope(a, b, cos, sin, *, backward=False, trans_b=False, tile_shape=TileShape(128, 128),
              reduction_tile_n=128, precision=PrecisionMode.EXACT64, ledger=None, tile_order=None):
    """K1: GEMM + pairwise rotation."""
    return _launch(traffic.K_ROPE, a, b, [PairwiseRope("cos", "sin", backward=backward)],
                   {"cos": cos, "sin": sin}, trans_b=trans_b, tile_shape=tile_shape,
                   reduction_tile_n=reduction_tile_n, precision=precision, ledger=ledger, tile_order=tile_order)


def gemm_swiglu(a, b, *, save_preact=False, trans_b=False, tile_shape=TileShape(128, 128), reduction_tile_n=128,
                precision=PrecisionMode.EXACT64, ledger=None, tile_order=None):
    """K2: GEMM over interleaved (gate, up) + gated activation (optionally saving the preactivation)."""
    prims = ([AuxTileStore("preact")] if save_preact else []) + [PairwiseSwiglu()]
    return _launch(traffic.K_SWIGLU, a, b, prims, {}, trans_b=trans_b, tile_shape=tile_shape,
                   reduction_tile_n=reduction_tile_n, precision=precision, ledger=ledger, tile_order=tile_order)


def gemm_partial_xent(a, b, labels, *, store_logits=True, trans_b=False, tile_shape=TileShape(128, 128),
                      reduction_tile_n=128, precision=PrecisionMode.EXACT64, ledger=None, tile_order=None):
    """K3: logit GEMM + target gather + streamed LSE pairs."""
    return _launch(traffic.K_PARTIAL_XENT, a, b, [TargetGather("labels", "target"), OnlineLse("lse")],
                   {"labels": labels}, trans_b=trans_b, tile_shape=tile_shape, reduction_tile_n=reduction_tile_n,
                   precision=precision, ledger=ledger, tile_order=tile_order, store_main=store_logits)


def gemm_residual_partial_rms(a, b, residual, gamma, *, trans_b=False, tile_shape=TileShape(128, 128),
                              reduction_tile_n=128, precision=PrecisionMode.EXACT64, ledger=None,
                              tile_order=None, gamma_folded=False):
    """K4: GEMM + residual + pre-norm save + sum-of-squares partials + gain.

    `gamma_folded=True` (B200 extension) skips the RowVecMul because the gain
    has already been folded into the consuming weight matrix.
    """
    prims = [ResidualAdd("residual"), AuxTileStore("pre_norm"), PartialSumSq("sumsq")]
    binds = {"residual": residual}
    if not gamma_folded:
        prims.append(RowVecMul("gamma"))
        binds["gamma"] = gamma
    return _launch(traffic.K_RESIDUAL_RMS, a, b, prims, binds, trans_b=trans_b, tile_shape=tile_shape,
                   reduction_tile_n=reduction_tile_n, precision=precision, ledger=ledger, tile_order=tile_order,
                   store_main=not gamma_folded)


def gemm_row_scale(a, b, scale, *, trans_b=False, tile_shape=TileShape(128, 128), reduction_tile_n=128,
                   precision=PrecisionMode.EXACT64, ledger=None, tile_order=None):
    """K5: GEMM + deferred per-row scale."""
    return _launch(traffic.K_ROW_SCALE, a, b, [RowScale("scale")], {"scale": scale}, trans_b=trans_b,
                   tile_shape=tile_shape, reduction_tile_n=reduction_tile_n, precision=precision, ledger=ledger,
                   tile_order=tile_order)


def gemm_rms_swiglu(a, b, scale, *, trans_b=False, tile_shape=TileShape(128, 128), reduction_tile_n=128,
                    precision=PrecisionMode.EXACT64, ledger=None, tile_order=None):
    """K6: row scale + preactivation save + gated activation."""
    return _launch(traffic.K_RMS_SWIGLU, a, b, [RowScale("scale"), AuxTileStore("preact"), PairwiseSwiglu()],
                   {"scale": scale}, trans_b=trans_b, tile_shape=tile_shape, reduction_tile_n=reduction_tile_n,
                   precision=precision, ledger=ledger, tile_order=tile_order)


def gemm_rms_rope(a, b, scale, cos, sin, *, trans_b=False, tile_shape=TileShape(128, 128), reduction_tile_n=128,
                  precision=PrecisionMode.EXACT64, ledger=None, tile_order=None):
    """K7: row scale + pairwise rotation."""
    return _launch(traffic.K_RMS_ROPE, a, b, [RowScale("scale"), PairwiseRope("cos", "sin")],
                   {"scale": scale, "cos": cos, "sin": sin}, trans_b=trans_b, tile_shape=tile_shape,
                   reduction_tile_n=reduction_tile_n, precision=precision, ledger=ledger, tile_order=tile_order)


def gemm_rms_partial_xent(a, b, scale, labels, *, store_logits=False, trans_b=False,
                          tile_shape=TileShape(128, 128), reduction_tile_n=128, precision=PrecisionMode.EXACT64,
                          ledger=None, tile_order=None):
    """K8: row scale + target gather + streamed LSE; logits stay on chip unless stored."""
    return _launch(traffic.K_RMS_XENT, a, b,
                   [RowScale("scale"), TargetGather("labels", "target"), OnlineLse("lse")],
                   {"scale": scale, "labels": labels}, trans_b=trans_b, tile_shape=tile_shape,
                   reduction_tile_n=reduction_tile_n, precision=precision, ledger=ledger, tile_order=tile_order,
                   store_main=store_logits)


def gemm_rmsnorm_backward(a, b, pre_norm, inv_rms, gamma, stat, *, grad_in=None, trans_a=False, trans_b=False,
                          tile_shape=TileShape(128, 128), reduction_tile_n=128, precision=PrecisionMode.EXACT64,
                          ledger=None, tile_order=None):
    """K9: gradient GEMM fused with the normalization backward (+ residual gradient)."""
    acc = "grad_in" if grad_in is not None else None
    binds = {"pre_norm": pre_norm, "inv_rms": inv_rms, "gamma": gamma, "stat": stat}
    if grad_in is not None:
        binds["grad_in"] = grad_in
    prim = RmsNormBackwardLocal("pre_norm", "inv_rms", "gamma", "stat", accumulate=acc, normed_out="normed",
                                gamma_grad="gamma_grad")
    return _launch(traffic.K_RMSNORM_BWD, a, b, [prim], binds, trans_a=trans_a, trans_b=trans_b,
                   tile_shape=tile_shape, reduction_tile_n=reduction_tile_n, precision=precision, ledger=ledger,
                   tile_order=tile_order)


def gemm_swiglu_backward(a, b, preact, *, trans_b=False, tile_shape=TileShape(128, 128), reduction_tile_n=128,
                         precision=PrecisionMode.EXACT64, ledger=None, tile_order=None):
    """K10: gradient GEMM fused with the gated-activation backward (width x2)."""
    return _launch(traffic.K_SWIGLU_BWD, a, b, [PairwiseSwigluBackward("preact", "recompute", "rowdot")],
                   {"preact": preact}, trans_b=trans_b, tile_shape=tile_shape, reduction_tile_n=reduction_tile_n,
                   precision=precision, ledger=ledger, tile_order=tile_order)


def rope_backward_stat(grad: DenseMatrix, rotated: DenseMatrix, cos: DenseMatrix, sin: DenseMatrix, *,
                       tile_n: int = 128, reduction_tile_n: int = 128,
                       precision: PrecisionMode = PrecisionMode.EXACT64,
                       ledger: Optional[TrafficLedger] = None) -> tuple[DenseMatrix, PartialSlot]:
    """Boundary pass: counter-rotate the qkv gradient and emit <rotated, grad> row-block partials.

    Rotation preserves row dot products, so these partials are those of
    <preact, grad_preact> (kernels.py:560-617).  One HBM-bound kernel.
    """
    import ctypes
    import torch

    from .engine import storage_tensor

    if precision is PrecisionMode.EXACT64:
        raise ConfigError("EXACT64 runs only in the CPU oracle; the GPU engine supports SIM32 and SIMBF16")
    m, n = grad.shape
    for name, t in (("rotated", rotated), ("cos", cos), ("sin", sin)):
        if t.shape != (m, n):
            raise DimensionError(f"{name} has shape {t.shape}, expected {(m, n)}")
    if n % 2:
        raise DimensionError(f"rotary width must be even, got {n}")
    ts = [storage_tensor(x, precision) for x in (grad, rotated, cos, sin)]
    dev = ts[0].device
    gz = alloc_matrix(m, n, precision.torch_dtype, dev)
    bst, nb, counts = block_starts(n, tile_n, reduction_tile_n, dev)
    rowdot = torch.empty((m, nb), dtype=torch.float32, device=dev)
    descs = [nat.tensor_desc(t) for t in ts]
    gzd = nat.tensor_desc(gz)
    uniform128 = all(int(w) == 128 for w in counts[:-1]) and int(counts[-1]) <= 128
    spec = rope_compact_of(cos, sin) if precision is PrecisionMode.SIMBF16 else None
    stream = torch.cuda.current_stream(dev).cuda_stream
    if spec is not None and uniform128 and 2 * spec.hidden <= n:
        cd_, sd_ = nat.tensor_desc(spec.cos), nat.tensor_desc(spec.sin)
        nat.call("coda_rope_backward_stat_compact", ctypes.byref(descs[0]), ctypes.byref(descs[1]),
                 ctypes.byref(cd_), ctypes.byref(sd_), spec.hidden, ctypes.byref(gzd), rowdot.data_ptr(),
                 rowdot.stride(0), stream, tag="rope_backward_stat", flops=0.0)
    else:
        nat.call("coda_rope_backward_stat", *[ctypes.byref(d) for d in descs],
                 None if uniform128 else bst.data_ptr(), nb, ctypes.byref(gzd), rowdot.data_ptr(), rowdot.stride(0),
                 stream, tag="rope_backward_stat", flops=0.0)
    slot = PartialSlot(StoreKind.ROW_SUM, rowdot, counts, precision).freeze()
    w, pw = precision.storage_bytes, precision.partial_bytes
    rec = LaunchRecord(traffic.K_ROPE_BWD_STAT, 4 * m * n * w, m * n * w + m * nb * pw)
    if ledger is not None:
        ledger.add(rec)
    return DenseMatrix._wrap(gz, precision), slot


# ---------------------------------------------------------------------------
# GEMM -> residual -> normalize -> GEMM (kernels.py:624-713)


@dataclass
class GrrgResult:
    y: DenseMatrix
    pre_norm: DenseMatrix
    normed: DenseMatrix
    inv_rms: Vector
    ledger: TrafficLedger


def pipeline_grrg_forward(x, w0, z, gamma, w1, *, config: PipelineConfig) -> GrrgResult:
    """K4 -> finalize_rms -> K5: three launches, no full-width re-read of the normalized rows."""
    ledger = TrafficLedger()
    kw = config.launch_kw(ledger)
    k4 = gemm_residual_partial_rms(x, w0, z, gamma, **kw)
    r = finalize_rms(k4.aux["sumsq"], config.eps, ledger=ledger)
    k5 = gemm_row_scale(k4.main, w1, r, **kw)
    return GrrgResult(y=k5.main, pre_norm=k4.aux["pre_norm"], normed=k4.main, inv_rms=r, ledger=ledger)


def pipeline_grrg_canonical(x, w0, z, gamma, w1, *, config: PipelineConfig):
    """Unfused reference schedule (kernels.py:677-713) on cuBLAS + torch elementwise.

    A comparator, not the product path: four standalone ops with every
    intermediate stored at the storage precision.  Returns (y, canonical ledger).
    """
    from . import unfused

    if config.precision is PrecisionMode.EXACT64:
        raise ConfigError("EXACT64 runs only in the CPU oracle; the GPU engine supports SIM32 and SIMBF16")
    P = config.precision
    t = lambda m: m.tensor.to(P.torch_dtype)  # noqa: E731
    y = unfused.grrg(t(x), t(w0), t(z), gamma.tensor.float(), t(w1), config.eps)
    m, k = x.shape
    d, n = w0.shape[1], w1.shape[1]
    ledger = TrafficLedger()
    w, pw = P.storage_bytes, P.partial_bytes
    ledger.record("gemm", (m * k + k * d) * w, m * d * w)
    ledger.record("residual_add", 2 * m * d * w, m * d * w)
    ledger.record("rmsnorm", (m * d + d) * w, m * d * w)
    ledger.record("gemm", (m * d + d * n) * w, m * n * w)
    out = alloc_matrix(y.shape[0], y.shape[1], y.dtype, y.device)
    out.copy_(y)
    return DenseMatrix._wrap(out, P), ledger


# ---------------------------------------------------------------------------
# transformer layer (kernels.py:716-1013)


@dataclass(frozen=True)
class LayerWeights:
    """Out-proj, interleaved gated FFN and packed qkv weights of one block."""

    w_out: DenseMatrix        # (d, d)
    gamma_ffn: Vector         # (d,)
    w_gate_up: DenseMatrix    # (d, ffn) interleaved gate/up
    w_down: DenseMatrix       # (ffn/2, d)
    gamma_qkv: Vector         # (d,)
    w_qkv: DenseMatrix        # (d, d + 2 kv) = (d, 3d) for the reference layout

    def check(self, config: PipelineConfig) -> None:
        d, f, qw = config.hidden, config.ffn_resolved, config.qkv_width
        for name, got, want in (
            ("w_out", self.w_out.shape, (d, d)),
            ("gamma_ffn", (len(self.gamma_ffn),), (d,)),
            ("w_gate_up", self.w_gate_up.shape, (d, f)),
            ("w_down", self.w_down.shape, (f // 2, d)),
            ("gamma_qkv", (len(self.gamma_qkv),), (d,)),
            ("w_qkv", self.w_qkv.shape, (d, qw)),
        ):
            if got != want:
                raise DimensionError(f"{name} has shape {got}, expected {want}")

    @classmethod
    def random(cls, rng: np.random.Generator, config: PipelineConfig, scale: float = 0.2) -> "LayerWeights":
        """Same draw order as the reference (kernels.py:750-767): N(0,1)*scale, gains 1+0.1N."""
        d, f, p = config.hidden, config.ffn_resolved, config.precision

        def mk(*shape):
            return DenseMatrix.from_array(rng.standard_normal(shape) * scale, p)

        w_out = mk(d, d)
        g_ffn = Vector.from_array(1.0 + 0.1 * rng.standard_normal(d), p)
        w_gu = mk(d, f)
        w_down = mk(f // 2, d)
        g_qkv = Vector.from_array(1.0 + 0.1 * rng.standard_normal(d), p)
        w_qkv = mk(d, config.qkv_width)
        return cls(w_out=w_out, gamma_ffn=g_ffn, w_gate_up=w_gu, w_down=w_down, gamma_qkv=g_qkv, w_qkv=w_qkv)


@dataclass
class LayerTape:
    """Forward state saved for layer_backward."""

    x: DenseMatrix
    pre_norm_a: DenseMatrix
    inv_rms_a: Vector
    preact: DenseMatrix
    pre_norm_b: DenseMatrix
    inv_rms_b: Vector
    qkv: DenseMatrix
    cos: DenseMatrix
    sin: DenseMatrix
    folded: Optional[FoldedGains] = None   # fold_gamma: the folded weights the forward used

    def check(self, config: PipelineConfig) -> None:
        m, d = self.x.shape
        if config.fold_gamma and self.folded is None:
            raise TapeError("fold_gamma backward needs the folded weights of its forward (tape.folded)")
        f, qw = config.ffn_resolved, config.qkv_width
        for name, got, want in (
            ("pre_norm_a", self.pre_norm_a.shape, (m, d)),
            ("preact", self.preact.shape, (m, f)),
            ("pre_norm_b", self.pre_norm_b.shape, (m, d)),
            ("qkv", self.qkv.shape, (m, qw)),
            ("cos", self.cos.shape, (m, qw)),
            ("sin", self.sin.shape, (m, qw)),
        ):
            if got != want:
                raise TapeError(f"tape entry {name} has shape {got}, expected {want}")
        if len(self.inv_rms_a) != m or len(self.inv_rms_b) != m:
            raise TapeError("tape inverse-RMS vectors must have one entry per row")


@dataclass
class LayerForwardResult:
    qkv: DenseMatrix
    residual: DenseMatrix
    tape: LayerTape
    ledger: TrafficLedger


def layer_forward(x: DenseMatrix, z: DenseMatrix, weights: LayerWeights, cos: DenseMatrix, sin: DenseMatrix, *,
                  config: PipelineConfig, folded: Optional[FoldedGains] = None) -> LayerForwardResult:
    """Six launches: K4 -> finalize -> K6 -> K4 -> finalize -> K7 (kernels.py:810-869).

    With `config.fold_gamma` the K4 launches store only pre_norm (no gained copy) and K6/K7
    read pre_norm against the folded weights; `folded` (from fold_gains) may be passed when
    the weights did not change since it was formed, otherwise two fold launches run first."""
    weights.check(config)
    if x.shape != z.shape:
        raise DimensionError(f"x and z shapes differ: {x.shape} vs {z.shape}")
    ledger = TrafficLedger()
    kw = config.launch_kw(ledger)
    if config.fold_gamma:
        if folded is None:
            folded = fold_gains(weights)
        k4a = gemm_residual_partial_rms(x, weights.w_out, z, weights.gamma_ffn, gamma_folded=True, **kw)
        ra = finalize_rms(k4a.aux["sumsq"], config.eps, ledger=ledger)
        k6 = gemm_rms_swiglu(k4a.aux["pre_norm"], folded.w_gate_up, ra, **kw)
        k4b = gemm_residual_partial_rms(k6.main, weights.w_down, k4a.aux["pre_norm"], weights.gamma_qkv,
                                        gamma_folded=True, **kw)
        rb = finalize_rms(k4b.aux["sumsq"], config.eps, ledger=ledger)
        k7 = gemm_rms_rope(k4b.aux["pre_norm"], folded.w_qkv, rb, cos, sin, **kw)
    else:
        k4a = gemm_residual_partial_rms(x, weights.w_out, z, weights.gamma_ffn, **kw)
        ra = finalize_rms(k4a.aux["sumsq"], config.eps, ledger=ledger)
        k6 = gemm_rms_swiglu(k4a.main, weights.w_gate_up, ra, **kw)
        k4b = gemm_residual_partial_rms(k6.main, weights.w_down, k4a.aux["pre_norm"], weights.gamma_qkv, **kw)
        rb = finalize_rms(k4b.aux["sumsq"], config.eps, ledger=ledger)
        k7 = gemm_rms_rope(k4b.main, weights.w_qkv, rb, cos, sin, **kw)
    tape = LayerTape(x=x, pre_norm_a=k4a.aux["pre_norm"], inv_rms_a=ra, preact=k6.aux["preact"],
                     pre_norm_b=k4b.aux["pre_norm"], inv_rms_b=rb, qkv=k7.main, cos=cos, sin=sin,
                     folded=folded if config.fold_gamma else None)
    return LayerForwardResult(qkv=k7.main, residual=k4b.aux["pre_norm"], tape=tape, ledger=ledger)


@dataclass
class LayerGrads:
    x: DenseMatrix
    z: DenseMatrix
    w_out: DenseMatrix
    gamma_ffn: Vector
    w_gate_up: DenseMatrix
    w_down: DenseMatrix
    gamma_qkv: Vector
    w_qkv: DenseMatrix
    ledger: TrafficLedger


WgradHook = Callable[[str, object], None]


def layer_backward(grad_qkv: DenseMatrix, tape: LayerTape, weights: LayerWeights, *,
                   grad_residual: Optional[DenseMatrix] = None, config: PipelineConfig,
                   wgrad_hook: Optional[WgradHook] = None) -> LayerGrads:
    """Thirteen launches (kernels.py:885-1013).

    Boundary statistic from rope_backward_stat, relocated statistics from the
    SwiGLU-backward launch, residual gradients accumulated inside the K9
    epilogues.  `wgrad_hook` (B200 extension for token-sharded data
    parallelism) receives each weight gradient as an unrounded float32
    tensor right after its GEMM is enqueued, in production order, and must
    leave the reduced sum in place; if the hook has a `wait()` (asynchronous
    reduction on another stream) it is called before returning (and before the
    single rounding to storage in SIMBF16), so the returned gradients are
    always complete on the caller's stream.
    """
    weights.check(config)
    tape.check(config)
    d = config.hidden
    ledger = TrafficLedger()
    kw = config.launch_kw(ledger)
    prec = config.precision
    f32 = wgrad_hook is not None and prec is PrecisionMode.SIMBF16 and getattr(wgrad_hook, "f32", True)

    # a hook that reduces inside the GEMM epilogue (parallel.PeerWgradReduce) launches the
    # weight gradients itself; bf16 storage only
    peer_gemm = getattr(wgrad_hook, "gemm", None) if prec is PrecisionMode.SIMBF16 else None

    # a hook that rounds after its own reduction (parallel.WgradReduceScatter) takes the
    # unrounded f32 weight gradients through reduce_unrounded() and hands back bf16 sums
    # through reduced(); otherwise the hook leaves the f32 sum in place and it is rounded here
    reduce_unrounded = getattr(wgrad_hook, "reduce_unrounded", None) if f32 else None

    def hand_over(name, t):
        if reduce_unrounded is not None:
            reduce_unrounded(name, t)
        else:
            wgrad_hook(name, t)

    def wgrad(name, a, b):
        if peer_gemm is not None:
            return peer_gemm(name, a, b, precision=prec)
        res = _launch(traffic.K_GEMM, a, b, [], {}, trans_a=True, tile_shape=config.tile_shape,
                      reduction_tile_n=config.reduction_tile_n, precision=prec, ledger=ledger, out_f32=f32)
        if wgrad_hook is not None:
            hand_over(name, res.main.tensor)
        return res.main

    fold = config.fold_gamma
    ones = _ones(d, prec, grad_qkv.tensor.device) if fold else None

    def wgrad_gain(name, gname, a, b, weight, gain):
        # folded gain: dW = diag(gain) (a^T b) and dgain = rowsum(W * a^T b) in one epilogue
        res = gemm_wgrad_gain(a, b, weight, gain, precision=prec, tile_shape=config.tile_shape,
                              reduction_tile_n=config.reduction_tile_n, ledger=ledger, out_f32=f32)
        g_gain = finalize_rowdot(res.aux["gain_dot"], 1, ledger=ledger)
        g_gain.tensor   # no later launch consumes the gain gradient: finalize it now, inside the step
        if wgrad_hook is not None:
            hand_over(name, res.main.tensor)
            wgrad_hook(gname, g_gain.tensor)
        return res.main, g_gain

    grad_zb, rowdot_b = rope_backward_stat(grad_qkv, tape.qkv, tape.cos, tape.sin, tile_n=config.tile_n,
                                           reduction_tile_n=config.reduction_tile_n, precision=prec, ledger=ledger)
    s_b = finalize_rowdot(rowdot_b, d, ledger=ledger)
    if fold:
        # K9 against W' = diag(gamma) W: its GEMM already yields D * gamma, so the local
        # backward runs with unit gains and `normed` is the un-gained c_n = c * r
        k9b = gemm_rmsnorm_backward(grad_zb, tape.folded.w_qkv, tape.pre_norm_b, tape.inv_rms_b, ones, s_b,
                                    grad_in=grad_residual, trans_b=True, **kw)
        grad_h1b = k9b.main
        g_wqkv, g_gqkv = wgrad_gain("w_qkv", "gamma_qkv", k9b.aux["normed"], grad_zb, weights.w_qkv,
                                    weights.gamma_qkv)
    else:
        k9b = gemm_rmsnorm_backward(grad_zb, weights.w_qkv, tape.pre_norm_b, tape.inv_rms_b, weights.gamma_qkv,
                                    s_b, grad_in=grad_residual, trans_b=True, **kw)
        grad_h1b = k9b.main
        g_wqkv = wgrad("w_qkv", k9b.aux["normed"], grad_zb)
        g_gqkv = reduce_row_partials(k9b.aux["gamma_grad"], ledger=ledger)
        if wgrad_hook is not None:
            wgrad_hook("gamma_qkv", g_gqkv.tensor)

    k10 = gemm_swiglu_backward(grad_h1b, weights.w_down, tape.preact, trans_b=True, **kw)
    grad_za = k10.main
    s_a = finalize_rowdot(k10.aux["rowdot"], d, ledger=ledger)
    g_wdown = wgrad("w_down", k10.aux["recompute"], grad_h1b)

    if fold:
        k9a = gemm_rmsnorm_backward(grad_za, tape.folded.w_gate_up, tape.pre_norm_a, tape.inv_rms_a, ones, s_a,
                                    grad_in=grad_h1b, trans_b=True, **kw)
        grad_h1a = k9a.main
        g_wgu, g_gffn = wgrad_gain("w_gate_up", "gamma_ffn", k9a.aux["normed"], grad_za, weights.w_gate_up,
                                   weights.gamma_ffn)
    else:
        k9a = gemm_rmsnorm_backward(grad_za, weights.w_gate_up, tape.pre_norm_a, tape.inv_rms_a,
                                    weights.gamma_ffn, s_a, grad_in=grad_h1b, trans_b=True, **kw)
        grad_h1a = k9a.main
        g_wgu = wgrad("w_gate_up", k9a.aux["normed"], grad_za)
        g_gffn = reduce_row_partials(k9a.aux["gamma_grad"], ledger=ledger)
        if wgrad_hook is not None:
            wgrad_hook("gamma_ffn", g_gffn.tensor)

    grad_x = _launch(traffic.K_GEMM, grad_h1a, weights.w_out, [], {}, trans_b=True, **kw).main
    g_wout = wgrad("w_out", tape.x, grad_h1a)

    if wgrad_hook is not None:
        # join an asynchronous reduction before anything reads the reduced gradients (and,
        # in SIMBF16, before their single rounding to storage) -- whatever the precision
        wait = getattr(wgrad_hook, "wait", None)
        if wait is not None:
            wait()
    if f32:
        reduced = getattr(wgrad_hook, "reduced", None) if reduce_unrounded is not None else None

        def storage(name, g):
            t = reduced(name) if reduced is not None else None
            return DenseMatrix._wrap(t, prec) if t is not None else to_storage(g, prec)

        g_wqkv, g_wdown, g_wgu, g_wout = (storage(n, g) for n, g in (("w_qkv", g_wqkv), ("w_down", g_wdown),
                                                                       ("w_gate_up", g_wgu), ("w_out", g_wout)))
    return LayerGrads(x=grad_x, z=grad_h1a, w_out=g_wout, gamma_ffn=g_gffn, w_gate_up=g_wgu, w_down=g_wdown,
                      gamma_qkv=g_gqkv, w_qkv=g_wqkv, ledger=ledger)


def to_storage(mat: DenseMatrix, precision: PrecisionMode) -> DenseMatrix:
    """Round an f32 result to the storage format once (csrc: convert_f32_bf16)."""
    import ctypes
    import torch

    t = mat.tensor
    if precision is not PrecisionMode.SIMBF16 or t.dtype != torch.float32:
        return mat
    out = alloc_matrix(t.shape[0], t.shape[1], torch.bfloat16, t.device)
    nat.call("coda_convert_f32_bf16", ctypes.byref(nat.tensor_desc(t)), ctypes.byref(nat.tensor_desc(out)),
             torch.cuda.current_stream(t.device).cuda_stream)
    return DenseMatrix._wrap(out, precision)


# ---------------------------------------------------------------------------
# lm head (kernels.py:1016-1076)


@dataclass
class LmHeadResult:
    losses: Vector
    mean_loss: float
    lse: Vector
    target: Vector
    pre_norm: DenseMatrix
    inv_rms: Vector
    logits: Optional[DenseMatrix]
    ledger: TrafficLedger
    # B200 extension: the gained normalized rows K8 consumed (K4's main output) and the
    # labels, kept for lm_head_backward
    normed: Optional[DenseMatrix] = None
    labels: object = None


def lm_head_forward(a, b, z, gamma, w_vocab, labels, *, config: PipelineConfig,
                    store_logits: bool = False) -> LmHeadResult:
    """K4 -> finalize -> K8 -> combine_lse -> cross_entropy_finalize."""
    ledger = TrafficLedger()
    kw = config.launch_kw(ledger)
    k4 = gemm_residual_partial_rms(a, b, z, gamma, **kw)
    r = finalize_rms(k4.aux["sumsq"], config.eps, ledger=ledger)
    k8 = gemm_rms_partial_xent(k4.main, w_vocab, r, labels, store_logits=store_logits, **kw)
    # one device->host read for the LSE / target checks and the mean (same errors, same order)
    lse = combine_lse(k8.aux["lse"], ledger=ledger, check=False)
    losses, mean = cross_entropy_finalize(k8.aux["target"], lse, ledger=ledger, check_lse=True)
    return LmHeadResult(losses=losses, mean_loss=mean, lse=lse, target=k8.aux["target"],
                        pre_norm=k4.aux["pre_norm"], inv_rms=r, logits=k8.main, ledger=ledger,
                        normed=k4.main, labels=labels)


def gemm_xent_backward(a, b, scale, lse, labels, *, grad_scale=1.0, trans_b=False, tile_shape=TileShape(128, 128),
                       reduction_tile_n=128, precision=PrecisionMode.EXACT64, ledger=None):
    """Logit-gradient launch (B200 extension): recompute the K8 logits tile r * (a @ b) and turn
    it into d loss / d logits = (softmax - onehot) * grad_scale in the epilogue; aux
    "xent_rowdot" carries the row-blocked <logits, d logits> partials."""
    return _launch(traffic.K_RMS_XENT, a, b,
                   [RowScale("scale"), CrossEntropyBackward("lse", "labels", "xent_rowdot", grad_scale)],
                   {"scale": scale, "lse": lse, "labels": labels}, trans_b=trans_b, tile_shape=tile_shape,
                   reduction_tile_n=reduction_tile_n, precision=precision, ledger=ledger)


@dataclass
class LmHeadGrads:
    a: DenseMatrix
    b: DenseMatrix
    z: DenseMatrix
    gamma: Vector
    w_vocab: DenseMatrix
    ledger: TrafficLedger


def lm_head_backward(res: LmHeadResult, a, b, gamma, w_vocab, *, config: PipelineConfig,
                     grad_loss: float = 1.0) -> LmHeadGrads:
    """Backward of lm_head_forward for the mean cross-entropy loss (B200 extension; the
    reference stops at the loss).  Five GEMM launches + two finalizers:

      1. logit gradient: recompute r * (normed @ w_vocab), (softmax - onehot) * grad_loss / m,
         with <logits, d logits> partials (the relocated RMSNorm statistic)
      2. finalize_rowdot -> s
      3. K9 gemm_rmsnorm_backward: d logits @ w_vocab^T through the normalization -> d h
         (h = a @ b + z), `normed`, gamma-grad partials (+ reduce_row_partials)
      4. w_vocab gradient: normed^T @ d logits
      5-6. d a = d h @ b^T, d b = a^T @ d h; d z = d h.
    """
    if res.normed is None or res.labels is None:
        raise TapeError("lm_head_backward needs the forward's normed rows and labels (lm_head_forward result)")
    ledger = TrafficLedger()
    kw = config.launch_kw(ledger)
    m = res.normed.rows
    k = gemm_xent_backward(res.normed, w_vocab, res.inv_rms, res.lse, res.labels, grad_scale=grad_loss / m, **kw)
    s = finalize_rowdot(k.aux["xent_rowdot"], res.normed.cols, ledger=ledger)
    k9 = gemm_rmsnorm_backward(k.main, w_vocab, res.pre_norm, res.inv_rms, gamma, s, trans_b=True, **kw)
    gh = k9.main
    g_gamma = reduce_row_partials(k9.aux["gamma_grad"], ledger=ledger)
    g_vocab = _launch(traffic.K_GEMM, k9.aux["normed"], k.main, [], {}, trans_a=True, **kw).main
    g_a = _launch(traffic.K_GEMM, gh, b, [], {}, trans_b=True, **kw).main
    g_b = _launch(traffic.K_GEMM, a, gh, [], {}, trans_a=True, **kw).main
    return LmHeadGrads(a=g_a, b=g_b, z=gh, gamma=g_gamma, w_vocab=g_vocab, ledger=ledger)
