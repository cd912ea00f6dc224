"""GEMM launch API: `GemmProblem`, `run_gemm`, `run_gemm_trans`, `KernelResult`.

Same call surface and validation as the reference engine
(tilefuse/engine.py:55-478).  Instead of a Python tile loop, `run_gemm`
lowers the epilogue program to device steps and enqueues ONE persistent
sm_100a kernel (csrc/coda_gemm.cuh) through the C-ABI on the current torch
stream.  Host work is validation, output allocation and slot bookkeeping;
there is no CPU execution path.

Precision modes:
  * SIMBF16 — bf16 operands and stores, f32 TMEM accumulation, f32 epilogue
    math and partials (tensors.py:40-54 of the reference);
  * SIM32   — f32 operands/stores; the GEMM runs on bf16 tensor cores over a
    6-term split of each f32 operand (error ~2^-24);
  * EXACT64 — CPU-oracle only; rejected with ConfigError.

Reference tile shapes (`GemmProblem.tile_shape`, `reduction_tile_n`) keep
their meaning for the *layout of partial results*; the GPU always computes in
128 x 256 tiles.  Partial blocks that straddle GPU tiles are produced as
pieces and folded back in ascending order by a tiny deterministic kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from fractions import Fraction
from typing import Optional, Sequence, Union

import numpy as np

from . import _native as nat
from .epilogue import (
    EpilogueProgram,
    OperandKind,
    PartialSlot,
    StoreKind,
    scaled_row_blocks,
    split_at,
)
from .errors import BindingError, ConfigError, DimensionError, LabelError, ProgramError
from .tensors import (
    DenseMatrix,
    PrecisionMode,
    TileShape,
    Vector,
    alloc_matrix,
    as_tma_ready,
    stat_mode,
    tile_coords,
)
from .traffic import LABEL_BYTES, LaunchRecord, TrafficLedger

Binding = Union[DenseMatrix, Vector, np.ndarray]


@dataclass(frozen=True)
class GemmProblem:
    """Shape, layout, tiling and precision of one launch (engine.py:55-76)."""

    m: int
    n: int
    k: int
    trans_a: bool = False
    trans_b: bool = False
    tile_shape: TileShape = TileShape(128, 128)
    reduction_tile_n: int = 128
    precision: PrecisionMode = PrecisionMode.EXACT64

    def __post_init__(self):
        if min(self.m, self.n, self.k) <= 0:
            raise DimensionError(f"problem dims must be positive, got {self.m}x{self.n}x{self.k}")
        if min(self.tile_shape[0], self.tile_shape[1]) <= 0:
            raise ConfigError(f"bad tile shape {self.tile_shape}")
        if self.reduction_tile_n <= 0:
            raise ConfigError("reduction_tile_n must be positive")


@dataclass
class KernelResult:
    """Outputs of one launch (engine.py:79-85)."""

    main: Optional[DenseMatrix]
    aux: dict
    record: LaunchRecord


# ----------------------------------------------------------------------------- layout caches

_map_cache: dict = {}


def _device_i32(arr: np.ndarray, device):
    import torch

    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32)).to(device)


def row_pieces(n: int, tile_n: int, rtn: int, scale: int, device):
    """Piece map for row-directed partials at integer width `scale`.

    Returns (map_dev[int32, n*scale], block_ptr_dev, n_pieces, n_blocks,
    counts).  Pieces are reference blocks split at GPU tile edges.
    """
    key = ("row", n, tile_n, rtn, scale, str(device))
    hit = _map_cache.get(key)
    if hit is not None:
        return hit
    blocks = scaled_row_blocks(n, tile_n, rtn, scale)
    # split at every 128-column half tile (each half belongs to one epilogue warp group)
    starts, ptr = split_at([(b.start, b.stop) for b in blocks], nat.GPU_TILE_N // 2 * scale)
    npieces = len(starts) - 1
    pmap = np.repeat(np.arange(npieces, dtype=np.int32), np.diff(starts))
    counts = np.array([b.width for b in blocks], dtype=np.int64)
    aligned = bool(np.all(starts[:-1] % (32 * scale) == 0))
    val = (_device_i32(pmap, device), _device_i32(ptr, device), npieces, len(blocks), counts, aligned)
    _map_cache[key] = val
    return val


def col_pieces(m: int, tile_m: int, device):
    """Row-piece map for column sums: reference tile rows split at GPU tile rows."""
    key = ("col", m, tile_m, str(device))
    hit = _map_cache.get(key)
    if hit is not None:
        return hit
    bounds = [(r, min(r + tile_m, m)) for r in range(0, m, tile_m)]
    starts, ptr = split_at(bounds, nat.GPU_TILE_M)
    npieces = len(starts) - 1
    pmap = np.repeat(np.arange(npieces, dtype=np.int32), np.diff(starts))
    counts = np.array([b - a for a, b in bounds], dtype=np.int64)
    aligned = bool(np.all(starts[:-1] % 32 == 0))
    val = (_device_i32(pmap, device), _device_i32(ptr, device), npieces, len(bounds), counts, aligned)
    _map_cache[key] = val
    return val


def block_starts(n: int, tile_n: int, rtn: int, device):
    key = ("bstart", n, tile_n, rtn, str(device))
    hit = _map_cache.get(key)
    if hit is not None:
        return hit
    blocks = scaled_row_blocks(n, tile_n, rtn, 1)
    st = np.array([b.start for b in blocks] + [n], dtype=np.int32)
    counts = np.array([b.width for b in blocks], dtype=np.int64)
    val = (_device_i32(st, device), len(blocks), counts)
    _map_cache[key] = val
    return val


# ----------------------------------------------------------------------------- helpers


def _tile_cols(n: int, tile_n: int) -> list[tuple[int, int]]:
    """(col0, width) of every reference tile column; only these matter for pairing."""
    key = ("cols", n, tile_n)
    hit = _map_cache.get(key)
    if hit is None:
        hit = [(c0, min(tile_n, n - c0)) for c0 in range(0, n, tile_n)]
        _map_cache[key] = hit
    return hit


def storage_tensor(mat: DenseMatrix, precision: PrecisionMode):
    """Device payload of `mat` in the storage dtype of `precision`."""
    t = mat.tensor
    want = precision.torch_dtype
    if t.dtype != want:
        conv = alloc_matrix(t.shape[0], t.shape[1], want, t.device)
        conv.copy_(t)
        t = conv
    return as_tma_ready(t)


# The six products a_i*b_j with i+j <= 2, smallest first: the tensor-core f32
# accumulator truncates each MMA's sum relative to the running magnitude, so
# the tiny terms are accumulated while it is still small and the dominant
# a0*b0 term comes last.
_A_PATTERN = (2, 1, 0, 1, 0, 0)
_B_PATTERN = (0, 1, 2, 0, 1, 0)
# SIM32 K-chunk: each chunk's product is summed into an f32 accumulator input
# (software RNE adds), bounding the number of MMA accumulations per sum.
SIM32_K_CHUNK = 256


def split_f32(t, k_axis: int, kp: int, pattern):
    """SIM32 operand -> 6 K-blocks of bf16 split terms (csrc/coda_aux.cuh)."""
    import ctypes
    import torch

    rows, cols = t.shape
    drows, dcols = (rows, 6 * kp) if k_axis == 1 else (6 * kp, cols)
    dst = alloc_matrix(drows, dcols, torch.bfloat16, t.device)
    pat = (ctypes.c_int32 * 6)(*pattern)
    nat.call("coda_split_operand", ctypes.byref(nat.tensor_desc(t)), k_axis, kp, pat,
             ctypes.byref(nat.tensor_desc(dst)), torch.cuda.current_stream(t.device).cuda_stream)
    return dst


def _stream(device):
    import torch

    return torch.cuda.current_stream(device).cuda_stream


# ----------------------------------------------------------------------------- run_gemm


def run_gemm(
    problem: GemmProblem,
    a: DenseMatrix,
    b: DenseMatrix,
    program: Optional[EpilogueProgram] = None,
    bindings: Optional[dict] = None,
    *,
    kernel_name: str = "gemm",
    ledger: Optional[TrafficLedger] = None,
    tile_order: Optional[Sequence[tuple[int, int]]] = None,
    store_main: bool = True,
    out_f32: bool = False,
) -> KernelResult:
    """One fused GEMM launch on the B200 (engine.py:376-464).

    `tile_order` is validated like the reference (a permutation of the
    reference tile grid) but has no effect: tiles are independent and the
    persistent kernel's schedule never changes results.  `out_f32` (not in
    the reference) keeps the main output unrounded in float32, used for
    weight gradients that are all-reduced before their single rounding.
    """
    import ctypes
    import torch

    if program is None:
        program = EpilogueProgram(())
    if bindings is None:
        bindings = {}
    p = problem
    if p.precision is PrecisionMode.EXACT64:
        raise ConfigError("EXACT64 runs only in the CPU oracle; the GPU engine supports SIM32 and SIMBF16")

    want_a = (p.k, p.m) if p.trans_a else (p.m, p.k)
    want_b = (p.n, p.k) if p.trans_b else (p.k, p.n)
    if not isinstance(a, DenseMatrix) or not isinstance(b, DenseMatrix):
        raise BindingError("a and b must be DenseMatrix")
    if a.shape != want_a:
        raise DimensionError(f"a has shape {a.shape}, problem wants {want_a}")
    if b.shape != want_b:
        raise DimensionError(f"b has shape {b.shape}, problem wants {want_b}")

    tm_ref, tn_ref = int(p.tile_shape[0]), int(p.tile_shape[1])
    pair_factors = tuple(s.entry_factor for s in program.steps if s.primitive.needs_pair_alignment)
    if pair_factors:
        key = ("pairing", pair_factors, p.n, tn_ref)
        if key not in _map_cache:
            program.check_pairing(_tile_cols(p.n, tn_ref))
            _map_cache[key] = True
    n_out = program.scaled_width(p.n) if store_main else None

    unknown = set(bindings) - set(program.operands)
    if unknown:
        raise BindingError(f"bindings not used by the program: {sorted(unknown)}")
    if tile_order is not None:
        grid = sorted((c.i, c.j) for c in tile_coords(p.m, p.n, p.tile_shape))
        if sorted(tuple(x) for x in tile_order) != grid:
            raise ConfigError("tile_order must be a permutation of the launch's (i, j) grid")

    steps, onames, snames = program.lower()
    dev = a.tensor.device
    prec = p.precision
    sdt = prec.torch_dtype
    scode = nat.BF16 if prec is PrecisionMode.SIMBF16 else nat.F32
    read_bytes = a.rows * a.cols * a.precision.storage_bytes + b.rows * b.cols * b.precision.storage_bytes
    write_bytes = 0

    # deferred finalizers (reductions.PendingFinalize): a pending statistic vector bound once,
    # as a RowScale operand or as RmsNormBackwardLocal's stat, is computed by this launch
    fin_targets = {}
    for si, (op, wd, args) in enumerate(steps):
        slot = args[0] if op == nat.OP_ROW_SCALE else args[3] if op == nat.OP_RMSNORM_BWD else None
        if slot is not None:
            fin_targets.setdefault(slot, []).append(si)
    bound_ids = [id(bindings.get(n)) for n in onames]

    # ---- operands
    keep = []
    descs = []
    deferred = []       # (operand slot, consuming step, vector, PendingFinalize)
    for i, name in enumerate(onames):
        op = program.operands[name]
        if name not in bindings:
            raise BindingError(f"program operand {name!r} is not bound")
        val = bindings[name]
        want = Fraction(p.n) * op.factor
        if op.kind is OperandKind.TILE:
            if not isinstance(val, DenseMatrix):
                raise BindingError(f"operand {name!r} must be a DenseMatrix")
            if want.denominator != 1:
                raise ProgramError(f"operand {name!r} scale {op.factor} does not divide n={p.n}")
            if val.shape != (p.m, int(want)):
                raise DimensionError(f"operand {name!r} has shape {val.shape}, expected {(p.m, int(want))}")
            t = storage_tensor(val, prec)
            read_bytes += val.rows * val.cols * val.precision.storage_bytes
        elif op.kind in (OperandKind.ROW_VEC, OperandKind.COL_VEC):
            if not isinstance(val, Vector):
                raise BindingError(f"operand {name!r} must be a Vector")
            if op.kind is OperandKind.ROW_VEC:
                if want.denominator != 1 or len(val) != int(want):
                    raise DimensionError(f"operand {name!r} has length {len(val)}, expected {want}")
            elif len(val) != p.m:
                raise DimensionError(f"operand {name!r} has length {len(val)}, expected {p.m}")
            pend = getattr(val, "_pending", None)
            if (pend is not None and op.kind is OperandKind.COL_VEC and len(fin_targets.get(i, ())) == 1
                    and bound_ids.count(id(val)) == 1):
                t = val._t                       # written by this launch
                deferred.append((i, fin_targets[i][0], val, pend))
            else:
                t = val.tensor if val.tensor.dtype == torch.float32 else val.tensor.float()
                t = t.contiguous()
            read_bytes += len(val) * val.precision.storage_bytes
        else:  # LABELS
            if isinstance(val, torch.Tensor):
                arr_dev = val
                if arr_dev.dim() != 1 or arr_dev.shape[0] != p.m:
                    raise DimensionError(f"labels {name!r} must have shape ({p.m},), got {tuple(arr_dev.shape)}")
                if arr_dev.dtype.is_floating_point:
                    raise LabelError(f"labels {name!r} must be integers")
                lo, hi = int(arr_dev.min()), int(arr_dev.max())
            else:
                arr = np.asarray(val)
                if arr.ndim != 1 or arr.shape[0] != p.m:
                    raise DimensionError(f"labels {name!r} must have shape ({p.m},), got {arr.shape}")
                if not np.issubdtype(arr.dtype, np.integer):
                    raise LabelError(f"labels {name!r} must be integers")
                lo, hi = int(arr.min()), int(arr.max())
                arr_dev = torch.from_numpy(arr.astype(np.int64))
            if lo < 0 or hi >= p.n:
                raise LabelError(f"labels {name!r} must lie in [0, {p.n}), got range [{lo}, {hi}]")
            t = arr_dev.to(device=dev, dtype=torch.int64).contiguous()
            read_bytes += p.m * LABEL_BYTES
        keep.append(t)
        descs.append(nat.tensor_desc(t))

    # ---- compact RoPE tables (qkv_rope_tables pairs): extra operands the specialised
    # kernel loads instead of the full (m, n) tables; the generic interpreter ignores them
    steps = list(steps)   # the lowering is memoized on the program: never edit it in place
    if prec is PrecisionMode.SIMBF16:
        from .kernels import rope_compact_of

        for si, (op, wd, args) in enumerate(steps):
            if op != nat.OP_ROPE or len(descs) + 2 > nat.MAX_OPERANDS:
                continue
            spec = rope_compact_of(bindings[onames[args[0]]], bindings[onames[args[1]]])
            # the compact rule covers n columns when n >= 2 hidden (packed qkv) or n == hidden
            # (a plain table over the whole width)
            if spec is None or (2 * spec.hidden > p.n and spec.hidden != p.n) or spec.cos.shape[0] != p.m:
                continue
            nops = len(descs)
            descs += [nat.tensor_desc(spec.cos), nat.tensor_desc(spec.sin)]
            keep.extend((spec.cos, spec.sin))
            steps[si] = (op, wd, list(args[:3]) + [nops + 1, nops + 2, spec.hidden, 0])
    # ---- deferred finalizers: the partials become an extra operand of the consuming step
    fin = {}
    for slot, si, vec, pend in deferred:
        if len(descs) + 1 > nat.MAX_OPERANDS:
            vec.tensor                               # no operand slot left: finalize standalone
            continue
        descs.append(nat.tensor_desc(pend.partials, nat.F32))
        keep.append(pend.partials)
        fin[si] = (len(descs), pend.kind, pend.d, pend.eps)
    nops = len(descs)
    op_descs = (nat.Tensor * max(1, nops))(*descs)

    # ---- stores
    st_descs = (nat.Store * max(1, len(snames)))()
    outputs = {}
    folds = []          # (name, kind, pieces tensor, ptr, nb, counts, np, n_or_m)
    pw = prec.partial_bytes
    for i, name in enumerate(snames):
        st = program.stores[name]
        want = Fraction(p.n) * st.factor
        if want.denominator != 1:
            raise ProgramError(f"store {name!r} scale {st.factor} does not divide n={p.n}")
        width = int(want)
        if st.kind is StoreKind.TILE:
            t = alloc_matrix(p.m, width, sdt, dev)
            outputs[name] = ("tile", t)
            st_descs[i] = nat.Store(nat.tensor_desc(t), None, nat.STORE_TILE, 0)
            write_bytes += p.m * width * prec.storage_bytes
        elif st.kind in (StoreKind.ROW_SUM, StoreKind.ROW_PAIR):
            if st.factor.denominator != 1:
                raise ProgramError(f"partial stores need an integer width scale, got {st.factor}")
            pmap, ptr, npc, nb, counts, aligned = row_pieces(p.n, p.tile_shape[1], p.reduction_tile_n,
                                                             st.factor.numerator, dev)
            pair = st.kind is StoreKind.ROW_PAIR
            t = torch.empty((p.m, npc * (2 if pair else 1)), dtype=torch.float32, device=dev)
            st_descs[i] = nat.Store(nat.tensor_desc(t), pmap.data_ptr(),
                                    nat.STORE_ROW_PAIR if pair else nat.STORE_ROW_SUM, int(aligned))
            keep.append(pmap)
            folds.append((name, st.kind, t, ptr, nb, counts, npc))
            write_bytes += (2 if pair else 1) * p.m * nb * pw
        elif st.kind is StoreKind.COL_SUM:
            pmap, ptr, npc, nb, counts, aligned = col_pieces(p.m, p.tile_shape[0], dev)
            t = torch.empty((npc, width), dtype=torch.float32, device=dev)
            st_descs[i] = nat.Store(nat.tensor_desc(t), pmap.data_ptr(), nat.STORE_COL_SUM, int(aligned))
            keep.append(pmap)
            folds.append((name, st.kind, t, ptr, nb, counts, npc))
            write_bytes += nb * width * pw
        else:  # GATHER
            t = torch.full((p.m,), float("nan"), dtype=torch.float32, device=dev)
            outputs[name] = ("gather", t)
            st_descs[i] = nat.Store(nat.tensor_desc(t), None, nat.STORE_GATHER, 0)
            write_bytes += p.m * pw

    main_t = None
    main_desc = None
    if store_main:
        odt = torch.float32 if out_f32 else sdt
        main_t = alloc_matrix(p.m, n_out, odt, dev)
        main_desc = nat.tensor_desc(main_t)
        write_bytes += p.m * n_out * prec.storage_bytes
    step_arr = (nat.Step * max(1, len(steps)))()
    for i, (op, wd, args) in enumerate(steps):
        fs, fk, fd, fe = fin.get(i, (0, 0, 0, 0.0))
        step_arr[i] = nat.Step(op, wd, (ctypes.c_int32 * 7)(*args), fs, fk, fd, fe, 0)

    def enqueue(ta, tb, kk, program_on, mdesc, acc_t, odtype):
        ws = nat.workspace(dev)
        prob = nat.Problem(p.m, p.n, kk, int(p.trans_a), int(p.trans_b), scode, odtype,
                           int(mdesc is not None), nat.sm_limit(),
                           ws.data_ptr() if ws is not None else None, ws.numel() * 4 if ws is not None else 0)
        acc_desc = nat.tensor_desc(acc_t) if acc_t is not None else None
        nat.call("coda_gemm_epilogue", ctypes.byref(prob), ctypes.byref(nat.tensor_desc(ta)),
                 ctypes.byref(nat.tensor_desc(tb)), step_arr, len(steps) if program_on else 0, op_descs,
                 nops if program_on else 0, st_descs, len(snames) if program_on else 0,
                 ctypes.byref(mdesc) if mdesc is not None else None,
                 ctypes.byref(acc_desc) if acc_desc is not None else None, _stream(dev),
                 tag=f"{kernel_name} {p.m}x{p.n}x{p.k}{' TN' if p.trans_a else ''}{' NT' if p.trans_b else ''}",
                 flops=2.0 * p.m * p.n * (kk if scode == nat.BF16 else kk // 6))

    out_code = nat.F32 if (out_f32 or scode == nat.F32) else nat.BF16
    if prec is PrecisionMode.SIMBF16:
        enqueue(storage_tensor(a, prec), storage_tensor(b, prec), p.k, True, main_desc, None, out_code)
    else:
        # SIM32: f32 operands as 6-term bf16 splits, K chunked with an f32 running sum
        fa, fb = storage_tensor(a, prec), storage_tensor(b, prec)
        acc = None
        for k0 in range(0, p.k, SIM32_K_CHUNK):
            k1 = min(p.k, k0 + SIM32_K_CHUNK)
            kp = -(-(k1 - k0) // 8) * 8
            sa = fa[k0:k1, :] if p.trans_a else fa[:, k0:k1]
            sb = fb[:, k0:k1] if p.trans_b else fb[k0:k1, :]
            ta = split_f32(sa, 0 if p.trans_a else 1, kp, _A_PATTERN)
            tb = split_f32(sb, 1 if p.trans_b else 0, kp, _B_PATTERN)
            if k1 < p.k:
                part = alloc_matrix(p.m, p.n, torch.float32, dev)
                enqueue(ta, tb, 6 * kp, False, nat.tensor_desc(part), acc, nat.F32)
                keep.append(part)
                acc = part
            else:
                enqueue(ta, tb, 6 * kp, True, main_desc, acc, out_code)

    for _, si, vec, pend in deferred:
        if si in fin:
            pend.adopt(vec)                          # the enqueued launch writes the vector

    # ---- fold pieces into the reference block layout
    aux: dict = {}
    for name, (kind, t) in outputs.items():
        if kind == "tile":
            aux[name] = DenseMatrix._wrap(t, prec)
        else:
            aux[name] = Vector._wrap(t, stat_mode(prec))
    for name, kind, t, ptr, nb, counts, npc in folds:
        if kind is StoreKind.COL_SUM:
            if npc != nb:
                out = torch.empty((nb, t.shape[1]), dtype=torch.float32, device=dev)
                nat.call("coda_combine_col_pieces", t.data_ptr(), npc, t.shape[1], t.stride(0), ptr.data_ptr(),
                         nb, out.data_ptr(), out.stride(0), _stream(dev))
                t = out
            aux[name] = PartialSlot(kind, t, counts, prec).freeze()
        else:
            pair = kind is StoreKind.ROW_PAIR
            if npc != nb:
                out = torch.empty((p.m, nb * (2 if pair else 1)), dtype=torch.float32, device=dev)
                nat.call("coda_combine_row_pieces", t.data_ptr(), p.m, npc, t.stride(0), ptr.data_ptr(), nb,
                         int(pair), out.data_ptr(), out.stride(0), _stream(dev))
                t = out
            if pair:
                t = t.view(p.m, nb, 2)
            aux[name] = PartialSlot(kind, t, counts, prec).freeze()

    main = DenseMatrix._wrap(main_t, PrecisionMode.SIM32 if (out_f32 and prec is PrecisionMode.SIMBF16) else prec) \
        if store_main else None
    record = LaunchRecord(kernel_name, read_bytes, write_bytes)
    if ledger is not None:
        ledger.add(record)
    return KernelResult(main=main, aux=aux, record=record)


def run_gemm_trans(problem: GemmProblem, a: DenseMatrix, b: DenseMatrix, program=None, bindings=None,
                   **kwargs) -> KernelResult:
    """run_gemm with B interpreted as stored (n, k) (engine.py:467-478)."""
    return run_gemm(replace(problem, trans_b=True), a, b, program, bindings, **kwargs)
