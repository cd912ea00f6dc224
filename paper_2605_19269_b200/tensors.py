"""Device-resident, precision-tagged containers.

Mirrors the container API of the reference (tilefuse/tensors.py:28-257) but
stores payloads in HBM in their real storage format instead of float64
arrays constrained to a grid:

  ============  ===================  ============================
  precision     matrix storage       vector / statistic storage
  ============  ===================  ============================
  EXACT64       float64 (CPU-only)   float64
  SIM32         float32              float32
  SIMBF16       bfloat16             float32 (values on the grid)
  ============  ===================  ============================

Rounding to bfloat16 is round-to-nearest-even (`cvt.rn.bf16.f32` on the
device, torch's RNE cast for uploads), which is exactly the reference's
bit-trick rounding (tensors.py:64-79) for finite values.  `.data` returns a
float64 numpy copy (downloaded lazily) so code written against the reference
keeps reading results the same way; `.tensor` is the device payload.

Row strides are padded to 16 bytes so every matrix can feed TMA.
"""

from __future__ import annotations

import enum
from typing import NamedTuple, Optional

import numpy as np

from .errors import ConfigError, DegenerateError, DimensionError


class PrecisionMode(enum.Enum):
    """Storage / accumulation regime (tensors.py:28-61)."""

    EXACT64 = "exact64"
    SIM32 = "sim32"
    SIMBF16 = "simbf16"

    @property
    def storage_bytes(self) -> int:
        return {"exact64": 8, "sim32": 4, "simbf16": 2}[self.value]

    @property
    def partial_bytes(self) -> int:
        return 8 if self is PrecisionMode.EXACT64 else 4

    @property
    def acc_dtype(self) -> np.dtype:
        return np.dtype(np.float64 if self is PrecisionMode.EXACT64 else np.float32)

    @property
    def partial_dtype(self) -> np.dtype:
        return self.acc_dtype

    @property
    def torch_dtype(self):
        import torch

        return {"exact64": torch.float64, "sim32": torch.float32, "simbf16": torch.bfloat16}[self.value]

    @property
    def vector_torch_dtype(self):
        import torch

        return torch.float64 if self is PrecisionMode.EXACT64 else torch.float32

    @classmethod
    def parse(cls, text: str) -> "PrecisionMode":
        try:
            return cls(text.strip().lower())
        except ValueError:
            raise ConfigError(f"unknown precision mode: {text!r}") from None


def _bf16_rne(values: np.ndarray) -> np.ndarray:
    """Host bf16 RNE on the f32 bit pattern (same rule as the device cvt.rn)."""
    f = np.ascontiguousarray(values, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32).view(np.float32)
    return np.where(np.isfinite(f), r, f)


def quantize(values, mode: PrecisionMode):
    """Host projection of values onto the grid of `mode` (float64 result).

    Utility for preparing inputs and comparing results; device kernels do
    their own rounding at every store.
    """
    scalar = np.ndim(values) == 0
    arr = np.asarray(values, dtype=np.float64)
    if mode is PrecisionMode.EXACT64:
        out = arr.copy()
    elif mode is PrecisionMode.SIM32:
        out = arr.astype(np.float32).astype(np.float64)
    else:
        out = _bf16_rne(arr.astype(np.float32)).astype(np.float64)
    return float(out.reshape(-1)[0]) if scalar else out


class TileShape(NamedTuple):
    rows: int
    cols: int


class TileCoord(NamedTuple):
    i: int
    j: int
    row0: int
    col0: int
    rows: int
    cols: int


def tile_coords(m: int, n: int, shape: TileShape) -> list[TileCoord]:
    """Row-major enumeration of (possibly ragged) output tiles (tensors.py:118-136)."""
    tm, tn = int(shape[0]), int(shape[1])
    if tm <= 0 or tn <= 0:
        raise ConfigError(f"tile dims must be positive, got {shape}")
    if m <= 0 or n <= 0:
        raise DimensionError(f"output dims must be positive, got {m}x{n}")
    out = []
    for i, r0 in enumerate(range(0, m, tm)):
        for j, c0 in enumerate(range(0, n, tn)):
            out.append(TileCoord(i, j, r0, c0, min(tm, m - r0), min(tn, n - c0)))
    return out


def stat_mode(mode: PrecisionMode) -> PrecisionMode:
    """Row statistics are float32 in both simulated modes (tensors.py:227-235)."""
    return PrecisionMode.EXACT64 if mode is PrecisionMode.EXACT64 else PrecisionMode.SIM32


# --------------------------------------------------------------------- device helpers


def default_device():
    import torch

    if not torch.cuda.is_available():
        from ._native import NativeUnavailable

        raise NativeUnavailable("no CUDA device: the CODA engine has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def alloc_matrix(rows: int, cols: int, dtype, device=None, zero: bool = False):
    """(rows, cols) view of a row-padded allocation (16-byte aligned rows)."""
    import torch

    device = device if device is not None else default_device()
    esize = torch.empty((), dtype=dtype).element_size()
    per = max(1, 16 // esize)
    ld = -(-cols // per) * per
    fn = torch.zeros if zero else torch.empty
    base = fn((rows, ld), dtype=dtype, device=device)
    return base if ld == cols else base[:, :cols]


def tma_ready(t) -> bool:
    """True if a 2-D tensor has unit column stride and 16-byte aligned rows."""
    es = t.element_size()
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        return False
    if t.data_ptr() % 16:
        return False
    return t.shape[0] == 1 or (t.stride(0) * es) % 16 == 0


def as_tma_ready(t):
    """Return `t` or a row-padded device copy of it."""
    if tma_ready(t):
        return t
    out = alloc_matrix(t.shape[0], t.shape[1], t.dtype, t.device)
    out.copy_(t)
    return out


class DenseMatrix:
    """Row-major 2-D device tensor tagged with its storage precision.

    Treated as immutable by the engine: launches always write fresh outputs.
    `_rope` optionally carries a compact form of a RoPE table (set only by
    `qkv_rope_tables`, which builds both forms from the same values).
    """

    __slots__ = ("_t", "precision", "_host", "_rope")

    def __init__(self, data, precision: PrecisionMode = PrecisionMode.EXACT64):
        import torch

        self.precision = precision
        self._host = None
        self._rope = None
        if isinstance(data, np.ndarray):
            if data.ndim != 2:
                raise DimensionError(f"DenseMatrix needs a 2-D array, got ndim={data.ndim}")
            if min(data.shape) < 1:
                raise DimensionError(f"DenseMatrix dims must be positive, got {data.shape}")
            self._t = _upload(np.asarray(data, dtype=np.float64), precision)
        elif isinstance(data, torch.Tensor):
            if data.dim() != 2:
                raise DimensionError(f"DenseMatrix needs a 2-D tensor, got ndim={data.dim()}")
            if min(data.shape) < 1:
                raise DimensionError(f"DenseMatrix dims must be positive, got {tuple(data.shape)}")
            if data.dtype != precision.torch_dtype:
                raise ConfigError(f"tensor dtype {data.dtype} does not store {precision.value}")
            if not data.is_cuda:
                raise ConfigError("DenseMatrix tensors must be device-resident (use from_array)")
            self._t = as_tma_ready(data)
        else:
            raise DimensionError(f"DenseMatrix needs an ndarray or tensor, got {type(data).__name__}")

    @classmethod
    def from_array(cls, values, precision: PrecisionMode = PrecisionMode.EXACT64) -> "DenseMatrix":
        arr = np.array(values, dtype=np.float64, order="C", ndmin=2)
        return cls(arr, precision)

    @classmethod
    def from_tensor(cls, tensor, precision: PrecisionMode) -> "DenseMatrix":
        return cls(tensor, precision)

    @classmethod
    def zeros(cls, rows: int, cols: int, precision: PrecisionMode = PrecisionMode.EXACT64) -> "DenseMatrix":
        t = alloc_matrix(rows, cols, precision.torch_dtype, zero=True)
        return cls(t, precision)

    @classmethod
    def _wrap(cls, tensor, precision: PrecisionMode) -> "DenseMatrix":
        obj = cls.__new__(cls)
        obj._t = tensor
        obj.precision = precision
        obj._host = None
        obj._rope = None
        return obj

    @property
    def tensor(self):
        return self._t

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            import torch

            t = self._t.detach()
            if t.dtype != torch.float64:
                t = t.float()
            arr = np.ascontiguousarray(t.cpu().numpy(), dtype=np.float64)
            arr.setflags(write=False)
            self._host = arr
        return self._host

    @property
    def rows(self) -> int:
        return int(self._t.shape[0])

    @property
    def cols(self) -> int:
        return int(self._t.shape[1])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    def to_array(self) -> np.ndarray:
        return self.data.copy()

    def __repr__(self) -> str:
        return f"DenseMatrix(shape={self.shape}, precision={self.precision.value})"


class Vector:
    """1-D device tensor (float32 in simulated modes) tagged with a precision."""

    __slots__ = ("_t", "precision", "_host", "_pending")

    def __init__(self, data, precision: PrecisionMode = PrecisionMode.EXACT64):
        import torch

        self.precision = precision
        self._host = None
        self._pending = None
        if isinstance(data, np.ndarray):
            if data.ndim != 1:
                raise DimensionError(f"Vector needs a 1-D array, got ndim={data.ndim}")
            if data.shape[0] < 1:
                raise DimensionError("Vector length must be positive")
            q = quantize(data, precision)
            self._t = torch.from_numpy(np.ascontiguousarray(q)).to(
                device=default_device(), dtype=precision.vector_torch_dtype)
        elif isinstance(data, torch.Tensor):
            if data.dim() != 1:
                raise DimensionError(f"Vector needs a 1-D tensor, got ndim={data.dim()}")
            if data.shape[0] < 1:
                raise DimensionError("Vector length must be positive")
            if not data.is_cuda:
                raise ConfigError("Vector tensors must be device-resident (use from_array)")
            if data.dtype != precision.vector_torch_dtype:
                data = data.to(precision.vector_torch_dtype)
            self._t = data.contiguous()
        else:
            raise DimensionError(f"Vector needs an ndarray or tensor, got {type(data).__name__}")

    @classmethod
    def from_array(cls, values, precision: PrecisionMode = PrecisionMode.EXACT64) -> "Vector":
        return cls(np.array(values, dtype=np.float64).reshape(-1), precision)

    @classmethod
    def from_tensor(cls, tensor, precision: PrecisionMode) -> "Vector":
        return cls(tensor, precision)

    @classmethod
    def zeros(cls, length: int, precision: PrecisionMode = PrecisionMode.EXACT64) -> "Vector":
        import torch

        return cls(torch.zeros(length, dtype=precision.vector_torch_dtype, device=default_device()), precision)

    @classmethod
    def _wrap(cls, tensor, precision: PrecisionMode) -> "Vector":
        obj = cls.__new__(cls)
        obj._t = tensor
        obj.precision = precision
        obj._host = None
        obj._pending = None
        return obj

    @property
    def tensor(self):
        # a deferred finalizer result (reductions.py) that no consuming launch has taken over
        # yet is computed now, by its standalone kernel
        if self._pending is not None:
            self._pending.materialize(self)
        return self._t

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            arr = np.ascontiguousarray(self.tensor.detach().cpu().double().numpy())
            arr.setflags(write=False)
            self._host = arr
        return self._host

    def __len__(self) -> int:
        return int(self._t.shape[0])

    @property
    def length(self) -> int:
        return len(self)

    def to_array(self) -> np.ndarray:
        return self.data.copy()

    def __repr__(self) -> str:
        return f"Vector(len={len(self)}, precision={self.precision.value})"


def _upload(arr: np.ndarray, precision: PrecisionMode):
    """Host float64 -> device storage format (f64 -> f32 RNE -> bf16 RNE)."""
    import torch

    dev = default_device()
    rows, cols = arr.shape
    out = alloc_matrix(rows, cols, precision.torch_dtype, dev)
    if precision is PrecisionMode.EXACT64:
        src = torch.from_numpy(np.ascontiguousarray(arr))
    else:
        src = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32))
    out.copy_(src.to(dev))   # f32 -> bf16 cast on device is RNE
    return out


def _payload(obj) -> np.ndarray:
    if isinstance(obj, (DenseMatrix, Vector)):
        return obj.data
    return np.asarray(obj, dtype=np.float64)


def rel_error(value, reference) -> float:
    """||value - reference||_F / ||reference||_F in float64 (tensors.py:244-257)."""
    a = _payload(value).astype(np.float64, copy=False)
    b = _payload(reference).astype(np.float64, copy=False)
    if a.shape != b.shape:
        raise DimensionError(f"shape mismatch {a.shape} vs {b.shape}")
    ref = float(np.linalg.norm(b))
    if ref == 0.0:
        raise DegenerateError("reference norm is zero; relative error undefined")
    return float(np.linalg.norm(a - b)) / ref


def max_abs_error(value, reference) -> float:
    a = _payload(value).astype(np.float64, copy=False)
    b = _payload(reference).astype(np.float64, copy=False)
    if a.shape != b.shape:
        raise DimensionError(f"shape mismatch {a.shape} vs {b.shape}")
    return float(np.max(np.abs(a - b))) if a.size else 0.0
