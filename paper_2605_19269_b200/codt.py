"""CODT binary tensor container (golden-vector exchange).

Byte-compatible with the reference container (tilefuse/codt.py:3-13):

    b"CODT" | u32 rank (1 or 2) | rank x u64 dims | u8 precision tag
    (0 exact64, 1 sim32, 2 simbf16) | little-endian row-major payload
    (f64 / f32 / the upper 16 bits of the f32 pattern for bfloat16)

Here the payload moves between the file and HBM without a float64 detour: a
bf16 device tensor is written as its raw 16-bit patterns and read back into a
bf16 device tensor, so round trips are bit-exact by construction.  The byte
codec (`encode` / `decode`) is host-only and usable without a GPU.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import ContainerError
from .tensors import DenseMatrix, PrecisionMode, Vector, alloc_matrix, default_device

MAGIC = b"CODT"
TAGS = {PrecisionMode.EXACT64: 0, PrecisionMode.SIM32: 1, PrecisionMode.SIMBF16: 2}
MODES = {v: k for k, v in TAGS.items()}
WIDTH = {0: 8, 1: 4, 2: 2}
CODEC = {0: "<f8", 1: "<f4", 2: "<u2"}


def encode(dims: tuple, precision: PrecisionMode, payload: np.ndarray) -> bytes:
    """Header + payload.  `payload` holds f64/f32 values or raw bf16 bit patterns (uint16)."""
    if len(dims) not in (1, 2):
        raise ContainerError(f"unsupported rank {len(dims)}")
    tag = TAGS[precision]
    body = np.ascontiguousarray(payload).reshape(-1).astype(CODEC[tag], copy=False)
    if body.size != int(np.prod(dims)):
        raise ContainerError("payload size does not match dims")
    return MAGIC + struct.pack("<I", len(dims)) + struct.pack(f"<{len(dims)}Q", *dims) + bytes([tag]) + body.tobytes()


def decode(raw: bytes, name: str = "<bytes>") -> tuple[tuple, PrecisionMode, np.ndarray]:
    """(dims, precision, payload) with payload in the codec dtype (f8 / f4 / u2 bit patterns)."""
    if len(raw) < 9 or raw[:4] != MAGIC:
        raise ContainerError(f"{name}: not a CODT container")
    (rank,) = struct.unpack_from("<I", raw, 4)
    if rank not in (1, 2):
        raise ContainerError(f"{name}: unsupported rank {rank}")
    off = 8 + 8 * rank
    if len(raw) < off + 1:
        raise ContainerError(f"{name}: truncated header")
    dims = struct.unpack_from(f"<{rank}Q", raw, 8)
    tag = raw[off]
    if tag not in MODES:
        raise ContainerError(f"{name}: unknown precision tag {tag}")
    count = int(np.prod(dims))
    body = raw[off + 1:]
    if len(body) != count * WIDTH[tag]:
        raise ContainerError(f"{name}: payload holds {len(body)} bytes, expected {count * WIDTH[tag]}")
    return tuple(int(d) for d in dims), MODES[tag], np.frombuffer(body, dtype=CODEC[tag], count=count)


def bf16_bits_to_float(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def write_tensor(path, tensor) -> None:
    """Serialize a device DenseMatrix or Vector (reference: codt.write_tensor)."""
    import torch

    if isinstance(tensor, DenseMatrix):
        dims = tensor.shape
        t = tensor.tensor
    elif isinstance(tensor, Vector):
        dims = (len(tensor),)
        t = tensor.tensor
    else:
        raise ContainerError(f"cannot serialize {type(tensor).__name__}")
    p = tensor.precision
    host = t.detach().contiguous().cpu()
    if p is PrecisionMode.SIMBF16:
        if host.dtype != torch.bfloat16:
            host = host.to(torch.bfloat16)   # vectors live in f32 holding bf16-grid values
        payload = host.view(torch.int16).numpy().view(np.uint16)
    elif p is PrecisionMode.SIM32:
        payload = host.float().numpy()
    else:
        payload = host.double().numpy()
    Path(path).write_bytes(encode(dims, p, payload))


def read_tensor(path):
    """Deserialize into a device DenseMatrix (rank 2) or Vector (rank 1)."""
    import torch

    dims, p, payload = decode(Path(path).read_bytes(), str(path))
    dev = default_device()
    if p is PrecisionMode.SIMBF16:
        src = torch.from_numpy(payload.view(np.int16).copy()).view(torch.bfloat16)
    elif p is PrecisionMode.SIM32:
        src = torch.from_numpy(payload.astype(np.float32))
    else:
        src = torch.from_numpy(payload.astype(np.float64))
    if len(dims) == 1:
        return Vector._wrap(src.to(dev).to(p.vector_torch_dtype), p)
    out = alloc_matrix(dims[0], dims[1], p.torch_dtype, dev)
    out.copy_(src.view(dims).to(dev))
    return DenseMatrix._wrap(out, p)
