"""ctypes bridge to the C-ABI declared in include/coda.h.

This is the only module that touches the shared library.  There is no
fallback: if `libcoda.so` is missing or cannot be loaded, every GPU entry
point raises `NativeUnavailable` (the product path must fail loudly).
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from . import errors

import os

# CODA_LIB=exp selects the experiment build, CODA_LIB=<variant> an experiment variant
# (_build.VARIANTS) -- tools/ only: measurement knobs, see coda.h
_LIB_NAME = os.environ.get("CODA_LIB", "")
LIB_PATH = Path(__file__).resolve().parent / "_lib" / (f"libcoda_{_LIB_NAME}.so" if _LIB_NAME else "libcoda.so")

# ---- constants mirrored from include/coda.h ----
BF16, F32, I64, I32 = 0, 1, 2, 3

OP_ROW_VEC_MUL = 1
OP_ROW_SCALE = 2
OP_RESIDUAL_ADD = 3
OP_AUX_TILE_STORE = 4
OP_PARTIAL_SUMSQ = 5
OP_PARTIAL_ROWDOT = 6
OP_PARTIAL_COLSUM = 7
OP_ONLINE_LSE = 8
OP_TARGET_GATHER = 9
OP_ROPE = 10
OP_SWIGLU = 11
OP_SWIGLU_BWD = 12
OP_RMSNORM_BWD = 13
OP_XENT_BWD = 14

FIN_RMS, FIN_ROWDOT = 1, 2   # deferred finalizer kinds (coda_step_t.fin_kind)

STORE_TILE, STORE_ROW_SUM, STORE_ROW_PAIR, STORE_COL_SUM, STORE_GATHER = 0, 1, 2, 3, 4

MAX_STEPS = 16
MAX_OPERANDS = 16
MAX_STORES = 16
MAX_ROW_STREAMS = 4
MAX_PEERS = 8

# GPU tile geometry of the persistent kernel (csrc/coda_gemm.cuh)
GPU_TILE_M = 128
GPU_TILE_N = 256

EXPORTS = (
    "coda_gemm_epilogue",
    "coda_finalize_rms",
    "coda_finalize_rowdot",
    "coda_reduce_row_partials",
    "coda_combine_lse",
    "coda_cross_entropy_finalize",
    "coda_rope_backward_stat",
    "coda_rope_backward_stat_compact",
    "coda_combine_row_pieces",
    "coda_combine_col_pieces",
    "coda_split_operand",
    "coda_convert_f32_bf16",
    "coda_scale_rows",
    "coda_peer_reduce_sizes",
    "coda_gemm_peer_reduce",
    "coda_num_sms",
    "coda_set_option",
    "coda_version",
    "coda_last_error",
)


class Tensor(ctypes.Structure):
    _fields_ = [
        ("ptr", ctypes.c_void_p),
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("ld", ctypes.c_int64),
        ("dtype", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
    ]


class Problem(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("k", ctypes.c_int64),
        ("trans_a", ctypes.c_int32),
        ("trans_b", ctypes.c_int32),
        ("storage", ctypes.c_int32),
        ("out_dtype", ctypes.c_int32),
        ("store_main", ctypes.c_int32),
        ("sm_limit", ctypes.c_int32),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_int64),
    ]


class Step(ctypes.Structure):
    _fields_ = [
        ("op", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("arg", ctypes.c_int32 * 7),
        ("fin_src", ctypes.c_int32),
        ("fin_kind", ctypes.c_int32),
        ("fin_d", ctypes.c_int32),
        ("fin_eps", ctypes.c_float),
        ("_pad", ctypes.c_int32),
    ]


class Store(ctypes.Structure):
    _fields_ = [
        ("t", Tensor),
        ("piece_map", ctypes.c_void_p),
        ("kind", ctypes.c_int32),
        ("aligned", ctypes.c_int32),
    ]


class PeerReduce(ctypes.Structure):
    """coda_peer_reduce_t: the cross-rank weight-gradient sum fused into the GEMM epilogue."""

    _fields_ = [
        ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("slots", ctypes.c_void_p * MAX_PEERS),
        ("counters", ctypes.c_void_p * MAX_PEERS),
        ("out", ctypes.c_void_p * MAX_PEERS),
        ("ld_out", ctypes.c_int64),
        ("slot_bytes", ctypes.c_int64),
        ("counter_bytes", ctypes.c_int64),
    ]


class NativeUnavailable(errors.TileFuseError):
    """The CUDA library could not be loaded (no silent CPU fallback exists)."""


_lock = threading.Lock()
_lib = None

_ERRMAP = {
    -1: errors.DimensionError,
    -2: errors.BindingError,
    -3: errors.ProgramError,
    -4: errors.PairingError,
    -5: errors.ConfigError,
    -6: errors.LabelError,
    -7: errors.DegenerateError,
}


def _declare(lib) -> None:
    vp, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
    P = ctypes.POINTER
    lib.coda_gemm_epilogue.argtypes = [P(Problem), P(Tensor), P(Tensor), P(Step), i32, P(Tensor), i32,
                                       P(Store), i32, P(Tensor), P(Tensor), vp]
    lib.coda_finalize_rms.argtypes = [vp, i64, i64, i64, i64, f32, vp, vp]
    lib.coda_finalize_rowdot.argtypes = [vp, i64, i64, i64, i64, vp, vp]
    lib.coda_reduce_row_partials.argtypes = [vp, i64, i64, i64, vp, vp]
    lib.coda_combine_lse.argtypes = [vp, i64, i64, i64, vp, vp]
    lib.coda_cross_entropy_finalize.argtypes = [vp, vp, i64, vp, vp]
    lib.coda_rope_backward_stat.argtypes = [P(Tensor), P(Tensor), P(Tensor), P(Tensor), vp, i64, P(Tensor),
                                            vp, i64, vp]
    lib.coda_rope_backward_stat_compact.argtypes = [P(Tensor), P(Tensor), P(Tensor), P(Tensor), i64, P(Tensor),
                                                    vp, i64, vp]
    lib.coda_combine_row_pieces.argtypes = [vp, i64, i64, i64, vp, i64, i32, vp, i64, vp]
    lib.coda_combine_col_pieces.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, vp]
    lib.coda_split_operand.argtypes = [P(Tensor), i32, i64, P(ctypes.c_int32), P(Tensor), vp]
    lib.coda_convert_f32_bf16.argtypes = [P(Tensor), P(Tensor), vp]
    lib.coda_scale_rows.argtypes = [P(Tensor), vp, P(Tensor), vp]
    lib.coda_peer_reduce_sizes.argtypes = [i64, i64, ctypes.c_int32, P(i64), P(i64)]
    lib.coda_gemm_peer_reduce.argtypes = [P(Problem), P(Tensor), P(Tensor), P(PeerReduce), vp]
    lib.coda_num_sms.argtypes = []
    lib.coda_set_option.argtypes = [ctypes.c_char_p, i32]
    lib.coda_version.argtypes = []
    lib.coda_version.restype = ctypes.c_char_p
    lib.coda_last_error.argtypes = []
    lib.coda_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("coda_version", "coda_last_error"):
            getattr(lib, name).restype = ctypes.c_int


def load(path: Path | None = None):
    """Load (once) and return the ctypes handle of libcoda.so."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise NativeUnavailable(
                f"CUDA library {p} is missing; run __graft_entry__.build() "
                f"(there is no CPU fallback)"
            )
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:  # pragma: no cover - depends on the box
            raise NativeUnavailable(f"cannot load {p}: {exc}") from exc
        _declare(lib)
        if path is None:
            _lib = lib
        return lib


def check(rc: int) -> None:
    """Raise the reference error class that a non-zero return code maps to."""
    if rc == 0:
        return
    msg = (_lib.coda_last_error() or b"").decode(errors="replace") if _lib is not None else ""
    cls = _ERRMAP.get(rc)
    if cls is None:
        raise RuntimeError(f"CUDA error in CODA library ({rc}): {msg}")
    raise cls(msg)


_launches = 0
_profile = None   # list of (tag, flops, start_event, end_event) while profiling
_tags = None      # list of launch tags while recording (no events)


def record_tags(rows) -> None:
    """Start (rows = a list) or stop (None) recording the tag of every launch."""
    global _tags
    _tags = rows


def call(name: str, *args, tag: str | None = None, flops: float = 0.0) -> None:
    """Invoke one C-ABI entry point; every call enqueues exactly one kernel."""
    global _launches
    lib = load()
    if _tags is not None:
        _tags.append(tag or name)
    if _profile is not None:
        import torch

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        check(getattr(lib, name)(*args))
        e1.record()
        _profile.append((tag or name, flops, e0, e1))
    else:
        check(getattr(lib, name)(*args))
    _launches += 1


def set_option(name: str, value: int) -> None:
    """Process-wide engine schedule option ("pdl", "cg", "generic", "raster", "split",
    "split_min_k"); see include/coda.h.  Measurement knobs ("ring", "prefetch", "ablate")
    exist only in experiment builds (libcoda_exp.so, CODA_LIB=exp)."""
    check(load().coda_set_option(name.encode(), int(value)))


_tls = threading.local()


def sm_limit() -> int:
    """SM cap of the GEMM launches enqueued by this thread (0 = every SM)."""
    return getattr(_tls, "sm_limit", 0)


class limit_sms:
    """Context manager: GEMM launches enqueued inside use at most `n` SMs (0 = all).

    Used around the backward of a data-parallel step so the NCCL all-reduce of
    the weight gradients, running on a side stream, keeps SMs of its own instead
    of waiting for gaps between persistent launches.  Thread-local; results are
    identical with any cap."""

    def __init__(self, n: int):
        if n < 0:
            raise errors.ConfigError(f"SM limit must be >= 0, got {n}")
        self.n = int(n)

    def __enter__(self):
        self.prev = sm_limit()
        _tls.sm_limit = self.n
        return self

    def __exit__(self, *exc):
        _tls.sm_limit = self.prev
        return False


WORKSPACE_BYTES = 96 << 20
_workspaces: dict = {}


def workspace(device):
    """Zeroed scratch for wave-tail splitting, one per (device, current stream), or None.

    The split-K counters are reset by the launch that consumes them, so consecutive
    launches on one stream can share the buffer; launches on different streams may
    run concurrently and therefore get their own.  A stream that is being captured
    into a CUDA graph without a workspace of its own gets None (the launch runs
    unsplit): borrowing another stream's buffer would let the graph's replay and
    eager launches on the owner stream race on the same counters.  Call
    `prepare_stream_workspace()` on the capture stream before capturing to keep
    the split inside graphs."""
    import torch

    key = (str(device), torch.cuda.current_stream(device).cuda_stream)
    ws = _workspaces.get(key)
    if ws is None:
        if torch.cuda.is_current_stream_capturing():
            return None
        ws = torch.zeros(WORKSPACE_BYTES // 4, dtype=torch.int32, device=device)
        _workspaces[key] = ws
    return ws


def prepare_stream_workspace(device, stream) -> None:
    """Allocate (outside capture) the split workspace owned by `stream`."""
    import torch

    with torch.cuda.stream(stream):
        workspace(device)
    torch.cuda.synchronize(device)


def num_sms() -> int:
    """SM count of the current device as the library sees it (0 without a device)."""
    return int(load().coda_num_sms())


def launch_count() -> int:
    """Number of CODA kernels enqueued by this process so far."""
    return _launches


def profile_launches(fn, reps: int = 2, lead: int = 1) -> dict:
    """Run fn() `reps` times recording CUDA events around every launch.

    Returns {tag: {name, count, avg_ms, total_ms, flops}} (flops per launch).
    Events are recorded on the launching (current) stream.  `lead` unrecorded calls
    are enqueued first, without a sync, so the recorded launches sit behind queued
    device work: on an idle GPU the first launch's interval would also contain the
    host time between its start event and the kernel (validation, allocation).
    """
    import torch

    global _profile
    for _ in range(lead):
        fn()
    _profile = []
    try:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        rows = _profile
    finally:
        _profile = None
    out: dict = {}
    for tag, flops, e0, e1 in rows:
        r = out.setdefault(tag, {"name": tag, "count": 0, "total_ms": 0.0, "flops": flops})
        r["count"] += 1
        r["total_ms"] += e0.elapsed_time(e1)
    for r in out.values():
        r["avg_ms"] = r["total_ms"] / r["count"]
        r["total_ms"] /= reps
        r["count"] //= reps
    return out


def tensor_desc(t, dtype_code: int | None = None) -> Tensor:
    """Describe a 1-D or 2-D torch CUDA tensor (row-major, unit column stride)."""
    import torch

    code = dtype_code if dtype_code is not None else dtype_of(t)
    if t.dim() == 1:
        if t.stride(0) != 1:
            raise errors.BindingError("vector operands must be contiguous")
        return Tensor(t.data_ptr(), 1, t.shape[0], t.shape[0], code, 0)
    if t.dim() != 2:
        raise errors.DimensionError(f"expected a 1-D or 2-D tensor, got {t.dim()}-D")
    if t.stride(1) != 1 and t.shape[1] > 1:
        raise errors.BindingError("matrices must have unit column stride")
    ld = t.stride(0) if t.shape[0] > 1 else max(t.stride(0), t.shape[1])
    return Tensor(t.data_ptr(), t.shape[0], t.shape[1], ld, code, 0)


def dtype_of(t) -> int:
    import torch

    m = {torch.bfloat16: BF16, torch.float32: F32, torch.int64: I64, torch.int32: I32}
    if t.dtype not in m:
        raise errors.BindingError(f"unsupported device dtype {t.dtype}")
    return m[t.dtype]


def peer_reduce_sizes(m: int, n: int, world: int) -> tuple[int, int]:
    """Bytes of the f32 landing buffer and of the counter buffer every rank of a
    `world`-rank peer-reduced (m, n) weight gradient needs (coda_peer_reduce_sizes)."""
    sb, cb = ctypes.c_int64(0), ctypes.c_int64(0)
    check(load().coda_peer_reduce_sizes(int(m), int(n), int(world), ctypes.byref(sb), ctypes.byref(cb)))
    return int(sb.value), int(cb.value)
