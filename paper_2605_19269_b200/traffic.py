"""Modeled HBM-traffic ledger of launches.

Same accounting convention as the reference ledger
(tilefuse/traffic.py:1-108): each bound operand is charged once at its
storage width, each store event at the problem's storage width (tiles) or
partial width (partials, gathers), labels at 4 bytes.  On the GPU these are
the *algorithmic* bytes of a launch; measured `dram__bytes` from ncu are
compared against them (profiles/).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable

from .errors import ConfigError

LABEL_BYTES = 4

K_RESIDUAL_RMS = "gemm_residual_partial_rms"
K_ROW_SCALE = "gemm_row_scale"
K_RMS_SWIGLU = "gemm_rms_swiglu"
K_RMS_ROPE = "gemm_rms_rope"
K_RMS_XENT = "gemm_rms_partial_xent"
K_PARTIAL_XENT = "gemm_partial_xent"
K_ROPE = "gemm_rope"
K_SWIGLU = "gemm_swiglu"
K_RMSNORM_BWD = "gemm_rmsnorm_backward"
K_SWIGLU_BWD = "gemm_swiglu_backward"
K_GEMM = "gemm"
K_ROPE_BWD_STAT = "rope_backward_stat"
R_FINALIZE_RMS = "finalize_rms"
R_FINALIZE_ROWDOT = "finalize_rowdot"
R_COMBINE_LSE = "combine_lse"
R_REDUCE_ROWVEC = "reduce_row_partials"
R_XENT_FINALIZE = "cross_entropy_finalize"


@dataclass(frozen=True)
class LaunchRecord:
    name: str
    read_bytes: int
    write_bytes: int

    @property
    def total_bytes(self) -> int:
        return self.read_bytes + self.write_bytes


@dataclass
class TrafficLedger:
    records: list[LaunchRecord] = field(default_factory=list)

    def record(self, name: str, read_bytes: int, write_bytes: int) -> LaunchRecord:
        if read_bytes < 0 or write_bytes < 0:
            raise ConfigError("byte counts cannot be negative")
        rec = LaunchRecord(name, int(read_bytes), int(write_bytes))
        self.records.append(rec)
        return rec

    def add(self, rec: LaunchRecord) -> None:
        self.records.append(rec)

    def extend(self, recs: Iterable[LaunchRecord]) -> None:
        self.records.extend(recs)

    @property
    def launches(self) -> int:
        return len(self.records)

    @property
    def read_bytes(self) -> int:
        return sum(r.read_bytes for r in self.records)

    @property
    def write_bytes(self) -> int:
        return sum(r.write_bytes for r in self.records)

    @property
    def total_bytes(self) -> int:
        return self.read_bytes + self.write_bytes

    def merged(self, other: "TrafficLedger") -> "TrafficLedger":
        return TrafficLedger(self.records + other.records)

    def __repr__(self) -> str:
        return f"TrafficLedger(launches={self.launches}, read={self.read_bytes}, write={self.write_bytes})"
