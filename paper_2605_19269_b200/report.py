"""Machine-readable verification reports (reference cli.py:104-148, checks.py:44-62).

The reference's `verify` command writes a JSON report of named invariant checks:
{"version", "seed", "checks": [{"name", "metric", "tolerance", "pass"}] sorted by
name, "environment": {"precision", ...}} plus free extra keys.  This module keeps
that schema byte-compatible (same keys, sort order, `json.dumps(indent=2,
sort_keys=True)` rendering, same validation errors) so reports from GPU runs of
this engine and from the reference can be read by the same tooling.  The GPU
checks themselves compare against the CPU oracle, which is test infrastructure:
they live in tests/gpu_verify.py and run under `pytest -m gpu`.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Sequence

from .errors import TileFuseError
from .tensors import PrecisionMode

REPORT_VERSION = "0.1.0"   # the reference package's __version__ (cli.py:41)


@dataclass(frozen=True)
class CheckResult:
    """Outcome of one named check (checks.py:44-62)."""

    name: str
    metric: float
    tolerance: float

    @property
    def passed(self) -> bool:
        return bool(self.metric <= self.tolerance)

    def as_dict(self) -> dict:
        return {"name": self.name, "metric": self.metric, "tolerance": self.tolerance, "pass": self.passed}


def build_report(seed: int, checks: Sequence[CheckResult], precision: PrecisionMode, **extra) -> dict:
    """cli.py:105-114: checks sorted by name, environment.precision, extra keys merged."""
    report = {
        "version": REPORT_VERSION,
        "seed": seed,
        "checks": [c.as_dict() for c in sorted(checks, key=lambda c: c.name)],
        "environment": {"precision": precision.value},
    }
    report.update(extra)
    return report


def render_report(report: dict) -> str:
    return json.dumps(report, indent=2, sort_keys=True) + "\n"


def parse_report(text: str) -> dict:
    """Validate and load a JSON report (cli.py:121-148, same error messages)."""
    try:
        report = json.loads(text)
    except ValueError as exc:
        raise TileFuseError(f"malformed report: {exc}") from None
    if not isinstance(report, dict):
        raise TileFuseError("report is not an object")
    for key, kind in (("version", str), ("seed", int), ("checks", list), ("environment", dict)):
        if key not in report:
            raise TileFuseError(f"report is missing {key!r}")
        if not isinstance(report[key], kind):
            raise TileFuseError(f"report field {key!r} has the wrong type")
    if "precision" not in report["environment"]:
        raise TileFuseError("report environment is missing 'precision'")
    for entry in report["checks"]:
        if not isinstance(entry, dict):
            raise TileFuseError("check entries must be objects")
        for key, kinds in (("name", (str,)), ("metric", (int, float)), ("tolerance", (int, float)),
                           ("pass", (bool,))):
            if key not in entry or not isinstance(entry[key], kinds):
                raise TileFuseError(f"check entry field {key!r} missing or wrong type")
    names = [e["name"] for e in report["checks"]]
    if names != sorted(names):
        raise TileFuseError("check entries must be ordered by name")
    return report


def all_passed(report: dict) -> bool:
    return all(bool(e["pass"]) for e in report["checks"])
