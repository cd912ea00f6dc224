"""Shared loader for the random-program golden fixtures (tests/golden/make_programs.py)."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load_programs(mode: str, kind: str = "programs"):
    """kind: "programs" (random compositions, make_programs.py) or "programs_ext" (widened device
    program space: >2 row streams, factors down to 1/32, > 8 steps/operands/stores)."""
    z = np.load(GOLDEN / f"{kind}_{mode}.npz")
    specs = json.loads(bytes(z["specs"]).decode())
    return z, specs


def build_program(cd, steps):
    return cd.EpilogueProgram([getattr(cd, name)(**kw) for name, kw in steps])
