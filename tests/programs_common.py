"""Shared loader for the random-program golden fixtures (tests/golden/make_programs.py)."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load_programs(mode: str):
    z = np.load(GOLDEN / f"programs_{mode}.npz")
    specs = json.loads(bytes(z["specs"]).decode())
    return z, specs


def build_program(cd, steps):
    return cd.EpilogueProgram([getattr(cd, name)(**kw) for name, kw in steps])
