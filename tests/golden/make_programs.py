"""Golden vectors for RANDOM epilogue-program compositions, from the REFERENCE engine.

The reference's tests compose primitives freely (tests/test_epilogue.py); this script
draws seeded random programs from the primitive set, runs each through the
reference's own `run_gemm` (tilefuse, read-only from /root/reference) on ragged
shapes in the reference's tile contexts, and stores program specs + inputs +
outputs in programs_<mode>.npz.  tests/test_gpu_programs.py replays every program
through the CUDA path; tests/test_programs_host.py checks that the same programs
validate and lower on the host.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_programs.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import tilefuse as tf  # noqa: E402

OUT = Path(__file__).resolve().parent
TILES = [((16, 24), 10), ((32, 32), 32), ((8, 24), 4), ((128, 128), 128)]   # test_acceptance.py:64-69
N_PROGRAMS = 16


def draw_program(rng):
    """A random valid composition as a list of (primitive, kwargs) specs.

    Running width factor f starts at 1; partial emitters only at f == 1 (the
    reference rule), SwiGLU halves f, SwiGLU-backward doubles it; at most two
    row-partial streams per program (the GPU epilogue's limit)."""
    steps, f, k = [], 1, 0
    row_parts = 0
    lse_gather = False
    for _ in range(int(rng.integers(1, 6))):
        k += 1
        if f == 1:
            pool = ["RowVecMul", "RowScale", "ResidualAdd", "AuxTileStore", "PairwiseRope", "PartialColSum",
                    "PairwiseSwiglu", "PairwiseSwigluBackward", "RmsNormBackwardLocal"]
            if row_parts < 2:
                pool += ["PartialSumSq", "PartialRowDot"]
            if row_parts < 2 and not lse_gather:
                pool += ["OnlineLse"]
        else:
            pool = ["RowVecMul", "RowScale", "ResidualAdd", "AuxTileStore"]
        p = pool[int(rng.integers(len(pool)))]
        if p == "RowVecMul":
            steps.append((p, {"operand": f"v{k}"}))
        elif p == "RowScale":
            steps.append((p, {"operand": f"c{k}"}))
        elif p == "ResidualAdd":
            steps.append((p, {"operand": f"t{k}"}))
        elif p == "AuxTileStore":
            steps.append((p, {"name": f"aux{k}"}))
        elif p == "PairwiseRope":
            steps.append((p, {"cos": f"cos{k}", "sin": f"sin{k}", "backward": bool(rng.integers(2))}))
        elif p == "PartialColSum":
            steps.append((p, {"name": f"colsum{k}"}))
        elif p == "PartialSumSq":
            steps.append((p, {"name": f"sumsq{k}"}))
            row_parts += 1
        elif p == "PartialRowDot":
            steps.append((p, {"operand": f"t{k}", "name": f"rowdot{k}"}))
            row_parts += 1
        elif p == "OnlineLse":
            steps.append((p, {"name": f"lse{k}"}))
            steps.append(("TargetGather", {"labels": f"labels{k}", "name": f"target{k}"}))
            row_parts += 1
            lse_gather = True
        elif p == "PairwiseSwiglu":
            steps.append((p, {}))
            f = 0.5
        elif p == "PairwiseSwigluBackward":
            if row_parts >= 2:
                continue
            steps.append((p, {"preact": f"pre{k}", "recompute": f"rec{k}", "name": f"srowdot{k}"}))
            row_parts += 1
            f = 2
        elif p == "RmsNormBackwardLocal":
            acc = f"acc{k}" if rng.integers(2) else None
            steps.append((p, {"pre": f"pn{k}", "inv_rms": f"r{k}", "gamma": f"g{k}", "stat": f"s{k}",
                              "accumulate": acc, "normed_out": f"normed{k}", "gamma_grad": f"gg{k}"}))
            break   # its output is a dgrad; end the program here
    return steps


def bind(rng, program, steps, m, n, mode):
    """Reference bindings for every operand the program declares, at its factor."""
    b, arrays = {}, {}
    for name, op in program.operands.items():
        w = int(n * op.factor)
        kind = op.kind.name
        if kind == "TILE":
            scale = 0.7 if name.startswith(("cos", "sin")) else 1.0
            x = rng.standard_normal((m, w)) * scale
            if name.startswith(("cos", "sin")):
                x = np.repeat(x[:, 0::2], 2, axis=1)[:, :w]    # one angle per pair, like rope tables
            b[name] = tf.DenseMatrix.from_array(x, mode)
            arrays[name] = b[name].data
        elif kind == "ROW_VEC":
            b[name] = tf.Vector.from_array(1.0 + 0.1 * rng.standard_normal(w), mode)
            arrays[name] = b[name].data
        elif kind == "COL_VEC":
            b[name] = tf.Vector.from_array(0.5 + rng.random(m), tf.stat_mode(mode))
            arrays[name] = b[name].data
        elif kind == "LABELS":
            lab = rng.integers(0, n, m).astype(np.int64)
            b[name] = lab
            arrays[name] = lab
        else:
            raise AssertionError(kind)
    return b, arrays


def main():
    for mode_name, mode in (("simbf16", tf.PrecisionMode.SIMBF16), ("sim32", tf.PrecisionMode.SIM32)):
        rng = np.random.default_rng([2605, 19269, 0 if mode_name == "simbf16" else 1])
        out, specs = {}, []
        i = 0
        while i < N_PROGRAMS:
            steps = draw_program(rng)
            cls = {nm: getattr(tf, nm) for nm in {s for s, _ in steps}}
            try:
                program = tf.EpilogueProgram([cls[s](**kw) for s, kw in steps])
            except tf.TileFuseError:
                continue
            (tm, tn), rtn = TILES[i % len(TILES)]
            m = int(rng.integers(40, 170))
            k = int(rng.integers(16, 96))
            n = 2 * int(rng.integers(16, 90))
            a = tf.DenseMatrix.from_array(rng.standard_normal((m, k)), mode)
            bm = tf.DenseMatrix.from_array(rng.standard_normal((k, n)) / np.sqrt(k), mode)
            bindings, arrays = bind(rng, program, steps, m, n, mode)
            prob = tf.GemmProblem(m=m, n=n, k=k, tile_shape=tf.TileShape(tm, tn), reduction_tile_n=rtn,
                                  precision=mode)
            try:
                res = tf.run_gemm(prob, a, bm, program, bindings)
            except tf.TileFuseError:
                continue
            p = f"p{i}_"
            out[p + "a"], out[p + "b"] = a.data, bm.data
            for name, arr in arrays.items():
                out[p + "in_" + name] = arr
            out[p + "main"] = res.main.data
            auxes = {}
            for name, val in res.aux.items():
                if isinstance(val, tf.PartialSlot):
                    out[p + "aux_" + name] = np.asarray(val.data)
                    out[p + "cnt_" + name] = np.asarray(val.counts)
                    auxes[name] = "slot"
                else:
                    out[p + "aux_" + name] = val.data
                    auxes[name] = "tile" if isinstance(val, tf.DenseMatrix) else "vector"
            specs.append({"steps": steps, "m": m, "n": n, "k": k, "tile": [tm, tn], "rtn": rtn, "aux": auxes})
            i += 1
        for key, v in out.items():   # simulated modes: every value lies on the f32 grid (lossless)
            if v.dtype == np.float64:
                assert np.array_equal(v.astype(np.float32).astype(np.float64), v, equal_nan=True), key
                out[key] = v.astype(np.float32)
        out["specs"] = np.frombuffer(json.dumps(specs).encode(), dtype=np.uint8)
        np.savez_compressed(OUT / f"programs_{mode_name}.npz", **out)
        print(mode_name, [" + ".join(s for s, _ in sp["steps"]) for sp in specs])


if __name__ == "__main__":
    main()
