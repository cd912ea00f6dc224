"""Golden vectors for the program shapes beyond round 1's device limits, from the REFERENCE engine.

VERDICT r01 (missing #5): the reference accepts any number of row-partial emitters,
any reachable width factor and any program length (tilefuse epilogue.py:626-660);
the GPU epilogue previously stopped at 2 row streams, factors {1/2, 1, 2} and 8
steps / operands / stores.  These programs exercise the widened device program
space: 3 and 4 row-partial streams, chained SwiGLUs down to factor 1/32, a
backward-then-forward factor path, 12- and 16-step programs with more than 8
operands or stores.  Each runs through the reference's own run_gemm (read-only
/root/reference) and is stored like make_programs.py's fixtures
(programs_ext_<mode>.npz), replayed on the GPU by tests/test_gpu_programs.py.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_programs_ext.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, str(Path(__file__).resolve().parent))

from make_programs import OUT, bind, tf  # noqa: E402

PROGRAMS = [
    # (steps, m, n, k, tile, rtn)
    ([("PartialSumSq", {"name": "ss1"}), ("PartialRowDot", {"operand": "t2", "name": "rd2"}),
      ("OnlineLse", {"name": "lse3"}), ("TargetGather", {"labels": "lab3", "name": "tg3"})],
     150, 200, 48, (32, 32), 32),
    ([("PartialSumSq", {"name": "ss1"}), ("PartialRowDot", {"operand": "t2", "name": "rd2"}),
      ("RowScale", {"operand": "c3"}), ("PartialSumSq", {"name": "ss4"}),
      ("PartialRowDot", {"operand": "t5", "name": "rd5"})],
     140, 264, 40, (128, 128), 128),
    ([("PairwiseSwiglu", {}), ("PairwiseSwiglu", {})], 130, 256, 64, (128, 128), 128),
    ([("AuxTileStore", {"name": "a0"}), ("PairwiseSwiglu", {}), ("RowVecMul", {"operand": "v2"}),
      ("PairwiseSwiglu", {}), ("ResidualAdd", {"operand": "t4"}), ("AuxTileStore", {"name": "a5"}),
      ("PairwiseSwiglu", {}), ("RowScale", {"operand": "c7"})],
     100, 512, 32, (128, 128), 128),
    ([("PairwiseSwiglu", {}), ("PairwiseSwiglu", {}), ("PairwiseSwiglu", {}), ("PairwiseSwiglu", {}),
      ("PairwiseSwiglu", {})], 70, 256, 40, (128, 128), 128),
    ([("PairwiseSwigluBackward", {"preact": "p1", "recompute": "r1", "name": "d1"}), ("PairwiseSwiglu", {}),
      ("PairwiseSwiglu", {}), ("AuxTileStore", {"name": "a4"})], 90, 192, 24, (32, 32), 32),
    ([("RowScale", {"operand": "c1"}), ("RowVecMul", {"operand": "v2"}), ("ResidualAdd", {"operand": "t3"}),
      ("AuxTileStore", {"name": "a4"}), ("RowVecMul", {"operand": "v5"}), ("RowScale", {"operand": "c6"}),
      ("PartialSumSq", {"name": "ss7"}), ("ResidualAdd", {"operand": "t8"}), ("RowVecMul", {"operand": "v9"}),
      ("AuxTileStore", {"name": "a10"}), ("PairwiseRope", {"cos": "cos11", "sin": "sin11", "backward": True}),
      ("RowScale", {"operand": "c12"})],
     120, 160, 40, (16, 24), 10),
    ([("AuxTileStore", {"name": f"s{i}"}) if i % 2 == 0 else ("RowScale", {"operand": f"c{i}"})
      for i in range(16)] + [], 80, 96, 32, (32, 32), 32),
]


def main():
    for mode_name, mode in (("simbf16", tf.PrecisionMode.SIMBF16), ("sim32", tf.PrecisionMode.SIM32)):
        rng = np.random.default_rng([2605, 19269, 7, 0 if mode_name == "simbf16" else 1])
        out, specs = {}, []
        for i, (steps, m, n, k, (tm, tn), rtn) in enumerate(PROGRAMS):
            cls = {nm: getattr(tf, nm) for nm in {s for s, _ in steps}}
            program = tf.EpilogueProgram([cls[s](**kw) for s, kw in steps])
            a = tf.DenseMatrix.from_array(rng.standard_normal((m, k)), mode)
            bm = tf.DenseMatrix.from_array(rng.standard_normal((k, n)) / np.sqrt(k), mode)
            bindings, arrays = bind(rng, program, steps, m, n, mode)
            prob = tf.GemmProblem(m=m, n=n, k=k, tile_shape=tf.TileShape(tm, tn), reduction_tile_n=rtn,
                                  precision=mode)
            res = tf.run_gemm(prob, a, bm, program, bindings)
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
        for key, v in out.items():
            if v.dtype == np.float64:
                assert np.array_equal(v.astype(np.float32).astype(np.float64), v, equal_nan=True), key
                out[key] = v.astype(np.float32)
        out["specs"] = np.frombuffer(json.dumps(specs).encode(), dtype=np.uint8)
        np.savez_compressed(OUT / f"programs_ext_{mode_name}.npz", **out)
        print(mode_name, [" + ".join(s for s, _ in sp["steps"]) for sp in specs])


if __name__ == "__main__":
    main()
