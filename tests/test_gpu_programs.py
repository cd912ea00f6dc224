"""GPU parity of RANDOM epilogue-program compositions against the reference engine.

Programs, inputs and outputs come from the reference's own run_gemm
(tests/golden/make_programs.py): 16 seeded compositions per precision over the
whole primitive set (row/col scaling, residual, aux stores, sum-of-squares /
row-dot / column-sum partials, online LSE + target gather, RoPE, SwiGLU and its
backward, the RMSNorm backward), ragged shapes, the reference's four tile
contexts.  Every main output, auxiliary tile and partial slot (data and
per-block counts) is compared.
"""

import numpy as np
import pytest

from oracle import coda_oracle as O
from programs_common import build_program, load_programs

pytestmark = pytest.mark.gpu

TOL = {"sim32": 1e-5, "simbf16": 2e-2}


@pytest.mark.parametrize("kind", ["programs", "programs_ext"])
@pytest.mark.parametrize("mode", ["simbf16", "sim32"])
def test_reference_programs_on_gpu(cuda_ready, mode, kind):
    """kind "programs_ext": 3-4 row-partial streams, SwiGLU chains down to factor 1/32, a
    12- and a 16-step program with > 8 operands / stores (tests/golden/make_programs_ext.py)."""
    import paper_2605_19269_b200 as cd

    z, specs = load_programs(mode, kind)
    P = cd.PrecisionMode.SIMBF16 if mode == "simbf16" else cd.PrecisionMode.SIM32
    worst = {}
    for i, sp in enumerate(specs):
        p = f"p{i}_"
        prog = build_program(cd, sp["steps"])
        bindings = {}
        for name, op in prog.operands.items():
            arr = z[p + "in_" + name]
            kind = op.kind.name
            if kind == "TILE":
                bindings[name] = cd.DenseMatrix.from_array(arr.astype(np.float64), P)
            elif kind == "ROW_VEC":
                bindings[name] = cd.Vector.from_array(arr.astype(np.float64), P)
            elif kind == "COL_VEC":
                bindings[name] = cd.Vector.from_array(arr.astype(np.float64), cd.stat_mode(P))
            else:
                bindings[name] = arr.astype(np.int64)
        a = cd.DenseMatrix.from_array(z[p + "a"].astype(np.float64), P)
        b = cd.DenseMatrix.from_array(z[p + "b"].astype(np.float64), P)
        prob = cd.GemmProblem(m=sp["m"], n=sp["n"], k=sp["k"], tile_shape=cd.TileShape(*sp["tile"]),
                              reduction_tile_n=sp["rtn"], precision=P)
        res = cd.run_gemm(prob, a, b, prog, bindings)
        label = " + ".join(s for s, _ in sp["steps"])
        errs = {"main": O.rel_error(res.main.data, z[p + "main"])}
        for name, kind in sp["aux"].items():
            want = z[p + "aux_" + name].astype(np.float64)
            got = res.aux[name]
            if kind == "slot":
                assert np.array_equal(np.asarray(got.counts), z[p + "cnt_" + name]), (i, label, name)
                gd = np.asarray(got.data, dtype=np.float64)
                if "lse" in name:
                    # (max, scaled-sum) pairs are only defined up to the pair's own scale: compare the
                    # per-block log-sum-exp they encode
                    enc = lambda d: d[..., 0] + np.log(d[..., 1])  # noqa: E731
                    errs[name] = O.rel_error(enc(gd), enc(want))
                else:
                    errs[name] = O.rel_error(gd, want)
            else:
                errs[name] = O.rel_error(np.asarray(got.data, dtype=np.float64), want)
        w = max(errs.values())
        worst[f"{i}: {label}"] = w
        assert w <= TOL[mode], (i, label, errs)
    print(f"\n[{mode}] worst rel err per program: " + "; ".join(f"{k} {v:.1e}" for k, v in worst.items()))
