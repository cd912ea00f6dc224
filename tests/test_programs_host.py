"""Random epilogue-program compositions drawn and run by the REFERENCE engine
(tests/golden/make_programs.py) are accepted, validated and lowered by this
package's host API exactly as the reference built them (no GPU needed)."""

from fractions import Fraction

import pytest

import paper_2605_19269_b200 as cd
from programs_common import build_program, load_programs


@pytest.mark.parametrize("kind", ["programs", "programs_ext"])
@pytest.mark.parametrize("mode", ["simbf16", "sim32"])
def test_reference_programs_lower(mode, kind):
    z, specs = load_programs(mode, kind)
    assert len(specs) >= (16 if kind == "programs" else 8)
    for i, sp in enumerate(specs):
        prog = build_program(cd, sp["steps"])
        steps, onames, snames = prog.lower()
        assert len(steps) == len(sp["steps"])
        # every operand the reference bound is declared, at the width the fixture holds
        for name in onames:
            arr = z[f"p{i}_in_{name}"]
            op = prog.operands[name]
            want = Fraction(sp["n"]) * op.factor
            if op.kind.name == "TILE":
                assert arr.shape == (sp["m"], int(want)), (i, name)
        # and every auxiliary output the reference produced has a store of that name
        assert set(sp["aux"]) == set(snames), (i, sp["aux"], snames)
