"""The verification-report schema (reference cli.py:104-148) on the host: a report written
by the reference's own `verify` command (tests/golden/reference_verify_report.json, made in
the build container with tilefuse.cli.main(["verify", "--seed", "0", "--json-out", ...]))
parses with this package's parse_report, and build/render reproduce its format."""

import json
from pathlib import Path

import pytest

import paper_2605_19269_b200 as cd
from paper_2605_19269_b200 import report as R

GOLDEN = Path(__file__).parent / "golden" / "reference_verify_report.json"


def test_reference_report_parses_and_rerenders_identically():
    text = GOLDEN.read_text()
    rep = R.parse_report(text)
    assert [c["name"] for c in rep["checks"]] == sorted(c["name"] for c in rep["checks"])
    assert R.all_passed(rep)
    checks = [R.CheckResult(c["name"], c["metric"], c["tolerance"]) for c in rep["checks"]]
    extra = {k: v for k, v in rep.items() if k not in ("version", "seed", "checks", "environment")}
    ours = R.build_report(rep["seed"], checks, cd.PrecisionMode.EXACT64, **extra)
    ours["version"] = rep["version"]
    assert R.render_report(ours) == text


@pytest.mark.parametrize("mutate,msg", [
    (lambda r: r.pop("seed"), "missing 'seed'"),
    (lambda r: r.__setitem__("checks", {}), "wrong type"),
    (lambda r: r["environment"].pop("precision"), "missing 'precision'"),
    (lambda r: r["checks"][0].pop("pass"), "'pass' missing"),
    (lambda r: r["checks"].reverse(), "ordered by name"),
])
def test_parse_report_rejections(mutate, msg):
    rep = json.loads(GOLDEN.read_text())
    mutate(rep)
    with pytest.raises(cd.TileFuseError, match=msg):
        R.parse_report(json.dumps(rep))
    with pytest.raises(cd.TileFuseError, match="malformed"):
        R.parse_report("{not json")
