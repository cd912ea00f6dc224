"""GPU verification report (f3): the reference's eight named checks run through the CUDA path
against the float64 oracle, serialized in the reference's JSON schema and re-parsed.  The
report is also written to gpurun_out/verify_report_<precision>.json when run on the box."""

import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["sim32", "simbf16"])
def test_gpu_verify_report(cuda_ready, precision):
    import gpu_verify

    from paper_2605_19269_b200 import report as R

    rep = gpu_verify.make_report(precision, seed=0)
    text = R.render_report(rep)
    assert R.parse_report(text) == rep
    names = [c["name"] for c in rep["checks"]]
    assert names == ["gradients_fd", "gradients_oracle", "kernel_oracles", "lse_blocking", "pipeline_oracles",
                     "scale_commutation", "statistic_relocation", "tile_invariance"]
    out = Path(__file__).resolve().parents[1] / "gpurun_out"
    if out.is_dir():
        (out / f"verify_report_{precision}.json").write_text(text)
    print("\n" + "\n".join(f"{c['name']}: {c['metric']:.3e} <= {c['tolerance']:g}" for c in rep["checks"]))
    assert R.all_passed(rep), rep["checks"]
