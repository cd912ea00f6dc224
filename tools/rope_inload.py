"""rope_backward_stat at C4 timed alone and right after a power-heavy GEMM (the in-step
condition of the block's backward), CUDA events around each rope launch."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import os  # noqa: E402

os.environ.setdefault("CODA_LIB", "exp")   # rope_u lives in the experiment build
from paper_2605_19269_b200 import _build  # noqa: E402

_build.build(experiments=True)
import bench  # noqa: E402
import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import _native  # noqa: E402

P = cd.PrecisionMode.SIMBF16
dev = torch.device("cuda", 0)
m, d = 16384, 4096
q = 3 * d
cos, sin = cd.qkv_rope_tables(m, d, precision=P)
g = cd.DenseMatrix.from_tensor(torch.randn(m, q, device=dev).to(torch.bfloat16), P)
r = cd.DenseMatrix.from_tensor(torch.randn(m, q, device=dev).to(torch.bfloat16), P)
a = cd.DenseMatrix.from_tensor((torch.randn(m, d, device=dev) * 0.05).to(torch.bfloat16), P)
b = cd.DenseMatrix.from_tensor((torch.randn(d, q, device=dev) * 0.05).to(torch.bfloat16), P)
prob = cd.GemmProblem(m, q, d, precision=P)
byts = 2 * m * q * 2 + 2 * m * (d // 2) * 2 + m * q * 2 + m * (q // 128) * 4
peak = bench.peaks()["hbm_gbs"]
out = {}
for variant in (0, 3, 6, 1):
  _native.set_option("rope_u", variant)
  for mode in ("alone", "after_gemm"):
    ts = []
    for it in range(40):
        if mode == "after_gemm":
            for _ in range(3):
                cd.run_gemm(prob, a, b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cd.rope_backward_stat(g, r, cos, sin, precision=P)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts[5:])
    out[f"u{variant}_{mode}"] = {"ms": round(ms, 4), "frac": round(byts / ms / 1e6 / peak, 3)}
print(json.dumps(out))
