"""DRAM bytes of the K9a-shape plain GEMM (16384x4096x28672 NT): this engine vs cuBLAS (run under ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import os  # noqa: E402

os.environ.setdefault("CODA_LIB", "exp")
from paper_2605_19269_b200 import _build  # noqa: E402

_build.build(experiments=True)
import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import _native  # noqa: E402

P = cd.PrecisionMode.SIMBF16
m, n, k = 16384, 4096, 28672
A = (torch.randn(m, k, device="cuda") * 0.05).to(torch.bfloat16)
B = (torch.randn(n, k, device="cuda") * 0.05).to(torch.bfloat16)
prob = cd.GemmProblem(m=m, n=n, k=k, trans_b=True, precision=P)
a, b = cd.DenseMatrix.from_tensor(A, P), cd.DenseMatrix.from_tensor(B, P)
for _ in range(2):
    cd.run_gemm(prob, a, b)
    torch.matmul(A, B.t())
    _native.set_option("persist", 0)
    cd.run_gemm(prob, a, b)
    _native.set_option("persist", 1)
    for pct in (50, 90):
        _native.set_option("wave_sync", pct)
        cd.run_gemm(prob, a, b)
        _native.set_option("wave_sync", 0)
torch.cuda.synchronize()
