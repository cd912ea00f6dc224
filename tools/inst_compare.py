"""Plain GEMM instruction / pipe activity: this engine vs cuBLAS at the K9a and K6 shapes (run under ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2605_19269_b200 as cd  # noqa: E402

P = cd.PrecisionMode.SIMBF16
for m, n, k, tb in ((16384, 4096, 28672, True), (16384, 28672, 4096, False)):
    A = (torch.randn(m, k, device="cuda") * 0.05).to(torch.bfloat16)
    B = (torch.randn(n, k, device="cuda") if tb else torch.randn(k, n, device="cuda")).mul(0.05).to(torch.bfloat16)
    prob = cd.GemmProblem(m=m, n=n, k=k, trans_b=tb, precision=P)
    a, b = cd.DenseMatrix.from_tensor(A, P), cd.DenseMatrix.from_tensor(B, P)
    cd.run_gemm(prob, a, b)
    torch.matmul(A, B.t() if tb else B)
torch.cuda.synchronize()
