"""Quick GPU sanity run: one GEMM per operand layout, printed errors (debug aid)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2605_19269_b200 as cd

P = cd.PrecisionMode.SIMBF16
for (m, n, k) in ((128, 256, 64), (256, 512, 256), (130, 264, 96)):
    for ta in (False, True):
        for tb in (False, True):
            A = torch.randn((k, m) if ta else (m, k), device="cuda").to(torch.bfloat16)
            B = torch.randn((n, k) if tb else (k, n), device="cuda").to(torch.bfloat16)
            t0 = time.time()
            res = cd.run_gemm(cd.GemmProblem(m=m, n=n, k=k, trans_a=ta, trans_b=tb, precision=P),
                              cd.DenseMatrix.from_tensor(A, P), cd.DenseMatrix.from_tensor(B, P), out_f32=True)
            torch.cuda.synchronize()
            ref = (A.float().T if ta else A.float()) @ (B.float().T if tb else B.float())
            got = res.main.tensor
            err = float((got - ref).norm() / ref.norm())
            print(f"m={m} n={n} k={k} ta={ta} tb={tb} rel={err:.3e} t={time.time()-t0:.3f}s", flush=True)
