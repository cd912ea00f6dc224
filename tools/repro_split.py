"""Debug aid: run each fused launch of tests/test_gpu_kernels.py::test_tail_split_matches_unsplit
one at a time (sync after each) under the chosen engine options."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import _native  # noqa: E402

for kv in sys.argv[1:]:
    k_, v_ = kv.split("=")
    _native.set_option(k_, int(v_))
rng = np.random.default_rng(8)
P = cd.PrecisionMode.SIMBF16
m, k, n = 1000, 2048, 1536
M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
a, b = M(rng.standard_normal((m, k)) / 40), M(rng.standard_normal((k, n)) / 40)
bt = M(rng.standard_normal((n, k)) / 40)
z, pre, gin = M(rng.standard_normal((m, n))), M(rng.standard_normal((m, n))), M(rng.standard_normal((m, n)))
pre2 = M(rng.standard_normal((m, 2 * n)))
cos, sin = cd.rope_tables(m, n, precision=P)
r = cd.Vector.from_array(0.5 + rng.random(m), cd.PrecisionMode.SIM32)
s = cd.Vector.from_array(0.1 * rng.standard_normal(m), cd.PrecisionMode.SIM32)
gamma = cd.Vector.from_array(1 + 0.1 * rng.standard_normal(n), P)
labels = rng.integers(0, n, m).astype(np.int64)
steps = [
    ("k4", lambda: cd.gemm_residual_partial_rms(a, b, z, gamma, precision=P)),
    ("k6", lambda: cd.gemm_rms_swiglu(a, b, r, precision=P)),
    ("k7", lambda: cd.gemm_rms_rope(a, b, r, cos, sin, precision=P)),
    ("k9", lambda: cd.gemm_rmsnorm_backward(a, bt, pre, r, gamma, s, grad_in=gin, trans_b=True, precision=P)),
    ("k10", lambda: cd.gemm_swiglu_backward(a, bt, pre2, trans_b=True, precision=P)),
    ("k8", lambda: cd.gemm_rms_partial_xent(a, b, r, labels, precision=P)),
]
for it in range(2):
    for name, fn in steps:
        t0 = time.time()
        fn()
        torch.cuda.synchronize()
        print(it, name, "ok", round(time.time() - t0, 4), flush=True)
