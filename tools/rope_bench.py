"""rope_backward_stat timing on the C4 boundary shape and a same-bytes shape that takes the
3-sweep variant; CUDA-graph replays of 20 launches, HBM fraction of MEASURED_PEAKS."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_19269_b200 as cd  # noqa: E402

P = cd.PrecisionMode.SIMBF16
dev = torch.device("cuda", 0)
peak = bench.peaks()["hbm_gbs"]
out = []
for m, d in ((16384, 4096), (32768, 2048), (8192, 2048)):
    q = 3 * d
    cos, sin = cd.qkv_rope_tables(m, d, precision=P)
    g = cd.DenseMatrix.from_tensor(torch.randn(m, q, device=dev).to(torch.bfloat16), P)
    r = cd.DenseMatrix.from_tensor(torch.randn(m, q, device=dev).to(torch.bfloat16), P)
    for _ in range(3):
        cd.rope_backward_stat(g, r, cos, sin, precision=P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        cd.rope_backward_stat(g, r, cos, sin, precision=P)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nb = q // 128
    byts = 2 * m * q * 2 + 2 * m * (d // 2) * 2 + m * q * 2 + m * nb * 4
    out.append({"m": m, "d": d, "ms": ms, "GB": byts / 1e9, "GBps": byts / ms / 1e6, "frac": byts / ms / 1e6 / peak})
print(json.dumps(out))
