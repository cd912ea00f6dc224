"""LM-head cross entropy: fused K4 -> finalize -> K8 -> combine_lse -> CE
finalize (logits never stored) vs unfused cuBLAS logits + torch cross_entropy.

    python tools/lm_head_bench.py [--m 16384] [--d 4096] [--vocab 32768]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import paper_2605_19269_b200 as cd  # noqa: E402
from paper_2605_19269_b200 import unfused  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--vocab", type=int, default=32768)
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    m, d, v = args.m, args.d, args.vocab
    dev = torch.device("cuda", 0)
    P = cd.PrecisionMode.SIMBF16
    g = torch.Generator(device=dev).manual_seed(0)
    mk = lambda *s, sc=1.0: (torch.randn(s, generator=g, device=dev) * sc).to(torch.bfloat16)  # noqa: E731
    A, B, Z = mk(m, d), mk(d, d, sc=0.02), mk(m, d)
    Wv = mk(d, v, sc=0.02)
    gamma = (1 + 0.1 * torch.randn(d, generator=g, device=dev)).float()
    labels = torch.randint(0, v, (m,), generator=g, device=dev)
    a, b, z, wv = (cd.DenseMatrix.from_tensor(t, P) for t in (A, B, Z, Wv))
    gm = cd.Vector.from_tensor(gamma, P)
    cfg = cd.PipelineConfig(hidden=d, precision=P)

    def fused():
        return cd.lm_head_forward(a, b, z, gm, wv, labels, config=cfg)

    def unfused_run():
        h = A @ B + Z
        n, _ = unfused.rmsnorm(h, gamma, cfg.eps)
        logits = n @ Wv
        return F.cross_entropy(logits.float(), labels)

    rf = fused()
    lu = float(unfused_run())
    rel = abs(rf.mean_loss - lu) / abs(lu)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps

    tf, tu = timed(fused), timed(unfused_run)
    flops = 2.0 * m * d * (d + v)
    print(json.dumps({"workload": f"lm head m={m} d={d} vocab={v}", "fused_ms": tf, "unfused_ms": tu,
                      "speedup": tu / tf, "fused_tflops": flops / tf / 1e9, "mean_loss_fused": rf.mean_loss,
                      "mean_loss_unfused": lu, "rel_err_loss": rel}), flush=True)


if __name__ == "__main__":
    main()
