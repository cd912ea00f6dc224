"""GPU verification report: the reference's named invariant checks (tilefuse checks.py:82-322)
run through the CUDA path against the CPU oracle, reported in the reference's JSON schema
(paper_2605_19269_b200.report, cli.py:104-148).  Test infrastructure: imports oracle/.

The reference runs its checks in EXACT64 with tolerance 1e-12; the GPU engine computes in
SIM32 (tolerance 1e-5, the north-star fp32 bound) or SIMBF16 (2e-2), on inputs quantized to
that precision's storage grid, against the float64 oracle on the same quantized values.

    python tests/gpu_verify.py [--precision sim32|simbf16] [--seed 0] [--json-out PATH]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from oracle import coda_oracle as O  # noqa: E402

TOL = {"sim32": 1e-5, "simbf16": 2e-2}


def _cd():
    import paper_2605_19269_b200 as cd

    return cd


def _mk(cd, rng, P, *shape, scale=1.0):
    return cd.DenseMatrix.from_array(rng.standard_normal(shape) * scale, P)


def _mode(cd, P):
    return O.SIM32 if P is cd.PrecisionMode.SIM32 else O.SIMBF16


def check_kernel_oracles(cd, P, seed, sizes=((128, 128, 64), (130, 266, 72), (256, 512, 128))):
    """gemm_rope / gemm_swiglu against the oracle compositions (checks.py:82-100)."""
    rng = np.random.default_rng(seed)
    worst = 0.0
    for m, n, k in sizes:
        n2 = n + (n % 2)
        a, b = _mk(cd, rng, P, m, k), _mk(cd, rng, P, k, n2, scale=1 / np.sqrt(k))
        cos, sin = cd.rope_tables(m, n2, precision=P)
        t = O.gemm(a.data, b.data, O.EXACT64)
        worst = max(worst, O.rel_error(cd.gemm_rope(a, b, cos, sin, precision=P).main.data,
                                       O.rope(t, cos.data, sin.data)))
        worst = max(worst, O.rel_error(cd.gemm_swiglu(a, b, precision=P).main.data, O.swiglu(t)))
    return "kernel_oracles", worst


def check_commutation(cd, P, seed):
    """Fused GRRG equals the canonical-order schedule (checks.py:103-116)."""
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(3):
        m, k, d, n = 200, 96, 256, 130
        x, w0, z = _mk(cd, rng, P, m, k, scale=0.3), _mk(cd, rng, P, k, d, scale=0.3), _mk(cd, rng, P, m, d)
        gamma = cd.Vector.from_array(1 + 0.1 * rng.standard_normal(d), P)
        w1 = _mk(cd, rng, P, d, n, scale=0.3)
        cfg = cd.PipelineConfig(hidden=d, precision=P)
        fused = cd.pipeline_grrg_forward(x, w0, z, gamma, w1, config=cfg)
        canon, _ = cd.pipeline_grrg_canonical(x, w0, z, gamma, w1, config=cfg)
        worst = max(worst, O.rel_error(fused.y.data, canon.data))
    return "scale_commutation", worst


def check_statistic_relocation(cd, P, seed):
    """Row dots relocated through the consuming weight (checks.py:119-132): the GPU's
    PartialRowDot of grad_y against h2 @ W vs the direct (grad_y W^T) . h2."""
    rng = np.random.default_rng(seed)
    m, d, n = 128, 256, 384
    h2, w = _mk(cd, rng, P, m, d), _mk(cd, rng, P, d, n, scale=1 / 16)
    gy = _mk(cd, rng, P, m, n)
    prog = cd.EpilogueProgram([cd.PartialRowDot("gy", "dots")])
    res = cd.run_gemm(cd.GemmProblem(m, n, d, precision=P), h2, w, prog, {"gy": gy})
    relocated = cd.finalize_rowdot(res.aux["dots"], d).data
    direct = np.sum((gy.data @ w.data.T) * h2.data, axis=1) / d
    return "statistic_relocation", O.rel_error(relocated, direct)


def check_lse(cd, P, seed):
    """Blocked streamed LSE equals the direct log-sum-exp (checks.py:135-147)."""
    rng = np.random.default_rng(seed)
    m, k, d, v = 256, 64, 128, 1000
    a, b, z = _mk(cd, rng, P, m, k, scale=0.3), _mk(cd, rng, P, k, d, scale=0.3), _mk(cd, rng, P, m, d)
    gamma = cd.Vector.from_array(np.ones(d), P)
    wv = _mk(cd, rng, P, d, v, scale=0.3)
    labels = rng.integers(0, v, size=m)
    cfg = cd.PipelineConfig(hidden=d, precision=P)
    res = cd.lm_head_forward(a, b, z, gamma, wv, labels, config=cfg, store_logits=True)
    lg = res.logits.data
    mx = lg.max(axis=1)
    direct = mx + np.log(np.exp(lg - mx[:, None]).sum(axis=1))
    return "lse_blocking", O.rel_error(res.lse.data, direct)


def _layer(cd, P, seed, m=256, d=256, ffn=1024):
    rng = np.random.default_rng(seed)
    mode = _mode(cd, P)
    w = O.random_layer(rng, d, ffn, mode)
    x, z = (O.q(rng.standard_normal((m, d)), mode) for _ in range(2))
    cos, sin = O.qkv_rope_tables(m, d, mode)
    gq, gr = O.q(rng.standard_normal((m, 3 * d)), mode), O.q(rng.standard_normal((m, d)), mode)
    M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
    V = lambda a: cd.Vector.from_array(a, P)  # noqa: E731
    lw = cd.LayerWeights(w_out=M(w["w_out"]), gamma_ffn=V(w["gamma_ffn"]), w_gate_up=M(w["w_gate_up"]),
                         w_down=M(w["w_down"]), gamma_qkv=V(w["gamma_qkv"]), w_qkv=M(w["w_qkv"]))
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, precision=P)
    fwd = cd.layer_forward(M(x), M(z), lw, M(cos), M(sin), config=cfg)
    bwd = cd.layer_backward(M(gq), fwd.tape, lw, grad_residual=M(gr), config=cfg)
    return dict(w=w, x=x, z=z, cos=cos, sin=sin, gq=gq, gr=gr, fwd=fwd, bwd=bwd)


def check_gradients_oracle(cd, P, seed):
    """layer_backward against the analytic float64 backward (checks.py:150-175)."""
    L = _layer(cd, P, seed)
    rf = O.layer_ref_forward(L["x"], L["z"], L["w"], L["cos"], L["sin"])
    rb = O.layer_ref_backward(L["gq"], L["gr"], rf, L["x"], L["w"], L["cos"], L["sin"])
    return "gradients_oracle", max(O.rel_error(getattr(L["bwd"], k).data, rb[k]) for k in O.GRAD_KEYS)


def check_gradients_fd(cd, P, seed, probes=2, h=1e-4):
    """Directional central differences of the float64 layer (checks.py:178-238)."""
    L = _layer(cd, P, seed, m=64, d=64, ffn=256)
    rng = np.random.default_rng([seed, 1])
    params = {"x": L["x"], "z": L["z"], **{k: L["w"][k] for k in ("w_out", "gamma_ffn", "w_gate_up", "w_down",
                                                                   "gamma_qkv", "w_qkv")}}
    worst = 0.0
    for name, value in params.items():
        grad = getattr(L["bwd"], name).data

        def f(val):
            p = dict(params)
            p[name] = val
            xx, zz = p.pop("x"), p.pop("z")
            out = O.layer_ref_forward(xx, zz, p, L["cos"], L["sin"])
            return float(np.sum(out["qkv"] * L["gq"]) + np.sum(out["h1b"] * L["gr"]))

        for _ in range(probes):
            v = rng.standard_normal(value.shape)
            v /= np.linalg.norm(v)
            quotient = (f(value + h * v) - f(value - h * v)) / (2 * h)
            want = float(np.sum(grad * v))
            # the reference divides by |quotient| (exact arithmetic); a random unit direction has
            # |<g, v>| ~ ||g|| / sqrt(numel), so that magnitude also bounds the denominator from
            # below -- otherwise a near-orthogonal probe turns the bf16 storage error of the GPU
            # gradient into an arbitrarily large relative error
            scale = max(abs(quotient), float(np.linalg.norm(grad)) / np.sqrt(grad.size), 1e-8)
            worst = max(worst, abs(quotient - want) / scale)
    return "gradients_fd", worst


def check_tile_invariance(cd, P, seed):
    """Pipeline outputs are independent of the reference tile shape (checks.py:241-254)."""
    rng = np.random.default_rng(seed)
    m, k, d, n = 200, 96, 256, 130
    x, w0, z = _mk(cd, rng, P, m, k, scale=0.3), _mk(cd, rng, P, k, d, scale=0.3), _mk(cd, rng, P, m, d)
    gamma = cd.Vector.from_array(1 + 0.1 * rng.standard_normal(d), P)
    w1 = _mk(cd, rng, P, d, n, scale=0.3)
    outs = []
    for tm, tn in ((16, 24), (32, 32), (128, 128)):
        cfg = cd.PipelineConfig(hidden=d, tile_m=tm, tile_n=tn, reduction_tile_n=tn, precision=P)
        outs.append(cd.pipeline_grrg_forward(x, w0, z, gamma, w1, config=cfg).y.data)
    return "tile_invariance", max(O.rel_error(o, outs[0]) for o in outs[1:])


def check_pipeline_oracles(cd, P, seed):
    """GRRG and the layer forward against naive float64 compositions (checks.py:257-282)."""
    rng = np.random.default_rng(seed)
    m, d = 192, 256
    x, w0, z = _mk(cd, rng, P, m, 96, scale=0.3), _mk(cd, rng, P, 96, d, scale=0.3), _mk(cd, rng, P, m, d)
    gamma = cd.Vector.from_array(1 + 0.1 * rng.standard_normal(d), P)
    w1 = _mk(cd, rng, P, d, 130, scale=0.3)
    cfg = cd.PipelineConfig(hidden=d, precision=P)
    fused = cd.pipeline_grrg_forward(x, w0, z, gamma, w1, config=cfg)
    h1 = x.data @ w0.data + z.data
    r = 1.0 / np.sqrt(np.mean(h1 * h1, axis=1) + cfg.eps)
    ref = (h1 * r[:, None] * gamma.data[None, :]) @ w1.data
    worst = O.rel_error(fused.y.data, ref)
    L = _layer(cd, P, seed)
    rf = O.layer_ref_forward(L["x"], L["z"], L["w"], L["cos"], L["sin"])
    worst = max(worst, O.rel_error(L["fwd"].qkv.data, rf["qkv"]), O.rel_error(L["fwd"].residual.data, rf["h1b"]))
    return "pipeline_oracles", worst


CHECKS = (check_kernel_oracles, check_commutation, check_statistic_relocation, check_lse, check_gradients_oracle,
          check_gradients_fd, check_tile_invariance, check_pipeline_oracles)


def run_checks(precision: str = "sim32", seed: int = 0):
    """Every named check on the GPU; CheckResults sorted by name (checks.py:285-308)."""
    cd = _cd()
    from paper_2605_19269_b200.report import CheckResult

    P = cd.PrecisionMode.SIM32 if precision == "sim32" else cd.PrecisionMode.SIMBF16
    out = [CheckResult(*fn(cd, P, seed), TOL[precision]) for fn in CHECKS]
    return P, sorted(out, key=lambda r: r.name)


def make_report(precision: str = "sim32", seed: int = 0) -> dict:
    import torch

    from paper_2605_19269_b200 import _native
    from paper_2605_19269_b200.report import build_report

    P, checks = run_checks(precision, seed)
    return build_report(seed, checks, P, device=torch.cuda.get_device_name(0),
                        engine=_native.load().coda_version().decode(), oracle="oracle/coda_oracle.py (float64)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", choices=("sim32", "simbf16"), default="sim32")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--json-out", default="-")
    args = ap.parse_args()
    from paper_2605_19269_b200.report import all_passed, render_report

    rep = make_report(args.precision, args.seed)
    text = render_report(rep)
    if args.json_out == "-":
        sys.stdout.write(text)
    else:
        Path(args.json_out).write_text(text)
    for c in rep["checks"]:
        print(f"{'PASS' if c['pass'] else 'FAIL'} {c['name']}: {c['metric']:.3e} <= {c['tolerance']:g}",
              file=sys.stderr)
    return 0 if all_passed(rep) else 1


if __name__ == "__main__":
    sys.exit(main())
