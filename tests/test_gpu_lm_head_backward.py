"""LM-head cross-entropy backward on the GPU (row f4 of SURVEY §8; a B200 extension -- the
reference stops at the loss): logit-gradient launch with the CrossEntropyBackward
epilogue, the relocated RMSNorm statistic, K9, the vocabulary / input weight gradients.
Compared with the fused-order oracle (oracle/coda_oracle.lm_head_backward, itself pinned by
finite differences of the float64 loss) in both precisions."""

import numpy as np
import pytest

from oracle import coda_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"sim32": 1e-5, "simbf16": 2e-2}


def _case(P, mode, m, k, d, v, seed):
    import paper_2605_19269_b200 as cd

    rng = np.random.default_rng(seed)
    qz = lambda x: O.q(x, mode)  # noqa: E731
    a, b, z = qz(rng.standard_normal((m, k)) * 0.5), qz(rng.standard_normal((k, d)) / np.sqrt(k)), \
        qz(rng.standard_normal((m, d)))
    gamma = qz(1 + 0.1 * rng.standard_normal(d))
    wv = qz(rng.standard_normal((d, v)) / np.sqrt(d))
    labels = rng.integers(0, v, m)
    M = lambda x: cd.DenseMatrix.from_array(x, P)  # noqa: E731
    return dict(a=a, b=b, z=z, gamma=gamma, wv=wv, labels=labels, A=M(a), B=M(b), Z=M(z),
                G=cd.Vector.from_array(gamma, P), WV=M(wv))


@pytest.mark.parametrize("mode,shape", [("sim32", (300, 96, 256, 1000)), ("simbf16", (300, 96, 256, 1000)),
                                        ("simbf16", (2048, 1024, 2048, 8192))])
def test_lm_head_backward_vs_oracle(cuda_ready, mode, shape):
    import torch

    import paper_2605_19269_b200 as cd

    P = cd.PrecisionMode.SIM32 if mode == "sim32" else cd.PrecisionMode.SIMBF16
    m, k, d, v = shape
    c = _case(P, mode, m, k, d, v, seed=3)
    cfg = cd.PipelineConfig(hidden=d, precision=P)
    fwd = cd.lm_head_forward(c["A"], c["B"], c["Z"], c["G"], c["WV"], c["labels"], config=cfg)
    grads = cd.lm_head_backward(fwd, c["A"], c["B"], c["G"], c["WV"], config=cfg)
    torch.cuda.synchronize()
    of = O.lm_head_forward(c["a"], c["b"], c["z"], c["gamma"], c["wv"], c["labels"], mode)
    ob = O.lm_head_backward(of, c["a"], c["b"], c["gamma"], c["wv"], c["labels"], mode)
    errs = {n: O.rel_error(getattr(grads, n).data, ob[n]) for n in ("a", "b", "z", "gamma", "w_vocab")}
    errs["loss"] = abs(fwd.mean_loss - of["mean"]) / abs(of["mean"])
    print(f"\n[{mode} {shape}] " + ", ".join(f"{n}={e:.2e}" for n, e in errs.items()))
    assert max(errs.values()) <= TOL[mode], errs


def test_lm_head_backward_finite_differences(cuda_ready):
    """SIM32 GPU gradients against central differences of the float64 loss."""
    import paper_2605_19269_b200 as cd

    P = cd.PrecisionMode.SIM32
    c = _case(P, O.SIM32, 64, 32, 64, 300, seed=5)
    cfg = cd.PipelineConfig(hidden=64, precision=P)
    fwd = cd.lm_head_forward(c["A"], c["B"], c["Z"], c["G"], c["WV"], c["labels"], config=cfg)
    grads = cd.lm_head_backward(fwd, c["A"], c["B"], c["G"], c["WV"], config=cfg)
    params = {"a": c["a"], "b": c["b"], "z": c["z"], "gamma": c["gamma"], "w_vocab": c["wv"]}
    rng = np.random.default_rng(9)
    h = 1e-5
    worst = 0.0
    for name, val in params.items():
        g = getattr(grads, name).data
        for _ in range(2):
            u = rng.standard_normal(val.shape)
            u /= np.linalg.norm(u)
            p1, p2 = dict(params), dict(params)
            p1[name], p2[name] = val + h * u, val - h * u
            fd = (O.lm_head_loss64(**p1, labels=c["labels"]) - O.lm_head_loss64(**p2, labels=c["labels"])) / (2 * h)
            scale = max(abs(fd), float(np.linalg.norm(g)) / np.sqrt(g.size))
            worst = max(worst, abs(fd - float(np.sum(g * u))) / scale)
    assert worst <= 1e-4, worst


def test_lm_head_forward_full_size_sampled_rows(cuda_ready):
    """The LM head at the benchmarked size (16384 tokens, d 4096, vocabulary 32768: K8 runs
    16384 x 32768 x 4096 with the logits never stored): every statistic is per row, so 256
    sampled rows of the GPU's per-token losses and log-sum-exps are checked against the
    fused-order oracle run on exactly those rows over the whole vocabulary."""
    import torch

    import paper_2605_19269_b200 as cd

    P = cd.PrecisionMode.SIMBF16
    m, k, d, v = 16384, 4096, 4096, 32768
    rng = np.random.default_rng(17)
    qz = lambda x: O.q(x, O.SIMBF16)  # noqa: E731
    a = qz(rng.standard_normal((m, k), dtype=np.float32))
    b = qz(rng.standard_normal((k, d), dtype=np.float32) * 0.02)
    z = qz(rng.standard_normal((m, d), dtype=np.float32))
    gamma = qz(1 + 0.1 * rng.standard_normal(d))
    wv = qz(rng.standard_normal((d, v), dtype=np.float32) * 0.02)
    labels = rng.integers(0, v, m)
    M = lambda x: cd.DenseMatrix.from_array(x, P)  # noqa: E731
    cfg = cd.PipelineConfig(hidden=d, precision=P)
    fwd = cd.lm_head_forward(M(a), M(b), M(z), cd.Vector.from_array(gamma, P), M(wv), labels, config=cfg)
    torch.cuda.synchronize()
    rows = np.sort(rng.choice(m, 256, replace=False))
    of = O.lm_head_forward(a[rows], b, z[rows], gamma, wv, labels[rows], O.SIMBF16)
    got_loss = fwd.losses.tensor.double().cpu().numpy()[rows]
    got_lse = fwd.lse.tensor.double().cpu().numpy()[rows]
    assert O.rel_error(got_lse, of["lse"]) <= 1e-5, O.rel_error(got_lse, of["lse"])
    assert O.rel_error(got_loss, of["losses"]) <= 2e-2, O.rel_error(got_loss, of["losses"])
    assert np.isfinite(fwd.mean_loss) and abs(fwd.mean_loss - np.log(v)) < 2.0
