"""Whole-step CUDA graphs (paper_2605_19269_b200.graphs.StepGraph).

A captured fused block step (forward + backward, 15 kernels) replayed over static input
buffers refilled in place must give the same bits as the eager step on the same
inputs, including the split-K weight gradients (K = tokens >= 8192)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

GRADS = ("x", "z", "w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv", "w_qkv")


def _case(m=8192, d=256, ffn=1024, seed=5):
    sys.path.insert(0, str(ROOT))
    from oracle import coda_oracle as O

    rng = np.random.default_rng(seed)
    mode = O.SIMBF16
    w = O.random_layer(rng, d, ffn, mode, scale=0.05)
    acts = [{k: O.q(rng.standard_normal(shape), mode) for k, shape in
             (("x", (m, d)), ("z", (m, d)), ("grad_qkv", (m, 3 * d)), ("grad_residual", (m, d)))}
            for _ in range(2)]
    return m, d, ffn, w, acts


@pytest.mark.parametrize("fold", [False, True])
def test_step_graph_replays_bit_identical(cuda_ready, fold):
    import torch

    import paper_2605_19269_b200 as cd

    m, d, ffn, w, acts = _case()
    P = cd.PrecisionMode.SIMBF16
    M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
    V = lambda a: cd.Vector.from_array(a, P)  # noqa: E731
    weights = cd.LayerWeights(w_out=M(w["w_out"]), gamma_ffn=V(w["gamma_ffn"]), w_gate_up=M(w["w_gate_up"]),
                              w_down=M(w["w_down"]), gamma_qkv=V(w["gamma_qkv"]), w_qkv=M(w["w_qkv"]))
    cfg = cd.PipelineConfig(hidden=d, ffn=ffn, precision=P, fold_gamma=fold)
    cos, sin = cd.qkv_rope_tables(m, d, precision=P)

    def step(a):
        fwd = cd.layer_forward(a["x"], a["z"], weights, cos, sin, config=cfg)
        bwd = cd.layer_backward(a["grad_qkv"], fwd.tape, weights, grad_residual=a["grad_residual"], config=cfg)
        return fwd, bwd

    def snapshot(fwd, bwd):
        # read the device tensors (DenseMatrix.data caches its first download, and the
        # graph's outputs are rewritten by every replay)
        torch.cuda.synchronize()
        out = {k: getattr(bwd, k).tensor.float().cpu().numpy() for k in GRADS}
        out["qkv"] = fwd.qkv.tensor.float().cpu().numpy()
        return out

    static = {k: M(v) for k, v in acts[0].items()}
    sg = cd.StepGraph(lambda: step(static))
    if not fold:
        assert sg.launches == 15
    for a in acts:
        for k, v in a.items():
            static[k].tensor.copy_(M(v).tensor)
        got = snapshot(*sg.replay())
        want = snapshot(*step({k: M(v) for k, v in a.items()}))
        for k in want:
            assert np.array_equal(got[k], want[k]), k
    # the two input sets differ, so the replays really recomputed
    assert not np.array_equal(snapshot(*sg.outputs)["w_out"], snapshot(*step({k: M(v) for k, v in acts[0].items()}))["w_out"])
