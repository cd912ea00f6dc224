"""Multi-block stack driver (BASELINE config 5: LLaMA-3-8B 4-block stack).

The reference stops a block at the post-RoPE packed QKV (SPEC.md:413 — the
attention core is out of scope) and has no stack driver.  Blocks are chained
with the glue SURVEY §7.3-7 recommends, an identity "attention":

    x_{l+1} = V span of qkv_l        (columns [2d, 3d))
    z_{l+1} = residual_l             (pre_norm_b of block l)

so the backward feeds block l-1 with grad_qkv = [0 | 0 | grad_x_l] and
grad_residual = grad_z_l.  Every block runs its 6 + 13 fused launches; the
oracle chains `layer_forward/backward` identically for parity.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

from .errors import ConfigError
from .kernels import LayerGrads, LayerTape, LayerWeights, PipelineConfig, layer_backward, layer_forward
from .tensors import DenseMatrix, alloc_matrix


@dataclass
class StackForwardResult:
    qkv: DenseMatrix
    residual: DenseMatrix
    tapes: list


def v_span(qkv: DenseMatrix, d: int) -> DenseMatrix:
    """(m, d) view of the V columns of a packed (m, 3d) projection (no copy)."""
    return DenseMatrix._wrap(qkv.tensor[:, 2 * d:3 * d], qkv.precision)


def _check_glue(config: PipelineConfig) -> None:
    if config.kv_resolved != config.hidden:
        raise ConfigError("the identity-attention stack glue needs a V span of hidden width (kv_width=None)")


def stack_forward(x: DenseMatrix, z: DenseMatrix, weights: Sequence[LayerWeights], cos: DenseMatrix,
                  sin: DenseMatrix, *, config: PipelineConfig) -> StackForwardResult:
    _check_glue(config)
    d = config.hidden
    tapes: list[LayerTape] = []
    fwd = None
    for w in weights:
        fwd = layer_forward(x, z, w, cos, sin, config=config)
        tapes.append(fwd.tape)
        x, z = v_span(fwd.qkv, d), fwd.residual
    return StackForwardResult(qkv=fwd.qkv, residual=fwd.residual, tapes=tapes)


def stack_backward(grad_qkv: DenseMatrix, grad_residual: Optional[DenseMatrix], result: StackForwardResult,
                   weights: Sequence[LayerWeights], *, config: PipelineConfig, wgrad_hook=None) -> list[LayerGrads]:
    """Gradients of every block, returned in block order (index 0 = first block)."""
    _check_glue(config)
    d = config.hidden
    grads: list[LayerGrads] = [None] * len(weights)
    gq, gr = grad_qkv, grad_residual
    for l in range(len(weights) - 1, -1, -1):
        g = layer_backward(gq, result.tapes[l], weights[l], grad_residual=gr, config=config, wgrad_hook=wgrad_hook)
        grads[l] = g
        if l > 0:
            t = g.x.tensor
            full = alloc_matrix(t.shape[0], 3 * d, t.dtype, t.device)
            full[:, :2 * d].zero_()
            full[:, 2 * d:].copy_(t)
            gq, gr = DenseMatrix._wrap(full, config.precision), g.z
    return grads
