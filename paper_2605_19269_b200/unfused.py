"""Unfused comparator: cuBLAS GEMMs + standalone elementwise ops (NOT the product path).

The CODA claim is measured against "an unfused cuBLAS-plus-elementwise
sequence" (BASELINE.json north star).  This module runs exactly the reference's
canonical op lists (tilefuse/traffic.py:338-459: canonical_grrg_ops,
canonical_layer_forward_ops, canonical_layer_backward_ops) on the GPU with
`torch.matmul` (cuBLAS, bf16 in / f32 accumulate / bf16 out) and one torch op
per elementwise step, storing every intermediate in the storage dtype like the
reference's canonical schedule (kernels.py:677-713).  It is used by
tools/primitive_sweep.py and tools/unfused_block.py for time and ncu-measured
HBM bytes; nothing in the fused pipelines calls it.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F


def rmsnorm(x: torch.Tensor, gamma: torch.Tensor, eps: float):
    """(x * r * gamma, r) with r = 1/sqrt(mean(x^2) + eps) computed in f32."""
    xf = x.float()
    r = torch.rsqrt(xf.pow(2).mean(dim=1) + eps)
    return (xf * r[:, None] * gamma[None, :]).to(x.dtype), r


def swiglu(z: torch.Tensor) -> torch.Tensor:
    return (F.silu(z[:, 0::2].float()) * z[:, 1::2].float()).to(z.dtype)


def rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor, backward: bool = False) -> torch.Tensor:
    xf, c, s = x.float(), cos.float(), sin.float()
    if backward:
        s = -s
    out = torch.empty_like(xf)
    out[:, 0::2] = xf[:, 0::2] * c[:, 0::2] - xf[:, 1::2] * s[:, 0::2]
    out[:, 1::2] = xf[:, 0::2] * s[:, 1::2] + xf[:, 1::2] * c[:, 1::2]
    return out.to(x.dtype)


def grrg(x, w0, z, gamma, w1, eps=1e-6):
    """gemm -> residual_add -> rmsnorm -> gemm (canonical_grrg_ops)."""
    h = x @ w0
    h = h + z
    n, r = rmsnorm(h, gamma, eps)
    return n @ w1


def layer_forward(x, z, w, cos, sin, eps=1e-6) -> dict:
    """canonical_layer_forward_ops: 4 cuBLAS GEMMs + 6 elementwise/normalization ops."""
    h1a = x @ w["w_out"]
    h1a = h1a + z
    na, ra = rmsnorm(h1a, w["gamma_ffn"], eps)
    za = na @ w["w_gate_up"]
    oa = swiglu(za)
    h1b = oa @ w["w_down"]
    h1b = h1b + h1a
    nb, rb = rmsnorm(h1b, w["gamma_qkv"], eps)
    zb = nb @ w["w_qkv"]
    qkv = rope(zb, cos, sin)
    return {"h1a": h1a, "na": na, "ra": ra, "za": za, "oa": oa, "h1b": h1b, "nb": nb, "rb": rb, "qkv": qkv}


def _rmsnorm_backward(gout, x, r, gamma):
    gf, xf = gout.float(), x.float()
    n = xf * r[:, None]
    s = (gf * n * gamma[None, :]).mean(dim=1)
    gx = r[:, None] * (gf * gamma[None, :] - n * s[:, None])
    return gx.to(x.dtype), (gf * n).sum(dim=0)


def _swiglu_backward(dout, z):
    g, u, d = z[:, 0::2].float(), z[:, 1::2].float(), dout.float()
    sg = torch.sigmoid(g)
    sl = g * sg
    out = torch.empty(z.shape, dtype=torch.float32, device=z.device)
    out[:, 0::2] = d * u * (sg + sl * (1 - sg))
    out[:, 1::2] = d * sl
    return out.to(z.dtype)


def layer_backward(grad_qkv, grad_residual, fwd: dict, x, w, cos, sin) -> dict:
    """canonical_layer_backward_ops: 8 cuBLAS GEMMs + 6 elementwise/normalization ops."""
    gzb = rope(grad_qkv, cos, sin, backward=True)
    gnb = gzb @ w["w_qkv"].t()
    g_wqkv = fwd["nb"].t() @ gzb
    gh1b, g_gqkv = _rmsnorm_backward(gnb, fwd["h1b"], fwd["rb"], w["gamma_qkv"])
    gh1b = gh1b + grad_residual
    goa = gh1b @ w["w_down"].t()
    gza = _swiglu_backward(goa, fwd["za"])
    g_wdown = fwd["oa"].t() @ gh1b
    gna = gza @ w["w_gate_up"].t()
    g_wgu = fwd["na"].t() @ gza
    gh1a, g_gffn = _rmsnorm_backward(gna, fwd["h1a"], fwd["ra"], w["gamma_ffn"])
    gh1a = gh1a + gh1b
    gx = gh1a @ w["w_out"].t()
    g_wout = x.t() @ gh1a
    return {"x": gx, "z": gh1a, "w_out": g_wout, "gamma_ffn": g_gffn, "w_gate_up": g_wgu, "w_down": g_wdown,
            "gamma_qkv": g_gqkv, "w_qkv": g_wqkv}
