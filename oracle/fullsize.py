"""CPU ORACLE, full-size driver — test infrastructure only.

The reference's fused-order layer (tilefuse kernels.py:810-1013, restated in
coda_oracle.layer_forward / layer_backward) run token-chunked, so the
benchmarked configurations (BASELINE configs 2 and 3: C3 8192 x 2048, C4
16384 x 4096) can be checked against the oracle in full, including the
weight gradients whose contraction runs over every token (K = M = 16384 at
C4) — SURVEY.md §8c "Big shapes".

Chunking is exact for everything row-local and for the reductions:
  * forward outputs, the activation gradients and every row statistic (r, s)
    depend only on their own token row (kernels.py:810-869, 885-1013);
  * the gain gradients reduce per-128-row tile partials in ascending tile order
    (reductions.py:134-145); chunks are multiples of 128 rows, so concatenating
    the chunk partials reproduces the unchunked partial array and the same
    ordered f32 total (reduce_row_partials below is the unchunked function);
  * the weight gradients are A^T B over all tokens: each chunk contributes its
    float32 product (the reference's accumulator dtype, engine.py:436-438) and
    the chunk products are summed in float64, then rounded to storage once
    (engine.py:443-447).  This differs from one K=M float32 product only by
    accumulation order.

Only `tests/` (and the fixture generator in tests/golden/) import this; the
product path never does.

Inputs are generated here, deterministically per tensor (numpy PCG64 seeded
with [seed, tensor index]), on the storage grid, so the GPU test regenerates
bit-identical operands on the box without shipping them.
"""

from __future__ import annotations

import numpy as np

from . import coda_oracle as O

# BASELINE.json configs -> (tokens M, hidden d, LLaMA intermediate I); F = 2I interleaved gate/up
CONFIGS = {
    "c1": (128, 256, 1024),
    "c3": (8192, 2048, 8192),
    "c4": (16384, 4096, 14336),
    "c5": (8192, 4096, 14336),     # per block of the 4-block stack, 8192 tokens per GPU
    "c4gqa": (16384, 4096, 14336),  # C4 with the GQA extension: k / v spans 1024 wide
}
BLOCKS = {"c5": 4}
KV = {"c4gqa": 1024}               # k / v span width (default: hidden, the reference's packed 3d)

# order of the generated tensors (stream index = position)
TENSORS = ("w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv", "w_qkv", "x", "z", "grad_qkv",
           "grad_residual")

OUTPUTS = ("qkv", "residual", "x", "z", "w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv", "w_qkv")


def _normal(seed: int, idx: int, shape, scale: float) -> np.ndarray:
    rng = np.random.default_rng([seed, idx])
    a = rng.standard_normal(shape, dtype=np.float32)
    if scale != 1.0:
        a *= np.float32(scale)
    return a


def make_stack_inputs(name: str, seed: int = 0, mode: str = O.SIMBF16, scale: float = 0.02) -> tuple[list, dict]:
    """Per-block weights (stream indices offset by 10 per block) and the stack's activations."""
    m, d, inter = CONFIGS[name]
    blocks = BLOCKS.get(name, 1)
    base = make_inputs(name, seed, mode, scale)
    ws = [weights_of(base)]
    for b in range(1, blocks):
        ws.append(weights_of(make_inputs(name, seed, mode, scale, stream_offset=10 * b, weights_only=True)))
    acts = {k: base[k] for k in ("x", "z", "grad_qkv", "grad_residual")}
    return ws, acts


def make_inputs(name: str, seed: int = 0, mode: str = O.SIMBF16, scale: float = 0.02, stream_offset: int = 0,
                weights_only: bool = False) -> dict:
    """Weights N(0, scale^2) with gains 1 + 0.1 N(0,1) (kernels.py:750-767 draw rules; per-tensor
    streams instead of one sequential stream), activations and incoming gradients N(0, 1), all
    quantized to the storage grid of `mode`.  Float32 arrays (every grid value is exact in f32)."""
    m, d, inter = CONFIGS[name]
    f = 2 * inter
    qw = d + 2 * KV.get(name, d)     # packed q | k | v width
    shapes = {"w_out": (d, d), "gamma_ffn": (d,), "w_gate_up": (d, f), "w_down": (inter, d), "gamma_qkv": (d,),
              "w_qkv": (d, qw), "x": (m, d), "z": (m, d), "grad_qkv": (m, qw), "grad_residual": (m, d)}
    out = {}
    for i, key in enumerate(TENSORS):
        if weights_only and not (key.startswith("w_") or key.startswith("gamma")):
            continue
        if key.startswith("gamma"):
            a = 1.0 + 0.1 * _normal(seed, i + stream_offset, shapes[key], 1.0)
        else:
            a = _normal(seed, i + stream_offset, shapes[key], scale if key.startswith("w_") else 1.0)
        out[key] = _grid(a, mode)
    return out


def _grid(a: np.ndarray, mode: str) -> np.ndarray:
    if mode == O.SIMBF16:
        return O.bf16_round(a)
    return np.asarray(a, dtype=np.float32 if mode == O.SIM32 else np.float64)


def weights_of(inp: dict) -> dict:
    return {k: inp[k] for k in ("w_out", "gamma_ffn", "w_gate_up", "w_down", "gamma_qkv", "w_qkv")}


# ----------------------------------------------------------------------------- chunked layer


def _backward_parts(grad_qkv, tape: dict, w: dict, mode, grad_residual, tile_m=128, tile_n=128, rtn=128):
    """coda_oracle.layer_backward (kernels.py:885-1013) with the cross-token sums left open:
    row-local outputs rounded as stored, weight-gradient products unrounded (accumulator dtype),
    gain gradients as their per-tile-row partial arrays."""
    d = w["w_out"].shape[0]
    gzb, rd_b = O.rope_backward_stat(grad_qkv, tape["qkv"], tape["cos"], tape["sin"], mode, tile_n, rtn)
    s_b = O.finalize_rowdot(rd_b, d, mode)
    k9b = O.k_rmsnorm_backward(gzb, w["w_qkv"], tape["pre_norm_b"], tape["inv_rms_b"], w["gamma_qkv"], s_b, mode,
                               grad_in=grad_residual, tile_m=tile_m, trans_b=True)
    gh1b = k9b["main"]
    k10 = O.k_swiglu_backward(gh1b, w["w_down"], tape["preact"], mode, tile_n, rtn, trans_b=True)
    gza = k10["main"]
    s_a = O.finalize_rowdot(k10["rowdot"], d, mode)
    k9a = O.k_rmsnorm_backward(gza, w["w_gate_up"], tape["pre_norm_a"], tape["inv_rms_a"], w["gamma_ffn"], s_a,
                               mode, grad_in=gh1b, tile_m=tile_m, trans_b=True)
    gh1a = k9a["main"]
    return {
        "x": O.q(O.gemm(gh1a, w["w_out"], mode, trans_b=True), mode),
        "z": gh1a,
        "w_qkv": O.gemm(k9b["normed"], gzb, mode, trans_a=True),
        "w_down": O.gemm(k10["recompute"], gh1b, mode, trans_a=True),
        "w_gate_up": O.gemm(k9a["normed"], gza, mode, trans_a=True),
        "w_out": O.gemm(tape["x"], gh1a, mode, trans_a=True),
        "gamma_qkv": k9b["gamma_grad"][0],
        "gamma_ffn": k9a["gamma_grad"][0],
    }


ROW_LOCAL = ("qkv", "residual", "x", "z")
WGRADS = ("w_out", "w_gate_up", "w_down", "w_qkv")
GAINS = ("gamma_ffn", "gamma_qkv")


def run_layer_chunked(inp: dict, mode: str = O.SIMBF16, chunk: int = 1024, eps: float = 1e-6,
                      on_rows=None) -> dict:
    """Full fused-order forward + backward of one block over all M tokens, `chunk` rows at a time.

    `on_rows(r0, r1, outs)` (optional) receives each chunk's row-local outputs {qkv, residual, x, z}
    so a caller can sketch / sample them without holding (M, 3d) arrays.  Returns the reduced
    weight gradients and gains (rounded to storage like the reference) and, when `on_rows` is
    None, the assembled row-local outputs too.
    """
    if chunk % 128:
        raise ValueError("chunk must be a multiple of the 128-row tile (gain-gradient partials)")
    w = weights_of(inp)
    m, d = inp["x"].shape
    kv = (w["w_qkv"].shape[1] - d) // 2
    kv_width = None if kv == d else kv      # GQA extension: the k / v span width
    acc = {k: None for k in WGRADS}
    gparts = {k: [] for k in GAINS}
    rows = {k: [] for k in ROW_LOCAL} if on_rows is None else None
    for r0 in range(0, m, chunk):
        r1 = min(m, r0 + chunk)
        cos, sin = O.qkv_rope_tables(r1 - r0, d, mode, start=r0, kv_width=kv_width)
        f = O.layer_forward(inp["x"][r0:r1], inp["z"][r0:r1], w, cos, sin, mode, eps=eps)
        b = _backward_parts(inp["grad_qkv"][r0:r1], f, w, mode, inp["grad_residual"][r0:r1])
        for k in WGRADS:
            part = np.asarray(b[k], dtype=np.float64)
            acc[k] = part if acc[k] is None else acc[k] + part
        for k in GAINS:
            gparts[k].append(b[k])
        outs = {"qkv": f["qkv"], "residual": f["residual"], "x": b["x"], "z": b["z"]}
        if on_rows is not None:
            on_rows(r0, r1, outs)
        else:
            for k in ROW_LOCAL:
                rows[k].append(outs[k])
    res = {k: O.q(acc[k], mode) for k in WGRADS}
    for k in GAINS:
        res[k] = O.reduce_row_partials((np.concatenate(gparts[k], axis=0), None), mode)
    if rows is not None:
        for k in ROW_LOCAL:
            res[k] = np.concatenate(rows[k], axis=0)
    return res


def run_stack_chunked(ws: list, acts: dict, mode: str = O.SIMBF16, chunk: int = 1024, eps: float = 1e-6,
                      on_rows=None) -> dict:
    """The identity-attention block stack (paper_2605_19269_b200/stack.py glue: x_{l+1} = V span
    of qkv_l, z_{l+1} = residual_l; backward feeds grad_qkv = [0 | 0 | grad_x_l], grad_residual =
    grad_z_l) token-chunked like run_layer_chunked -- every block is row-local in the same way.
    Returns per-block reduced gradients under keys "<name>.<block>"; `on_rows` receives the
    final qkv / residual and block 0's x / z gradients per chunk."""
    if chunk % 128:
        raise ValueError("chunk must be a multiple of the 128-row tile")
    m, d = acts["x"].shape
    nb = len(ws)
    acc = {(k, b): None for k in WGRADS for b in range(nb)}
    gparts = {(k, b): [] for k in GAINS for b in range(nb)}
    for r0 in range(0, m, chunk):
        r1 = min(m, r0 + chunk)
        cos, sin = O.qkv_rope_tables(r1 - r0, d, mode, start=r0)
        x, z = acts["x"][r0:r1], acts["z"][r0:r1]
        tapes = []
        for w in ws:
            f = O.layer_forward(x, z, w, cos, sin, mode, eps=eps)
            tapes.append(f)
            x, z = f["qkv"][:, 2 * d:3 * d], f["residual"]
        gq, gr = acts["grad_qkv"][r0:r1], acts["grad_residual"][r0:r1]
        for b in range(nb - 1, -1, -1):
            parts = _backward_parts(gq, tapes[b], ws[b], mode, gr)
            for k in WGRADS:
                p = np.asarray(parts[k], dtype=np.float64)
                acc[(k, b)] = p if acc[(k, b)] is None else acc[(k, b)] + p
            for k in GAINS:
                gparts[(k, b)].append(parts[k])
            if b > 0:
                gq = np.concatenate([np.zeros((r1 - r0, 2 * d)), parts["x"]], axis=1)
                gr = parts["z"]
        if on_rows is not None:
            on_rows(r0, r1, {"qkv": tapes[-1]["qkv"], "residual": tapes[-1]["residual"], "x": parts["x"],
                             "z": parts["z"]})
    res = {}
    for (k, b), v in acc.items():
        res[f"{k}.{b}"] = O.q(v, mode)
    for (k, b), v in gparts.items():
        res[f"{k}.{b}"] = O.reduce_row_partials((np.concatenate(v, axis=0), None), mode)
    return res


# ----------------------------------------------------------------------------- sketches


SKETCH_ROWS = 6
SAMPLE_ROWS = 4


def _output_index(name: str) -> int:
    """OUTPUTS index; per-block stack outputs "<name>.<b>" get their own streams."""
    base, _, blk = name.partition(".")
    return OUTPUTS.index(base) + (100 * (int(blk) + 1) if blk else 0)


def sketch_matrix(name: str, rows: int, k: int = SKETCH_ROWS, seed: int = 1234) -> np.ndarray:
    """Gaussian JL sketch S (k, rows), float32, deterministic per output name."""
    idx = _output_index(name)
    return np.random.default_rng([seed, 99, idx]).standard_normal((k, rows), dtype=np.float32)


def sample_rows(name: str, rows: int, k: int = SAMPLE_ROWS, seed: int = 1234) -> np.ndarray:
    """First, last and k-2 seeded interior rows (sorted)."""
    idx = _output_index(name)
    inner = np.random.default_rng([seed, 77, idx]).choice(np.arange(1, rows - 1), size=k - 2, replace=False)
    return np.sort(np.concatenate([[0, rows - 1], inner])).astype(np.int64)


def fingerprint(name: str, full: np.ndarray, k: int = SKETCH_ROWS, rows: int = SAMPLE_ROWS) -> dict:
    """Sketch (k rows), Frobenius norm and `rows` sampled rows of one full output (vectors are
    kept whole)."""
    a = np.asarray(full, dtype=np.float64)
    if a.ndim == 1:
        return {"full": a, "norm": float(np.linalg.norm(a))}
    S = sketch_matrix(name, a.shape[0], k).astype(np.float64)
    ri = sample_rows(name, a.shape[0], rows)
    return {"sketch": S @ a, "norm": float(np.linalg.norm(a)), "rows": a[ri], "row_idx": ri}


class RowLocalSketcher:
    """Accumulates fingerprints of the row-local outputs chunk by chunk (run_layer_chunked on_rows)."""

    def __init__(self, m: int, k: int = SKETCH_ROWS, rows: int = SAMPLE_ROWS):
        self.m = m
        self.k = k
        self.rows = rows
        self.acc: dict = {}

    def __call__(self, r0: int, r1: int, outs: dict) -> None:
        for k, v in outs.items():
            a = np.asarray(v, dtype=np.float64)
            st = self.acc.get(k)
            if st is None:
                st = self.acc[k] = {"sketch": 0.0, "sq": 0.0, "rows": {},
                                    "row_idx": sample_rows(k, self.m, self.rows)}
            S = sketch_matrix(k, self.m, self.k)[:, r0:r1].astype(np.float64)
            st["sketch"] = st["sketch"] + S @ a
            st["sq"] += float(np.sum(a * a))
            for r in st["row_idx"]:
                if r0 <= r < r1:
                    st["rows"][int(r)] = a[r - r0]

    def result(self) -> dict:
        out = {}
        for k, st in self.acc.items():
            out[k] = {"sketch": st["sketch"], "norm": float(np.sqrt(st["sq"])),
                      "rows": np.stack([st["rows"][int(r)] for r in st["row_idx"]]), "row_idx": st["row_idx"]}
        return out


def compare(name: str, got: np.ndarray | None, fp: dict, *, got_sketch=None, got_rows=None) -> dict:
    """Estimated Frobenius relative error and sampled-row max-abs error of one output.

    `got` (host array) or `got_sketch`/`got_rows` (computed on the device by the caller) plus the
    fixture fingerprint.  rel_est = ||S(G - O)|| / ||S O||; max_abs over the sampled rows."""
    if "full" in fp:
        g = np.asarray(got, dtype=np.float64)
        o = fp["full"]
        return {"rel": float(np.linalg.norm(g - o) / np.linalg.norm(o)), "max_abs": float(np.max(np.abs(g - o))),
                "max_ref": float(np.max(np.abs(o))), "exact": True}
    if got_sketch is None:
        g = np.asarray(got, dtype=np.float64)
        got_sketch = sketch_matrix(name, g.shape[0], fp["sketch"].shape[0]).astype(np.float64) @ g
        got_rows = g[fp["row_idx"]]
    rel = float(np.linalg.norm(got_sketch - fp["sketch"]) / np.linalg.norm(fp["sketch"]))
    dif = np.abs(np.asarray(got_rows, dtype=np.float64) - fp["rows"])
    rows_rel = float(np.linalg.norm(dif) / np.linalg.norm(fp["rows"]))
    return {"rel": rel, "rows_rel": rows_rel, "max_abs": float(np.max(dif)), "max_ref": float(np.max(np.abs(fp["rows"]))),
            "exact": False}
