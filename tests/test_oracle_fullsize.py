"""CPU checks of the token-chunked full-size oracle driver (oracle/fullsize.py).

Chunking must not change the reference algorithm: row-local outputs and the
gain gradients are bit-identical to the unchunked fused-order oracle, weight
gradients differ only by float32 accumulation order.  Also pins the fixture
format the GPU full-size parity tests read.
"""

import numpy as np
import pytest

from oracle import coda_oracle as O
from oracle import fullsize as FS


def _small_inputs(m=512, d=128, inter=256, mode=O.SIMBF16):
    FS.CONFIGS["_t"] = (m, d, inter)
    try:
        return FS.make_inputs("_t", seed=3, mode=mode, scale=0.2)
    finally:
        del FS.CONFIGS["_t"]


@pytest.mark.parametrize("mode", [O.SIMBF16, O.SIM32])
def test_chunked_equals_unchunked(mode):
    inp = _small_inputs(mode=mode)
    m, d = inp["x"].shape
    w = FS.weights_of(inp)
    cos, sin = O.qkv_rope_tables(m, d, mode)
    f = O.layer_forward(inp["x"], inp["z"], w, cos, sin, mode)
    b = O.layer_backward(inp["grad_qkv"], f, w, mode, grad_residual=inp["grad_residual"])
    res = FS.run_layer_chunked(inp, mode, chunk=128)
    assert np.array_equal(res["qkv"], f["qkv"])
    assert np.array_equal(res["residual"], f["residual"])
    for k in ("x", "z", "gamma_ffn", "gamma_qkv"):
        assert np.array_equal(res[k], b[k]), k
    for k in FS.WGRADS:
        assert O.rel_error(res[k], b[k]) < (2e-3 if mode == O.SIMBF16 else 1e-6), k


def test_row_local_sketcher_matches_fingerprint():
    inp = _small_inputs(m=384)
    m = inp["x"].shape[0]
    sk = FS.RowLocalSketcher(m)
    FS.run_layer_chunked(inp, O.SIMBF16, chunk=128, on_rows=sk)
    full = FS.run_layer_chunked(inp, O.SIMBF16, chunk=384)
    fps = sk.result()
    for k in FS.ROW_LOCAL:
        ref = FS.fingerprint(k, full[k])
        np.testing.assert_allclose(fps[k]["sketch"], ref["sketch"], rtol=1e-9, atol=1e-9)
        assert np.array_equal(fps[k]["rows"], ref["rows"])
        assert abs(fps[k]["norm"] - ref["norm"]) <= 1e-9 * ref["norm"]
        assert FS.compare(k, full[k], fps[k])["rel"] < 1e-12


def test_compare_estimates_relative_error():
    rng = np.random.default_rng(0)
    o = rng.standard_normal((4096, 64))
    g = o + 1e-3 * rng.standard_normal(o.shape)
    fp = FS.fingerprint("w_out", o)
    est = FS.compare("w_out", g, fp)["rel"]
    assert 0.5e-3 < est < 2e-3          # true value 1e-3; JL estimate with 6 sketch rows


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_fixture_format(name):
    from pathlib import Path

    p = Path(__file__).parent / "golden" / f"fullsize_{name}.npz"
    if not p.exists():
        pytest.skip("fixture not generated")
    z = np.load(p)
    m, d, inter = FS.CONFIGS[name]
    assert str(z["meta_config"]) == name
    for k in FS.OUTPUTS:
        if k.startswith("gamma"):
            assert z[f"{k}__full"].shape == (d,)
        else:
            assert z[f"{k}__sketch"].shape[0] == FS.SKETCH_ROWS
            assert z[f"{k}__rows"].shape[0] == FS.SAMPLE_ROWS


def test_stack_chunked_equals_chained_oracle():
    """The chunked stack driver reproduces the block-by-block chained oracle (stack.py glue)."""
    FS.CONFIGS["_s"] = (256, 64, 128)
    FS.BLOCKS["_s"] = 3
    try:
        ws, acts = FS.make_stack_inputs("_s", seed=4, scale=0.2)
    finally:
        del FS.CONFIGS["_s"], FS.BLOCKS["_s"]
    mode = O.SIMBF16
    m, d = acts["x"].shape
    res = FS.run_stack_chunked(ws, acts, mode, chunk=128)
    cos, sin = O.qkv_rope_tables(m, d, mode)
    x, z, tapes = acts["x"], acts["z"], []
    for w in ws:
        f = O.layer_forward(x, z, w, cos, sin, mode)
        tapes.append(f)
        x, z = f["qkv"][:, 2 * d:], f["residual"]
    gq, gr = acts["grad_qkv"], acts["grad_residual"]
    for b in range(len(ws) - 1, -1, -1):
        g = O.layer_backward(gq, tapes[b], ws[b], mode, grad_residual=gr)
        for k in FS.GAINS:
            assert np.array_equal(res[f"{k}.{b}"], g[k]), (k, b)
        for k in FS.WGRADS:
            assert O.rel_error(res[f"{k}.{b}"], g[k]) < 2e-3, (k, b)
        gq, gr = np.concatenate([np.zeros((m, 2 * d)), g["x"]], axis=1), g["z"]


def test_chunked_equals_unchunked_gqa():
    """The GQA extension layout (k / v spans narrower than hidden) through the chunked driver."""
    FS.CONFIGS["_g"], FS.KV["_g"] = (512, 128, 256), 32
    try:
        inp = FS.make_inputs("_g", seed=5, mode=O.SIMBF16, scale=0.2)
    finally:
        del FS.CONFIGS["_g"], FS.KV["_g"]
    m, d = inp["x"].shape
    assert inp["w_qkv"].shape == (d, d + 64) and inp["grad_qkv"].shape == (m, d + 64)
    w = FS.weights_of(inp)
    cos, sin = O.qkv_rope_tables(m, d, O.SIMBF16, kv_width=32)
    f = O.layer_forward(inp["x"], inp["z"], w, cos, sin, O.SIMBF16)
    b = O.layer_backward(inp["grad_qkv"], f, w, O.SIMBF16, grad_residual=inp["grad_residual"])
    res = FS.run_layer_chunked(inp, O.SIMBF16, chunk=128)
    assert np.array_equal(res["qkv"], f["qkv"])
    for k in ("x", "z", "gamma_ffn", "gamma_qkv"):
        assert np.array_equal(res[k], b[k]), k
    for k in FS.WGRADS:
        assert O.rel_error(res[k], b[k]) < 2e-3, k
