"""Generate the full-size parity fixtures tests/golden/fullsize_<cfg>.npz (test infrastructure).

Runs the token-chunked fused-order oracle (oracle/fullsize.py, a restatement of
tilefuse kernels.py:810-1013 pinned by the golden vectors of make_golden.py) over
the whole benchmarked block — C3 (8192 x 2048, ffn 2 x 8192) and C4 (16384 x 4096,
ffn 2 x 14336), bf16 storage — on this container's CPU, and stores, for every
output (qkv, residual, the eight gradients), a Gaussian sketch S·O, the Frobenius
norm and a few full sampled rows (gain gradients are stored whole).  The GPU test
(tests/test_gpu_fullsize_parity.py) regenerates the same bf16 inputs from the
same seeds on the box, runs the CUDA path, and compares against these.

    python tests/golden/make_fullsize.py [c3] [c4] [c5] [c4gqa]
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import coda_oracle as O  # noqa: E402
from oracle import fullsize as FS  # noqa: E402

SEED = 0


def make_stack(name: str) -> Path:
    """C5: the 4-block stack (identity-attention glue of stack.py), 8192 tokens; per-block
    weight / gain gradients under "<name>.<block>", block 0's x / z gradients and the last
    block's qkv / residual as row-local outputs."""
    t0 = time.time()
    ws, acts = FS.make_stack_inputs(name, seed=SEED)
    t1 = time.time()
    m = acts["x"].shape[0]
    sk = FS.RowLocalSketcher(m, k=4, rows=2)          # 28 outputs: smaller fingerprints
    res = FS.run_stack_chunked(ws, acts, O.SIMBF16, chunk=1024, on_rows=sk)
    t2 = time.time()
    fps = sk.result()
    for k, v in res.items():
        fps[k] = FS.fingerprint(k, v, k=4, rows=2)
    arrays = {"meta_seed": np.array(SEED), "meta_config": np.array(name), "meta_mode": np.array(O.SIMBF16),
              "meta_oracle_s": np.array(t2 - t1), "meta_blocks": np.array(len(ws))}
    for k, fp in fps.items():
        for field, v in fp.items():
            a = np.asarray(v)
            if a.dtype == np.float64 and a.ndim > 0 and field in ("rows", "sketch"):
                a = a.astype(np.float32)
            arrays[f"{k}__{field}"] = a
    out = ROOT / "tests" / "golden" / f"fullsize_{name}.npz"
    np.savez_compressed(out, **arrays)
    print(f"{name}: inputs {t1 - t0:.1f}s, oracle {t2 - t1:.1f}s -> {out} ({out.stat().st_size / 1e6:.2f} MB)")
    return out


def make(name: str) -> Path:
    if name in FS.BLOCKS:
        return make_stack(name)
    t0 = time.time()
    inp = FS.make_inputs(name, seed=SEED)
    t1 = time.time()
    m = inp["x"].shape[0]
    sk = FS.RowLocalSketcher(m)
    res = FS.run_layer_chunked(inp, O.SIMBF16, chunk=1024, on_rows=sk)
    t2 = time.time()
    fps = sk.result()
    for k in FS.WGRADS + FS.GAINS:
        fps[k] = FS.fingerprint(k, res[k])
    arrays = {"meta_seed": np.array(SEED), "meta_config": np.array(name), "meta_mode": np.array(O.SIMBF16),
              "meta_oracle_s": np.array(t2 - t1)}
    for k, fp in fps.items():
        for field, v in fp.items():
            a = np.asarray(v)
            if a.dtype == np.float64 and a.ndim > 0:
                a = a.astype(np.float32) if field == "rows" else a
            arrays[f"{k}__{field}"] = a
    out = ROOT / "tests" / "golden" / f"fullsize_{name}.npz"
    np.savez_compressed(out, **arrays)
    print(f"{name}: inputs {t1 - t0:.1f}s, oracle {t2 - t1:.1f}s -> {out} ({out.stat().st_size / 1e6:.2f} MB)")
    return out


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c3", "c4", "c5"]:
        make(n)
