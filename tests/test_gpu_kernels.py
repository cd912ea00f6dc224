"""GPU parity of every fused launch against the reference's golden vectors.

Inputs come from tests/golden (produced by the reference), the CUDA path runs
through the public API (-> C-ABI -> sm_100a kernels), and results are
compared with the reference outputs and with the CPU oracle.

Tolerances (BASELINE.json north star): SIM32 <= 1e-5 relative, SIMBF16 <= 2e-2
relative (Frobenius), max abs error reported.  Integer metadata (partial
counts / block layouts) must match exactly.
"""

import zlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import coda_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"sim32": 1e-5, "simbf16": 2e-2}


def _mods():
    import paper_2605_19269_b200 as cd

    return cd


def _mode(cd, name):
    return {"sim32": cd.PrecisionMode.SIM32, "simbf16": cd.PrecisionMode.SIMBF16}[name]


def _check(name, got, want, tol, report):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    nrm = np.linalg.norm(want)
    err = float(np.linalg.norm(got - want) / nrm) if nrm else float(np.max(np.abs(got)))
    report[name] = (err, float(np.max(np.abs(got - want))) if got.size else 0.0)
    assert err <= tol, f"{name}: rel {err:.3e} > {tol:.1e} (max abs {report[name][1]:.3e})"


@pytest.mark.parametrize("tag", ["ragged", "default"])
@pytest.mark.parametrize("mode", ["sim32", "simbf16"])
def test_kernels_vs_reference_golden(cuda_ready, tag, mode):
    cd = _mods()
    g = load_golden(f"kernels_{tag}_{mode}")
    m, k, n, tm, tn, rtn = (int(v) for v in g["meta"])
    P = _mode(cd, mode)
    kw = dict(tile_shape=cd.TileShape(tm, tn), reduction_tile_n=rtn, precision=P)
    M = lambda key: cd.DenseMatrix.from_array(g[key], P)  # noqa: E731
    V = lambda key: cd.Vector.from_array(g[key], cd.stat_mode(P))  # noqa: E731
    a, b, bt, z, cos, sin, pre, gin, pre2 = (M(x) for x in ("a", "b", "bt", "z", "cos", "sin", "pre", "gin",
                                                           "preact2"))
    gamma = cd.Vector.from_array(g["gamma"], P)
    r, s = V("r"), V("s")
    tol = TOL[mode]
    rep = {}
    _check("k1", cd.gemm_rope(a, b, cos, sin, **kw).main.data, g["k1"], tol, rep)
    _check("k1_bwd", cd.gemm_rope(a, b, cos, sin, backward=True, **kw).main.data, g["k1_bwd"], tol, rep)
    k2 = cd.gemm_swiglu(a, b, save_preact=True, **kw)
    _check("k2", k2.main.data, g["k2"], tol, rep)
    _check("k2_preact", k2.aux["preact"].data, g["k2_preact"], tol, rep)
    k3 = cd.gemm_partial_xent(a, b, g["labels"].astype(np.int64), store_logits=True, **kw)
    _check("k3", k3.main.data, g["k3"], tol, rep)
    _check("k3_target", k3.aux["target"].data, g["k3_target"], tol, rep)
    assert np.array_equal(k3.aux["lse"].counts, g["k3_lse_counts"])
    _check("k3_lse", cd.combine_lse(k3.aux["lse"]).data, g["k3_lse"], tol, rep)
    k4 = cd.gemm_residual_partial_rms(a, b, z, gamma, **kw)
    _check("k4", k4.main.data, g["k4"], tol, rep)
    _check("k4_pre_norm", k4.aux["pre_norm"].data, g["k4_pre_norm"], tol, rep)
    assert np.array_equal(k4.aux["sumsq"].counts, g["k4_sumsq_counts"])
    _check("k4_sumsq", k4.aux["sumsq"].data, g["k4_sumsq_data"], tol, rep)
    _check("k4_r", cd.finalize_rms(k4.aux["sumsq"], 1e-6).data, g["k4_r"], tol, rep)
    _check("k5", cd.gemm_row_scale(a, b, r, **kw).main.data, g["k5"], tol, rep)
    k6 = cd.gemm_rms_swiglu(a, b, r, **kw)
    _check("k6", k6.main.data, g["k6"], tol, rep)
    _check("k6_preact", k6.aux["preact"].data, g["k6_preact"], tol, rep)
    _check("k7", cd.gemm_rms_rope(a, b, r, cos, sin, **kw).main.data, g["k7"], tol, rep)
    k8 = cd.gemm_rms_partial_xent(a, b, r, g["labels"].astype(np.int64), **kw)
    assert k8.main is None
    _check("k8_target", k8.aux["target"].data, g["k8_target"], tol, rep)
    _check("k8_lse", cd.combine_lse(k8.aux["lse"]).data, g["k8_lse"], tol, rep)
    k9 = cd.gemm_rmsnorm_backward(a, bt, pre, r, gamma, s, grad_in=gin, trans_b=True, **kw)
    _check("k9", k9.main.data, g["k9"], tol, rep)
    _check("k9_normed", k9.aux["normed"].data, g["k9_normed"], tol, rep)
    assert np.array_equal(k9.aux["gamma_grad"].counts, g["k9_gg_counts"])
    _check("k9_gamma_grad", k9.aux["gamma_grad"].data, g["k9_gg_data"], tol, rep)
    _check("k9_dgamma", cd.reduce_row_partials(k9.aux["gamma_grad"]).data, g["k9_dgamma"], tol, rep)
    k10 = cd.gemm_swiglu_backward(a, bt, pre2, trans_b=True, **kw)
    _check("k10", k10.main.data, g["k10"], tol, rep)
    _check("k10_recompute", k10.aux["recompute"].data, g["k10_recompute"], tol, rep)
    assert np.array_equal(k10.aux["rowdot"].counts, g["k10_rowdot_counts"])
    _check("k10_rowdot", k10.aux["rowdot"].data, g["k10_rowdot_data"], tol, rep)
    _check("k10_s", cd.finalize_rowdot(k10.aux["rowdot"], 7).data, g["k10_s"], tol, rep)
    gz, rd = cd.rope_backward_stat(z, pre, cos, sin, tile_n=tn, reduction_tile_n=rtn, precision=P)
    _check("rbs_gz", gz.data, g["rbs_gz"], tol, rep)
    assert np.array_equal(rd.counts, g["rbs_counts"])
    _check("rbs_rowdot", rd.data, g["rbs_data"], tol, rep)
    at = M("at")
    prob = cd.GemmProblem(m=m, n=n, k=k, trans_a=True, precision=P, tile_shape=cd.TileShape(tm, tn),
                          reduction_tile_n=rtn)
    _check("wgrad", cd.run_gemm(prob, at, b).main.data, g["wgrad"], tol, rep)
    print(f"\n[{tag}/{mode}] worst rel {max(v[0] for v in rep.values()):.3e}; "
          + ", ".join(f"{k}={v[0]:.1e}" for k, v in rep.items()))


@pytest.mark.parametrize("layout", ["nn", "nt", "tn", "tt"])
@pytest.mark.parametrize("shape", [(128, 256, 64), (300, 520, 200), (1024, 768, 1000), (7, 9, 5)])
def test_plain_gemm_vs_torch_fp32(cuda_ready, layout, shape):
    """Mainloop numerics for every operand majorness against a torch fp32 matmul."""
    import torch

    cd = _mods()
    m, n, k = shape
    ta, tb = layout[0] == "t", layout[1] == "t"
    gen = torch.Generator(device="cuda").manual_seed(zlib.crc32(f"{layout}{shape}".encode()))
    A = torch.randn((k, m) if ta else (m, k), device="cuda", generator=gen).to(torch.bfloat16)
    B = torch.randn((n, k) if tb else (k, n), device="cuda", generator=gen).to(torch.bfloat16)
    P = cd.PrecisionMode.SIMBF16
    res = cd.run_gemm(cd.GemmProblem(m=m, n=n, k=k, trans_a=ta, trans_b=tb, precision=P),
                      cd.DenseMatrix.from_tensor(A, P), cd.DenseMatrix.from_tensor(B, P), out_f32=True)
    ref = (A.float().T if ta else A.float()) @ (B.float().T if tb else B.float())
    got = res.main.tensor
    err = float((got - ref).norm() / ref.norm())
    assert err < 1e-5, f"{layout} {shape}: rel {err:.3e}"


def test_exact64_is_rejected(cuda_ready):
    cd = _mods()
    a = cd.DenseMatrix.from_array(np.ones((4, 4)), cd.PrecisionMode.SIMBF16)
    with pytest.raises(cd.ConfigError):
        cd.gemm_row_scale(a, a, cd.Vector.from_array(np.ones(4)))


def test_launch_is_deterministic(cuda_ready):
    cd = _mods()
    g = load_golden("kernels_default_simbf16")
    P = cd.PrecisionMode.SIMBF16
    a, bt, pre, gin = (cd.DenseMatrix.from_array(g[x], P) for x in ("a", "bt", "pre", "gin"))
    r = cd.Vector.from_array(g["r"], cd.PrecisionMode.SIM32)
    s = cd.Vector.from_array(g["s"], cd.PrecisionMode.SIM32)
    gamma = cd.Vector.from_array(g["gamma"], P)
    outs = [cd.gemm_rmsnorm_backward(a, bt, pre, r, gamma, s, grad_in=gin, trans_b=True, precision=P)
            for _ in range(3)]
    for o in outs[1:]:
        assert np.array_equal(o.main.data, outs[0].main.data)
        assert np.array_equal(o.aux["gamma_grad"].data, outs[0].aux["gamma_grad"].data)


def test_tile_shape_invariance(cuda_ready):
    """Reference tile shapes change only the partial layout, never the finalized statistics."""
    cd = _mods()
    rng = np.random.default_rng(3)
    P = cd.PrecisionMode.SIM32
    a = cd.DenseMatrix.from_array(rng.standard_normal((200, 96)), P)
    b = cd.DenseMatrix.from_array(rng.standard_normal((96, 300)) / 10, P)
    z = cd.DenseMatrix.from_array(rng.standard_normal((200, 300)), P)
    gamma = cd.Vector.from_array(np.ones(300), P)
    rs = []
    for tile, rtn in (((128, 128), 128), ((16, 24), 10), ((32, 300), 7), ((8, 512), 512)):
        k4 = cd.gemm_residual_partial_rms(a, b, z, gamma, tile_shape=cd.TileShape(*tile), reduction_tile_n=rtn,
                                          precision=P)
        rs.append(cd.finalize_rms(k4.aux["sumsq"]).data)
    for r in rs[1:]:
        assert O.rel_error(r, rs[0]) < 1e-6


def test_specialised_and_generic_epilogues_agree(cuda_ready):
    """The flag-specialised kernels and the generic interpreter compute the same launch."""
    import os
    import subprocess
    import sys

    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import load_golden
import paper_2605_19269_b200 as cd
g = load_golden("kernels_default_simbf16")
P = cd.PrecisionMode.SIMBF16
M = lambda k: cd.DenseMatrix.from_array(g[k], P)
a, b, bt, z, cos, sin, pre, gin, pre2 = (M(x) for x in ("a","b","bt","z","cos","sin","pre","gin","preact2"))
r = cd.Vector.from_array(g["r"], cd.PrecisionMode.SIM32); s = cd.Vector.from_array(g["s"], cd.PrecisionMode.SIM32)
gamma = cd.Vector.from_array(g["gamma"], P)
kw = dict(precision=P)
outs = []
k4 = cd.gemm_residual_partial_rms(a, b, z, gamma, **kw); outs += [k4.main.data, k4.aux["pre_norm"].data, k4.aux["sumsq"].data]
k6 = cd.gemm_rms_swiglu(a, b, r, **kw); outs += [k6.main.data, k6.aux["preact"].data]
outs.append(cd.gemm_rms_rope(a, b, r, cos, sin, **kw).main.data)
k9 = cd.gemm_rmsnorm_backward(a, bt, pre, r, gamma, s, grad_in=gin, trans_b=True, **kw)
outs += [k9.main.data, k9.aux["normed"].data, k9.aux["gamma_grad"].data]
k10 = cd.gemm_swiglu_backward(a, bt, pre2, trans_b=True, **kw)
outs += [k10.main.data, k10.aux["recompute"].data, k10.aux["rowdot"].data]
lab = g["labels"].astype(np.int64)
k3 = cd.gemm_partial_xent(a, b, lab, store_logits=True, **kw)
outs += [k3.main.data, k3.aux["target"].data, cd.combine_lse(k3.aux["lse"]).data]
k8 = cd.gemm_rms_partial_xent(a, b, r, lab, **kw)
outs += [k8.aux["target"].data, cd.combine_lse(k8.aux["lse"]).data]
np.savez(sys.argv[1], *outs)
'''
    res = {}
    variants = {"fast-2cta": ("0", "2"), "fast-1cta": ("0", "1"), "generic": ("1", "2")}
    for name, (generic, cg) in variants.items():
        out = f"/tmp/coda_epi_{name}.npz"
        env = dict(os.environ, CODA_FORCE_GENERIC=generic, CODA_CG=cg)
        subprocess.run([sys.executable, "-c", code, out], check=True, env=env, cwd=str(__import__("conftest").ROOT))
        with np.load(out) as z:
            res[name] = [z[k] for k in z.files]
    for other in ("fast-1cta", "fast-2cta"):
        for x, y in zip(res[other], res["generic"]):
            assert x.shape == y.shape
            assert O.rel_error(x, y) < 1e-5 if np.linalg.norm(y) else np.all(x == y)


def _split_programs(cd, m, k, n, seed=8):
    """Every fast-path program family (K4, K6, K7, K9 + grad_in, K10, K8, a TN plain GEMM) on
    one set of seeded operands; returns a function that runs them and returns the outputs."""
    import torch

    rng = np.random.default_rng(seed)
    P = cd.PrecisionMode.SIMBF16
    M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
    a, b = M(rng.standard_normal((m, k)) / 40), M(rng.standard_normal((k, n)) / 40)
    bt = M(rng.standard_normal((n, k)) / 40)
    z, pre, gin = M(rng.standard_normal((m, n))), M(rng.standard_normal((m, n))), M(rng.standard_normal((m, n)))
    pre2 = M(rng.standard_normal((m, 2 * n)))
    cos, sin = cd.rope_tables(m, n, precision=P)
    r = cd.Vector.from_array(0.5 + rng.random(m), cd.PrecisionMode.SIM32)
    s = cd.Vector.from_array(0.1 * rng.standard_normal(m), cd.PrecisionMode.SIM32)
    gamma = cd.Vector.from_array(1 + 0.1 * rng.standard_normal(n), P)
    labels = rng.integers(0, n, m).astype(np.int64)
    at = M(rng.standard_normal((k, m)) / 40)

    def run():
        outs = []
        k4 = cd.gemm_residual_partial_rms(a, b, z, gamma, precision=P)
        outs += [k4.main.data, k4.aux["pre_norm"].data, cd.finalize_rms(k4.aux["sumsq"]).data]
        k6 = cd.gemm_rms_swiglu(a, b, r, precision=P)
        outs += [k6.main.data, k6.aux["preact"].data]
        outs.append(cd.gemm_rms_rope(a, b, r, cos, sin, precision=P).main.data)
        k9 = cd.gemm_rmsnorm_backward(a, bt, pre, r, gamma, s, grad_in=gin, trans_b=True, precision=P)
        outs += [k9.main.data, k9.aux["normed"].data, cd.reduce_row_partials(k9.aux["gamma_grad"]).data]
        k10 = cd.gemm_swiglu_backward(a, bt, pre2, trans_b=True, precision=P)
        outs += [k10.main.data, k10.aux["recompute"].data, cd.finalize_rowdot(k10.aux["rowdot"], n).data]
        k8 = cd.gemm_rms_partial_xent(a, b, r, labels, precision=P)
        outs += [k8.aux["target"].data, cd.combine_lse(k8.aux["lse"]).data]
        prob = cd.GemmProblem(m=m, n=n, k=k, trans_a=True, precision=P)
        outs.append(cd.run_gemm(prob, at, b).main.data)
        torch.cuda.synchronize()
        return outs

    return run


def test_tail_split_matches_unsplit(cuda_ready):
    """Wave-tail split-K (partial last wave folded in fixed order) equals the unsplit launch."""
    cd = _mods()
    from paper_2605_19269_b200 import _native

    run = _split_programs(cd, 1000, 2048, 1536)    # 4 x 6 = 24 pair tiles < 74 units -> every tile split
    try:
        _native.set_option("split_min_k", 0)     # split every eligible launch of this test
        _native.set_option("split", 0)
        ref = run()
        _native.set_option("split", 1)
        got = run()
        got2 = run()
    finally:
        _native.set_option("split", 1)
        _native.set_option("split_min_k", 8192)
    for i, (x, y, y2) in enumerate(zip(ref, got, got2)):
        assert np.array_equal(y, y2), f"output {i}: split launch not deterministic"
        assert O.rel_error(y, x) < 5e-3, (i, O.rel_error(y, x))



def test_concurrent_streams_with_tail_split(cuda_ready):
    """Two split-K launches running concurrently on two streams use separate workspaces
    and give the same bits as when run one after the other."""
    import torch

    cd = _mods()
    from paper_2605_19269_b200 import _native

    rng = np.random.default_rng(5)
    P = cd.PrecisionMode.SIMBF16
    M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
    m, k, n = 2304, 8192, 2560            # 90 pair tiles: a full wave plus a split tail
    pairs = [(M(rng.standard_normal((m, k)) / 64), M(rng.standard_normal((k, n)) / 64)) for _ in range(2)]
    prob = cd.GemmProblem(m=m, n=n, k=k, precision=P)
    try:
        _native.set_option("split_min_k", 0)
        ref = [cd.run_gemm(prob, a, b).main.data for a, b in pairs]
        streams = [torch.cuda.Stream() for _ in pairs]
        outs = []
        torch.cuda.synchronize()
        for (a, b), s in zip(pairs, streams):
            with torch.cuda.stream(s):
                outs.append(cd.run_gemm(prob, a, b))
        torch.cuda.synchronize()
    finally:
        _native.set_option("split_min_k", 8192)
    for r, o in zip(ref, outs):
        assert np.array_equal(r, o.main.data)


@pytest.mark.parametrize("n", [33, 258, 262, 1000])
@pytest.mark.parametrize("out_f32", [False, True])
def test_ragged_columns_copy_out(cuda_ready, n, out_f32):
    """The epilogue's coalesced copy-out of a staged box whose last 16-B chunk is partial
    (N not a multiple of 8 bf16 / 4 f32 values): every column, the ragged last ones
    included, matches the product (f32) or its bf16 rounding."""
    import torch

    cd = _mods()
    P = cd.PrecisionMode.SIMBF16
    rng = np.random.default_rng(n)
    m, k = 300, 256
    a = cd.DenseMatrix.from_array(rng.standard_normal((m, k)) / 16, P)
    b = cd.DenseMatrix.from_array(rng.standard_normal((k, n)) / 16, P)
    prob = cd.GemmProblem(m=m, n=n, k=k, precision=P)
    t = cd.run_gemm(prob, a, b, out_f32=out_f32).main.tensor
    torch.cuda.synchronize()
    got = t.float().cpu().numpy().astype(np.float64)
    exact = O.gemm(a.data, b.data, O.SIMBF16)
    want = exact if out_f32 else O.q(exact, O.SIMBF16)
    scale = np.max(np.abs(want))
    tol = 1e-5 if out_f32 else 8e-3            # f32 accumulation order / one bf16 ulp
    assert np.max(np.abs(got - want)) <= tol * scale
    tail = slice(max(0, n - 9), n)             # the partial chunk and the one before it
    assert np.max(np.abs(got[:, tail] - want[:, tail])) <= tol * scale
