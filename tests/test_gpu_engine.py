"""run_gemm engine behaviour on the GPU, mirroring the reference's tests/test_engine.py:
tile-order irrelevance, ledger accounting, store_main=False, output on the precision
grid, and the binding / label error taxonomy raised before any launch."""

import numpy as np
import pytest

from oracle import coda_oracle as O

pytestmark = pytest.mark.gpu


def _cd():
    import paper_2605_19269_b200 as cd

    return cd


def _rand(cd, rng, r, c, P):
    return cd.DenseMatrix.from_array(rng.standard_normal((r, c)), P)


def _problem(cd, m, n, k, P, tile=(128, 128), **kw):
    return cd.GemmProblem(m=m, n=n, k=k, tile_shape=cd.TileShape(*tile), precision=P, **kw)


@pytest.fixture
def P(cuda_ready):
    return _cd().PrecisionMode.SIMBF16


def test_tile_order_is_irrelevant_bit_for_bit(P):
    cd = _cd()
    rng = np.random.default_rng(4)
    a, b = _rand(cd, rng, 10, 6, P), _rand(cd, rng, 6, 9, P)
    p = _problem(cd, 10, 9, 6, P, tile=(4, 4))
    base = cd.run_gemm(p, a, b).main.data
    grid = [(i, j) for i in range(3) for j in range(3)]
    for order in (list(reversed(grid)), grid[1::2] + grid[0::2]):
        assert np.array_equal(cd.run_gemm(p, a, b, tile_order=order).main.data, base)


def test_tile_order_must_be_a_permutation(P):
    cd = _cd()
    rng = np.random.default_rng(5)
    a, b = _rand(cd, rng, 4, 4, P), _rand(cd, rng, 4, 4, P)
    with pytest.raises(cd.ConfigError):
        cd.run_gemm(_problem(cd, 4, 4, 4, P), a, b, tile_order=[(0, 0), (0, 0)])


def test_ledger_accounting_and_row_vec(P):
    cd = _cd()
    rng = np.random.default_rng(6)
    m, n, k = 6, 10, 7
    a, b = _rand(cd, rng, m, k, P), _rand(cd, rng, k, n, P)
    ledger = cd.TrafficLedger()
    res = cd.run_gemm(_problem(cd, m, n, k, P), a, b, kernel_name="gemm", ledger=ledger)
    assert res.record.read_bytes == (m * k + k * n) * 2
    assert res.record.write_bytes == m * n * 2
    assert ledger.launches == 1 and ledger.records[0] is res.record
    g = cd.Vector.from_array(rng.standard_normal(n), P)
    prog = cd.EpilogueProgram([cd.RowVecMul("gamma")])
    res = cd.run_gemm(_problem(cd, m, n, k, P), a, b, prog, {"gamma": g})
    assert res.record.read_bytes == (m * k + k * n) * 2 + n * 2
    want = O.q(O.gemm(a.data, b.data, O.SIMBF16) * g.data[None, :], O.SIMBF16)
    assert O.rel_error(res.main.data, want) < 1e-2


def test_store_main_false_writes_nothing(P):
    cd = _cd()
    rng = np.random.default_rng(8)
    a, b = _rand(cd, rng, 4, 4, P), _rand(cd, rng, 4, 4, P)
    res = cd.run_gemm(_problem(cd, 4, 4, 4, P), a, b, store_main=False)
    assert res.main is None and res.record.write_bytes == 0


def test_reduced_precision_output_lives_on_grid(cuda_ready):
    cd = _cd()
    rng = np.random.default_rng(9)
    for mode, om in ((cd.PrecisionMode.SIM32, O.SIM32), (cd.PrecisionMode.SIMBF16, O.SIMBF16)):
        a, b = _rand(cd, rng, 5, 6, mode), _rand(cd, rng, 6, 4, mode)
        out = cd.run_gemm(_problem(cd, 5, 4, 6, mode), a, b).main
        assert out.precision is mode
        assert np.array_equal(O.q(out.data, om), out.data)


class TestBindingErrors:
    @pytest.fixture(autouse=True)
    def _setup(self, P):
        cd = _cd()
        rng = np.random.default_rng(11)
        self.cd, self.P = cd, P
        self.a, self.b = _rand(cd, rng, 4, 3, P), _rand(cd, rng, 3, 5, P)
        self.p = _problem(cd, 4, 5, 3, P)

    def test_missing_operand(self):
        prog = self.cd.EpilogueProgram([self.cd.RowVecMul("gamma")])
        with pytest.raises(self.cd.BindingError):
            self.cd.run_gemm(self.p, self.a, self.b, prog, {})

    def test_unused_binding(self):
        extra = {"stray": self.cd.Vector.from_array(np.ones(5), self.P)}
        with pytest.raises(self.cd.BindingError):
            self.cd.run_gemm(self.p, self.a, self.b, None, extra)

    def test_wrong_container_kind(self):
        prog = self.cd.EpilogueProgram([self.cd.RowVecMul("gamma")])
        bad = {"gamma": self.cd.DenseMatrix.from_array(np.ones((1, 5)), self.P)}
        with pytest.raises(self.cd.BindingError):
            self.cd.run_gemm(self.p, self.a, self.b, prog, bad)

    def test_wrong_vector_length(self):
        prog = self.cd.EpilogueProgram([self.cd.RowVecMul("gamma")])
        bad = {"gamma": self.cd.Vector.from_array(np.ones(4), self.P)}
        with pytest.raises(self.cd.DimensionError):
            self.cd.run_gemm(self.p, self.a, self.b, prog, bad)

    def test_operand_shape_mismatch(self):
        with pytest.raises(self.cd.DimensionError):
            self.cd.run_gemm(self.p, self.b, self.a)

    def test_operands_must_be_matrices(self):
        with pytest.raises(self.cd.BindingError):
            self.cd.run_gemm(self.p, self.a.data, self.b.data)


class TestLabels:
    def make(self, labels):
        cd = _cd()
        P = cd.PrecisionMode.SIMBF16
        rng = np.random.default_rng(12)
        a, b = _rand(cd, rng, 4, 3, P), _rand(cd, rng, 3, 5, P)
        prog = cd.EpilogueProgram([cd.OnlineLse(), cd.TargetGather()])
        return cd.run_gemm(_problem(cd, 4, 5, 3, P), a, b, prog, {"labels": labels}, store_main=False)

    def test_valid_labels_gather(self, cuda_ready):
        res = self.make(np.array([0, 4, 2, 2]))
        assert len(res.aux["target"]) == 4

    @pytest.mark.parametrize("labels", [[0, 5, 2, 2], [0, -1, 2, 2], [0.0, 1.0, 2.0, 3.0]])
    def test_bad_labels(self, cuda_ready, labels):
        import paper_2605_19269_b200 as cd

        with pytest.raises(cd.LabelError):
            self.make(np.array(labels))
