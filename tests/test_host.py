"""Host-side logic of the drop-in that needs no GPU."""
import numpy as np
import pytest

import paper_2308_01037_b200 as mc
from paper_2308_01037_b200 import errors, series, sparsemat, walker
from tests import golden_io


def test_walkconfig_validation():
    with pytest.raises(errors.ArgumentError):
        walker.WalkConfig(0)
    with pytest.raises(errors.ArgumentError):
        walker.WalkConfig(10, weight_cutoff=1.0)
    with pytest.raises(errors.ArgumentError):
        walker.WalkConfig(10, weight_cutoff=0.0)
    with pytest.raises(errors.ArgumentError):
        walker.WalkConfig(10, max_steps=0)
    c = walker.WalkConfig(5.0)
    assert c.n_walks == 5 and c.weight_cutoff == 1e-6 and c.max_steps == 10_000 and c.seed == 0


def test_series_kats():
    k = golden_io.kats()
    assert [series.EXPONENTIAL.coeff(i) for i in range(6)] == k["coeff_exp_0_5"]
    assert series.EXPONENTIAL.prefix(32).tolist() == k["prefix_exp_32"]
    assert series.RESOLVENT.coeff(7) == 1.0 and series.RESOLVENT.ratio(5) == 1.0
    assert series.EXPONENTIAL.ratio(9) == 0.1
    assert 0.0 <= series.EXPONENTIAL.coeff(170) < 1e-300
    with pytest.raises(errors.ArgumentError):
        series.CoefficientStream("sine")
    assert series.as_stream("resolvent") == series.RESOLVENT


def test_sparse_matrix_contract():
    with pytest.raises(errors.ArgumentError):
        sparsemat.SparseMatrix.from_coo([0, 0], [1, 1], [1.0, 2.0], 2)   # duplicate
    with pytest.raises(errors.ArgumentError):
        sparsemat.SparseMatrix.from_coo([0], [1], [0.0], 2)              # explicit zero
    with pytest.raises(errors.ArgumentError):
        sparsemat.SparseMatrix.from_coo([0], [2], [1.0], 2)              # out of range
    a = sparsemat.SparseMatrix.from_dense([[0, 2, -1], [0, 0, 0], [5, 0, 0]])
    assert sparsemat.row_abs_sums(a).tolist() == [3, 0, 5]
    s = sparsemat.scale(a, 0.5)
    assert s.csr.data.tolist() == [1.0, -0.5, 2.5] and s.meta["gamma"] == 0.5
    with pytest.raises(errors.ArgumentError):
        sparsemat.scale(a, 0.0)
    c4 = sparsemat.SparseMatrix.from_dense(np.roll(np.eye(4), 1, 1) + np.roll(np.eye(4), -1, 1), True)
    assert walker.alpha_diagnostic(sparsemat.scale(c4, 0.1)) == pytest.approx(0.04)


def test_error_codes_map_to_reference_hierarchy():
    assert errors.BY_CODE[1] is errors.ArgumentError
    assert issubclass(errors.BY_CODE[2], errors.DataError) and errors.BY_CODE[2].exit_code == 2
    assert errors.BY_CODE[3].exit_code == 3 and errors.BY_CODE[4].exit_code == 4


def test_product_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    a = sparsemat.SparseMatrix.from_dense([[0, 1], [1, 0]], True)
    with pytest.raises(errors.McfunmError):
        mc.rand_funm_action(a, series.EXPONENTIAL, np.ones(2), walker.WalkConfig(10))
    with pytest.raises(errors.McfunmError):
        mc.subgraph_centrality(a, 0.1, walker.WalkConfig(10))


def test_zero_matrix_is_h_term_only():
    # A = 0 needs no device: d = zeta_0, y = zeta_0 v exactly
    z = sparsemat.SparseMatrix(sparsemat.sparse.csr_array((3, 3)), sparsemat.sparse.csc_array((3, 3)))
    d = mc.rand_funm_diag(z, series.EXPONENTIAL, walker.WalkConfig(10))
    assert d.values.tolist() == [1.0, 1.0, 1.0]
    y = mc.rand_funm_action(z, series.EXPONENTIAL, np.array([1.0, -2.0, 3.0]), walker.WalkConfig(10))
    assert y.values.tolist() == [1.0, -2.0, 3.0]
