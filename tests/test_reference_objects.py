"""Genuine reference objects through the drop-in's host boundary (CPU only).

The reference package (/root/reference/pkg/src/mcfunm) exists only in the build
container; on the GPU box these tests skip.  What is checked: the reference's
own WalkConfig, CoefficientStream and SparseMatrix instances are accepted by
check_config / as_stream / the estimator and centrality input checks, with
the same values and the same errors as this package's types."""
import os
import sys

import numpy as np
import pytest

import paper_2308_01037_b200 as mc
from paper_2308_01037_b200 import errors, series, walker

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "mcfunm")), reason="reference not present")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    try:
        import mcfunm.series as rs
        import mcfunm.sparsemat as rsm
        import mcfunm.walker as rw
        yield rw, rs, rsm
    finally:
        sys.path.remove(REF)


def test_reference_walkconfig_accepted(ref):
    rw, _, _ = ref
    c = walker.check_config(rw.WalkConfig(1234, 1e-7, 25, 9))
    assert (c.n_walks, c.weight_cutoff, c.max_steps, c.seed) == (1234, 1e-7, 25, 9)
    # the same validation errors as the reference (walker.py:60-67)
    with pytest.raises(Exception):
        rw.WalkConfig(0)
    with pytest.raises(errors.ArgumentError):
        walker.WalkConfig(0)


def test_reference_coefficient_streams_accepted(ref):
    _, rs, _ = ref
    for stream in (rs.EXPONENTIAL, rs.RESOLVENT):
        s = series.as_stream(stream)
        assert s.tag == stream.tag
        assert np.array_equal(s.prefix(40), stream.prefix(40))
        assert [s.coeff(k) for k in range(12)] == [stream.coeff(k) for k in range(12)]


def _ref_matrix(rsm, n=5):
    rows = np.array([0, 1, 1, 2, 3, 4, 2, 4])
    cols = np.array([1, 0, 2, 1, 4, 3, 4, 2])
    return rsm.SparseMatrix.from_coo(rows, cols, np.ones(rows.size), n, symmetric_hint=True)


def test_reference_sparsematrix_input_checks(ref):
    rw, rs, rsm = ref
    a = _ref_matrix(rsm)
    cfg = rw.WalkConfig(100, 1e-6, 10, 0)
    # wrong v length is rejected before any device work
    with pytest.raises(errors.ArgumentError):
        mc.rand_funm_action(a, rs.EXPONENTIAL, np.ones(4), cfg)
    # entry index outside [0, n)
    with pytest.raises(errors.ArgumentError):
        mc.rand_funm_entry(a, rs.EXPONENTIAL, np.ones(5), 7, cfg)
    # alpha diagnostic on the reference matrix equals the reference's own
    scaled = rsm.scale(a, 0.3)
    assert walker.alpha_diagnostic(scaled) == rw.alpha_diagnostic(scaled)
    # Katz with an explicit gamma whose alpha >= 1 is rejected
    with pytest.raises(errors.ArgumentError, match="alpha"):
        mc.katz_centrality(a, 0.5, cfg, gamma=1.0)


def test_reference_zero_matrix_h_term(ref):
    """A = 0: the H-term only, no device needed."""
    rw, rs, rsm = ref
    z = rsm.SparseMatrix.from_coo(np.array([], dtype=np.int64), np.array([], dtype=np.int64), np.array([]), 4)
    cfg = rw.WalkConfig(10, 1e-6, 5, 0)
    d = mc.rand_funm_diag(z, rs.EXPONENTIAL, cfg)
    assert np.array_equal(d.values, np.ones(4))
    y = mc.rand_funm_action(z, rs.RESOLVENT, np.arange(4.0), cfg)
    assert np.array_equal(y.values, np.arange(4.0))


def test_reference_matrix_needs_device(ref):
    """A nonzero reference matrix goes to the device; with no GPU the drop-in
    fails loudly (DeviceError), never a CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rw, rs, rsm = ref
    with pytest.raises(errors.DeviceError):
        mc.rand_funm_diag(_ref_matrix(rsm), rs.EXPONENTIAL, rw.WalkConfig(100, 1e-6, 10, 0))
