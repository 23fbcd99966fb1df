"""Oracle restatements of the SPEC-only estimators (rand_funm_entry,
mc_baseline): their SPEC examples and the exact
zero-variance cases.  These layers have no reference code to pin against, so
parity for them rests on the SPEC examples and on the shared, pinned walker."""
import numpy as np
import pytest

from oracle import port


def test_entry_empty_row_is_h_term_only():
    a = port.Csr.from_dense([[0, 1, 0], [1, 0, 0], [0, 0, 0]])
    v = np.array([2.0, 3.0, 5.0])
    r = port.funm_entry(a, "exponential", v, 2, 1000, 1e-6, 100, 0)
    assert r.payload[0] == 5.0 and r.walks == 0


@pytest.mark.parametrize("i", [0, 1])
def test_entry_involutory_exact(i):
    g = 0.1
    a = port.Csr.from_dense([[0, g], [g, 0]])
    ref = port.dense_funm(a, "exponential", 29).sum(1)[i]
    y = port.funm_entry(a, "exponential", np.ones(2), i, 500, 1e-300, 28, 3).payload[0]
    assert abs(y - ref) < 1e-14 and abs(y - np.exp(0.1)) < 1e-12


def test_entry_budgets_renormalised_over_row_support():
    a = port.Csr.from_dense([[0, 1, 1, 0], [1, 0, 0, 1], [1, 0, 0, 0], [0, 1, 0, 0]])
    t = port.transition_tables(a)
    ni = port.entry_budgets(t, a, 0, 1001)
    assert ni.sum() == 1001 and ni[0] == 0 and ni[3] == 0 and ni[1] > 0 and ni[2] > 0


def test_mc_baseline_spec_example():
    """2-node path, exponential, gamma = 0.1 -> diag within 1e-2 of cosh 0.1."""
    a = port.Csr.from_dense([[0, 0.1], [0.1, 0]])
    d = port.mc_baseline(a, "exponential", 10_000, 1e-10, 10_000, 0, "diag").payload
    np.testing.assert_allclose(d, np.cosh(0.1), atol=1e-2)
    y = port.mc_baseline(a, "exponential", 10_000, 1e-10, 10_000, 0, "action", v=np.ones(2)).payload
    np.testing.assert_allclose(y, np.exp(0.1), rtol=1e-12)  # zero-variance walks


def test_mc_baseline_zero_walk_terms_match_series():
    """One walk per row on the involutory 2x2 with the cap only: deterministic,
    equals the truncated series with max_steps terms (k = 0..M-1)."""
    g = 0.5
    a = port.Csr.from_dense([[0, g], [g, 0]])
    for m in (1, 4, 9):
        ref = port.dense_funm(a, "exponential", m - 1)
        d = port.mc_baseline(a, "exponential", 1, 1e-300, m, 0, "diag").payload
        np.testing.assert_allclose(d, np.diag(ref), rtol=1e-15)
