"""Pins the CPU oracle (oracle/port.py) to the real reference's outputs.

Every array here was produced by /root/reference's own code (see
tests/golden/make_golden.py); equality is bit-for-bit."""
import numpy as np
import pytest

from oracle import port
from tests import golden_io

CASES = golden_io.CASES


@pytest.mark.parametrize("name", CASES)
def test_tables_bitwise(name):
    c = golden_io.load(name)
    t = port.transition_tables(c.sa)
    for mine, ref in [(t.row_cdf, "m_row_cdf"), (t.cdf_key, "m_cdf_key"), (t.step_ratio, "m_step_ratio"),
                      (t.rsum, "m_row_abs_sum"), (t.col_norms, "m_col_norms"), (t.init_prob, "m_init_prob")]:
        assert np.array_equal(mine, c[ref]), ref


@pytest.mark.parametrize("name", CASES)
def test_allocation_bitwise(name):
    c = golden_io.load(name)
    t = port.transition_tables(c.sa)
    for ns in (1, 7, 1000, 12345, 10 * c.n + 3):
        assert np.array_equal(port.allocate(t, ns), c[f"ni_{ns}"])
        assert port.allocate(t, ns).sum() == ns  # SPEC.md:316 budget conservation


@pytest.mark.parametrize("name", CASES)
def test_estimates_and_streams_bitwise(name):
    c = golden_io.load(name)
    for j, r in enumerate(c.runs):
        p = f"r{j}_"
        if r["mode"] == "action":
            run = port.funm_action(c.sa, r["tag"], c[p + "v"], r["n_walks"], r["cutoff"], r["max_steps"],
                                   r["seed"], record=True)
            assert np.array_equal(run.payload, c[p + "y"])
            assert np.array_equal(run.aux["q"], c[p + "q"])
        else:
            run = port.funm_diag(c.sa, r["tag"], r["n_walks"], r["cutoff"], r["max_steps"], r["seed"], record=True)
            assert np.array_equal(run.payload, c[p + "d"])
        assert np.array_equal(run.ni, c[p + "ni"])
        assert run.emissions == int(c[p + "emissions"])
        assert run.truncated == int(c[p + "truncated"])
        assert np.array_equal(run.record.walk_off, c[p + "walk_off"])
        assert np.array_equal(run.record.entries, c[p + "entries"].astype(np.int64))


@pytest.mark.parametrize("name", ["spec3", "inv2", "signed6", "er300", "ba400"])
def test_replay_reproduces_reference(name):
    """A recorded entry stream alone determines the estimate (replay semantics the
    device kernels implement); summation order differs -> 1e-12 relative."""
    c = golden_io.load(name)
    for j, r in enumerate(c.runs):
        p = f"r{j}_"
        rec = c.record(j)
        if r["mode"] == "action":
            out = port.replay(c.sa, r["tag"], rec, r["max_steps"], r["cutoff"], "action", c[p + "v"])
            ref = c[p + "y"]
        else:
            out = port.replay(c.sa, r["tag"], rec, r["max_steps"], r["cutoff"], "diag")
            ref = c[p + "d"]
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-300)


def test_spec_kats_on_oracle():
    k = golden_io.kats()
    a3 = port.Csr.from_dense([[0, 1, 1], [1, 0, 0], [1, 0, 0]])
    t3 = port.transition_tables(a3)
    assert t3.row_cdf.tolist() == k["spec257_row_cdf"]
    assert t3.col_norms.tolist() == k["spec257_col_norms"]
    assert t3.init_prob.tolist() == k["spec257_init_prob"]
    assert port.allocate(t3, 1000).tolist() == k["spec268_alloc"] == [414, 293, 293]
    assert port.largest_remainder(np.array([0.9, 0.1]), 1).tolist() == k["spec269_alloc"] == [1, 0]
    assert port.largest_remainder(np.array([0.5, 0.5]), 10).tolist() == k["spec267_alloc"] == [5, 5]
    aw = port.Csr.from_dense([[0, 2, -1], [0, 0, 0], [5, 0, 0]])
    assert port.transition_tables(aw).step_ratio.tolist() == k["spec258_step_ratio"]
    assert port.row_abs_sums(aw).tolist() == k["spec80_row_abs_sums"] == [3, 0, 5]
    c4 = port.Csr.from_dense(np.roll(np.eye(4), 1, 1) + np.roll(np.eye(4), -1, 1))
    assert port.gershgorin_gamma(c4, 0.85) == k["spec466_gershgorin"] == 0.425
    s1 = port.transition_tables(port.Csr.from_dense([[0.5]]))
    assert list(port.single_walk(s1, "exponential", 0, 100, 0.1, lambda *x: None)) == k["spec287_run_walk"]
    assert list(port.batch_walks(s1, 0, 1, 100, 0.1, port.column_stream(0, 0), lambda *x: None)) == k["spec287_batch"]
    cw = port.Csr.from_dense([[0, 1], [1, 0]])
    tcw = port.transition_tables(cw)
    assert list(port.batch_walks(tcw, 0, 5, 17, 0.5, port.column_stream(0, 0), lambda *x: None)) == k["spec288_batch"]
    assert list(port.single_walk(tcw, "exponential", 0, 17, 0.5, lambda *x: None)) == k["spec288_run_walk"]
    np.testing.assert_array_equal(port.dense_funm(cw.scaled(0.1), "exponential", 30), k["spec447_cosh"])
    np.testing.assert_array_equal(port.dense_funm(cw.scaled(0.5), "resolvent", 60), k["spec448_resolvent"])
    np.testing.assert_array_equal(port.cg_solve(cw, 0.5, np.ones(2)), k["spec457_cg"])
    np.testing.assert_array_equal(port.zeta_prefix("exponential", 32), k["prefix_exp_32"])


@pytest.mark.parametrize("m", [1, 5, 28])
def test_truncation_mapping_kat(m):
    """on gamma*[[0,1],[1,0]] every walk is deterministic; with
    max_steps=M and W_c=1e-300 both estimators equal dense_funm(terms=M+1)."""
    for g in (0.5, 0.9):
        a = port.Csr.from_dense([[0, g], [g, 0]])
        ref = port.dense_funm(a, "exponential", m + 1)
        d = port.funm_diag(a, "exponential", 64, 1e-300, m, 0).payload
        y = port.funm_action(a, "exponential", np.ones(2), 64, 1e-300, m, 0).payload
        np.testing.assert_allclose(d, np.diag(ref), rtol=4e-15)
        np.testing.assert_allclose(y, ref.sum(1), rtol=4e-15)
