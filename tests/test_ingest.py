"""Graph ingest against the reference's own outputs
(tests/golden/ingest/, made by make_ingest_golden.py from the reference's
load_graph / symmetrize_digraph): parsers, filter order, id compaction,
Eq. 25 symmetrization and the ParseError messages.  The filters run with
torch on the CPU here and on the GPU in the -m gpu variant."""
import json
import os

import numpy as np
import pytest

from paper_2308_01037_b200.errors import McfunmError, ParseError
from paper_2308_01037_b200.ingest import GraphSource, load_graph, simple_graph_from_edges, symmetrize_digraph

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ingest")
GOLD = json.load(open(os.path.join(HERE, "ingest_golden.json")))
CASES = sorted(k for k in GOLD if "|" in k)


def _check(device):
    for key in CASES:
        name, directed, drop_isolated = key.split("|")
        fmt = "edgelist" if name.endswith(".txt") else ("matrix-market" if "general" in name else "mtx")
        ref = GOLD[key]
        a = load_graph(GraphSource(os.path.join(HERE, name), fmt, directed=directed == "True",
                                   drop_isolated=drop_isolated == "True"), device=device)
        assert a.n == ref["n"], key
        assert np.array_equal(a.csr.indptr, ref["indptr"]), key
        assert np.array_equal(a.csr.indices, ref["indices"]), key
        assert np.array_equal(a.csr.data, ref["data"]), key
        assert a.symmetric_hint == ref["symmetric_hint"], key
        if ref["original_ids"] is None:
            assert a.original_ids is None, key
        else:
            assert np.array_equal(a.original_ids, ref["original_ids"]), key
        # the CSC view holds the same triples
        assert np.array_equal(a.csc.toarray(), a.csr.toarray())
        if "sym" in ref:
            s = symmetrize_digraph(a)
            assert s.n == ref["sym"]["n"] and s.meta["symmetrized_blocks"] == ref["sym"]["symmetrized_blocks"]
            assert np.array_equal(s.csr.indptr, ref["sym"]["indptr"])
            assert np.array_equal(s.csr.indices, ref["sym"]["indices"])
            assert s.symmetric_hint and (abs(s.csr - s.csr.T)).nnz == 0


def test_load_graph_matches_reference_cpu():
    _check("cpu")


@pytest.mark.gpu
def test_load_graph_matches_reference_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    _check("cuda")


@pytest.mark.parametrize("name", ["bad_cols.txt", "bad_neg.txt", "bad_header.mtx"])
def test_parse_errors_match_reference(name):
    ref = GOLD[name]
    fmt = "mtx" if name.endswith(".mtx") else "edgelist"
    with pytest.raises(McfunmError) as exc:
        load_graph(GraphSource(os.path.join(HERE, name), fmt), device="cpu")
    assert type(exc.value).__name__ == ref["error"]
    assert str(exc.value).replace(HERE + os.sep, "") == ref["message"]


def test_filter_edge_cases():
    with pytest.raises(McfunmError):  # only loops -> empty
        simple_graph_from_edges([1, 2], [1, 2], device="cpu")
    with pytest.raises(McfunmError, match="duplicate"):
        simple_graph_from_edges([0, 0], [1, 1], directed=True, drop_duplicates=False, device="cpu")
    a = simple_graph_from_edges([0, 5], [5, 0], directed=True, drop_isolated=False, device="cpu")
    assert a.n == 6 and a.nnz == 2 and a.original_ids is None
    with pytest.raises(ParseError):
        load_graph(GraphSource(os.path.join(HERE, "bad_cols.txt")), device="cpu")
    with pytest.raises(McfunmError, match="not found"):
        load_graph(GraphSource(os.path.join(HERE, "missing.txt")), device="cpu")


@pytest.mark.gpu
def test_filter_kernels_match_torch_path():
    """mcf_edges_to_csr / mcf_csr_compact (GPU) against the torch path (CPU) on
    random edge lists with loops, duplicates, both directions and isolated
    ids: identical CSR, ids and errors."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2308_01037_b200.errors import ArgumentError
    rng = np.random.default_rng(11)
    for trial in range(6):
        n = int(rng.integers(50, 5000))
        m = int(rng.integers(10, 20 * n))
        u = rng.integers(0, n, m)
        v = np.where(rng.random(m) < 0.05, u, rng.integers(0, n, m))  # some loops
        u[: m // 10] = (u[: m // 10] % 7) * 3  # a few hubs
        for directed in (False, True):
            for iso in (True, False):
                a = simple_graph_from_edges(u, v, directed=directed, drop_isolated=iso, device="cpu")
                b = simple_graph_from_edges(u, v, directed=directed, drop_isolated=iso, device="cuda")
                assert a.n == b.n
                assert np.array_equal(a.csr.indptr, b.csr.indptr) and np.array_equal(a.csr.indices, b.csr.indices)
                assert (a.original_ids is None) == (b.original_ids is None)
                if a.original_ids is not None:
                    assert np.array_equal(a.original_ids, b.original_ids)
        with pytest.raises(ArgumentError):
            simple_graph_from_edges(np.r_[u, u[:1]], np.r_[v, v[:1]], drop_duplicates=False, device="cuda")


@pytest.mark.gpu
def test_generator_kernels():
    """R-MAT and Chung-Lu by the library kernels: symmetric, sorted rows, no
    loops or duplicates, and the same degree statistics as the torch recipes
    (same rule, different random streams)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from scipy import sparse
    from paper_2308_01037_b200 import graphs
    for kind in ("rmat", "chunglu"):
        if kind == "rmat":
            n, rp, ci = graphs.rmat_device(16, 16, seed=2)
            n2, rp2, ci2 = graphs.rmat_torch(16, 16, seed=2)
        else:
            n, rp, ci = graphs.chung_lu_device(200_000, seed=2)
            n2, rp2, ci2 = graphs.chung_lu_torch(200_000, seed=2)
        rp, ci = rp.cpu().numpy(), ci.cpu().numpy()
        a = sparse.csr_array((np.ones(ci.size), ci, rp), shape=(n, n))
        assert abs(a - a.T).nnz == 0
        rows = np.repeat(np.arange(n), np.diff(rp))
        assert not np.any(rows == ci)
        same_row = rows[1:] == rows[:-1]
        assert np.all(ci[1:][same_row] > ci[:-1][same_row])  # sorted, no duplicates
        nnz2 = int(ci2.numel())
        assert abs(ci.size - nnz2) < 0.01 * nnz2, (kind, ci.size, nnz2)
        d1, d2 = np.diff(rp).max(), int((rp2[1:] - rp2[:-1]).max())
        assert abs(d1 - d2) < 0.15 * d2, (kind, d1, d2)
