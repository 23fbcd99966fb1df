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
