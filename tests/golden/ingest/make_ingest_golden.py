"""Golden outputs of the reference's graph ingest (sparsemat.py:149-335) on
small files in this directory.  Run in the build container (the reference is
importable there, never on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/ingest/make_ingest_golden.py
"""
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def write_inputs():
    rng = np.random.default_rng(7)
    with open(os.path.join(HERE, "el_small.txt"), "w") as fh:
        fh.write("# comment line\n% another comment\n\n")
        for _ in range(60):
            u, v = rng.integers(0, 40, 2)
            fh.write(f"{u} {v}\n" if rng.random() > 0.2 else f"  {u}\t{v}  extra\n")
        fh.write("3 3\n5 7\n5 7\n100 101\n")  # a loop, a duplicate, and ids forming an isolated gap
    with open(os.path.join(HERE, "mm_general.mtx"), "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n% c\n12 12 9\n")
        for i, j, x in [(1, 2, 1.5), (2, 1, 1.0), (3, 4, 0.0), (5, 5, 2.0), (6, 7, -1.0),
                        (7, 6, 1.0), (12, 1, 3.0), (4, 9, 1e-3), (9, 4, 2e2)]:
            fh.write(f"{i} {j} {x}\n")
    with open(os.path.join(HERE, "mm_sym_pattern.mtx"), "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate pattern symmetric\n10 10 6\n2 1\n3 1\n4 4\n7 5\n9 8\n10 9\n")
    with open(os.path.join(HERE, "bad_cols.txt"), "w") as fh:
        fh.write("1 2\n3\n")
    with open(os.path.join(HERE, "bad_neg.txt"), "w") as fh:
        fh.write("1 2\n-3 4\n")
    with open(os.path.join(HERE, "bad_header.mtx"), "w") as fh:
        fh.write("%%NotMM matrix coordinate real general\n2 2 1\n1 1 1\n")


def main():
    from mcfunm.errors import McfunmError
    from mcfunm.sparsemat import GraphSource, load_graph, symmetrize_digraph
    write_inputs()
    cases = {}
    for name, fmt in (("el_small.txt", "edgelist"), ("mm_general.mtx", "matrix-market"),
                      ("mm_sym_pattern.mtx", "mtx")):
        for directed in (False, True):
            for drop_isolated in (True, False):
                key = f"{name}|{directed}|{drop_isolated}"
                try:
                    a = load_graph(GraphSource(os.path.join(HERE, name), fmt, directed=directed,
                                               drop_isolated=drop_isolated))
                except McfunmError as exc:
                    cases[key] = {"error": type(exc).__name__}
                    continue
                rec = {"n": int(a.n), "indptr": a.csr.indptr.tolist(), "indices": a.csr.indices.tolist(),
                       "data": a.csr.data.tolist(), "symmetric_hint": bool(a.symmetric_hint),
                       "original_ids": None if a.original_ids is None else a.original_ids.tolist()}
                if directed:
                    s = symmetrize_digraph(a)
                    rec["sym"] = {"n": int(s.n), "indptr": s.csr.indptr.tolist(), "indices": s.csr.indices.tolist(),
                                  "symmetrized_blocks": s.meta.get("symmetrized_blocks")}
                cases[key] = rec
    for name, fmt in (("bad_cols.txt", "edgelist"), ("bad_neg.txt", "edgelist"), ("bad_header.mtx", "mtx")):
        try:
            load_graph(GraphSource(os.path.join(HERE, name), fmt))
            cases[name] = {"error": None}
        except McfunmError as exc:
            cases[name] = {"error": type(exc).__name__, "message": str(exc).replace(HERE + os.sep, "")}
    with open(os.path.join(HERE, "ingest_golden.json"), "w") as fh:
        json.dump(cases, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
