"""Loader for the committed reference fixtures (tests/golden/*.npz)."""
import json
import os

import numpy as np

from oracle.port import Csr, Record

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["spec3", "inv2", "signed6", "er300", "kron8", "ba400", "sw64_katz"]


class Case:
    def __init__(self, name):
        self.name = name
        self.z = np.load(os.path.join(HERE, f"{name}.npz"))
        z = self.z
        self.n = int(z["n"])
        self.gamma = float(z["gamma"])
        self.a = Csr(self.n, z["row_ptr"], z["col_ids"], z["vals"], z["csc_ptr"], z["csc_rows"], z["csc_vals"])
        self.sa = self.a.scaled(self.gamma)
        self.runs = json.loads(str(z["runs_json"]))
        self.symmetric = bool(z["symmetric"])

    def record(self, j):
        p = f"r{j}_"
        return Record(self.z[p + "walk_pre"], self.z[p + "walk_off"], self.z[p + "entries"].astype(np.int64))

    def __getitem__(self, k):
        return self.z[k]


def load(name):
    return Case(name)


def kats():
    with open(os.path.join(HERE, "kats.json")) as fh:
        return json.load(fh)
