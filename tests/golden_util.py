"""Loader for tests/golden (vectors produced by the reference itself, see
tests/golden/make_golden.py)."""
import json
import os

import numpy as np

_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Case:
    def __init__(self, meta, arrays):
        self.meta = meta
        self.name = meta["name"]
        self.algo = meta["algo"]
        self.n = meta["n"]
        self.undirected = meta["undirected"]
        self.params = meta["params"]
        p = self.name + "/"
        self.rp = arrays[p + "rp"]
        self.col = arrays[p + "col"]
        self.w = arrays[p + "w"] if meta["weighted"] else None
        self.out = {k: arrays[p + k] for k in meta["outputs"]}

    def __repr__(self):
        return f"Case({self.name})"


class Golden:
    def __init__(self):
        with open(os.path.join(_DIR, "manifest.json")) as f:
            self.manifest = json.load(f)
        z = np.load(os.path.join(_DIR, "golden.npz"))
        arrays = {k: z[k] for k in z.files}
        self.cases = [Case(m, arrays) for m in self.manifest["cases"]]

    def by_algo(self, algo):
        return [c for c in self.cases if c.algo == algo]


def case_ids(algo):
    with open(os.path.join(_DIR, "manifest.json")) as f:
        return [c["name"] for c in json.load(f)["cases"] if c["algo"] == algo]
