"""Loader for the golden vectors in tests/golden (generated from the reference)."""
import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names(prefix):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


class Case:
    def __init__(self, name):
        self.name = name
        self.a = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        with open(os.path.join(GOLDEN, name + ".json")) as fh:
            self.meta = json.load(fh)

    def __getitem__(self, k):
        return self.a[k]

    # --- inputs -------------------------------------------------------------
    @property
    def p_loc(self):
        return np.column_stack([self.a["in_p_xyz"].reshape(-1, 3), self.a["in_p_t"]])

    @property
    def field(self):
        a = self.a
        return (tuple(int(v) for v in a["in_f_dims"]), a["in_f_origin"], a["in_f_spacing"],
                a["in_f_times"], a["in_f_values"])

    @property
    def n_field(self):
        return int(self.a["in_f_values"].size)

    @property
    def extent(self):
        e = self.meta["extent"]
        return (np.array([e["x"][0], e["y"][0], e["z"][0], e["t"][0]]),
                np.array([e["x"][1], e["y"][1], e["z"][1], e["t"][1]]))

    @property
    def params(self):
        return self.meta["params"]
