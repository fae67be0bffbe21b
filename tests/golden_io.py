"""Load the reference-made golden fixtures (tests/golden/*.npz) and rebuild their datasets.

Datasets are rebuilt with the oracle's bit-exact Philox generator and checked
against the sha256 the reference recorded (tests/golden/make_golden.py).
"""

from __future__ import annotations

import glob
import hashlib
import json
import os

import numpy as np

from oracle import cavi, philox

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def names(prefix=""):
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


class Golden:
    def __init__(self, name):
        self.name = name
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        self.z = {k: z[k] for k in z.files}
        self.recipe = json.loads(str(self.z["recipe"]))
        h = json.loads(str(self.z["hyper"]))
        self.hyper = cavi.Hyper(h["a0"], h["b0"], h["q0"], int(h["n0"]), np.array(h["K0"]),
                                np.array(h["Lambda0"]))
        self.fit_kw = json.loads(str(self.z["fit_kw"])) if "fit_kw" in self.z else None
        self._data = None

    def __getitem__(self, k):
        return self.z[k]

    def data(self, check=True):
        """(r, mu, D) rebuilt bit-exactly; asserts the reference's sha256."""
        if self._data is None:
            rc = self.recipe
            if rc["kind"] == "random":
                r, mu, D = philox.generate(rc["seed"], rc["V"], rc["N"], rc["K"], np.array(rc["Lam"]), rc["rho"])
            else:
                bits = np.array(rc["profiles"], dtype=float)
                mu = bits[:, -1].copy()
                D = bits[:, :-1] - mu[:, None]
                r = philox.synth(philox.Stream(rc["seed"]), rc["K"], np.array(rc["Lam"]), rc["rho"], mu, D)
            if check:
                assert sha(r) == rc["sha_r"] and sha(mu) == rc["sha_mu"] and sha(D) == rc["sha_D"], self.name
            self._data = (r, mu, D)
        return self._data
