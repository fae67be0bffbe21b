"""Golden fixtures for the posterior summaries, made by RUNNING THE REFERENCE's
tissuemix.analysis (reference analysis.py:58-188) on seeded inputs.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_kde_golden.py

Inputs are regenerated in the tests from the recipes below (numpy default_rng seeds,
or the posterior-draw goldens post_*.npz); tests/golden/kde/expected.npz holds what the
reference returned.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, ".."))
from tissuemix import analysis  # noqa: E402  (the reference)

from kde_cases import CASES, SUMMARY_CASES, inputs, summary_inputs  # noqa: E402


def main():
    out = {}
    meta = {}
    for name, c in CASES.items():
        x = inputs(c)
        kde = analysis.kde_fit(x, c.get("bw"))
        out[f"{name}/bandwidth"] = np.float64(kde.bandwidth)
        n = c.get("grid", 512)
        lo, hi = c.get("lo"), c.get("hi")
        mode, multi = analysis.kde_mode(kde, n=n, lo=lo, hi=hi)
        out[f"{name}/mode"] = np.float64(mode)
        out[f"{name}/multimodal"] = np.bool_(multi)
        g = analysis.kde_grid(kde, lo=lo, hi=hi, n=n)
        out[f"{name}/grid_x"] = g.x
        out[f"{name}/grid_density"] = g.density
        q = np.linspace(float(x.min()) - 1.0, float(x.max()) + 1.0, 97)
        out[f"{name}/density_q"] = analysis.kde_density(kde, q)
        meta[name] = {"mode": mode, "multimodal": multi}
    for name, c in SUMMARY_CASES.items():
        s = summary_inputs(c, HERE)
        rep = analysis.summarize(s, c.get("bw"))
        out[f"{name}/report"] = np.array(json.dumps(rep))
        meta[name] = rep
    np.savez(os.path.join(HERE, "kde", "expected.npz"), **out)
    print(json.dumps(meta, indent=1)[:3000])


if __name__ == "__main__":
    main()
