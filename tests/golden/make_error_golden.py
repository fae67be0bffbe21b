"""Error goldens made by RUNNING THE REFERENCE (tissuemix) on inputs that drive its linear-
algebra guards (row a11: linalg.py:111-153 adjugate |det| guard, 279-298 jitter retry):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_error_golden.py

Writes tests/golden/errors.json: per case the recipe (dataset = random_profiles + synth_generate
on RngStream(seed), rebuilt bit-exactly by oracle/philox.generate) and the exception class and
message the reference's vb_fit raises."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from tissuemix import model, vb  # noqa: E402  (the reference)
from tissuemix.samplers import RngStream  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def case(seed, V, N, K, lam, rho, lambda0_scale):
    rng = RngStream(seed)
    truth = model.ModelParams(K=np.asarray(K, float), Lam=np.asarray(lam, float), rho=rho)
    ds = model.synth_generate(rng, truth, model.random_profiles(rng, V, N))
    d = N - 1
    hp = model.HyperParams(a0=0.5, b0=0.5, q0=0.001, n0=1, K0=np.full(d, 1 / 3), Lambda0=lambda0_scale * np.eye(d))
    try:
        vb.vb_fit(ds, hp)
        out = {"error": None}
    except Exception as e:  # noqa: BLE001
        out = {"error": type(e).__name__, "message": str(e)}
    out["recipe"] = {"seed": seed, "V": V, "N": N, "K": list(K), "Lam": np.asarray(lam).tolist(), "rho": rho,
                     "lambda0_scale": lambda0_scale}
    return out


def main():
    lam2 = np.linalg.inv(model.REFERENCE_LAMBDA_INV)
    cases = {
        # |det Lambda0| = 1e-320 < 1e-300: vb_init's per-gene adjugate inverse raises (no retry there)
        "tiny_lambda0_n3": case(3, 5, 3, [0.1, 0.3], lam2, 100.0, 1e-160),
        "tiny_lambda0_n4": case(4, 7, 4, [0.2, 0.2, 0.2], 100.0 * np.eye(3), 100.0, 1e-110),
        "tiny_lambda0_n2": case(2, 6, 2, [0.3], [[100.0]], 100.0, 1e-305),
    }
    with open(os.path.join(HERE, "errors.json"), "w") as fh:
        json.dump(cases, fh, indent=1, sort_keys=True)
    for k, v in cases.items():
        print(k, v["error"], v.get("message"))


if __name__ == "__main__":
    main()
