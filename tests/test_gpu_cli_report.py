"""`tissuemix fit --method vb` end to end on the drop-in vs the reference on the CPU (SURVEY
8(a) row a19: cli._fit_vb, cli.py:235-268): the CLI is the reference's own (baseline/_ref);
one process runs it unchanged, the other after vb.install() (vb_fit, vb_posterior_sample with
the default 10,000 draws, summarize and the dataset reader on the B200).  report.json,
trace.csv and samples.csv must agree."""

import csv
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

SCRIPT = """
import sys
sys.path[:0] = [{ref!r}, {root!r}]
if {install}:
    from paper_2401_10068_b200 import vb
    vb.install()
from tissuemix import cli
assert cli.main(["synth", "--genes", "400", "--true-k", "0.1,0.3", "--rho", "100", "--lambda", "default",
                 "--seed", "5", "--out", {ds!r}]) == 0
sys.exit(cli.main(["fit", "--method", "vb", "--dataset", {ds!r}, "--out", {out!r}, "--seed", "1"]))
"""


def run_cli(tmp, install):
    out = os.path.join(tmp, "gpu" if install else "cpu")
    code = SCRIPT.format(ref=REF, root=ROOT, install=install, ds=os.path.join(tmp, f"ds{int(install)}.csv"), out=out)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return out


def numbers(x, path=""):
    """Flatten a JSON document into {path: number}; strings must match exactly."""
    out = {}
    if isinstance(x, dict):
        for k, v in x.items():
            out.update(numbers(v, f"{path}/{k}"))
    elif isinstance(x, list):
        for i, v in enumerate(x):
            out.update(numbers(v, f"{path}[{i}]"))
    elif isinstance(x, (int, float)) and not isinstance(x, bool):
        out[path] = float(x)
    else:
        out[path] = x
    return out


def read_csv(path):
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    return rows[0], np.array(rows[1:], dtype=float)


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tissuemix")), reason="baseline/_ref not installed")
def test_cli_fit_vb_report_matches_the_reference_run(tmp_path):
    cpu = run_cli(str(tmp_path), install=False)
    gpu = run_cli(str(tmp_path), install=True)
    a = numbers(json.load(open(os.path.join(cpu, "report.json"))))
    b = numbers(json.load(open(os.path.join(gpu, "report.json"))))
    assert a.keys() == b.keys()
    timing = [k for k in a if "wall" in k or "seconds" in k or "elapsed" in k or "time" in k.lower()]
    worst = 0.0
    for k in a:
        if k in timing or "dataset" in k or k.endswith("/out"):
            continue
        if isinstance(a[k], float):
            # posterior summaries of 10,000 draws: the draws themselves agree to ~1e-12 (same
            # Philox stream, states equal to ~1e-13), so KDE modes and quantiles do as well
            rel = abs(a[k] - b[k]) / max(abs(a[k]), 1e-300)
            worst = max(worst, rel if abs(a[k]) > 1e-12 else abs(a[k] - b[k]))
        else:
            assert a[k] == b[k], k
    assert worst < 1e-9, worst
    ha, ta = read_csv(os.path.join(cpu, "trace.csv"))
    hb, tb = read_csv(os.path.join(gpu, "trace.csv"))
    assert ha == hb and ta.shape == tb.shape  # same sweep count to the stop rule
    np.testing.assert_allclose(tb[:, 1], ta[:, 1], rtol=1e-9)  # the bound
    sa, xa = read_csv(os.path.join(cpu, "samples.csv"))
    sb, xb = read_csv(os.path.join(gpu, "samples.csv"))
    assert sa == sb and xa.shape == xb.shape == (10000, xa.shape[1])
    np.testing.assert_allclose(xb, xa, rtol=1e-9, atol=1e-12)
