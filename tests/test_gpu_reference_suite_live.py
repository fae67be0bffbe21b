"""The reference's OWN test suite (reference pkg/tests, installed unmodified into the
git-ignored baseline/_ref by tools/install_reference.sh) run against the drop-in on a B200:
a pytest subprocess loads tests/refsuite_plugin.py, which calls vb.install() before the
reference's modules are collected, so their `vb.vb_fit`, `em.em_fit`, `analysis.summarize`
and `cli.main([...])` calls go through the CUDA engine.

Covered: test_vb.py in full -- including the Monte-Carlo ELBO oracle
(:115-131) and the quadrature-evidence bound (:133-144) -- test_em.py, test_analysis.py,
the CLI's `fit --method vb` / `bench` paths (test_cli.py; cli.py:235-268, 382-445), and the
acceptance criteria on this path (C01, C04, C05, C08).  Every selected test must pass; the
few deselected ones are listed with the reason in DESELECT."""

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "tests")

SELECT = ["test_vb.py", "test_em.py", "test_analysis.py", "test_cli.py::TestFit", "test_cli.py::TestBench",
          "test_cli.py::TestDensity",
          "test_acceptance.py::test_c01_synthetic_recovery", "test_acceptance.py::test_c04_vb_convergence_profile",
          "test_acceptance.py::test_c05_em_ascent", "test_acceptance.py::test_c08_elbo_cross_validation"]
DESELECT = {}


def run_suite(tmp_path, select):
    xml = tmp_path / "ref.xml"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, TESTS, os.path.join(ROOT, "tests"), ROOT]))
    args = [sys.executable, "-m", "pytest", "-p", "refsuite_plugin", "-q", "-x", "--no-header", "-p", "no:cacheprovider",
            f"--junitxml={xml}", "--rootdir", TESTS, *[os.path.join(TESTS, s) for s in select]]
    for k in DESELECT:
        args += ["--deselect", os.path.join(TESTS, k)]
    out = subprocess.run(args, cwd=TESTS, env=env, capture_output=True, text=True, timeout=1800)
    return out, ET.parse(xml).getroot() if xml.exists() else None


@pytest.mark.skipif(not os.path.isdir(TESTS), reason="baseline/_ref not installed (tools/install_reference.sh)")
def test_reference_suite_passes_on_the_drop_in(tmp_path):
    out, root = run_suite(tmp_path, SELECT)
    assert root is not None, out.stdout[-3000:] + out.stderr[-3000:]
    cases = root.iter("testcase")
    failed = [f"{c.get('classname')}::{c.get('name')}" for c in cases
              if c.find("failure") is not None or c.find("error") is not None]
    n = int(sum(int(s.get("tests", 0)) for s in root.iter("testsuite")))
    assert out.returncode == 0 and not failed, "\n".join(failed) + "\n" + out.stdout[-6000:]
    assert n >= 60, f"only {n} reference tests ran"
