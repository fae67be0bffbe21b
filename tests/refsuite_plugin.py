"""pytest plugin (-p refsuite_plugin): run the reference's own test suite with the drop-in
installed.  Before the reference's test modules are collected, vb.install() rebinds
tissuemix.vb / em / analysis and the CLI's dataset readers to the CUDA engine, so every
`vb.vb_fit(...)`, `cli.main([...])` etc. in those tests runs on the B200."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import tissuemix  # noqa: F401  (from baseline/_ref, on PYTHONPATH)

    from paper_2401_10068_b200 import vb

    vb.install()
    config._refsuite_installed = True
