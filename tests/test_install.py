"""install() rebinds the reference's module attributes (the CLI's call sites, cli.py:238/386)
to the engine.  Needs the reference importable (this container only; skipped elsewhere)."""

import importlib
import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")
def test_install_rebinds_vb_and_em():
    sys.path.insert(0, REF_SRC)
    try:
        ref_vb = importlib.import_module("tissuemix.vb")
        ref_em = importlib.import_module("tissuemix.em")
        ref_linalg = importlib.import_module("tissuemix.linalg")
        saved = {m: dict(vars(m)) for m in (ref_vb, ref_em)}
        from paper_2401_10068_b200 import em, linalg, vb

        saved_err = (linalg.NumericError, linalg.BatchItemError)
        try:
            vb.install()
            for name in ("vb_init", "vb_step", "vb_elbo", "vb_fit", "vb_posterior_sample"):
                assert getattr(ref_vb, name) is getattr(vb, name)
            for name in ("em_step", "em_fit"):
                assert getattr(ref_em, name) is getattr(em, name)
            assert linalg.NumericError is ref_linalg.NumericError
        finally:
            for m, d in saved.items():
                for k, v in d.items():
                    setattr(m, k, v)
            linalg.NumericError, linalg.BatchItemError = saved_err
    finally:
        sys.path.remove(REF_SRC)
