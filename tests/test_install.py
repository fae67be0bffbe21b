"""install() rebinds the reference's module attributes (the CLI's call sites, cli.py:238/386)
to the engine.  Needs the reference importable (this container only; skipped elsewhere)."""

import importlib
import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")
def test_install_rebinds_reference_entry_points():
    sys.path.insert(0, REF_SRC)
    try:
        ref_vb = importlib.import_module("tissuemix.vb")
        ref_em = importlib.import_module("tissuemix.em")
        ref_linalg = importlib.import_module("tissuemix.linalg")
        ref_an = importlib.import_module("tissuemix.analysis")
        ref_cli = importlib.import_module("tissuemix.cli")
        saved = {m: dict(vars(m)) for m in (ref_vb, ref_em, ref_an, ref_cli)}
        from paper_2401_10068_b200 import _lib, analysis, em, ingest, linalg, vb

        saved_usage = _lib.UsageError

        saved_err = (linalg.NumericError, linalg.BatchItemError)
        try:
            vb.install()
            for name in ("vb_init", "vb_step", "vb_elbo", "vb_fit", "vb_posterior_sample"):
                assert getattr(ref_vb, name) is getattr(vb, name)
            for name in ("em_step", "em_fit"):
                assert getattr(ref_em, name) is getattr(em, name)
            assert linalg.NumericError is ref_linalg.NumericError
            for name in ("kde_fit", "kde_density", "kde_grid", "kde_mode", "summarize"):
                assert getattr(ref_an, name) is getattr(analysis, name)
            assert ref_cli.read_dataset_csv is ingest.read_dataset_csv
            assert _lib.UsageError is ref_cli.UsageError
        finally:
            for m, d in saved.items():
                for k, v in d.items():
                    setattr(m, k, v)
            linalg.NumericError, linalg.BatchItemError = saved_err
            _lib.UsageError = ingest.UsageError = saved_usage
    finally:
        sys.path.remove(REF_SRC)
