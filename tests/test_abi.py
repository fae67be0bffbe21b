"""The C-ABI library loads and exports every symbol include/cavi.h declares (no GPU needed)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cavi.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cv_[a-z_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ("cv_dataset_create", "cv_dataset_generate", "cv_init", "cv_step", "cv_elbo", "cv_fit",
                 "cv_materialize", "cv_last_error"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    from paper_2401_10068_b200 import _lib

    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) <= set(_lib.EXPORTS)
    assert lib.cv_abi_version() == 1


def test_ctypes_layout_matches_c(tmp_path):
    """sizeof/offsetof of the ABI structs as gcc sees them == the ctypes mirror."""
    from paper_2401_10068_b200 import _lib

    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stddef.h>\n#include <stdio.h>\n#include "cavi.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu\\n\", sizeof(cv_state), sizeof(cv_hyper),"
        " offsetof(cv_state, gen_e_rho), offsetof(cv_state, resid), offsetof(cv_hyper, Lambda0));return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(_lib.CvState), ctypes.sizeof(_lib.CvHyper), _lib.CvState.gen_e_rho.offset,
            _lib.CvState.resid.offset, _lib.CvHyper.Lambda0.offset]
    assert got == want


def test_product_has_no_cpu_fallback(monkeypatch, tmp_path):
    """Without the CUDA library the engine refuses to load instead of computing on the CPU."""
    from paper_2401_10068_b200 import _lib

    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.load(str(tmp_path / "missing.so"))
    src = open(os.path.join(ROOT, "paper_2401_10068_b200", "vb.py")).read()
    assert "oracle" not in src


def test_status_codes_match_header():
    """_lib's exception mapping uses the header's status values (cavi.h enum)."""
    import re

    from paper_2401_10068_b200 import _lib

    with open(os.path.join(ROOT, "include", "cavi.h")) as fh:
        text = fh.read()
    codes = {m.group(1): int(m.group(2)) for m in re.finditer(r"(CV_(?:OK|ERR_\w+))\s*=\s*(\d+)", text)}
    want = {"CV_OK": _lib.OK, "CV_ERR_NUMERIC": _lib.ERR_NUMERIC, "CV_ERR_NONFINITE": _lib.ERR_NONFINITE,
            "CV_ERR_ARG": _lib.ERR_ARG, "CV_ERR_CUDA": _lib.ERR_CUDA, "CV_ERR_IMPROPER": _lib.ERR_IMPROPER,
            "CV_ERR_FORMAT": _lib.ERR_FORMAT, "CV_ERR_PEER": _lib.ERR_PEER, "CV_ERR_SINGULAR": _lib.ERR_SINGULAR}
    assert codes == want
