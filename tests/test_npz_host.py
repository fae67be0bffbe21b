"""Binary dataset files: the host-side validation of the np.savez container (cv_npz_probe) --
runs without a GPU.  The device load is checked in tests/test_gpu_ingest.py."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _ds(V=1000, d=3, seed=0):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(V), rng.integers(0, 2, V).astype(float), rng.integers(-1, 2, (V, d)).astype(float)


def test_probe_reads_what_np_savez_writes(tmp_path):
    from paper_2401_10068_b200 import ingest, model

    r, mu, D = _ds()
    p = tmp_path / "ds.npz"
    ingest.write_dataset_npz(p, model.Dataset(r=r, mu=mu, D=D, n_networks=4))
    assert ingest.npz_info(p) == (1000, 3)
    z = np.load(p)  # and it is an ordinary numpy file
    assert np.array_equal(z["r"], r) and np.array_equal(z["D"], D)


@pytest.mark.parametrize("case", ["compressed", "missing", "dtype", "fortran", "shape", "not_zip"])
def test_probe_rejects_other_files(tmp_path, case):
    from paper_2401_10068_b200 import ingest

    r, mu, D = _ds()
    p = str(tmp_path / f"{case}.npz")
    with open(p, "wb") as fh:
        if case == "compressed":
            np.savez_compressed(fh, r=r, mu=mu, D=D)
        elif case == "missing":
            np.savez(fh, r=r, D=D)
        elif case == "dtype":
            np.savez(fh, r=r.astype(np.float32), mu=mu, D=D)
        elif case == "fortran":
            np.savez(fh, r=r, mu=mu, D=np.asfortranarray(D))
        elif case == "shape":
            np.savez(fh, r=r, mu=mu[:-1], D=D)
        else:
            fh.write(b"r,d_1,d_2\\n0.5,1,0\\n")
    with pytest.raises(ingest.UsageError):
        ingest.npz_info(p)


def test_probe_missing_file_raises_like_open(tmp_path):
    from paper_2401_10068_b200 import ingest

    with pytest.raises(FileNotFoundError):
        ingest.npz_info(tmp_path / "nope.npz")
