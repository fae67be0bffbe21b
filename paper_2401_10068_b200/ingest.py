"""Dataset files on the GPU: drop-ins for the reference's `cli.read_dataset_csv` /
`cli.write_dataset_csv` (reference cli.py:47-75) + `model.transform` (model.py:174-189),
SURVEY §8(f) row 2.

The reference reads a dataset by building one Python object per row; here the file
body goes to HBM once and is parsed there (`cv_dataset_load_csv`: terminator scan,
row numbering, one thread per row converting with Python float() semantics, correctly
rounded) straight into the dataset's stream layout, so `load_dataset_csv` returns a
`DeviceDataset` ready for `vb_fit` without a host-side transform.  `read_dataset_csv`
returns the host `Dataset` the reference's reader returns (bit-identical arrays).
`write_dataset_csv` formats every value exactly as Python's repr(float) (byte-identical
files), multithreaded in native code.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib, model
from ._lib import UsageError

__all__ = ["UsageError", "load_dataset_csv", "load_dataset_npz", "read_dataset_csv", "read_dataset_npz",
           "write_dataset_csv", "write_dataset_npz"]


def _open_check(path) -> bytes:
    path = os.fspath(path)
    with open(path, "rb"):  # the reference's open() errors (FileNotFoundError, ...) first
        pass
    return path.encode()


def load_dataset_csv(path, storage: str = "f64", device: int | None = None) -> model.DeviceDataset:
    """Parse a dataset CSV (header r,d_1,...,d_N) on the GPU into an HBM-resident dataset."""
    p = _open_check(path)
    h, n = C.c_void_p(), C.c_int32()
    _lib.check(_lib.lib().cv_dataset_load_csv(p, model._STORAGE[storage],
                                              _lib.default_device() if device is None else device,
                                              C.byref(h), C.byref(n)))
    return model.DeviceDataset(h.value, n.value)


def read_dataset_csv(path) -> model.Dataset:
    """The reference's reader (cli.py:58-75): the working-transform Dataset on the host.  The
    parsed HBM stream stays attached to it (vb.keep_resident), so the vb_fit that follows
    (cli._fit_vb, cli.py:235-268) starts from it instead of uploading the arrays again."""
    from . import vb  # noqa: PLC0415

    dd = load_dataset_csv(path)
    ds = dd.to_host()
    vb.keep_resident(ds, dd)
    return ds


def write_dataset_csv(path, ds, threads: int = 0) -> None:
    """The reference's writer (cli.py:47-56), byte-identical output."""
    if isinstance(ds, model.DeviceDataset):
        r, mu, D = ds.download()
    else:
        r = np.ascontiguousarray(ds.r, dtype=np.float64)
        mu = np.ascontiguousarray(ds.mu, dtype=np.float64)
        D = np.ascontiguousarray(np.atleast_2d(ds.D), dtype=np.float64)
        if D.shape[0] != r.shape[0]:
            D = D.reshape(r.shape[0], -1)
    V, d = D.shape
    _lib.check(_lib.lib().cv_write_dataset_csv(os.fspath(path).encode(), _lib.dptr(r), _lib.dptr(mu), _lib.dptr(D),
                                               V, d, int(threads)))


# ---------------------------------------------------------------- binary (.npz) dataset files
def write_dataset_npz(path, ds) -> None:
    """The Dataset's working arrays r (V,), mu (V,), D (V, d) as an uncompressed np.savez file
    (any numpy reads it back with np.load); the fast path for datasets too large for CSV."""
    if isinstance(ds, model.DeviceDataset):
        r, mu, D = ds.download()
    else:
        r, mu, D = (np.ascontiguousarray(a, dtype=np.float64) for a in (ds.r, ds.mu, np.atleast_2d(ds.D)))
    with open(os.fspath(path), "wb") as fh:  # an open file: np.savez does not append ".npz"
        np.savez(fh, r=r, mu=mu, D=D)


def npz_info(path):
    """(V, d) of a dataset .npz, validated on the host (no GPU needed)."""
    p = _open_check(path)
    V, d = C.c_int64(), C.c_int32()
    _lib.check(_lib.lib().cv_npz_probe(p, C.byref(V), C.byref(d)))
    return V.value, d.value


def load_dataset_npz(path, storage: str = "f64", device: int | None = None) -> model.DeviceDataset:
    """A dataset .npz (write_dataset_npz / np.savez of r, mu, D) streamed into HBM."""
    p = _open_check(path)
    h, n = C.c_void_p(), C.c_int32()
    _lib.check(_lib.lib().cv_dataset_load_npz(p, model._STORAGE[storage],
                                              _lib.default_device() if device is None else device,
                                              C.byref(h), C.byref(n)))
    return model.DeviceDataset(h.value, n.value)


def read_dataset_npz(path) -> model.Dataset:
    """The host Dataset of a dataset .npz, its HBM stream attached (as read_dataset_csv)."""
    from . import vb  # noqa: PLC0415

    dd = load_dataset_npz(path)
    ds = dd.to_host()
    vb.keep_resident(ds, dd)
    return ds
