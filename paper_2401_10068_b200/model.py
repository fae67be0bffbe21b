"""Observed-layer and prior types on both sides of the CAVI path, plus the
device-resident dataset and the on-device synthetic generator.

Mirrors the reference's `tissuemix.model` types the hot path consumes
(reference model.py:89-151, 200-221): `Dataset`, `HyperParams`,
`ModelParams`, `default_hyperparams`, `full_weights`, `REFERENCE_LAMBDA_INV`.
Reference objects are accepted anywhere these are (duck typing on
r / mu / D / n_networks and a0 / b0 / q0 / n0 / K0 / Lambda0).

`DeviceDataset` is the measurement stream resident in HBM (one upload per
dataset); `generate()` builds it directly on the GPU with the reference's
Philox4x32-10 stream layout (model.py:224-270, samplers.py:47-147), which is
how datasets of 1e8-1e9 genes are made.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib, linalg

REFERENCE_LAMBDA_INV = np.array([[0.01, 0.005], [0.005, 0.008]])


def _freeze(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    a.flags.writeable = False
    return a


@dataclass(frozen=True, eq=False)
class Dataset:
    """r (V,), mu (V,), D (V, N-1): the working transform (reference model.py:89-123)."""

    r: np.ndarray
    mu: np.ndarray
    D: np.ndarray
    n_networks: int

    def __post_init__(self):
        r = _freeze(np.atleast_1d(self.r))
        mu = _freeze(np.atleast_1d(self.mu))
        D = _freeze(np.atleast_2d(self.D))
        if r.shape[0] == 0:
            raise ValueError("empty dataset")
        if not (r.shape[0] == mu.shape[0] == D.shape[0]):
            raise ValueError("inconsistent lengths")
        if D.shape[1] != self.n_networks - 1:
            raise ValueError(f"D width {D.shape[1]} != n_networks-1 = {self.n_networks - 1}")
        object.__setattr__(self, "r", r)
        object.__setattr__(self, "mu", mu)
        object.__setattr__(self, "D", D)

    @property
    def V(self) -> int:
        return self.r.shape[0]

    @property
    def dim(self) -> int:
        return self.D.shape[1]


@dataclass(frozen=True, eq=False)
class HyperParams:
    """Prior constants (reference model.py:126-151)."""

    a0: float
    b0: float
    q0: float
    n0: int
    K0: np.ndarray
    Lambda0: np.ndarray

    def __post_init__(self):
        if not (self.a0 > 0 and self.b0 > 0 and self.q0 > 0 and self.n0 >= 1):
            raise ValueError("hyperparameters must be positive")
        K0 = _freeze(np.atleast_1d(self.K0))
        L0 = _freeze(np.atleast_2d(self.Lambda0))
        if L0.shape != (K0.shape[0], K0.shape[0]):
            raise ValueError("Lambda0 shape inconsistent with K0")
        _spd_or_raise(L0)
        object.__setattr__(self, "K0", K0)
        object.__setattr__(self, "Lambda0", L0)
        object.__setattr__(self, "n0", int(self.n0))

    @property
    def dim(self) -> int:
        return self.K0.shape[0]


@dataclass(frozen=True, eq=False)
class ModelParams:
    """One point in parameter space: K, precision Lam, rho (reference model.py:154-171)."""

    K: np.ndarray
    Lam: np.ndarray
    rho: float

    def __post_init__(self):
        K = _freeze(np.atleast_1d(self.K))
        Lam = _freeze(np.atleast_2d(self.Lam))
        if Lam.shape != (K.shape[0], K.shape[0]):
            raise ValueError("Lam shape inconsistent with K")
        if not self.rho > 0:
            raise ValueError("rho must be positive")
        _spd_or_raise(Lam)
        object.__setattr__(self, "K", K)
        object.__setattr__(self, "Lam", Lam)


def _spd_or_raise(M: np.ndarray) -> None:
    # argument validation only (the reference runs cholesky_batched here, model.py:144)
    try:
        np.linalg.cholesky(M)
    except np.linalg.LinAlgError:
        raise linalg.BatchItemError("non-positive pivot", [0]) from None


def default_hyperparams(N: int) -> HyperParams:
    """Defaults for N networks (reference model.py:200-215)."""
    if N < 2:
        raise ValueError("need at least 2 networks")
    dim = N - 1
    lam0 = np.linalg.inv(REFERENCE_LAMBDA_INV) if N == 3 else np.linalg.inv(0.01 * np.eye(dim))
    return HyperParams(a0=0.5, b0=0.5, q0=0.001, n0=1, K0=np.full(dim, 1.0 / 3.0), Lambda0=lam0)


def full_weights(K) -> np.ndarray:
    """Append the implied last weight 1 - sum(K) (reference model.py:218-221)."""
    K = np.atleast_1d(np.asarray(K, dtype=np.float64))
    return np.concatenate([K, [1.0 - K.sum()]])


# ---------------------------------------------------------------- device datasets
class DeviceDataset:
    """A measurement stream resident in HBM (handle to a `cv_dataset`).

    Holds genes [gene_lo, gene_lo + V) of a dataset of V_total genes; for a
    single-GPU dataset gene_lo = 0 and V == V_total.  Layout: x = r - mu and
    the D columns, structure-of-arrays, fp64 (`storage="f64"`) or fp32
    (`storage="f32"`, the optional fp32 path; math stays fp64; `storage="f32m"`: fp32 per-gene
    math as well, fp64 sums).
    """

    def __init__(self, handle: int, n_networks: int):
        self._h = C.c_void_p(handle)
        self.n_networks = n_networks
        V, d, lo, Vt, st, nb = (C.c_int64(), C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32(), C.c_int64())
        _lib.check(_lib.lib().cv_dataset_info(self._h, C.byref(V), C.byref(d), C.byref(lo), C.byref(Vt),
                                              C.byref(st), C.byref(nb)))
        self.V, self.dim, self.gene_lo, self.V_total = V.value, d.value, lo.value, Vt.value
        self.storage = {_lib.STORE_F32: "f32", _lib.STORE_F32M: "f32m"}.get(st.value, "f64")
        self.device_bytes = nb.value
        self._fin = weakref.finalize(self, _lib.lib().cv_dataset_destroy, self._h)

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        self._fin()

    def download(self):
        """(r, mu, D) of this shard back on the host (r and mu exactly as stored)."""
        V, d = self.V, self.dim
        r, mu, D = np.empty(V), np.empty(V), np.empty((V, d))
        _lib.check(_lib.lib().cv_dataset_download(self._h, None, _lib.dptr(r), _lib.dptr(mu), _lib.dptr(D)))
        return r, mu, D

    def to_host(self) -> Dataset:
        r, mu, D = self.download()
        return Dataset(r=r, mu=mu, D=D, n_networks=self.n_networks)

    def stream_x(self) -> np.ndarray:
        x = np.empty(self.V)
        _lib.check(_lib.lib().cv_dataset_download(self._h, _lib.dptr(x), None, None, None))
        return x


_STORAGE = {"f64": _lib.STORE_F64, "f32": _lib.STORE_F32, "f32m": _lib.STORE_F32M}


def upload(ds, storage: str = "f64", device: int | None = None, gene_lo: int = 0, V_total: int | None = None):
    """Copy a host Dataset (ours or the reference's) into HBM."""
    r = np.ascontiguousarray(ds.r, dtype=np.float64)
    mu = np.ascontiguousarray(ds.mu, dtype=np.float64)
    D = np.ascontiguousarray(np.atleast_2d(ds.D), dtype=np.float64)
    V, d = D.shape
    h = C.c_void_p()
    _lib.check(_lib.lib().cv_dataset_create(
        _lib.dptr(r), _lib.dptr(mu), _lib.dptr(D), V, d, gene_lo, V if V_total is None else V_total,
        _STORAGE[storage], _lib.default_device() if device is None else device, C.byref(h)))
    return DeviceDataset(h.value, int(ds.n_networks))


def generate(seed: int, V: int, N: int, K, Lam, rho: float, storage: str = "f64", device: int | None = None,
             gene_lo: int = 0, V_total: int | None = None) -> DeviceDataset:
    """random_profiles(RngStream(seed), V_total, N) + synth_generate(ModelParams(K, Lam, rho)),
    genes [gene_lo, gene_lo + V), built on the GPU (reference model.py:224-270)."""
    K = np.ascontiguousarray(np.atleast_1d(K), dtype=np.float64)
    Lam = np.ascontiguousarray(np.atleast_2d(Lam), dtype=np.float64)
    if K.shape[0] != N - 1 or Lam.shape != (N - 1, N - 1):
        raise ValueError(f"profiles have {N} networks but truth implies {K.shape[0] + 1}")
    h = C.c_void_p()
    _lib.check(_lib.lib().cv_dataset_generate(
        seed & 0xFFFFFFFFFFFFFFFF, gene_lo, V, V if V_total is None else V_total, N, _lib.dptr(K), _lib.dptr(Lam),
        float(rho), _STORAGE[storage], _lib.default_device() if device is None else device, C.byref(h)))
    return DeviceDataset(h.value, N)


def regime(V: int, seed: int = 0, N: int = 3, K=None, rho: float = 100.0, **kw) -> DeviceDataset:
    """The reference test-suite regime (reference tests/conftest.py:15-26), on the device."""
    if N == 3:
        lam = np.linalg.inv(REFERENCE_LAMBDA_INV)
        K = np.array([0.1, 0.3]) if K is None else np.asarray(K, dtype=float)
    else:
        lam = np.linalg.inv(0.01 * np.eye(N - 1))
        if K is None or len(K) != N - 1:
            K = np.full(N - 1, 0.2)
    return generate(seed, V, N, K, lam, rho, **kw)
