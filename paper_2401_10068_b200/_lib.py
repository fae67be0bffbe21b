"""ctypes binding of libcavi.so (the C ABI in include/cavi.h).

The library is built in-tree (`make`, or `__graft_entry__.build()`); importing
this module without it raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import linalg

MAX_D = 15
MAX_D2 = MAX_D * MAX_D

OK, ERR_NUMERIC, ERR_NONFINITE, ERR_ARG, ERR_CUDA, ERR_IMPROPER, ERR_FORMAT, ERR_PEER, ERR_SINGULAR = range(9)
STORE_F64, STORE_F32, STORE_F32M = 0, 1, 2

_LIB_PATH = os.environ.get("CAVI_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcavi.so"))


class CvHyper(C.Structure):
    _fields_ = [
        ("a0", C.c_double), ("b0", C.c_double), ("q0", C.c_double),
        ("n0", C.c_int32), ("d", C.c_int32),
        ("K0", C.POINTER(C.c_double)), ("Lambda0", C.POINTER(C.c_double)),
    ]


class CvState(C.Structure):
    _fields_ = [
        ("d", C.c_int32), ("n_iter", C.c_int32), ("status", C.c_int32), ("elbo_status", C.c_int32),
        ("V", C.c_int64),
        ("a_rho", C.c_double), ("b_rho", C.c_double), ("e_rho", C.c_double),
        ("k0k", C.c_double * MAX_D),
        ("lam0l_inv", C.c_double * MAX_D2),
        ("e_lam", C.c_double * MAX_D2),
        ("e_lamk", C.c_double * MAX_D),
        ("ln_det_lam0l_inv", C.c_double),
        ("elbo", C.c_double),
        ("resid", C.c_double),
        ("gen_c", C.c_double * MAX_D),
        ("gen_A", C.c_double * MAX_D2),
        ("gen_Ainv", C.c_double * MAX_D2),
        ("gen_lnA", C.c_double),
        ("gen_e_rho", C.c_double),
    ]

    def vec(self, name: str) -> np.ndarray:
        return np.array(getattr(self, name)[: self.d], dtype=np.float64)

    def mat(self, name: str) -> np.ndarray:
        d = self.d
        return np.array(getattr(self, name)[: d * d], dtype=np.float64).reshape(d, d)

    def copy(self) -> "CvState":
        out = CvState()
        C.memmove(C.byref(out), C.byref(self), C.sizeof(CvState))
        return out


_P = C.POINTER
_D = _P(C.c_double)
_SIGS = {
    "cv_abi_version": (C.c_int32, []),
    "cv_last_error": (C.c_char_p, []),
    "cv_device_count": (C.c_int32, [_P(C.c_int32)]),
    "cv_dataset_create": (C.c_int32, [_D, _D, _D, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int32,
                                      C.c_int32, _P(C.c_void_p)]),
    "cv_dataset_generate": (C.c_int32, [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, _D, _D,
                                        C.c_double, C.c_int32, C.c_int32, _P(C.c_void_p)]),
    "cv_dataset_download": (C.c_int32, [C.c_void_p, _D, _D, _D, _D]),
    "cv_dataset_info": (C.c_int32, [C.c_void_p, _P(C.c_int64), _P(C.c_int32), _P(C.c_int64), _P(C.c_int64),
                                    _P(C.c_int32), _P(C.c_int64)]),
    "cv_dataset_destroy": (None, [C.c_void_p]),
    "cv_init": (C.c_int32, [C.c_void_p, _P(CvHyper), _P(CvState)]),
    "cv_step": (C.c_int32, [C.c_void_p, _P(CvHyper), _P(CvState), _P(CvState)]),
    "cv_elbo": (C.c_int32, [C.c_void_p, _P(CvHyper), _P(CvState), _D]),
    "cv_fit": (C.c_int32, [C.c_void_p, _P(CvHyper), C.c_int32, C.c_double, C.c_int32, C.c_double, _P(CvState),
                           _D, _D, _D, _D, _P(C.c_int32)]),
    "cv_materialize": (C.c_int32, [C.c_void_p, _P(CvHyper), _P(CvState), C.c_int64, C.c_int64, _D, _D, _D, _D,
                                   _D]),
    "cv_nccl_unique_id": (C.c_int32, [C.c_char_p]),
    "cv_comm_create": (C.c_int32, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, _P(C.c_void_p)]),
    "cv_comm_destroy": (None, [C.c_void_p]),
    "cv_comm_fused": (C.c_int32, [C.c_void_p]),
    "cv_comm_drop_publish": (C.c_int32, [C.c_void_p, C.c_int32]),
    "cv_dataset_set_comm": (C.c_int32, [C.c_void_p, C.c_void_p]),
    "cv_dataset_set_shard": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32]),
    "cv_shard_stats": (C.c_int32, [C.c_void_p, _P(CvHyper), _P(CvState), _D]),
    "cv_em_fit": (C.c_int32, [C.c_void_p, _D, _D, C.c_double, C.c_int32, C.c_double, _D, _D, _D, _D, _D, _D,
                              _P(C.c_int32)]),
    "cv_dataset_load_csv": (C.c_int32, [C.c_char_p, C.c_int32, C.c_int32, _P(C.c_void_p), _P(C.c_int32)]),
    "cv_dataset_load_npz": (C.c_int32, [C.c_char_p, C.c_int32, C.c_int32, _P(C.c_void_p), _P(C.c_int32)]),
    "cv_npz_probe": (C.c_int32, [C.c_char_p, _P(C.c_int64), _P(C.c_int32)]),
    "cv_write_dataset_csv": (C.c_int32, [C.c_char_p, _D, _D, _D, C.c_int64, C.c_int32, C.c_int32]),
    "cv_parse_number_host": (C.c_int32, [C.c_char_p, C.c_int64, _D]),
    "cv_format_repr": (C.c_int32, [C.c_double, C.c_char_p]),
    "cv_csv_records_host": (C.c_int32, [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, _P(C.c_int64)]),
    "cv_kde_columns": (C.c_int32, [_D, C.c_int64, C.c_int32, _D, C.c_double, C.c_double, C.c_double, C.c_int32, _D,
                                   C.c_double, C.c_double, C.c_int32, C.c_int32, _D, _D]),
    "cv_kde_density": (C.c_int32, [_D, C.c_int64, C.c_double, C.c_double, _D, C.c_int64, C.c_int32, _D]),
    "cv_summarize": (C.c_int32, [_D, _D, _D, C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double,
                                 C.c_double, C.c_double, C.c_int32, _D, _D]),
    "cv_em_step": (C.c_int32, [C.c_void_p, _D, _D, C.c_double, _D, _D, _D, _D, _D]),
    "cv_batched_fit": (C.c_int32, [_D, _D, _D, _P(C.c_int64), C.c_int64, C.c_int32, _P(CvHyper), C.c_int32,
                                   C.c_double, C.c_int32, C.c_double, C.c_int32, _P(CvState), _D]),
    "cv_batch_run": (C.c_int32, [_D, _D, _D, _P(C.c_int64), C.c_int64, C.c_int32, _P(CvHyper), C.c_int32, C.c_double,
                                 C.c_int32, C.c_double, C.c_int32, _P(C.c_int32), _P(C.c_void_p)]),
    "cv_batch_states": (C.c_int32, [C.c_void_p, C.c_int64, C.c_int64, _P(CvState)]),
    "cv_batch_traces": (C.c_int32, [C.c_void_p, C.c_int64, C.c_int64, _D]),
    "cv_batch_destroy": (None, [C.c_void_p]),
    "cv_posterior_sample": (C.c_int32, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, C.c_double,
                                        C.c_int64, C.c_double, C.c_double, _D, _D, C.c_int64, C.c_int32, _D, _D, _D,
                                        _P(C.c_uint64)]),
    "cv_test_rate_inverse": (C.c_int32, [_D, C.c_int32, C.c_int32, _D, _D, _P(C.c_int32)]),
    "cv_host_alloc": (C.c_int32, [C.c_int64, _P(C.c_void_p)]),
    "cv_host_free": (None, [C.c_void_p]),
    "cv_bench_sweeps": (C.c_int32, [C.c_void_p, _P(CvHyper), _P(CvState), C.c_int32, C.c_int32, _D, _D,
                                    _P(C.c_int32)]),
}

EXPORTS = tuple(_SIGS)


def load(path: str = _LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"libcavi.so not found at {path}: build it with `make -j` (or __graft_entry__.build()); "
            "the CAVI engine has no CPU fallback"
        )
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


class UsageError(ValueError):
    """A malformed dataset file (the reference's cli.UsageError, cli.py:40-41)."""


class PeerTimeoutError(RuntimeError):
    """Multi-GPU: a peer's per-sweep statistics did not arrive within CAVI_PEER_TIMEOUT_S
    (a stalled or failed rank).  The next shard call resyncs the communicator."""


def check(rc: int, n_items: int | None = None) -> None:
    """Map a status code to the reference's exception types (linalg.py:46-69).  n_items: the
    batch a singular-item error refers to (vb_init's V per-gene precisions, vb.py:94-96)."""
    if rc == OK:
        return
    msg = lib().cv_last_error().decode(errors="replace")
    if rc == ERR_SINGULAR:  # BatchItemError(msg, every item): the reference's exact message
        raise linalg.BatchItemError(msg, [np.int64(i) for i in range(n_items or 0)])
    if rc in (ERR_NUMERIC, ERR_IMPROPER):
        raise linalg.NumericError(msg)
    if rc == ERR_NONFINITE:
        raise FloatingPointError(msg)
    if rc == ERR_ARG:
        raise ValueError(msg)
    if rc == ERR_FORMAT:
        raise UsageError(msg)
    if rc == ERR_PEER:
        raise PeerTimeoutError(msg)
    raise RuntimeError(f"libcavi: {msg}")


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def hyper_struct(hp):
    """CvHyper for reference-shaped HyperParams; returns (struct, keepalive)."""
    K0 = np.ascontiguousarray(np.atleast_1d(hp.K0), dtype=np.float64)
    L0 = np.ascontiguousarray(np.atleast_2d(hp.Lambda0), dtype=np.float64)
    s = CvHyper(float(hp.a0), float(hp.b0), float(hp.q0), int(hp.n0), int(K0.shape[0]), dptr(K0), dptr(L0))
    return s, (K0, L0)


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """numpy array in page-locked host memory (cudaMallocHost), freed with the array."""
    import weakref  # noqa: PLC0415

    count = int(np.prod(shape))
    nbytes = max(1, count * np.dtype(dtype).itemsize)
    p = C.c_void_p()
    check(lib().cv_host_alloc(nbytes, C.byref(p)))
    buf = (C.c_char * nbytes).from_address(p.value)
    weakref.finalize(buf, lib().cv_host_free, p)
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)


def default_device() -> int:
    for key in ("CAVI_DEVICE", "LOCAL_RANK"):
        if key in os.environ:
            return int(os.environ[key])
    return 0
