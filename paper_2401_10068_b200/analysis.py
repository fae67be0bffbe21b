"""Posterior summaries on the GPU: drop-in for the reference's `tissuemix.analysis`
(reference analysis.py:17-188), SURVEY §8(f) row 4.

Same names, arguments and errors: `KdeModel`, `DensityGrid`, `kde_fit`, `kde_density`,
`kde_grid`, `kde_mode`, `summarize`.  The kernel sums (every grid point against every
sample, the golden-section refinements, the per-column moments and order statistics)
run in csrc/kde.cu; the host only validates arguments and formats the report.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["DensityGrid", "KdeModel", "kde_density", "kde_fit", "kde_grid", "kde_mode", "summarize"]

_GOLDEN = (np.sqrt(5.0) - 1.0) / 2.0
_SQRT2PI = float(np.sqrt(2.0 * np.pi))


def _dev():
    return _lib.default_device()


@dataclass(frozen=True)
class KdeModel:
    """Samples plus a Gaussian-kernel bandwidth (scalar, one dimension) -- analysis.py:29-44."""

    samples: np.ndarray
    bandwidth: float

    def __post_init__(self):
        s = np.asarray(self.samples, dtype=np.float64)
        if s.ndim != 1 or s.shape[0] < 2:
            raise ValueError("need at least 2 one-dimensional samples")
        if not np.all(np.isfinite(s)):
            raise ValueError("samples contain non-finite values")
        if not self.bandwidth > 0:
            raise ValueError("bandwidth must be positive")
        object.__setattr__(self, "samples", np.ascontiguousarray(s))


@dataclass(frozen=True)
class DensityGrid:
    x: np.ndarray
    density: np.ndarray
    mode: float

    @property
    def integral(self) -> float:
        return float(np.trapezoid(self.density, self.x))


def _columns(cols: np.ndarray, bw=None, grid_n=0, rng=None, find_mode=False, qlo=0.5, qhi=0.5, grid=False):
    cols = np.ascontiguousarray(np.atleast_2d(cols), dtype=np.float64)  # (C, n)
    Cn, n = cols.shape
    out = np.empty((Cn, 10))
    g = np.empty((Cn, grid_n)) if grid and grid_n > 0 else None
    bwa = None if bw is None else np.ascontiguousarray(np.broadcast_to(np.asarray(bw, float), (Cn,)))
    ra = None if rng is None else np.ascontiguousarray(np.asarray(rng, float).reshape(Cn, 2))
    _lib.check(_lib.lib().cv_kde_columns(_lib.dptr(cols), n, Cn, _lib.dptr(bwa), float(n ** (-1.0 / 5.0)), _SQRT2PI,
                                         float(_GOLDEN), int(grid_n), _lib.dptr(ra), float(qlo), float(qhi),
                                         int(find_mode), _dev(), _lib.dptr(out), _lib.dptr(g)))
    return out, g


def kde_fit(samples, bandwidth: float | None = None) -> KdeModel:
    """1-d Gaussian KDE; default bandwidth by Scott's rule h = sd * n^(-1/5) (analysis.py:58-71)."""
    s = np.asarray(samples, dtype=np.float64)
    if s.ndim != 1 or s.shape[0] < 2:
        raise ValueError("need at least 2 one-dimensional samples")
    if bandwidth is None:
        if not np.all(np.isfinite(s)):
            raise ValueError("samples contain non-finite values")
        out, _ = _columns(s[None, :])  # sample sd on the device
        sd = float(out[0, 1])
        if sd == 0.0:
            raise ValueError("zero-variance samples: pass an explicit bandwidth")
        bandwidth = sd * len(s) ** (-1.0 / 5.0)
    return KdeModel(samples=s, bandwidth=float(bandwidth))


def kde_density(model: KdeModel, x) -> np.ndarray:
    """Density values at the query points (analysis.py:74-85)."""
    x = np.ascontiguousarray(np.atleast_1d(np.asarray(x, dtype=np.float64)))
    out = np.empty_like(x)
    flat = x.reshape(-1)
    smp = np.ascontiguousarray(model.samples, dtype=np.float64)
    _lib.check(_lib.lib().cv_kde_density(_lib.dptr(smp), len(smp), float(model.bandwidth),
                                         _SQRT2PI, _lib.dptr(flat), flat.shape[0], _dev(), _lib.dptr(out.reshape(-1))))
    return out


def _range(model, lo, hi):
    if lo is None:
        lo = float(model.samples.min()) - 4.0 * model.bandwidth
    if hi is None:
        hi = float(model.samples.max()) + 4.0 * model.bandwidth
    return lo, hi


def kde_grid(model: KdeModel, lo: float | None = None, hi: float | None = None, n: int = 512) -> DensityGrid:
    """Density on linspace(lo, hi, n), default span = samples +- 4 bandwidths (analysis.py:88-95)."""
    lo, hi = _range(model, lo, hi)
    x = np.linspace(lo, hi, n)
    if n < 256:  # the reference's kde_mode raises for coarse grids; the density itself is fine
        return DensityGrid(x=x, density=kde_density(model, x), mode=kde_mode(model, n=n, lo=lo, hi=hi)[0])
    out, g = _columns(model.samples[None, :], bw=model.bandwidth, grid_n=n, rng=[lo, hi], find_mode=True, grid=True)
    return DensityGrid(x=x, density=g[0], mode=float(out[0, 3]))


def kde_mode(model: KdeModel, n: int = 512, lo: float | None = None, hi: float | None = None) -> tuple[float, bool]:
    """Grid argmax refined by three golden-section steps; (mode, multimodal) (analysis.py:98-139)."""
    if n < 256:
        raise ValueError("grid resolution must be >= 256")
    lo, hi = _range(model, lo, hi)
    out, _ = _columns(model.samples[None, :], bw=model.bandwidth, grid_n=n, rng=[lo, hi], find_mode=True)
    return float(out[0, 3]), bool(out[0, 4])


def summarize(samples: dict, bandwidth: float | None = None) -> dict:
    """Mode / mean / central 95% interval per parameter, plus full weights (analysis.py:147-188)."""
    K = np.ascontiguousarray(samples["K"], dtype=np.float64)
    rho = np.ascontiguousarray(samples["rho"], dtype=np.float64)
    if K.shape[0] < 100:
        raise ValueError("need at least 100 samples")
    n, d = K.shape
    lam = None
    if "Lambda" in samples:
        lam = np.ascontiguousarray(samples["Lambda"], dtype=np.float64)
    for a in (K, rho) + (() if lam is None else (lam,)):
        if not np.all(np.isfinite(a)):
            raise ValueError("samples contain non-finite values")
    if bandwidth is not None and not bandwidth > 0:
        raise ValueError("bandwidth must be positive")
    alpha = 0.5 * (1.0 - 0.95)  # _central_interval (analysis.py:142-144)
    out = np.empty((2 * d + 2, 10))
    lm = np.empty((d, d)) if lam is not None else None
    _lib.check(_lib.lib().cv_summarize(_lib.dptr(K), _lib.dptr(rho), _lib.dptr(lam), n, d,
                                       float(bandwidth) if bandwidth is not None else 0.0, float(n ** (-1.0 / 5.0)),
                                       _SQRT2PI, float(_GOLDEN), alpha, 1.0 - alpha, _dev(), _lib.dptr(out),
                                       _lib.dptr(lm)))

    def entry(row):
        return {"mode": float(row[3]), "mean": float(row[0]), "ci95": [float(row[5]), float(row[6])]}

    report: dict = {"parameters": {}, "full_weights": {}}
    for j in range(d):
        report["parameters"][f"K{j + 1}"] = entry(out[j])
    modes = []
    for j in range(d + 1):
        e = entry(out[d + j])
        report["full_weights"][f"w{j + 1}"] = e
        modes.append(e["mode"])
    report["full_weights"]["mode_vector"] = modes
    report["parameters"]["rho"] = entry(out[2 * d + 1])
    if lm is not None:
        report["parameters"]["Lambda_mean"] = lm.tolist()
    return report
