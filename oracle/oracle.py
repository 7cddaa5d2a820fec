"""CPU oracle for the per-frame segmentation hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
(``paper_1407_2089_b200``) never imports anything under ``oracle/``.

It restates the reference (ref = /root/reference/pkg/src/clonetrack) on top of
``liboracle.so`` (``ct_oracle.c``: the numerical kernels, restating the
scipy 1.18.1 / numpy 2.3.5 routines the reference calls) plus numpy glue for
array plumbing.  Every function names the reference lines it follows.  Parity
with the reference itself is pinned by ``tests/golden`` (fixtures produced by
``tests/golden/make_golden.py`` from the live reference) and by live
comparisons in ``tests/test_oracle.py`` when /root/reference is present.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


class OracleParameterError(ValueError):
    """Mirrors ref errors.py:16 ParameterError."""


class OracleDegenerateHistogramError(ValueError):
    """Mirrors ref errors.py:20 DegenerateHistogramError."""


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, U64, D, INT = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
        sig = {
            "ora_synth_base": (None, [P, INT, I64, I64, I64, U64, I64]),
            "ora_synth_balls": (None, [P, INT, I64, I64, I64, U64, I64, P, I64, I64]),
            "ora_synth_tubes": (None, [P, INT, I64, I64, I64, U64, I64, P, I64, I64]),
            "ora_gauss_axis": (None, [P, P, I64, I64, I64, INT, P, INT]),
            "ora_median": (None, [P, I64, I64, I64, INT, P]),
            "ora_histogram": (INT, [P, I64, P]),
            "ora_otsu": (INT, [P, I64, P]),
            "ora_closing": (None, [P, I64, I64, I64, INT, P]),
            "ora_label26": (I64, [P, I64, I64, I64, P]),
            "ora_centroid_seq": (None, [P, I64, D, D, D, P]),
            "ora_edt": (None, [P, I64, I64, I64, D, D, D, P]),
            "ora_pairwise_sum": (D, [P, I64]),
            "ora_intensity_step": (D, [P, I64]),
            "ora_noise_sigma": (INT, [P, I64, I64, I64, P]),
            "ora_sign_sum": (None, [P, I64, I64, I64, P]),
            "ora_mrf": (INT, [P, I64, I64, I64, INT, P, P, P, P, P]),
            "ora_num_threads": (INT, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def threads() -> int:
    return int(lib().ora_num_threads())


# ---------------------------------------------------------------------------
# Synthetic frames (counter-based; bit-identical to the CUDA generator)
# ---------------------------------------------------------------------------
def synth_frame(dims, dtype: str, seed: int, vmax: int, balls=None, tubes=None, amp_ball=0, amp_tube=0):
    nx, ny, nz = dims
    code = 1 if dtype == "u8" else 2
    out = np.empty(dims, dtype=np.uint8 if code == 1 else np.uint16)
    L = lib()
    L.ora_synth_base(_p(out), code, nx, ny, nz, seed, vmax)
    if tubes is not None and len(tubes):
        t = np.ascontiguousarray(tubes, dtype=np.int64)
        L.ora_synth_tubes(_p(out), code, nx, ny, nz, seed, vmax, _p(t), t.shape[0], amp_tube)
    if balls is not None and len(balls):
        b = np.ascontiguousarray(balls, dtype=np.int64)
        L.ora_synth_balls(_p(out), code, nx, ny, nz, seed, vmax, _p(b), b.shape[0], amp_ball)
    return out


# ---------------------------------------------------------------------------
# Cell channel denoise: ref denoise.py:58-89
# ---------------------------------------------------------------------------
def gaussian_weights(sigma: float, radius: int) -> np.ndarray:
    """w[j] = weight at tap distance j (scipy _filters.py:656-686, order 0)."""
    sigma2 = sigma * sigma
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / sigma2 * x**2)
    phi = phi / phi.sum()
    return np.ascontiguousarray(phi[radius:])


def gaussian_background(values: np.ndarray, sigmas) -> np.ndarray:
    """ref denoise.py:84-85: gaussian_filter(float64, sigma, 'nearest', truncate 4)."""
    x = np.ascontiguousarray(values, dtype=np.float64)
    nx, ny, nz = x.shape
    for axis, sigma in enumerate(sigmas):
        if not sigma > 1e-15:
            continue
        r = int(4.0 * float(sigma) + 0.5)
        w = gaussian_weights(float(sigma), r)
        y = np.empty_like(x)
        lib().ora_gauss_axis(_p(x), _p(y), nx, ny, nz, axis, _p(w), r)
        x = y
    return x


def median(values: np.ndarray, radius: int) -> np.ndarray:
    x = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty_like(x)
    lib().ora_median(_p(x), *x.shape, radius, _p(out))
    return out


def denoise_cell(values, spacing, sigma_um: float = 10.0, median_radius: int = 1):
    """ref denoise.py:67-89.  Returns dict(bg, residual, denoised)."""
    values = np.asarray(values)
    if values.size == 0:
        raise OracleParameterError("cannot denoise an empty grid")
    sig = tuple(sigma_um / s for s in spacing)
    for s, n in zip(sig, values.shape):
        if s > n:
            raise OracleParameterError(f"gaussian kernel scale {s:.1f} voxels exceeds grid extent {n}")
    v = values.astype(np.float64)
    bg = gaussian_background(v, sig)
    res = np.maximum(v - bg, 0.0)
    den = median(res, median_radius)
    return {"bg": bg, "residual": res, "denoised": den}


# ---------------------------------------------------------------------------
# Segmentation: ref segment.py:99-318
# ---------------------------------------------------------------------------
def histogram(values) -> np.ndarray:
    """ref segment.py:154-163 (256 or 65536 bins)."""
    x = np.ascontiguousarray(values, dtype=np.float64)
    h = np.zeros(65536, dtype=np.int64)
    nb = lib().ora_histogram(_p(x), x.size, _p(h))
    return h[:nb].copy()


def otsu(hist) -> int:
    """ref segment.py:99-151 (incl. int64 wrap of the float prefilter)."""
    h = np.ascontiguousarray(hist, dtype=np.int64)
    if h.ndim != 1:
        raise OracleDegenerateHistogramError("histogram must be 1-D")
    t = np.zeros(1, dtype=np.int64)
    st = lib().ora_otsu(_p(h), h.size, _p(t))
    if st == 2:
        raise OracleDegenerateHistogramError("histogram has fewer than 2 non-empty bins")
    return int(t[0])


def binarize(values) -> np.ndarray:
    """ref segment.py:192-204."""
    h = histogram(values)
    if np.count_nonzero(h) < 2:
        if h[0] == h.sum():
            return np.zeros(np.shape(values), dtype=bool)
        raise OracleDegenerateHistogramError("frame is constant")
    t = otsu(h)
    return np.rint(np.asarray(values, dtype=np.float64)) > t


def closing(mask, radius: int) -> np.ndarray:
    """ref segment.py:175-189."""
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    out = np.empty_like(m)
    lib().ora_closing(_p(m), *m.shape, radius, _p(out))
    return out.astype(bool)


def label26(mask):
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    lab = np.empty(m.shape, dtype=np.int32)
    n = lib().ora_label26(_p(m), *m.shape, _p(lab))
    return lab, int(n)


@dataclass
class OracleDetection:
    id: int
    frame: int
    voxels: np.ndarray
    centroid_um: np.ndarray
    volume_um3: float
    root: int
    bbox: np.ndarray  # (imin, jmin, kmin, imax, jmax, kmax)
    intensity_sum: float | None = None

    @property
    def voxel_count(self) -> int:
        return int(self.voxels.shape[0])


def centroid_seq(vox: np.ndarray, spacing) -> np.ndarray:
    v = np.ascontiguousarray(vox, dtype=np.int64)
    out = np.empty(3, dtype=np.float64)
    lib().ora_centroid_seq(_p(v), v.shape[0], float(spacing[0]), float(spacing[1]), float(spacing[2]), _p(out))
    return out


def detections(mask, spacing, frame: int = 0, min_volume_um3: float = 19.0, id_start: int = 0, intensity=None):
    """ref segment.py:242-276 without hulls (hulls stay host-side)."""
    lab, n = label26(mask)
    shape = lab.shape
    vv = (float(spacing[0]) * float(spacing[1])) * float(spacing[2])
    flat = lab.ravel()
    order = np.argsort(flat, kind="stable")  # stable: C order within a label
    counts = np.bincount(flat, minlength=n + 1)
    starts = np.concatenate([[0], np.cumsum(counts)])
    groups = []
    for c in range(1, n + 1):
        cnt = int(counts[c])
        if cnt * vv < min_volume_um3:
            continue
        lin = order[starts[c] : starts[c + 1]]
        groups.append((cnt, int(lin[0]), lin))
    groups.sort(key=lambda g: (-g[0], g[1]))
    dets = []
    ivals = None if intensity is None else np.asarray(intensity).ravel()
    for off, (cnt, root, lin) in enumerate(groups):
        vox = np.stack(np.unravel_index(lin, shape), axis=1).astype(np.int64)
        isum = None
        if ivals is not None:
            isum = float(np.sum(ivals[lin].astype(np.int64))) if ivals.dtype.kind in "iu" else None
        dets.append(
            OracleDetection(
                id=id_start + off,
                frame=frame,
                voxels=vox,
                centroid_um=centroid_seq(vox, spacing),
                volume_um3=cnt * vv,
                root=root,
                bbox=np.concatenate([vox.min(axis=0), vox.max(axis=0)]),
                intensity_sum=isum,
            )
        )
    return dets


def segment_cell(values, spacing, min_volume_um3=19.0, closing_radius=1, frame=0, id_start=0, intensity=None):
    """ref segment.py:279-289."""
    mask = closing(binarize(values), closing_radius)
    return detections(mask, spacing, frame, min_volume_um3, id_start, intensity=intensity)


def edt(mask, spacing) -> np.ndarray:
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    out = np.empty(m.shape, dtype=np.float64)
    lib().ora_edt(_p(m), *m.shape, float(spacing[0]), float(spacing[1]), float(spacing[2]), _p(out))
    return out


def distance_map(mask, spacing):
    """ref segment.py:292-304 -> (values, empty)."""
    m = np.asarray(mask, dtype=bool)
    if m.size == 0:
        raise OracleParameterError("mask has no voxels")
    if not m.any():
        return np.full(m.shape, np.inf), True
    return edt(m, spacing), False


def segment_vessel(values, spacing, closing_radius=1):
    """ref segment.py:307-318 -> (mask, dist, empty)."""
    mask = closing(binarize(values), closing_radius)
    dist, empty = distance_map(mask, spacing)
    return mask, dist, empty


# ---------------------------------------------------------------------------
# Vessel channel MRF: ref denoise.py:92-195
# ---------------------------------------------------------------------------
def pairwise_sum(a) -> float:
    x = np.ascontiguousarray(a, dtype=np.float64).ravel()
    return float(lib().ora_pairwise_sum(_p(x), x.size))


def intensity_step(values) -> float:
    x = np.ascontiguousarray(values, dtype=np.float64).ravel()
    return float(lib().ora_intensity_step(_p(x), x.size))


def noise_sigma(values) -> float:
    x = np.ascontiguousarray(values, dtype=np.float64)
    out = np.zeros(1)
    if lib().ora_noise_sigma(_p(x), *x.shape, _p(out)) != 0:
        raise OracleParameterError(f"grid dims {x.shape} leave fewer than 2 interior voxels")
    return float(out[0])


def sign_sum(values) -> np.ndarray:
    x = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty(x.shape, dtype=np.int64)
    lib().ora_sign_sum(_p(x), *x.shape, _p(out))
    return out


def mrf(values, max_iters: int = 1000) -> dict:
    """ref denoise.py:147-190.  'current' is None when delta == 0 (the
    reference then returns the input grid object unchanged)."""
    x = np.ascontiguousarray(values, dtype=np.float64)
    if x.size == 0:
        raise OracleParameterError("cannot denoise an empty grid")
    cur = np.empty_like(x)
    it = np.zeros(1, dtype=np.int32)
    conv = np.zeros(1, dtype=np.int32)
    sh = np.zeros(1)
    dl = np.zeros(1)
    st = lib().ora_mrf(_p(x), *x.shape, max_iters, _p(cur), _p(it), _p(conv), _p(sh), _p(dl))
    if st == 3:
        return {"current": None, "iteration": 0, "converged": True, "sigma_hat": 0.0, "delta": 0.0}
    return {
        "current": cur,
        "iteration": int(it[0]),
        "converged": bool(conv[0]),
        "sigma_hat": float(sh[0]),
        "delta": float(dl[0]),
    }
