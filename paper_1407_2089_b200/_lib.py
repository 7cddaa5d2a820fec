"""ctypes binding of libct (include/ct.h).

The product path has no CPU fallback: if ``libct.so`` is missing, or no CUDA
device is present when a kernel is called, this module raises.  Build the
library with ``python -c "import __graft_entry__ as g; g.build()"`` (or
``make -C paper_1407_2089_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ParameterError

_HERE = os.path.dirname(os.path.abspath(__file__))
# CT_LIB=debug loads the bounds-checked build (csrc: make debug), test tooling only
LIB_PATH = os.path.join(_HERE, "libct_debug.so" if os.environ.get("CT_LIB") == "debug" else "libct.so")

CT_U8, CT_U16, CT_I32, CT_F64 = 1, 2, 4, 8
CT_OK, CT_ERR_PARAM, CT_ERR_CUDA, CT_ERR_UNSUPPORTED, CT_ERR_IO = 0, 1, 3, 4, 5

# result / counter word indices (ct.h)
OTSU_T, OTSU_STATUS, OTSU_NBINS, OTSU_NONZERO = 0, 1, 2, 3
CNT_FG, CNT_COMPONENTS, CNT_KEPT, CNT_KEPT_VOXELS, CNT_OVERFLOW = 0, 1, 2, 3, 4
MRF_DELTA, MRF_SIGMA, MRF_SIGMA_STATUS, MRF_NNZ, MRF_NORM, MRF_DECISION = 0, 1, 2, 3, 4, 5
MRF_WORDS = 9

# ct_cell (16 x 8 bytes)
CELL_DTYPE = np.dtype(
    [
        ("id", "<i8"),
        ("count", "<i8"),
        ("root", "<i8"),
        ("bbox_lo", "<i8", (3,)),
        ("bbox_hi", "<i8", (3,)),
        ("intensity_sum", "<i8"),
        ("centroid_um", "<f8", (3,)),
        ("volume_um3", "<f8"),
        ("voxel_offset", "<i8"),
        ("mean_intensity", "<f8"),
    ]
)
assert CELL_DTYPE.itemsize == 128

_P, _I64, _U64, _D, _INT, _SZ = (
    ctypes.c_void_p,
    ctypes.c_int64,
    ctypes.c_uint64,
    ctypes.c_double,
    ctypes.c_int,
    ctypes.c_size_t,
)

SIGNATURES = {
    "ct_version": (ctypes.c_char_p, []),
    "ct_last_error": (ctypes.c_char_p, []),
    "ct_memset": (_INT, [_P, _INT, _I64, _P]),
    "ct_workspace_bytes": (_SZ, [_INT, _I64, _I64, _I64, _I64]),
    "ct_gaussian_residual": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _INT, _INT, _INT, _P, _P, _P, _P, _INT, _P]),
    "ct_gaussian_q": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _INT, _INT, _INT, _P, _P, _P, _I64, _D, _INT, _P]),
    "ct_voxel_runs": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P]),
    "ct_k1_path": (_INT, [_INT, _I64, _I64, _I64, _INT, _INT, _INT, _INT]),
    "ct_to_f64": (_INT, [_P, _INT, _I64, _P, _P]),
    "ct_median": (_INT, [_P, _INT, _I64, _I64, _I64, _INT, _P, _P, _P]),
    "ct_histogram": (_INT, [_P, _INT, _I64, _P, _P]),
    "ct_otsu": (_INT, [_P, _I64, _P, _P]),
    "ct_threshold_close": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _I64, _INT, _P, _P, _P]),
    "ct_closing": (_INT, [_P, _I64, _I64, _I64, _INT, _P, _P, _P]),
    "ct_ccl26": (_INT, [_P, _I64, _I64, _I64, _P, _P, _P, _P]),
    "ct_threshold_close_rows": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _I64, _P, _P, _P, _P]),
    "ct_ccl26_rows": (_INT, [_P, _I64, _I64, _I64, _P, _P, _P, _INT, _P]),
    "ct_cell_table": (
        _INT,
        [_P, _I64, _I64, _I64, _P, _P, _P, _INT, _D, _D, _D, _D, _I64, _I64, _P, _P, _P, _P],
    ),
    "ct_mrf": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _P, _P, _P]),
    "ct_mrf_decide": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _P, _P, _P]),
    "ct_mrf_step": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P]),
    "ct_sign_sum": (_INT, [_P, _INT, _I64, _I64, _I64, _P, _P]),
    "ct_edt": (_INT, [_P, _I64, _I64, _I64, _D, _D, _D, _P, _P, _P]),
    "ct_fp64_peak": (_INT, [_P, _INT, _P]),
    "ct_synth_frame": (_INT, [_P, _INT, _I64, _I64, _I64, _U64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P]),
}



class TiffInfo(ctypes.Structure):
    """ct_tiff_info (include/ct.h)."""

    _fields_ = [
        ("nx", ctypes.c_int64),
        ("ny", ctypes.c_int64),
        ("nz", ctypes.c_int64),
        ("bytes_per_sample", ctypes.c_int32),
        ("sample_format", ctypes.c_int32),
        ("big_endian", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("segments", ctypes.c_int64),
    ]


SIGNATURES.update({
    "ct_tiff_open": (_INT, [ctypes.c_char_p, ctypes.POINTER(TiffInfo), ctypes.POINTER(ctypes.c_void_p)]),
    "ct_tiff_read": (_INT, [_P, _P, _I64, ctypes.c_int32]),
    "ct_tiff_close": (None, [_P]),
    "ct_tiff_write": (_INT, [ctypes.c_char_p, _P, _I64, _I64, _I64, ctypes.c_int32, ctypes.c_int32]),
    "ct_transpose_xz": (_INT, [_P, _P, _I64, _I64, _I64, ctypes.c_int32, ctypes.c_int32, _P]),
})

_lib = None


class LibctError(RuntimeError):
    """A libct call failed for a reason that is not a reference-level error."""


def lib():
    """Load libct.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {os.path.join(_HERE, 'csrc')}` "
                "(there is no CPU fallback for the segmentation path)"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


# kernels each entry point launches (memsets excluded); used for the
# bench's gpu_launches count
LAUNCHES = {
    "ct_gaussian_residual": 3, "ct_gaussian_q": 7, "ct_to_f64": 1, "ct_median": 1, "ct_histogram": 1, "ct_otsu": 1,
    "ct_threshold_close": 2, "ct_closing": 2, "ct_ccl26": 4, "ct_threshold_close_rows": 2, "ct_ccl26_rows": 5, "ct_cell_table": 6, "ct_voxel_runs": 3, "ct_mrf": 5, "ct_mrf_decide": 8,
    "ct_mrf_step": 4, "ct_sign_sum": 1, "ct_edt": 4, "ct_synth_frame": 3, "ct_memset": 0,
}
launch_counter = {"enabled": False, "count": 0}


def call(name: str, *args) -> None:
    """Invoke ct_<name>; map status codes to exceptions."""
    fn = getattr(lib(), name)
    if launch_counter["enabled"]:
        launch_counter["count"] += LAUNCHES.get(name, 1)
    st = fn(*args)
    if st == CT_OK:
        return
    msg = lib().ct_last_error().decode(errors="replace")
    if st == CT_ERR_PARAM:
        raise ParameterError(msg)
    if st == CT_ERR_IO:
        from .errors import ManifestError

        raise ManifestError(msg)
    raise LibctError(f"{name} failed ({st}): {msg}")


def workspace_bytes(which: int, nx: int, ny: int, nz: int, cap: int = 0) -> int:
    return int(lib().ct_workspace_bytes(which, nx, ny, nz, cap))
