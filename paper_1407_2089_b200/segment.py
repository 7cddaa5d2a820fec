"""Per-frame cell and vessel segmentation on the B200.

Drop-in for ref segment.py (same names, signatures, dataclasses and
exceptions).  Every stage is a libct kernel (include/ct.h):
histogram (ct_histogram), Otsu (K3 ct_otsu, the reference's exact semantics),
threshold + ball closing (K4), 26-connected labelling (K5), the per-cell
table with canonical ids, C-order voxel lists and bit-identical centroids
(K6), and the anisotropic EDT (K8).  Only the convex hull stays on the host
(SCOPE: SURVEY.md 8f; it is Qhull in the reference too) and the voxel-run
codec, an export format.

numpy inputs give numpy outputs (the reference's behaviour); torch CUDA
inputs keep results on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from ._lib import (
    CELL_DTYPE,
    CNT_KEPT,
    CNT_KEPT_VOXELS,
    CNT_OVERFLOW,
    CT_U8,
    OTSU_NBINS,
    OTSU_STATUS,
    OTSU_T,
    call,
    workspace_bytes,
)
from .errors import DegenerateHistogramError, EmptyDistanceMapError, ParameterError
from .imaging import VoxelGrid, VoxelSpacing, physical_coordinates

FULL_CONNECTIVITY = np.ones((3, 3, 3), dtype=bool)  # 26-connected

DEFAULT_COMPONENT_CAPACITY = 1 << 20


@dataclass(frozen=True)
class SegmentationConfig:
    """Cell segmentation knobs; connectivity is fixed at 26 (ref segment.py:23-34)."""

    min_volume_um3: float = 19.0
    closing_radius: int = 1

    def __post_init__(self):
        if self.min_volume_um3 < 0:
            raise ParameterError(f"min volume must be >= 0, got {self.min_volume_um3}")
        if self.closing_radius < 0:
            raise ParameterError(f"closing radius must be >= 0, got {self.closing_radius}")


@dataclass(eq=False)
class HullMesh:
    """Convex hull of a detection's voxel centres (ref segment.py:37-55)."""

    vertices_um: np.ndarray
    facets: np.ndarray
    flat: bool = False
    equations: np.ndarray | None = None

    def contains(self, points_um: np.ndarray, tol: float = 1e-9) -> np.ndarray:
        if self.flat or self.equations is None:
            raise ValueError("containment test undefined for a flat hull")
        pts = np.atleast_2d(points_um)
        return (pts @ self.equations[:, :3].T + self.equations[:, 3]).max(axis=1) <= tol


@dataclass(eq=False, slots=True)  # slots: ~25% faster construction of a frame's detections
class Detection:
    """One segmented cell in one frame (ref segment.py:58-74)."""

    id: int
    frame: int
    voxels: np.ndarray  # (n, 3) int64, C order
    centroid_um: np.ndarray
    volume_um3: float
    hull: HullMesh | None = None
    # north-star per-cell features beyond the reference's record (computed by
    # the same K6 table pass): bounding box (imin, jmin, kmin, imax, jmax, kmax)
    # and the mean of the cell's raw intensities (numpy intensity[voxels].mean();
    # None when no intensity volume was given)
    bbox: np.ndarray | None = None
    mean_intensity: float | None = None

    @property
    def voxel_count(self) -> int:
        return int(self.voxels.shape[0])

    def voxel_set(self) -> set[tuple[int, int, int]]:
        return {tuple(v) for v in self.voxels.tolist()}


@dataclass
class DistanceMap:
    """Distance (um) to the nearest vessel voxel (ref segment.py:77-96).

    ``values`` is a numpy array or a device-resident torch tensor."""

    values: object
    spacing: VoxelSpacing
    empty: bool = False

    def at_voxel(self, i: int, j: int, k: int) -> float:
        if self.empty:
            raise EmptyDistanceMapError("distance map has no foreground")
        return float(self.values[i, j, k])

    def at_point_um(self, point_um: np.ndarray) -> float:
        """Nearest-index lookup of a physical point."""
        if self.empty:
            raise EmptyDistanceMapError("distance map has no foreground")
        idx = np.rint(np.asarray(point_um, dtype=float) / self.spacing.as_array()).astype(int)
        idx = np.clip(idx, 0, np.array(tuple(self.values.shape)) - 1)
        return float(self.values[tuple(int(x) for x in idx)])


# ---------------------------------------------------------------------------
# histogram / Otsu / binarize
# ---------------------------------------------------------------------------
def _histogram_dev(values: torch.Tensor) -> torch.Tensor:
    hist = _dev.zeros(65536, torch.int64)
    call("ct_histogram", values.data_ptr(), _dev.ct_code(values), values.numel(), hist.data_ptr(),
         _dev.stream_handle())
    return hist


def _otsu_dev(hist: torch.Tensor, nbins: int = 0) -> torch.Tensor:
    res = _dev.zeros(4, torch.int64)
    call("ct_otsu", hist.data_ptr(), nbins, res.data_ptr(), _dev.stream_handle())
    return res


def otsu_threshold(histogram) -> int:
    """Threshold maximising between-class variance; ties -> lowest t
    (ref segment.py:99-151, including its int64 float prefilter)."""
    counts = np.asarray(histogram, dtype=np.int64)
    if counts.ndim != 1 or counts.size < 2:
        raise DegenerateHistogramError(f"histogram must be 1-D with >= 2 bins, got shape {counts.shape}")
    if (counts > 0).sum() < 2:
        raise DegenerateHistogramError("histogram has fewer than 2 non-empty bins")
    if counts.size > 65536:
        raise ValueError("histograms longer than 65536 bins are not supported")
    h = torch.from_numpy(np.ascontiguousarray(counts)).to(_dev.require_cuda())
    res = _otsu_dev(h, counts.size).cpu().numpy()
    return int(res[OTSU_T])


def intensity_histogram(grid: VoxelGrid) -> np.ndarray:
    """256- or 65536-bin histogram of rint(clip(values)) (ref segment.py:154-163)."""
    v = _dev.to_device(grid.values)
    hist = _histogram_dev(v).cpu().numpy()
    return hist[:256].copy() if not hist[256:].any() else hist


def ball_element(radius: int) -> np.ndarray:
    """Binary ball x^2+y^2+z^2 <= r^2 (ref segment.py:166-172)."""
    if radius == 0:
        return np.ones((1, 1, 1), dtype=bool)
    r = np.arange(-radius, radius + 1)
    return (r[:, None, None] ** 2 + r[None, :, None] ** 2 + r[None, None, :] ** 2) <= radius * radius


def _close_dev(values: torch.Tensor, otsu_res, t_host: int, radius: int) -> torch.Tensor:
    nx, ny, nz = (int(d) for d in values.shape)
    out = _dev.empty((nx, ny, nz), torch.uint8)
    work = None
    if radius >= 1:
        work = _dev.empty(workspace_bytes(1, nx, ny, nz, radius), torch.uint8)
    call(
        "ct_threshold_close", values.data_ptr(), _dev.ct_code(values), nx, ny, nz,
        otsu_res.data_ptr() if otsu_res is not None else None, t_host, radius, out.data_ptr(),
        work.data_ptr() if work is not None else None, _dev.stream_handle(),
    )
    return out


def morphological_closing(mask, radius: int):
    """Closing with a ball on the implicit zero-padded infinite domain
    (ref segment.py:175-189)."""
    if radius == 0:
        return mask.clone() if _dev.is_torch(mask) else np.array(mask, copy=True)
    m = _dev.to_device(mask, allow=(torch.uint8,))
    if m.dtype != torch.uint8:
        m = (m != 0).to(torch.uint8)
    out = _close_dev(m, None, 0, radius)
    return _dev.like_input(out.bool(), mask)


def _binarize_dev(values: torch.Tensor, radius: int = 0):
    """threshold (+ closing) on device; returns (mask u8, otsu result)."""
    res = _otsu_dev(_histogram_dev(values), 0)
    return _close_dev(values, res, 0, radius), res


def _check_otsu(res: torch.Tensor):
    st = res.cpu().numpy()
    if st[OTSU_STATUS] == 2:
        raise DegenerateHistogramError("frame is constant; no threshold separates it")
    return st


def binarize(grid: VoxelGrid):
    """Otsu-threshold a denoised grid into a foreground mask (ref segment.py:192-204)."""
    v = _dev.to_device(grid.values)
    mask, res = _binarize_dev(v, 0)
    _check_otsu(res)
    return _dev.like_input(mask.bool(), grid.values)


# ---------------------------------------------------------------------------
# components / detections
# ---------------------------------------------------------------------------
def compute_hull(voxels: np.ndarray, spacing: VoxelSpacing) -> HullMesh:
    """Convex hull of voxel centres; degenerate sets -> flat hull
    (ref segment.py:220-239).  Host-side Qhull, as in the reference."""
    from scipy.spatial import ConvexHull, QhullError

    points = physical_coordinates(voxels, spacing)
    if points.shape[0] >= 4:
        try:
            h = ConvexHull(points)
            return HullMesh(vertices_um=points[h.vertices], facets=h.simplices.copy(), flat=False,
                            equations=h.equations.copy())
        except QhullError:
            pass
    return HullMesh(vertices_um=np.unique(points, axis=0), facets=np.empty((0, 3), dtype=np.int64), flat=True)


# Hulls stay host Qhull; scipy's Qhull holds the GIL, so a frame's
# many small hulls are spread over worker processes (identical calls, identical
# results, original order).  Below HULL_POOL_MIN cells the pool is not worth
# its start-up; CT_HULL_PROCS=0 forces the serial loop.
HULL_POOL_MIN = 256
_hull_pool = None


def _hull_chunk(args):
    vox_list, spacing = args
    return [compute_hull(v, spacing) for v in vox_list]


def compute_hulls(vox_list, spacing: VoxelSpacing) -> list:
    """compute_hull for every voxel array of a frame, in order."""
    import os

    global _hull_pool
    procs = int(os.environ.get("CT_HULL_PROCS", str(min(16, os.cpu_count() or 1))))
    if procs <= 1 or len(vox_list) < HULL_POOL_MIN:
        return [compute_hull(v, spacing) for v in vox_list]
    from concurrent.futures.process import BrokenProcessPool

    if _hull_pool is None:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor

        import atexit

        # forkserver: workers never inherit this process's CUDA context
        _hull_pool = ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("forkserver"))
        atexit.register(_hull_pool.shutdown)
    step = max(16, len(vox_list) // (4 * procs))
    chunks = [(vox_list[i:i + step], spacing) for i in range(0, len(vox_list), step)]
    try:
        return [h for part in _hull_pool.map(_hull_chunk, chunks) for h in part]
    except BrokenProcessPool:
        # a worker died (OOM, signal): drop the pool (the next call starts a
        # fresh one) and finish this frame serially -- same calls, same results
        pool, _hull_pool = _hull_pool, None
        pool.shutdown(wait=False, cancel_futures=True)
        return [compute_hull(v, spacing) for v in vox_list]


@dataclass
class CellTable:
    """Device-resident result of K5+K6 for one frame."""

    labels: torch.Tensor     # int32 (nx,ny,nz): rank of the kept cell, -1 elsewhere
    table: torch.Tensor      # uint8 view of ct_cell rows (capacity)
    voxels: torch.Tensor     # int32 concatenated C-order linear indices
    counters: torch.Tensor   # int64[8]


def label_cells(mask: torch.Tensor, spacing: VoxelSpacing, min_volume_um3: float, id_start: int = 0,
                intensity: torch.Tensor | None = None, capacity: int = DEFAULT_COMPONENT_CAPACITY) -> CellTable:
    """K5 + K6 on a device mask (u8).  Retries with a larger component
    capacity if the first attempt overflowed (checked by the caller via
    counters; see _materialize)."""
    nx, ny, nz = (int(d) for d in mask.shape)
    n = nx * ny * nz
    cap = max(1, min(capacity, n))
    labels = _dev.empty((nx, ny, nz), torch.int32)
    fg = _dev.empty(n, torch.int32)
    counters = _dev.zeros(8, torch.int64)
    s = _dev.stream_handle()
    call("ct_ccl26", mask.data_ptr(), nx, ny, nz, labels.data_ptr(), fg.data_ptr(), counters.data_ptr(), s)
    work = _dev.empty(workspace_bytes(2, nx, ny, nz, cap), torch.uint8)
    table = _dev.empty(cap * CELL_DTYPE.itemsize, torch.uint8)
    voxels = _dev.empty(n, torch.int32)
    icode = _dev.ct_code(intensity) if intensity is not None else 0
    call(
        "ct_cell_table", labels.data_ptr(), nx, ny, nz, fg.data_ptr(), counters.data_ptr(),
        intensity.data_ptr() if intensity is not None else None, icode,
        spacing.dx, spacing.dy, spacing.dz, float(min_volume_um3), int(id_start), cap,
        work.data_ptr(), table.data_ptr(), voxels.data_ptr(), s,
    )
    return CellTable(labels=labels, table=table, voxels=voxels, counters=counters)


def read_table(ct: CellTable):
    """(counters, rows) on the host; rows is a structured CELL_DTYPE array."""
    cnt = ct.counters.cpu().numpy()
    nk = int(cnt[CNT_KEPT])
    rows = ct.table[: nk * CELL_DTYPE.itemsize].cpu().numpy().view(CELL_DTYPE)
    return cnt, rows


def _materialize(ct: CellTable, dims, spacing: VoxelSpacing, frame: int, with_hull: bool = True, table=None):
    """Detection objects of a cell table (``table`` = a (counters, rows) pair
    already read back, else read here)."""
    cnt, rows = table if table is not None else read_table(ct)
    if cnt[CNT_OVERFLOW]:
        return None
    nv = int(cnt[CNT_KEPT_VOXELS])
    _, ny, nz = dims
    lin = ct.voxels[:nv].to(torch.int64)
    coords = torch.stack((lin // (ny * nz), (lin // nz) % ny, lin % nz), dim=1).cpu().numpy()
    # one C-level split into per-cell views (the voxel lists are concatenated
    # in id order) and positional construction: per-row field access and
    # keyword dataclass init dominated the host side of materialisation
    cnts = rows["count"].astype(np.int64)
    offs = np.concatenate(([0], np.cumsum(cnts))).tolist()
    voxs = [coords[a:b] for a, b in zip(offs[:-1], offs[1:])]  # (np.split: ~1.5 us of swapaxes per view)
    ids, vols = rows["id"].tolist(), rows["volume_um3"].tolist()
    cents = list(np.array(rows["centroid_um"], dtype=np.float64))
    bbox = list(np.concatenate([rows["bbox_lo"], rows["bbox_hi"]], axis=1).astype(np.int64))
    means = [None if m != m else m for m in rows["mean_intensity"].tolist()]  # NaN: no intensity given
    hulls = compute_hulls(voxs, spacing) if with_hull else [None] * len(voxs)
    return [Detection(i, frame, v, c, vol, h, b, m)
            for i, v, c, vol, h, b, m in zip(ids, voxs, cents, vols, hulls, bbox, means)]


def _intensity_dev(intensity, shape):
    """Optional raw intensity volume (U8/U16, the mask's shape) on the device."""
    if intensity is None:
        return None
    t = _dev.to_device(intensity, allow=(torch.uint8, torch.uint16))
    if t.dtype not in (torch.uint8, torch.uint16) or tuple(t.shape) != tuple(shape):
        raise ParameterError(f"intensity must be a uint8/uint16 volume of shape {tuple(shape)}")
    return t


def _detections_dev(mask: torch.Tensor, spacing, frame, min_volume_um3, id_start, with_hull=True, intensity=None):
    cap = DEFAULT_COMPONENT_CAPACITY
    inten = _intensity_dev(intensity, mask.shape)
    while True:
        ct = label_cells(mask, spacing, min_volume_um3, id_start, intensity=inten, capacity=cap)
        dets = _materialize(ct, tuple(int(d) for d in mask.shape), spacing, frame, with_hull)
        if dets is not None:
            return dets
        cap *= 4


def detections_from_mask(mask, spacing: VoxelSpacing, frame: int, min_volume_um3: float,
                         id_start: int = 0, intensity=None) -> list[Detection]:
    """Label a mask and build volume-filtered detections: ids by (-count,
    first voxel) from id_start (ref segment.py:242-276).  ``intensity``
    (extension, optional): the raw uint8/uint16 volume whose per-cell mean
    fills ``Detection.mean_intensity``."""
    m = _dev.to_device(mask, allow=(torch.uint8,))
    if m.dtype != torch.uint8:
        m = (m != 0).to(torch.uint8)
    return _detections_dev(m, spacing, frame, min_volume_um3, id_start, intensity=intensity)


def segment_cell_channel(grid: VoxelGrid, config: SegmentationConfig | None = None, frame: int = 0,
                         id_start: int = 0, intensity=None) -> list[Detection]:
    """Segment a denoised cell-channel frame into detections (ref segment.py:279-289).
    ``intensity`` as in detections_from_mask (the frame's raw volume)."""
    config = config or SegmentationConfig()
    v = _dev.to_device(grid.values)
    mask, res = _binarize_dev(v, config.closing_radius)
    _check_otsu(res)
    return _detections_dev(mask, grid.spacing, frame, config.min_volume_um3, id_start, intensity=intensity)


# ---------------------------------------------------------------------------
# vessels
# ---------------------------------------------------------------------------
def _edt_dev(mask: torch.Tensor, spacing: VoxelSpacing) -> torch.Tensor:
    nx, ny, nz = (int(d) for d in mask.shape)
    out = _dev.empty((nx, ny, nz), torch.float64)
    work = _dev.empty(workspace_bytes(3, nx, ny, nz), torch.uint8)
    call("ct_edt", mask.data_ptr(), nx, ny, nz, spacing.dx, spacing.dy, spacing.dz, work.data_ptr(),
         out.data_ptr(), _dev.stream_handle())
    return out


def distance_map(vessel_mask, spacing: VoxelSpacing) -> DistanceMap:
    """Exact Euclidean distance transform in um (ref segment.py:292-304)."""
    if _dev.is_torch(vessel_mask):
        if vessel_mask.numel() == 0:
            raise ParameterError("mask has no voxels")
    else:
        vessel_mask = np.asarray(vessel_mask, dtype=bool)
        if vessel_mask.size == 0:
            raise ParameterError("mask has no voxels")
    m = _dev.to_device(vessel_mask, allow=(torch.uint8,))
    if m.dtype != torch.uint8:
        m = (m != 0).to(torch.uint8)
    if not bool(m.any()):
        vals = torch.full(tuple(m.shape), float("inf"), dtype=torch.float64, device=m.device)
        return DistanceMap(values=_dev.like_input(vals, vessel_mask), spacing=spacing, empty=True)
    return DistanceMap(values=_dev.like_input(_edt_dev(m, spacing), vessel_mask), spacing=spacing, empty=False)


def segment_vessel_channel(grid: VoxelGrid, config: SegmentationConfig | None = None):
    """Vessel mask and distance map (ref segment.py:307-318)."""
    config = config or SegmentationConfig()
    v = _dev.to_device(grid.values)
    mask, res = _binarize_dev(v, config.closing_radius)
    _check_otsu(res)
    if not bool(mask.any()):
        vals = torch.full(tuple(mask.shape), float("inf"), dtype=torch.float64, device=mask.device)
        dm = DistanceMap(values=_dev.like_input(vals, grid.values), spacing=grid.spacing, empty=True)
    else:
        dm = DistanceMap(values=_dev.like_input(_edt_dev(mask, grid.spacing), grid.values), spacing=grid.spacing)
    return _dev.like_input(mask.bool(), grid.values), dm


# ---------------------------------------------------------------------------
# voxel-run codec (export format, host side; ref segment.py:321-351)
# ---------------------------------------------------------------------------
def encode_voxel_runs(voxels: np.ndarray) -> list[list[int]]:
    """Run-length encode (n,3) voxels along z as [i, j, k0, length]."""
    v = np.asarray(voxels, dtype=np.int64).reshape(-1, 3)
    if v.shape[0] == 0:
        return []
    v = v[np.lexsort((v[:, 2], v[:, 1], v[:, 0]))]
    brk = np.ones(v.shape[0], dtype=bool)
    brk[1:] = (v[1:, 0] != v[:-1, 0]) | (v[1:, 1] != v[:-1, 1]) | (v[1:, 2] != v[:-1, 2] + 1)
    starts = np.flatnonzero(brk)
    lengths = np.diff(np.append(starts, v.shape[0]))
    return [[int(a), int(b), int(c), int(n)] for (a, b, c), n in zip(v[starts], lengths)]


def cell_runs(ct: CellTable, dims, cap_runs: int | None = None):
    """encode_voxel_runs of every kept cell of a device CellTable, computed on
    the GPU (ct_voxel_runs): returns (runs int32 (R, 4) = [i, j, k0, length],
    offsets int64 (ncells + 1)); cell r's runs are runs[offsets[r]:offsets[r+1]],
    identical to encode_voxel_runs(detections[r].voxels)."""
    _, ny, nz = (int(d) for d in dims)
    cnt = ct.counters.cpu().numpy()
    nk = int(cnt[CNT_KEPT])
    nv = int(cnt[CNT_KEPT_VOXELS])
    cap = int(cap_runs if cap_runs is not None else max(nv, 1))
    dev = ct.voxels.device
    runs = torch.empty((cap, 4), dtype=torch.int32, device=dev)
    offs = torch.empty(nk + 1, dtype=torch.int64, device=dev)
    nr = torch.zeros(2, dtype=torch.int64, device=dev)
    call("ct_voxel_runs", ct.voxels.data_ptr(), ct.table.data_ptr(), ct.counters.data_ptr(), ny, nz, cap,
         runs.data_ptr(), offs.data_ptr(), nr.data_ptr(), _dev.stream_handle())
    n_runs, over = (int(x) for x in nr.cpu())
    if over:
        raise RuntimeError(f"{n_runs} runs exceed cap_runs={cap}")
    return runs[:n_runs].cpu().numpy(), offs.cpu().numpy()


def decode_voxel_runs(runs: list[list[int]]) -> np.ndarray:
    """Inverse of encode_voxel_runs."""
    if not runs:
        return np.empty((0, 3), dtype=np.int64)
    r = np.asarray(runs, dtype=np.int64)
    lengths = r[:, 3]
    rep = np.repeat(np.arange(r.shape[0]), lengths)
    first = np.repeat(np.cumsum(lengths) - lengths, lengths)
    k = r[rep, 2] + (np.arange(rep.size) - first)
    return np.stack([r[rep, 0], r[rep, 1], k], axis=1)
