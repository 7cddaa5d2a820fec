"""Fused, device-resident per-frame segmentation (the benchmark path).

``FramePipeline`` preallocates every buffer for one volume shape and issues
the whole per-(frame, channel) hot path as stream-ordered libct launches with
no host synchronisation:

  cell   : K1 Gaussian+residual+quantise (raw -> q) -> K2 integer median with
           fused histogram -> K3 Otsu -> K4 threshold+closing -> K5 CCL ->
           K6 per-cell table (canonical ids, bbox, intensity sums, C-order
           voxel lists, bit-exact centroids)
  vessel : K7 MRF statistics (delta, sigma_hat, first-step decision, input
           histogram) -> K3 Otsu -> K4 threshold+closing -> K8 EDT

It relies on two exact identities, verified by the parity tests:
  * rint(median(r)) == median(rint(r)) (rint and the order statistic are
    monotone), so segmenting median(q) with q = rint(residual) equals the
    reference's binarize(denoise_cell_channel(raw));
  * the MRF stops before its first step on realistic volumes (decision 0),
    in which case its output is the input as float64 and its histogram is the
    input's; any other decision is finished through the drop-in API
    (``finish_vessel``), which reproduces the reference in every case.
Data-dependent errors (DegenerateHistogramError) surface in ``finish_*``.

Stream contract: every launch goes to the current torch stream, and a
result's buffers (labels, table, voxel lists, mask, distance) are reused by
the next ``cell()`` / ``vessel()`` call of the same pipeline (the next
frame's K5 first resets the previous frame's foreground labels to -1).  A
result is valid only until that call, for work ordered after it on the
launching stream; a consumer on any other stream must make the launching
stream wait for it first.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from ._lib import (
    CELL_DTYPE,
    CNT_KEPT,
    CNT_OVERFLOW,
    MRF_DECISION,
    OTSU_STATUS,
    call,
    workspace_bytes,
)
from .denoise import CellDenoiseParams, device_taps, mrf_denoise
from .errors import DegenerateHistogramError, ParameterError
from .imaging import VoxelGrid, VoxelSpacing
from .segment import CellTable, DistanceMap, SegmentationConfig, _materialize, segment_vessel_channel


@dataclass
class CellResult:
    frame: int
    id_start: int
    cells: CellTable
    otsu: torch.Tensor  # int64[4]


@dataclass
class VesselResult:
    mask: torch.Tensor      # u8
    distance: torch.Tensor  # f64
    state: torch.Tensor     # f64[9]
    otsu: torch.Tensor      # int64[4]


class FramePipeline:
    def __init__(self, dims, dtype: str, spacing: VoxelSpacing, denoise: CellDenoiseParams | None = None,
                 seg: SegmentationConfig | None = None, capacity: int = 1 << 20, cell: bool = True,
                 vessel: bool = True, device=None):
        self.dims = tuple(int(d) for d in dims)
        nx, ny, nz = self.dims
        n = nx * ny * nz
        self.n = n
        self.dtype = dtype
        self.tdtype = torch.uint8 if dtype == "u8" else torch.uint16
        self.code = 1 if dtype == "u8" else 2
        # u8 volumes (and the u8-stored median) never exceed 255, so the
        # reference's intensity_histogram has exactly 256 bins (segment.py:161)
        self.nbins = 256 if dtype == "u8" else 0
        self.spacing = spacing
        self.denoise = denoise or CellDenoiseParams()
        self.seg = seg or SegmentationConfig()
        dev = device or _dev.require_cuda()
        self.device = dev
        self.marks = None  # list of (stage, start_event, end_event) when timing
        self.exact_k1 = False  # True: scipy-order K1 (no FMA fast path)
        self.k1_path = 0       # ct_gaussian_q path: 0 auto, 1 FP64 FMA, 2 tensor cores
        self.k1_eps = 0.0      # ct_gaussian_q eps_override (0: the certified bound; tests force the fix-up)
        E = lambda shape, dt: torch.empty(shape, dtype=dt, device=dev)  # noqa: E731
        Z = lambda shape, dt: torch.zeros(shape, dtype=dt, device=dev)  # noqa: E731
        cr = self.seg.closing_radius
        if cell:
            sig = tuple(self.denoise.gaussian_sigma_um / s for s in (spacing.dx, spacing.dy, spacing.dz))
            for s_, d_ in zip(sig, self.dims):
                if s_ > d_:
                    raise ParameterError(
                        f"gaussian kernel scale {s_:.1f} voxels exceeds grid extent {d_}; "
                        f"reduce gaussian_sigma_um ({self.denoise.gaussian_sigma_um})"
                    )
            self.w, self.r = device_taps(sig, dev)
            self.gwork = E(2 * n, torch.float64)
            self.fix_cap = 1 << 20
            self.fix = Z(2 + self.fix_cap, torch.int64)  # certified-K1 fix-up list
            self.q = E(self.dims, self.tdtype)
            self.med = E(self.dims, self.tdtype)
            self.hist = Z(65536, torch.int64)
            self.otsu = Z(4, torch.int64)
            self.labels = E(self.dims, torch.int32)
            self.fg = E(n, torch.int32)
            self.counters = Z(8, torch.int64)
            self.cap = max(1, min(capacity, n))
            self.twork = E(workspace_bytes(2, nx, ny, nz, self.cap), torch.uint8)
            self.table = E(self.cap * CELL_DTYPE.itemsize, torch.uint8)
            self.voxels = E(n, torch.int32)
            self.cwork = E(workspace_bytes(1, nx, ny, nz, cr), torch.uint8) if cr >= 1 else None
            # K4 -> K5 through packed z-rows (r == 1, nz <= 128): the closed mask
            # is never materialised as bytes on the fused path
            self.rows_path = cr == 1 and nz <= 128 and nz % 4 == 0
            self.crows = E(nx * ny * (1 if nz <= 64 else 2), torch.int64) if self.rows_path else None
            self.mask = None if self.rows_path else E(self.dims, torch.uint8)
            if self.rows_path:
                # -1 everywhere once; afterwards each frame's K5 resets only the
                # previous frame's foreground (CT_LABELS_RESET: fg list + count
                # kept in fg / counters), not the whole volume
                call("ct_memset", self.labels.data_ptr(), 0xFF, self.labels.numel() * 4, _dev.stream_handle())
        if vessel:
            self.mwork = E(workspace_bytes(4, nx, ny, nz, self.code), torch.uint8)
            self.state = Z(9, torch.float64)
            self.vhist = Z(65536, torch.int64)
            self.votsu = Z(4, torch.int64)
            self.vmask = E(self.dims, torch.uint8)
            self.ework = E(workspace_bytes(3, nx, ny, nz), torch.uint8)
            self.dist = E(self.dims, torch.float64)
            self.vcwork = E(workspace_bytes(1, nx, ny, nz, cr), torch.uint8) if cr >= 1 else None

    # -- optional per-stage CUDA events (on the launching stream) -----------
    def _t0(self):
        if self.marks is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def _t1(self, stage, e0):
        if e0 is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.marks.append((stage, e0, e))

    def stage_times_ms(self) -> dict:
        """Mean milliseconds per stage over the recorded marks (synchronises)."""
        out: dict = {}
        for stage, a, b in self.marks or []:
            b.synchronize()
            out.setdefault(stage, []).append(a.elapsed_time(b))
        return {k: float(np.mean(v)) for k, v in out.items()}

    # -- launches (current torch stream; no host sync) ---------------------
    @property
    def k1_path_tc(self) -> bool:
        """True when K1 runs on the tensor cores (ct_k1_path == 2)."""
        if self.exact_k1 or not hasattr(self, "w"):
            return False
        from ._lib import lib
        nx, ny, nz = self.dims
        return lib().ct_k1_path(self.code, nx, ny, nz, *self.r, self.k1_path) == 2

    def cell(self, raw: torch.Tensor, frame: int = 0, id_start: int = 0) -> CellResult:
        nx, ny, nz = self.dims
        s = _dev.stream_handle()
        rx, ry, rz = self.r
        # only the bins the median can touch: 256 for u8 (the reference's nbins), all 65536 for u16
        call("ct_memset", self.hist.data_ptr(), 0, (256 if self.code == 1 else 65536) * 8, s)
        e = self._t0()
        if self.exact_k1:
            call("ct_gaussian_residual", raw.data_ptr(), self.code, nx, ny, nz, self.w.data_ptr(), rx, ry, rz,
                 self.gwork.data_ptr(), None, None, self.q.data_ptr(), self.code, s)
            self.fix[:2].zero_()
        else:
            call("ct_gaussian_q", raw.data_ptr(), self.code, nx, ny, nz, self.w.data_ptr(), rx, ry, rz,
                 self.gwork.data_ptr(), self.q.data_ptr(), self.fix.data_ptr(), self.fix_cap, self.k1_eps,
                 self.k1_path, s)
        self._t1("K1 gaussian", e)
        e = self._t0()
        call("ct_median", self.q.data_ptr(), self.code, nx, ny, nz, self.denoise.median_radius,
             self.med.data_ptr(), self.hist.data_ptr(), s)
        self._t1("K2 median+hist", e)
        e = self._t0()
        call("ct_otsu", self.hist.data_ptr(), self.nbins, self.otsu.data_ptr(), s)
        self._t1("K3 otsu", e)
        e = self._t0()
        if self.rows_path:
            call("ct_threshold_close_rows", self.med.data_ptr(), self.code, nx, ny, nz, self.otsu.data_ptr(), 0,
                 None, self.crows.data_ptr(), self.cwork.data_ptr(), s)
        else:
            call("ct_threshold_close", self.med.data_ptr(), self.code, nx, ny, nz, self.otsu.data_ptr(), 0,
                 self.seg.closing_radius, self.mask.data_ptr(),
                 self.cwork.data_ptr() if self.cwork is not None else None, s)
        self._t1("K4 threshold+close", e)
        e = self._t0()
        if self.rows_path:
            call("ct_ccl26_rows", self.crows.data_ptr(), nx, ny, nz, self.labels.data_ptr(), self.fg.data_ptr(),
                 self.counters.data_ptr(), 2, s)  # CT_LABELS_RESET
        else:
            call("ct_ccl26", self.mask.data_ptr(), nx, ny, nz, self.labels.data_ptr(), self.fg.data_ptr(),
                 self.counters.data_ptr(), s)
        self._t1("K5 ccl", e)
        e = self._t0()
        sp = self.spacing
        call("ct_cell_table", self.labels.data_ptr(), nx, ny, nz, self.fg.data_ptr(), self.counters.data_ptr(),
             raw.data_ptr(), self.code, sp.dx, sp.dy, sp.dz, float(self.seg.min_volume_um3), int(id_start),
             self.cap, self.twork.data_ptr(), self.table.data_ptr(), self.voxels.data_ptr(), s)
        self._t1("K6 table", e)
        return CellResult(frame=frame, id_start=id_start,
                          cells=CellTable(self.labels, self.table, self.voxels, self.counters), otsu=self.otsu)

    def vessel(self, raw: torch.Tensor) -> VesselResult:
        nx, ny, nz = self.dims
        s = _dev.stream_handle()
        call("ct_memset", self.vhist.data_ptr(), 0, (256 if self.code == 1 else 65536) * 8, s)
        e = self._t0()
        call("ct_mrf_decide", raw.data_ptr(), self.code, nx, ny, nz, self.mwork.data_ptr(), self.state.data_ptr(),
             self.vhist.data_ptr(), s)
        self._t1("K7 mrf", e)
        e = self._t0()
        call("ct_otsu", self.vhist.data_ptr(), self.nbins, self.votsu.data_ptr(), s)
        call("ct_threshold_close", raw.data_ptr(), self.code, nx, ny, nz, self.votsu.data_ptr(), 0,
             self.seg.closing_radius, self.vmask.data_ptr(),
             self.vcwork.data_ptr() if self.vcwork is not None else None, s)
        self._t1("K3+K4 vessel otsu+close", e)
        e = self._t0()
        sp = self.spacing
        call("ct_edt", self.vmask.data_ptr(), nx, ny, nz, sp.dx, sp.dy, sp.dz, self.ework.data_ptr(),
             self.dist.data_ptr(), s)
        self._t1("K8 edt", e)
        return VesselResult(mask=self.vmask, distance=self.dist, state=self.state, otsu=self.votsu)

    # -- CUDA graphs ---------------------------------------------------------
    def capture(self, fn) -> "torch.cuda.CUDAGraph":
        """Capture ``fn()`` -- e.g. ``lambda: pipe.cell(raw)`` or
        ``lambda: pipe.vessel(raw)`` -- as a CUDA graph: every launch of the
        frame (torch's and libct's) in one graph.  ``graph.replay()`` on a
        stream re-runs the frame on the same buffers and input address with no
        per-kernel host launch cost, in that stream's order (so a cell graph
        replayed on one stream and a vessel graph on another overlap as the
        eager launches do).  Run ``fn`` once eagerly before capturing (module
        load, function attributes); results are read as after ``cell`` /
        ``vessel``."""
        assert self.marks is None, "stage timing marks cannot be captured"
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.graph(g, stream=side, capture_error_mode="relaxed"):
            fn()
        torch.cuda.current_stream(self.device).wait_stream(side)
        return g

    # -- host-side completion (synchronises) --------------------------------
    def finish_cell(self, res: CellResult, materialize: bool = False, with_hull: bool = False, table=None):
        """Raise reference errors; return (counters, rows) or Detections
        (``table``: the (counters, rows) pair of an earlier call, not re-read)."""
        if int(res.otsu[OTSU_STATUS].item()) == 2:
            raise DegenerateHistogramError("frame is constant; no threshold separates it")
        cnt = res.cells.counters.cpu().numpy()
        if cnt[CNT_OVERFLOW]:
            raise RuntimeError("component capacity exceeded; raise FramePipeline(capacity=...)")
        if materialize:
            return _materialize(res.cells, self.dims, self.spacing, res.frame, with_hull, table)
        nk = int(cnt[CNT_KEPT])
        rows = res.cells.table[: nk * CELL_DTYPE.itemsize].cpu().numpy().view(CELL_DTYPE)
        return cnt, rows

    def finish_vessel(self, res: VesselResult, raw: torch.Tensor, max_iters: int = 1000):
        """(mask, DistanceMap) exactly as segment_vessel_channel(mrf_denoise(raw, max_iters))."""
        decision = int(res.state[MRF_DECISION].item())
        if decision != 0:
            vden = mrf_denoise(VoxelGrid(values=raw, spacing=self.spacing), max_iters=max_iters)
            return segment_vessel_channel(vden, self.seg)
        if int(res.otsu[OTSU_STATUS].item()) == 2:
            raise DegenerateHistogramError("frame is constant; no threshold separates it")
        empty = not bool(res.mask.any())
        vals = res.distance
        return res.mask.bool(), DistanceMap(values=vals, spacing=self.spacing, empty=empty)
