"""Ingest: TIFF stacks -> device grids (the step before the path).

ref imaging.py:211-220 ``load_tiff_volume`` decodes with tifffile into (z, y, x)
pages and transposes to an (x, y, z) C-order grid on the host;
ref imaging.py:232-240 ``save_grid`` writes the (z, y, x) transpose.  Here:

* the host only moves page bytes -- ``ct_tiff_read`` (C++, libct) preads the
  strips of every page, several threads at once, into pinned memory;
* the bytes cross PCIe once, and ``ct_transpose_xz`` (CUDA) turns (z, y, x)
  into (x, y, z) in HBM (and byte-swaps big-endian files on the way);
* ``FrameIngest`` pipelines it over a frame sequence: a reader thread fills
  pinned slot k+1 while slot k is copied and the path runs on frame k-1.

Same names, argument meaning and errors as the reference: unreadable files
raise ``ManifestError("failed to read image <path>: ...")``; a single-page
file is a stack of one z-slice (ref imaging.py:217-218).  There is no CPU
fallback for the transpose: a missing CUDA device raises.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import numpy as np

from . import _lib
from .errors import ManifestError

_FMT_DTYPE = {
    (1, 1): np.uint8, (1, 2): np.int8, (2, 1): np.uint16, (2, 2): np.int16,
    (4, 1): np.uint32, (4, 2): np.int32, (4, 3): np.float32,
    (8, 1): np.uint64, (8, 2): np.int64, (8, 3): np.float64,
}
_DTYPE_FMT = {np.dtype(v): k for k, v in _FMT_DTYPE.items()}


class TiffStack:
    """An open TIFF stack (ct_tiff_open): page geometry without reading data."""

    def __init__(self, path):
        self.path = str(path)
        self.info = _lib.TiffInfo()
        h = ctypes.c_void_p()
        st = _lib.lib().ct_tiff_open(self.path.encode(), ctypes.byref(self.info), ctypes.byref(h))
        if st != _lib.CT_OK:
            msg = _lib.lib().ct_last_error().decode(errors="replace")
            raise ManifestError(msg)
        self._h = h

    @property
    def dims(self) -> tuple[int, int, int]:
        """Grid dims (nx, ny, nz) = (page width, page height, pages)."""
        return (self.info.nx, self.info.ny, self.info.nz)

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(_FMT_DTYPE[(self.info.bytes_per_sample, self.info.sample_format)])

    @property
    def big_endian(self) -> bool:
        return bool(self.info.big_endian)

    @property
    def nbytes(self) -> int:
        return self.info.nx * self.info.ny * self.info.nz * self.info.bytes_per_sample

    def read_into(self, ptr: int, nbytes: int, threads: int = 8) -> None:
        """All pages, (z, y, x) order, file byte order, into host memory at ptr."""
        _lib.call("ct_tiff_read", self._h, ptr, nbytes, threads)

    def close(self) -> None:
        if self._h:
            _lib.lib().ct_tiff_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_tiff_pages(path, threads: int = 8) -> np.ndarray:
    """Raw pages as a host (nz, ny, nx) array in native byte order (what
    tifffile.imread returns for a grayscale stack)."""
    with TiffStack(path) as ts:
        out = np.empty((ts.info.nz, ts.info.ny, ts.info.nx), dtype=ts.dtype)
        ts.read_into(out.ctypes.data, out.nbytes, threads)
        if ts.big_endian and out.itemsize > 1:
            out.byteswap(inplace=True)
        return out


def write_tiff_pages(path, pages_zyx: np.ndarray) -> None:
    """Write a host (nz, ny, nx) array (or (ny, nx): one page) as a TIFF stack."""
    a = np.ascontiguousarray(pages_zyx)
    if a.ndim == 2:
        a = a[np.newaxis]
    if a.ndim != 3:
        raise ValueError(f"pages must be 2-D or 3-D, got shape {a.shape}")
    a = a.astype(a.dtype.newbyteorder("="), copy=False)
    key = _DTYPE_FMT.get(np.dtype(a.dtype.str.replace(">", "<")))
    if key is None:
        raise ValueError(f"unsupported sample type {a.dtype}")
    Path(path).parent.mkdir(parents=True, exist_ok=True)
    _lib.call("ct_tiff_write", str(path).encode(), a.ctypes.data, a.shape[2], a.shape[1], a.shape[0], key[0], key[1])


# ---------------------------------------------------------------------------
# device side
# ---------------------------------------------------------------------------
def _torch_dtype(dt: np.dtype):
    import torch

    return {
        np.dtype(np.uint8): torch.uint8, np.dtype(np.int8): torch.int8, np.dtype(np.uint16): torch.uint16,
        np.dtype(np.int16): torch.int16, np.dtype(np.uint32): torch.uint32, np.dtype(np.int32): torch.int32,
        np.dtype(np.float32): torch.float32, np.dtype(np.uint64): torch.uint64, np.dtype(np.int64): torch.int64,
        np.dtype(np.float64): torch.float64,
    }[np.dtype(dt)]


def transpose_xz(src, dst, na: int, nb: int, nc: int, byteswap: bool = False) -> None:
    """dst[c, b, a] = src[a, b, c] on the current stream (ct_transpose_xz)."""
    from ._dev import stream_handle

    _lib.call("ct_transpose_xz", src.data_ptr(), dst.data_ptr(), na, nb, nc, src.element_size(), int(byteswap),
              stream_handle())


def load_tiff_volume(path, device=None, threads: int = 8):
    """ref imaging.py:211-220: a multi-page TIFF as an (nx, ny, nz) grid, page
    k = z-slice k.  Returns numpy (the reference's type) unless ``device`` is
    given, in which case the grid stays on that CUDA device."""
    import torch

    from ._dev import require_cuda

    dev = require_cuda() if device is None else torch.device(device)
    with TiffStack(path) as ts:
        nx, ny, nz = ts.dims
        tdt = _torch_dtype(ts.dtype)
        host = torch.empty(ts.nbytes, dtype=torch.uint8, pin_memory=True)
        ts.read_into(host.data_ptr(), ts.nbytes, threads)
        raw = host.to(dev, non_blocking=True).view(tdt)
        grid = torch.empty((nx, ny, nz), dtype=tdt, device=dev)
        with torch.cuda.device(dev):
            transpose_xz(raw, grid, nz, ny, nx, ts.big_endian)
        if device is not None:
            return grid
        out = grid.cpu()
        if tdt in (torch.uint16, torch.uint32, torch.uint64):
            return out.view({torch.uint16: torch.int16, torch.uint32: torch.int32,
                             torch.uint64: torch.int64}[tdt]).numpy().view(ts.dtype)
        return out.numpy()


def save_grid(grid, path) -> None:
    """ref imaging.py:232-240: write a grid as a multi-page TIFF, page k =
    z-slice k.  The (x, y, z) -> (z, y, x) transpose runs on the device."""
    import torch

    from ._dev import require_cuda

    v = grid.values if hasattr(grid, "values") else grid
    dev = require_cuda()
    if isinstance(v, torch.Tensor):
        t = v.to(dev).contiguous()
        if t.dtype == torch.bool:
            t = t.to(torch.uint8)
        dt = np.dtype(str(t.dtype).replace("torch.", ""))
    else:
        a = np.ascontiguousarray(v)
        dt = a.dtype
        if a.dtype == np.bool_:
            a, dt = a.astype(np.uint8), np.dtype(np.uint8)
        if dt in (np.dtype(np.uint16), np.dtype(np.uint32), np.dtype(np.uint64)):
            t = torch.from_numpy(a.view({2: np.int16, 4: np.int32, 8: np.int64}[dt.itemsize])).to(dev)
        else:
            t = torch.from_numpy(a).to(dev)
    nx, ny, nz = (int(s) for s in t.shape)
    pages = torch.empty((nz, ny, nx), dtype=t.dtype, device=dev)
    transpose_xz(t, pages, nx, ny, nz)
    signed = {torch.uint16: torch.int16, torch.uint32: torch.int32, torch.uint64: torch.int64}
    if pages.dtype in signed:
        pages = pages.view(signed[pages.dtype])
    host = pages.cpu().numpy().view(dt)
    write_tiff_pages(path, host)


class FrameIngest:
    """Pipelined TIFF -> device grid feed over a sequence of frame files.

    A reader thread preads file k+1 into pinned slot (k+1) % depth while file
    k crosses PCIe on a copy stream and is transposed into device grid slot
    k % depth.  Iterating yields (index, grid) with ``grid`` ready on the
    current stream; a grid stays valid until ``depth`` further frames were
    yielded.  All files must share dims and sample type (the manifest's
    contract, ref imaging.py:226-228)."""

    def __init__(self, paths, depth: int = 3, threads: int = 8, device=None):
        import torch

        from ._dev import require_cuda

        self.paths = [str(p) for p in paths]
        if not self.paths:
            raise ValueError("no frames")
        self.dev = require_cuda() if device is None else torch.device(device)
        self.depth = max(2, depth)
        self.threads = threads
        with TiffStack(self.paths[0]) as ts:
            self.dims, self.dtype, self.nbytes = ts.dims, ts.dtype, ts.nbytes
        self.tdt = _torch_dtype(self.dtype)
        nx, ny, nz = self.dims
        self.pinned = [torch.empty(self.nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(self.depth)]
        self.raw = [torch.empty(self.nbytes, dtype=torch.uint8, device=self.dev) for _ in range(self.depth)]
        self.grids = [torch.empty((nx, ny, nz), dtype=self.tdt, device=self.dev) for _ in range(self.depth)]
        self.copy_stream = torch.cuda.Stream(self.dev)
        self.h2d_done = [torch.cuda.Event() for _ in range(self.depth)]
        self.consumed = [torch.cuda.Event() for _ in range(self.depth)]
        self.bytes_read = 0

    def _read(self, k: int, slot: int, swap: list) -> None:
        self.h2d_done[slot].synchronize()  # the H2D of frame k - depth has left the pinned slot
        with TiffStack(self.paths[k]) as ts:
            if ts.dims != self.dims or ts.dtype != self.dtype:
                raise ManifestError(f"image {self.paths[k]} has dims {ts.dims} {ts.dtype}, "
                                    f"expected {self.dims} {self.dtype}")
            ts.read_into(self.pinned[slot].data_ptr(), self.nbytes, self.threads)
            swap[slot] = ts.big_endian
        self.bytes_read += self.nbytes

    def __iter__(self):
        import torch

        n, D = len(self.paths), self.depth
        swap = [False] * D
        errors: list = [None] * n
        done = [threading.Event() for _ in range(n)]
        issued = [threading.Event() for _ in range(n)]  # H2D of frame k enqueued
        stop = threading.Event()

        def worker():
            for k in range(n):
                if k >= D:
                    while not issued[k - D].wait(0.05):
                        if stop.is_set():
                            return
                if stop.is_set():
                    return
                try:
                    self._read(k, k % D, swap)
                except BaseException as e:  # surfaced on the consumer side
                    errors[k] = e
                done[k].set()
                if errors[k] is not None:
                    for j in range(k + 1, n):
                        done[j].set()
                    return

        for e in self.h2d_done + self.consumed:
            e.record()
        th = threading.Thread(target=worker, daemon=True)
        th.start()
        nx, ny, nz = self.dims
        main = torch.cuda.current_stream(self.dev)
        try:
            for k in range(n):
                slot = k % D
                done[k].wait()
                if errors[k] is not None:
                    raise errors[k]
                with torch.cuda.stream(self.copy_stream):
                    self.copy_stream.wait_event(self.consumed[slot])
                    self.raw[slot].copy_(self.pinned[slot], non_blocking=True)
                    self.h2d_done[slot].record()
                    issued[k].set()
                    transpose_xz(self.raw[slot].view(self.tdt), self.grids[slot], nz, ny, nx, swap[slot])
                main.wait_stream(self.copy_stream)
                yield k, self.grids[slot]
                self.consumed[slot].record(main)
        finally:
            stop.set()
            th.join()
