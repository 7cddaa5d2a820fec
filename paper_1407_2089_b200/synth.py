"""Synthetic 5-D stacks for parity tests and the benchmark.

The reference's own generator (ref synth.py) writes noiseless TIFF scenes; the
benchmark needs noisy frames at sizes where storing stacks is impractical, so
frames here are counter-based: voxel values are a pure function of
(seed, linear index, object lists), generated on the device by
``ct_synth_frame`` and bit-identically on the CPU by the oracle
(``oracle/ct_oracle.c``).  Object lists (cell balls, vessel tubes) are drawn
on the host with numpy's default_rng and expressed in 1/16-voxel fixed point
so both generators use integer arithmetic only.

  cell channel  : clip(0.08 vmax + 0.04 vmax (x/nx + y/ny) + noise + 0.6 vmax * ball, 0, vmax)
  vessel channel: the same background + 0.5 vmax inside x-aligned tubes
  noise         : Irwin-Hall of 4 hash bytes, std ~0.03 vmax
  seeds         : frame t, channel c -> 1000*c + t (+ 10^6 * scene seed)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from ._lib import CT_U8, CT_U16, call

# channels: the reference processes the first cell and the first vessel
# channel (ref session.py:286-289); CELL2 is C3's third channel, a second cell
# population segmented through the cell path directly (an extension)
CELL, VESSEL, CELL2 = 0, 1, 2


@dataclass(frozen=True)
class SceneSpec:
    nx: int
    ny: int
    nz: int
    dtype: str = "u8"          # "u8" or "u16" (12-bit)
    n_cells: int = 50
    r_min: float = 2.5         # ball radius range (voxels)
    r_max: float = 4.5
    drift: float = 2.0         # max centre drift per frame (voxels)
    n_tubes: int = 3
    tube_r: tuple = (2.0, 4.0)
    seed: int = 0

    @property
    def dims(self):
        return (self.nx, self.ny, self.nz)

    @property
    def vmax(self) -> int:
        return 255 if self.dtype == "u8" else 4095

    @property
    def np_dtype(self):
        return np.uint8 if self.dtype == "u8" else np.uint16

    @property
    def torch_dtype(self):
        return torch.uint8 if self.dtype == "u8" else torch.uint16

    @property
    def ct_code(self) -> int:
        return CT_U8 if self.dtype == "u8" else CT_U16

    @property
    def amp_cell(self) -> int:
        return (self.vmax * 6) // 10

    @property
    def amp_tube(self) -> int:
        return self.vmax // 2

    def frame_seed(self, t: int, channel: int) -> int:
        return 1000 * channel + t + 1_000_000 * self.seed

    def balls(self, t: int, channel: int = CELL) -> np.ndarray:
        """(n_cells, 4) int64: cx16, cy16, cz16, r16 at frame t (CELL2: another population)."""
        rng = np.random.default_rng(self.seed * 7919 + 17 + (104_729 if channel == CELL2 else 0))
        n = self.n_cells
        c = rng.uniform(0.0, 1.0, size=(n, 3)) * (np.array(self.dims, dtype=float) - 1.0)
        r = rng.uniform(self.r_min, self.r_max, size=n)
        v = rng.uniform(-self.drift, self.drift, size=(n, 3))
        c16 = np.rint(c * 16).astype(np.int64) + t * np.rint(v * 16).astype(np.int64)
        hi = (np.array(self.dims, dtype=np.int64) - 1) * 16
        c16 = np.clip(c16, 0, hi)
        out = np.empty((n, 4), dtype=np.int64)
        out[:, :3] = c16
        out[:, 3] = np.rint(r * 16).astype(np.int64)
        return out

    def tubes(self) -> np.ndarray:
        """(n_tubes, 3) int64: cy16, cz16, r16 (x-aligned, static)."""
        rng = np.random.default_rng(self.seed * 104729 + 29)
        n = self.n_tubes
        cy = rng.uniform(0.1, 0.9, size=n) * (self.ny - 1)
        cz = rng.uniform(0.3, 0.7, size=n) * (self.nz - 1)
        r = rng.uniform(self.tube_r[0], self.tube_r[1], size=n)
        return np.stack([np.rint(cy * 16), np.rint(cz * 16), np.rint(r * 16)], axis=1).astype(np.int64)


def generate(spec: SceneSpec, t: int, channel: int, out: torch.Tensor | None = None,
             objects: tuple | None = None) -> torch.Tensor:
    """Frame (t, channel) generated on the current CUDA device/stream."""
    dev = _dev.require_cuda()
    if out is None:
        out = torch.empty(spec.dims, dtype=spec.torch_dtype, device=dev)
    if objects is None:
        balls = torch.from_numpy(spec.balls(t, channel)).to(dev) if channel in (CELL, CELL2) else None
        tubes = torch.from_numpy(spec.tubes()).to(dev) if channel == VESSEL else None
    else:
        balls, tubes = objects
    call(
        "ct_synth_frame", out.data_ptr(), spec.ct_code, spec.nx, spec.ny, spec.nz,
        spec.frame_seed(t, channel), spec.vmax,
        balls.data_ptr() if balls is not None else None, 0 if balls is None else balls.shape[0], spec.amp_cell,
        tubes.data_ptr() if tubes is not None else None, 0 if tubes is None else tubes.shape[0], spec.amp_tube,
        _dev.stream_handle(),
    )
    return out


# benchmark / parity configurations of BASELINE.json.  Cell and vessel
# densities are those of C1 (50 cells per 256x256x32; 3 tubes per 256x32
# y-z cross-section): with only 3 tubes a 1024x1024 frame is 0.2% vessel and
# Otsu splits the background ramp instead (82% "vessel"), which the
# reference's vessel channel ("foreground covers large regions",
# ref denoise.py:5-7) is not.
C1 = SceneSpec(256, 256, 32, "u8", n_cells=50, n_tubes=3)
C2 = SceneSpec(1024, 1024, 64, "u8", n_cells=1600, n_tubes=24)
C3 = SceneSpec(1024, 1024, 64, "u16", n_cells=1600, n_tubes=24)
C4 = SceneSpec(4096, 4096, 96, "u8", n_cells=20000, r_min=3.0, r_max=6.0, n_tubes=144)
# a 1024 x 1024 x 96 crop of C4 at C4's density (parity-test size; nz = 96 kernels)
C4_CROP = SceneSpec(1024, 1024, 96, "u8", n_cells=1250, r_min=3.0, r_max=6.0, n_tubes=36, seed=4)
