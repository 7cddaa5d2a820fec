"""Boundary types of the segmentation path (ref imaging.py:25-79, 270-272).

``VoxelGrid.values`` may be a numpy array (host; results come back as numpy,
which is how the reference's tests drive the API) or a torch CUDA tensor
(device-resident; results stay on the device).  Grids are indexed
``values[i, j, k]`` for voxel (x, y, z), z fastest; voxel (i, j, k) sits at
(i*dx, j*dy, k*dz) micrometres.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ManifestError


@dataclass(frozen=True)
class VoxelSpacing:
    """Physical voxel pitch in micrometres along x, y, z."""

    dx: float
    dy: float
    dz: float

    def __post_init__(self):
        for name in ("dx", "dy", "dz"):
            v = getattr(self, name)
            if not (math.isfinite(v) and v > 0):
                raise ManifestError(f"spacing {name} must be finite and positive, got {v}")

    def as_array(self) -> np.ndarray:
        return np.array([self.dx, self.dy, self.dz], dtype=float)

    @property
    def voxel_volume_um3(self) -> float:
        # Python float product, left to right: the volume filter compares
        # count * this value in float64 (ref segment.py:250-255)
        return self.dx * self.dy * self.dz


@dataclass(frozen=True)
class VoxelGrid:
    """One channel of one time point: a 3-D intensity array with spacing."""

    values: object  # numpy.ndarray or torch.Tensor
    spacing: VoxelSpacing

    def __post_init__(self):
        if self.values.ndim != 3:
            raise ValueError(f"grid must be 3-D, got shape {tuple(self.values.shape)}")

    @property
    def dims(self) -> tuple[int, int, int]:
        return tuple(int(s) for s in self.values.shape)

    @property
    def voxel_count(self) -> int:
        n = 1
        for s in self.values.shape:
            n *= int(s)
        return n

    def with_values(self, values) -> "VoxelGrid":
        return VoxelGrid(values=values, spacing=self.spacing)


def physical_coordinates(voxels: np.ndarray, spacing: VoxelSpacing) -> np.ndarray:
    """Voxel-centre positions in micrometres for an (n, 3) index array."""
    return np.asarray(voxels, dtype=np.float64) * spacing.as_array()


def load_tiff_volume(path, device=None, threads: int = 8):
    """ref imaging.py:211-220 -- see ingest.load_tiff_volume (pread of the page
    bytes on the host, (z, y, x) -> (x, y, z) transpose on the device)."""
    from .ingest import load_tiff_volume as _load

    return _load(path, device=device, threads=threads)


def save_grid(grid: VoxelGrid, path) -> None:
    """ref imaging.py:232-240 -- see ingest.save_grid."""
    from .ingest import save_grid as _save

    _save(grid, path)
