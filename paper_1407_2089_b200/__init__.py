"""B200-native (sm_100a) per-frame 3-D segmentation for LEVER 3-D (arXiv 1407.2089).

A drop-in for the reference's hot path (clonetrack.denoise / clonetrack.segment):
same names, signatures, dataclasses and exceptions, computed by the CUDA kernels
of libct.so (include/ct.h).  ``pipeline.FramePipeline`` is the fused,
device-resident per-frame path; ``distributed`` shards frames over GPUs.
"""

from .denoise import CellDenoiseParams, MrfState, denoise_cell_channel, mrf_denoise, mrf_denoise_state
from .errors import (
    ClonetrackError,
    DegenerateHistogramError,
    EmptyDistanceMapError,
    ManifestError,
    ParameterError,
)
from .imaging import VoxelGrid, VoxelSpacing, load_tiff_volume, physical_coordinates, save_grid
from .segment import (
    Detection,
    DistanceMap,
    HullMesh,
    SegmentationConfig,
    segment_cell_channel,
    segment_vessel_channel,
)

__version__ = "0.1.0"

__all__ = [
    "CellDenoiseParams",
    "ClonetrackError",
    "DegenerateHistogramError",
    "Detection",
    "DistanceMap",
    "EmptyDistanceMapError",
    "HullMesh",
    "ManifestError",
    "MrfState",
    "ParameterError",
    "SegmentationConfig",
    "VoxelGrid",
    "VoxelSpacing",
    "denoise_cell_channel",
    "mrf_denoise",
    "mrf_denoise_state",
    "load_tiff_volume",
    "physical_coordinates",
    "save_grid",
    "segment_cell_channel",
    "segment_vessel_channel",
]
