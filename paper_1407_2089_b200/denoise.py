"""Channel-specific background and noise removal on the B200.

Drop-in for ref denoise.py (same names, signatures, dataclasses, exceptions);
every computation is a libct kernel (include/ct.h):

* cell channel (ref denoise.py:67-89): Gaussian background (K1, scipy's exact
  float64 accumulation order), residual clamp, median (K2);
* vessel channel (ref denoise.py:92-195): intensity step, noise estimate in
  numpy's pairwise-summation order, and the synchronous sign-sum iteration
  (K7), whose rare extra iterations are driven from here one launch each.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from ._lib import (
    CT_F64,
    CT_U8,
    CT_U16,
    MRF_DECISION,
    MRF_DELTA,
    MRF_SIGMA,
    MRF_SIGMA_STATUS,
    MRF_WORDS,
    call,
    workspace_bytes,
)
from .errors import ParameterError
from .imaging import VoxelGrid

logger = logging.getLogger(__name__)

GAUSSIAN_TRUNCATE = 4.0


@dataclass(frozen=True)
class CellDenoiseParams:
    """Cell-channel background model parameters (ref denoise.py:28-43)."""

    gaussian_sigma_um: float = 10.0
    median_radius: int = 1

    def __post_init__(self):
        if self.gaussian_sigma_um <= 0:
            raise ParameterError(f"gaussian sigma must be positive, got {self.gaussian_sigma_um}")
        if self.median_radius < 1:
            raise ParameterError(f"median radius must be >= 1, got {self.median_radius}")


@dataclass
class MrfState:
    """Result of the iterative vessel denoise (ref denoise.py:46-55)."""

    original: VoxelGrid
    current: VoxelGrid
    sigma_hat: float
    delta: float
    iteration: int
    converged: bool = True


def _sigma_voxels(params: CellDenoiseParams, grid: VoxelGrid) -> tuple[float, float, float]:
    s = grid.spacing
    return (params.gaussian_sigma_um / s.dx, params.gaussian_sigma_um / s.dy, params.gaussian_sigma_um / s.dz)


def gaussian_taps(sigma: float) -> tuple[np.ndarray, int]:
    """One-sided weights w[0..r] (w[j] = tap at distance j) and radius r of
    scipy's order-0 kernel (scipy _filters.py:656-686, radius int(4s+0.5));
    r = -1 when scipy skips the axis (sigma <= 1e-15)."""
    if not sigma > 1e-15:
        return np.zeros(0), -1
    r = int(GAUSSIAN_TRUNCATE * float(sigma) + 0.5)
    sigma2 = float(sigma) * float(sigma)
    x = np.arange(-r, r + 1)
    phi = np.exp(-0.5 / sigma2 * x**2)
    phi = phi / phi.sum()
    return np.ascontiguousarray(phi[r:]), r


def device_taps(sigmas, device=None) -> tuple[torch.Tensor, tuple[int, int, int]]:
    ws, rs = [], []
    for s in sigmas:
        w, r = gaussian_taps(s)
        ws.append(w)
        rs.append(r)
    w = np.concatenate(ws) if any(r >= 0 for r in rs) else np.zeros(1)
    return torch.from_numpy(w).to(device or _dev.require_cuda()), tuple(rs)


def _check_sigmas(params: CellDenoiseParams, grid: VoxelGrid):
    sigmas = _sigma_voxels(params, grid)
    for sigma, n in zip(sigmas, grid.dims):
        if sigma > n:
            raise ParameterError(
                f"gaussian kernel scale {sigma:.1f} voxels exceeds grid extent {n}; "
                f"reduce gaussian_sigma_um ({params.gaussian_sigma_um})"
            )
    return sigmas


def denoise_cell_channel(grid: VoxelGrid, params: CellDenoiseParams | None = None) -> VoxelGrid:
    """Remove low-frequency background and shot noise (ref denoise.py:67-89).

    Gaussian background (float64, scipy order) subtracted and clamped at 0,
    then the (2r+1)^3 median; returns a float64 grid like the reference.
    """
    params = params or CellDenoiseParams()
    if grid.voxel_count == 0:
        raise ParameterError("cannot denoise an empty grid")
    sigmas = _check_sigmas(params, grid)
    raw = _dev.to_device(grid.values)
    nx, ny, nz = grid.dims
    n = nx * ny * nz
    w, (rx, ry, rz) = device_taps(sigmas, raw.device)
    work = _dev.empty(2 * n, torch.float64)
    residual = _dev.empty((nx, ny, nz), torch.float64)
    s = _dev.stream_handle()
    call(
        "ct_gaussian_residual",
        raw.data_ptr(), _dev.ct_code(raw), nx, ny, nz, w.data_ptr(), rx, ry, rz,
        work.data_ptr(), None, residual.data_ptr(), None, 0, s,
    )
    del work
    out = _dev.empty((nx, ny, nz), torch.float64)
    call("ct_median", residual.data_ptr(), CT_F64, nx, ny, nz, params.median_radius, out.data_ptr(), None, s)
    return grid.with_values(_dev.like_input(out, grid.values))


# ---------------------------------------------------------------------------
# vessel channel
# ---------------------------------------------------------------------------
def _mrf_launch(values):
    """Run ct_mrf; returns (raw tensor, code, dims, work, state tensor, hist)."""
    raw = _dev.to_device(values)
    if raw.ndim != 3:
        raw = raw.reshape(-1, 1, 1)
    nx, ny, nz = (int(d) for d in raw.shape)
    code = _dev.ct_code(raw)
    work = _dev.empty(workspace_bytes(4, nx, ny, nz, code), torch.uint8)
    state = _dev.zeros(MRF_WORDS, torch.float64)
    hist = _dev.zeros(65536, torch.int64) if code in (CT_U8, CT_U16) else None
    call(
        "ct_mrf", raw.data_ptr(), code, nx, ny, nz, work.data_ptr(), state.data_ptr(),
        hist.data_ptr() if hist is not None else None, _dev.stream_handle(),
    )
    return raw, code, (nx, ny, nz), work, state, hist


def estimate_noise_variance(grid: VoxelGrid) -> float:
    """std of the interior 6-neighbour Laplacian / sqrt(42) (ref denoise.py:92-114)."""
    nx, ny, nz = grid.dims
    n_interior = max(nx - 2, 0) * max(ny - 2, 0) * max(nz - 2, 0)
    if n_interior < 2:
        raise ParameterError(f"grid dims {grid.dims} leave fewer than 2 interior voxels")
    st = _mrf_launch(grid.values)[4].cpu().numpy()
    return float(st[MRF_SIGMA])


def _neighbor_sign_sum(v) -> np.ndarray:
    """Six-direction sign sum with replicated edges (ref denoise.py:117-132)."""
    t = _dev.to_device(v)
    out = _dev.empty(tuple(t.shape), torch.int64)
    nx, ny, nz = (int(d) for d in t.shape)
    call("ct_sign_sum", t.data_ptr(), _dev.ct_code(t), nx, ny, nz, out.data_ptr(), _dev.stream_handle())
    return _dev.like_input(out, v)


def intensity_step(values) -> float:
    """Minimum gap between distinct values; 0.0 if constant (ref denoise.py:135-144)."""
    n = values.numel() if _dev.is_torch(values) else np.size(values)
    if n == 0:
        return 0.0
    st = _mrf_launch(values.reshape(-1, 1, 1))[4].cpu().numpy()
    return float(st[MRF_DELTA])


def _as_f64(raw: torch.Tensor, code: int) -> torch.Tensor:
    out = _dev.empty(tuple(raw.shape), torch.float64)
    call("ct_to_f64", raw.data_ptr(), code, raw.numel(), out.data_ptr(), _dev.stream_handle())
    return out


def mrf_denoise_state(grid: VoxelGrid, max_iters: int = 1000) -> MrfState:
    """Iterative edge-preserving vessel denoise (ref denoise.py:147-190)."""
    if grid.voxel_count == 0:
        raise ParameterError("cannot denoise an empty grid")
    raw, code, (nx, ny, nz), work, state, _ = _mrf_launch(grid.values)
    st = state.cpu().numpy()
    delta = float(st[MRF_DELTA])
    if int(st[MRF_DECISION]) == 2 or delta == 0.0:
        return MrfState(original=grid, current=grid, sigma_hat=0.0, delta=0.0, iteration=0)
    sigma_hat = 0.0 if st[MRF_SIGMA_STATUS] != 0 else float(st[MRF_SIGMA])
    iteration, converged = 0, True
    cur = None
    if int(st[MRF_DECISION]) == 0:
        if max_iters <= 0:
            converged = False
    else:
        s = _dev.stream_handle()
        bufs = [_dev.empty((nx, ny, nz), torch.float64), _dev.empty((nx, ny, nz), torch.float64)]
        out2 = _dev.zeros(2, torch.float64)
        while True:
            if iteration >= max_iters:
                converged = False
                logger.warning("vessel denoise did not terminate within %d iterations", max_iters)
                break
            nxt = bufs[iteration % 2]
            call(
                "ct_mrf_step", raw.data_ptr(), code, nx, ny, nz,
                cur.data_ptr() if cur is not None else None, state.data_ptr(), nxt.data_ptr(),
                work.data_ptr(), out2.data_ptr(), s,
            )
            norm, moved = out2.cpu().numpy()
            if norm > sigma_hat or moved == 0:
                break
            cur = nxt
            iteration += 1
    current = cur if cur is not None else _as_f64(raw, code)
    current = current.reshape(grid.dims)
    return MrfState(
        original=grid,
        current=grid.with_values(_dev.like_input(current, grid.values)),
        sigma_hat=sigma_hat,
        delta=delta,
        iteration=iteration,
        converged=converged,
    )


def mrf_denoise(grid: VoxelGrid, max_iters: int = 1000) -> VoxelGrid:
    """Edge-preserving vessel-channel denoise; see mrf_denoise_state."""
    return mrf_denoise_state(grid, max_iters=max_iters).current
