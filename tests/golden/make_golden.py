"""Generate the golden fixtures in tests/golden/ from the LIVE reference.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures pin both the CPU oracle (tests/test_oracle.py) and the CUDA
path (tests/test_gpu_parity.py) to the reference's own outputs; the GPU box
has no /root/reference, only these files.

Inputs come from the seeded synthetic generator (paper_1407_2089_b200.synth
object lists + oracle/ct_oracle.c frames) and seeded numpy RNGs; outputs are
whatever the reference (clonetrack @ /root/reference/pkg/src) returns.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import _refimport  # noqa: E402

ct = _refimport.clonetrack()
from clonetrack import denoise as D  # noqa: E402
from clonetrack import segment as S  # noqa: E402
from clonetrack.imaging import VoxelGrid, VoxelSpacing  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1407_2089_b200.synth import SceneSpec  # noqa: E402

ANISO = VoxelSpacing(0.8, 0.8, 1.0)
UNIT = VoxelSpacing(1.0, 1.0, 1.0)


def det_arrays(dets, prefix):
    """Flatten a Detection list into arrays."""
    out = {}
    out[prefix + "ids"] = np.array([d.id for d in dets], dtype=np.int64)
    out[prefix + "counts"] = np.array([d.voxel_count for d in dets], dtype=np.int64)
    out[prefix + "centroids"] = np.array([d.centroid_um for d in dets], dtype=np.float64).reshape(-1, 3)
    out[prefix + "volumes"] = np.array([d.volume_um3 for d in dets], dtype=np.float64)
    vox = [d.voxels for d in dets]
    out[prefix + "voxels"] = (np.concatenate(vox) if vox else np.empty((0, 3))).astype(np.int32)
    return out


def synth_cases():
    """Cell + vessel pipeline on synthetic frames."""
    specs = [
        ("c1crop_u8", SceneSpec(64, 64, 32, "u8", n_cells=12, seed=3), 10.0),
        ("small_u16", SceneSpec(48, 40, 24, "u16", n_cells=8, seed=5), 6.0),
        ("tiny_u8", SceneSpec(20, 18, 12, "u8", n_cells=3, r_min=2.0, r_max=3.0, seed=9), 3.0),
    ]
    for name, spec, sigma_um in specs:
        data = {"dims": np.array(spec.dims), "seed": spec.seed, "dtype": spec.dtype, "sigma_um": sigma_um,
                "n_cells": spec.n_cells}
        for t in range(2):
            raw_c = O.synth_frame(spec.dims, spec.dtype, spec.frame_seed(t, 0), spec.vmax, balls=spec.balls(t),
                                  amp_ball=spec.amp_cell)
            raw_v = O.synth_frame(spec.dims, spec.dtype, spec.frame_seed(t, 1), spec.vmax, tubes=spec.tubes(),
                                  amp_tube=spec.amp_tube)
            g = VoxelGrid(values=raw_c, spacing=ANISO)
            den = D.denoise_cell_channel(g, D.CellDenoiseParams(gaussian_sigma_um=sigma_um))
            dets = S.segment_cell_channel(den, S.SegmentationConfig(), frame=t, id_start=100 * t)
            data[f"t{t}_raw_cell"] = raw_c
            data[f"t{t}_raw_vessel"] = raw_v
            data[f"t{t}_denoised"] = den.values
            data.update(det_arrays(dets, f"t{t}_"))
            st = D.mrf_denoise_state(VoxelGrid(values=raw_v, spacing=ANISO))
            mask, dm = S.segment_vessel_channel(st.current)
            data[f"t{t}_mrf"] = np.array([st.sigma_hat, st.delta, st.iteration, float(st.converged)])
            data[f"t{t}_vmask"] = mask
            data[f"t{t}_vdist"] = dm.values
        np.savez_compressed(os.path.join(HERE, f"pipeline_{name}.npz"), **data)
        print("wrote", name, {k: v.shape for k, v in data.items() if hasattr(v, "shape")})


def otsu_cases():
    rng = np.random.default_rng(505)
    hists, ts = [], []
    for i in range(400):
        n_bins = 256 if i % 10 == 0 else int(rng.integers(2, 257))
        counts = rng.integers(0, 60, n_bins)
        counts[rng.random(n_bins) < rng.uniform(0.0, 0.8)] = 0
        if np.count_nonzero(counts) < 2:
            counts[0] += 1
            counts[-1] += 7
        h = np.zeros(256, dtype=np.int64)
        h[:n_bins] = counts
        hists.append(h)
        ts.append([n_bins, S.otsu_threshold(counts.astype(np.int64))])
    # wide / large-count histograms (65536 bins; int64 prefilter regime)
    big = []
    for i in range(6):
        h = np.zeros(65536, dtype=np.int64)
        idx = rng.integers(0, 65536, 40)
        h[idx] = rng.integers(1, 10**7, 40)
        big.append(h)
    # the wrap regime: ~1.6e9 voxels of u8
    wrap = np.zeros(256, dtype=np.int64)
    wrap[:40] = 30_000_000
    wrap[200:230] = 10_000_000
    wrap[100] = 77
    big_t = [S.otsu_threshold(h) for h in big] + [S.otsu_threshold(wrap)]
    np.savez_compressed(
        os.path.join(HERE, "otsu.npz"),
        hists=np.array(hists), meta=np.array(ts), big=np.array(big), wrap=wrap, big_t=np.array(big_t),
    )
    print("wrote otsu", len(hists), big_t)


def mask_cases():
    rng = np.random.default_rng(11)
    data = {}
    for i in range(6):
        shape = tuple(int(x) for x in rng.integers(6, 18, 3))
        m = rng.random(shape) > rng.uniform(0.55, 0.9)
        data[f"m{i}"] = m
        data[f"close1_{i}"] = S.morphological_closing(m, 1)
        data[f"close2_{i}"] = S.morphological_closing(m, 2)
        dets = S.detections_from_mask(m, ANISO, frame=1, min_volume_um3=1.5, id_start=7)
        data.update(det_arrays(dets, f"d{i}_"))
        if m.any():
            data[f"edt{i}"] = S.distance_map(m, ANISO).values
    np.savez_compressed(os.path.join(HERE, "masks.npz"), **data)
    print("wrote masks")


def mrf_cases():
    data = {}
    for seed in range(4):
        v = np.random.default_rng(seed).integers(0, 256, size=(16, 16, 16)).astype(float)
        st = D.mrf_denoise_state(VoxelGrid(values=v, spacing=UNIT))
        data[f"v{seed}"] = v
        data[f"cur{seed}"] = st.current.values
        data[f"meta{seed}"] = np.array([st.sigma_hat, st.delta, st.iteration, float(st.converged)])
    v = np.random.default_rng(23).normal(100.0, 6.0, size=(24, 25, 26))
    data["noise_v"] = v
    data["noise_sigma"] = np.array([D.estimate_noise_variance(VoxelGrid(values=v, spacing=UNIT))])
    data["noise_step"] = np.array([D.intensity_step(v)])
    data["noise_sign"] = D._neighbor_sign_sum(v)
    np.savez_compressed(os.path.join(HERE, "mrf.npz"), **data)
    print("wrote mrf")


if __name__ == "__main__":
    O.build()
    synth_cases()
    otsu_cases()
    mask_cases()
    mrf_cases()
