"""CPU oracle pinned against the reference: golden fixtures (always) and the
live reference (only where /root/reference exists, i.e. the build container)."""

import numpy as np
import pytest

import _refimport
from conftest import PIPELINE_CASES, golden
from paper_1407_2089_b200.synth import SceneSpec

ANISO = (0.8, 0.8, 1.0)


def check_dets(dets, g, prefix):
    assert [d.id for d in dets] == list(g[prefix + "ids"])
    assert [d.voxel_count for d in dets] == list(g[prefix + "counts"])
    vox = np.concatenate([d.voxels for d in dets]) if dets else np.empty((0, 3))
    np.testing.assert_array_equal(vox, g[prefix + "voxels"])
    cen = np.array([d.centroid_um for d in dets]).reshape(-1, 3)
    np.testing.assert_array_equal(cen, g[prefix + "centroids"])  # bit-exact
    np.testing.assert_array_equal(np.array([d.volume_um3 for d in dets]), g[prefix + "volumes"])


@pytest.mark.parametrize("case", PIPELINE_CASES)
def test_oracle_pipeline_matches_golden(oracle, case):
    g = golden(f"pipeline_{case}.npz")
    dtype = str(g["dtype"])
    spec = SceneSpec(*[int(x) for x in g["dims"]], dtype=dtype, n_cells=int(g["n_cells"]), seed=int(g["seed"]),
                     **({"r_min": 2.0, "r_max": 3.0} if case == "tiny_u8" else {}))
    for t in range(2):
        raw_c = oracle.synth_frame(spec.dims, dtype, spec.frame_seed(t, 0), spec.vmax, balls=spec.balls(t),
                                   amp_ball=spec.amp_cell)
        raw_v = oracle.synth_frame(spec.dims, dtype, spec.frame_seed(t, 1), spec.vmax, tubes=spec.tubes(),
                                   amp_tube=spec.amp_tube)
        # generator pinned: the frames the reference saw
        np.testing.assert_array_equal(raw_c, g[f"t{t}_raw_cell"])
        np.testing.assert_array_equal(raw_v, g[f"t{t}_raw_vessel"])
        den = oracle.denoise_cell(raw_c, ANISO, float(g["sigma_um"]))["denoised"]
        np.testing.assert_array_equal(den, g[f"t{t}_denoised"])  # bit-exact float64
        dets = oracle.segment_cell(den, ANISO, frame=t, id_start=100 * t)
        check_dets(dets, g, f"t{t}_")
        st = oracle.mrf(raw_v)
        meta = g[f"t{t}_mrf"]
        assert st["sigma_hat"] == meta[0] and st["delta"] == meta[1] and st["iteration"] == meta[2]
        cur = st["current"] if st["current"] is not None else raw_v
        mask, dist, empty = oracle.segment_vessel(cur, ANISO)
        np.testing.assert_array_equal(mask, g[f"t{t}_vmask"])
        np.testing.assert_allclose(dist, g[f"t{t}_vdist"], rtol=0, atol=1e-9)


def test_oracle_otsu_matches_golden(oracle):
    g = golden("otsu.npz")
    for h, (nb, t) in zip(g["hists"], g["meta"]):
        assert oracle.otsu(h[:nb]) == t
    for h, t in zip(list(g["big"]) + [g["wrap"]], g["big_t"]):
        assert oracle.otsu(h) == t


def test_oracle_masks_match_golden(oracle):
    g = golden("masks.npz")
    for i in range(6):
        m = g[f"m{i}"]
        np.testing.assert_array_equal(oracle.closing(m, 1), g[f"close1_{i}"])
        np.testing.assert_array_equal(oracle.closing(m, 2), g[f"close2_{i}"])
        check_dets(oracle.detections(m, ANISO, frame=1, min_volume_um3=1.5, id_start=7), g, f"d{i}_")
        if m.any():
            np.testing.assert_allclose(oracle.edt(m, ANISO), g[f"edt{i}"], rtol=0, atol=1e-9)


def test_oracle_mrf_matches_golden(oracle):
    g = golden("mrf.npz")
    for seed in range(4):
        st = oracle.mrf(g[f"v{seed}"])
        meta = g[f"meta{seed}"]
        assert (st["sigma_hat"], st["delta"], st["iteration"], float(st["converged"])) == tuple(meta)
        np.testing.assert_array_equal(st["current"], g[f"cur{seed}"])
    assert oracle.noise_sigma(g["noise_v"]) == g["noise_sigma"][0]
    assert oracle.intensity_step(g["noise_v"]) == g["noise_step"][0]
    np.testing.assert_array_equal(oracle.sign_sum(g["noise_v"]), g["noise_sign"])


def test_oracle_pairwise_sum_is_numpy_sum(oracle):
    rng = np.random.default_rng(4)
    for n in [1, 7, 8, 9, 127, 128, 129, 1000, 4097, 1_000_003]:
        x = rng.random(n) * 100
        assert oracle.pairwise_sum(x) == np.sum(x)
    x = rng.random((64, 61, 33))
    assert oracle.pairwise_sum(x) == np.sum(x)


live = pytest.mark.skipif(not _refimport.available(), reason="reference not mounted (GPU box)")


@live
def test_oracle_vs_live_reference_random(oracle):
    ct = _refimport.clonetrack()
    from clonetrack import segment as S
    from clonetrack.imaging import VoxelGrid, VoxelSpacing
    from clonetrack import denoise as D

    rng = np.random.default_rng(99)
    sp = VoxelSpacing(0.8, 0.8, 1.0)
    for _ in range(4):
        shape = tuple(int(x) for x in rng.integers(8, 24, 3))
        v = rng.integers(0, 256, size=shape).astype(np.uint8)
        sigma = float(rng.uniform(0.5, 3.0))
        ref = D.denoise_cell_channel(VoxelGrid(values=v, spacing=sp), D.CellDenoiseParams(gaussian_sigma_um=sigma))
        mine = oracle.denoise_cell(v, ANISO, sigma)["denoised"]
        np.testing.assert_array_equal(ref.values, mine)
        m = rng.random(shape) > 0.7
        np.testing.assert_array_equal(S.morphological_closing(m, 1), oracle.closing(m, 1))
        np.testing.assert_allclose(S.distance_map(m, sp).values if m.any() else 0, oracle.edt(m, ANISO) if m.any() else 0,
                                   atol=1e-9, rtol=0)
