"""The reference's own hot-path test cases (ref pkg/tests/test_segment.py,
test_denoise.py and the hot-path acceptance criteria of test_acceptance.py)
re-run against the drop-in API, which executes on the GPU.  Assertions follow
the reference tests; oracles are restated here independently."""

from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1407_2089_b200.denoise import (
    CellDenoiseParams,
    _neighbor_sign_sum,
    denoise_cell_channel,
    estimate_noise_variance,
    intensity_step,
    mrf_denoise,
    mrf_denoise_state,
)
from paper_1407_2089_b200.errors import DegenerateHistogramError, EmptyDistanceMapError, ParameterError
from paper_1407_2089_b200.imaging import VoxelGrid, VoxelSpacing
from paper_1407_2089_b200.segment import (
    SegmentationConfig,
    ball_element,
    binarize,
    compute_hull,
    decode_voxel_runs,
    detections_from_mask,
    distance_map,
    encode_voxel_runs,
    intensity_histogram,
    morphological_closing,
    otsu_threshold,
    segment_cell_channel,
    segment_vessel_channel,
)

pytestmark = pytest.mark.gpu

UNIT = VoxelSpacing(1.0, 1.0, 1.0)
ANISO = VoxelSpacing(0.8, 0.8, 1.0)


def grid(v, sp=UNIT):
    return VoxelGrid(values=np.asarray(v), spacing=sp)


def rational_otsu(counts):
    """argmax_t w0*w1*(mu0-mu1)^2 in exact rationals, lowest t on ties."""
    counts = [int(c) for c in counts]
    n = sum(counts)
    best, best_t = Fraction(-1), None
    for t in range(len(counts) - 1):
        w0 = sum(counts[: t + 1])
        w1 = n - w0
        if not w0 or not w1:
            continue
        m0 = Fraction(sum(i * c for i, c in enumerate(counts[: t + 1])), w0)
        m1 = Fraction(sum(i * c for i, c in enumerate(counts) if i > t), w1)
        score = Fraction(w0 * w1, n * n) * (m0 - m1) ** 2
        if score > best:
            best, best_t = score, t
    return best_t


def brute_edt(mask, sp):
    fg = np.argwhere(mask).astype(float) * sp.as_array()
    out = np.empty(mask.shape)
    for idx in np.ndindex(mask.shape):
        p = np.array(idx, dtype=float) * sp.as_array()
        out[idx] = np.sqrt(((fg - p) ** 2).sum(axis=1).min())
    return out


class TestOtsu:
    def test_two_spikes(self, cuda):
        c = np.zeros(256, dtype=np.int64)
        c[10] = c[200] = 500
        t = otsu_threshold(c)
        assert 10 <= t < 200 and t == rational_otsu(c)

    def test_random_histograms(self, cuda):
        rng = np.random.default_rng(7)
        for _ in range(60):
            c = rng.integers(0, 40, size=rng.integers(2, 64))
            if (c > 0).sum() >= 2:
                assert otsu_threshold(c) == rational_otsu(c)

    def test_symmetric_tie_lowest(self, cuda):
        c = np.array([5, 0, 0, 5])
        assert otsu_threshold(c) == rational_otsu(c) == 0

    def test_degenerate(self, cuda):
        c = np.zeros(16, dtype=np.int64)
        c[3] = 100
        with pytest.raises(DegenerateHistogramError):
            otsu_threshold(c)
        with pytest.raises(DegenerateHistogramError):
            otsu_threshold(np.zeros(8, dtype=np.int64))

    @given(st.lists(st.integers(0, 30), min_size=2, max_size=40).filter(lambda c: sum(v > 0 for v in c) >= 2))
    @settings(max_examples=60, deadline=None)
    def test_property(self, cuda, counts):
        assert otsu_threshold(np.array(counts)) == rational_otsu(counts)

    def test_acceptance_1000_histograms(self, cuda):
        rng = np.random.default_rng(505)
        for i in range(300):
            nb = 256 if i % 10 == 0 else int(rng.integers(2, 257))
            c = rng.integers(0, 60, nb)
            c[rng.random(nb) < rng.uniform(0.0, 0.8)] = 0
            if np.count_nonzero(c) < 2:
                c[0] += 1
                c[-1] += 7
            assert otsu_threshold(c) == rational_otsu(c)


class TestBinarize:
    def test_strictly_above(self, cuda):
        v = np.zeros((6, 6, 6))
        v[2:4, 2:4, 2:4] = 100.0
        m = binarize(grid(v))
        assert m.sum() == 8 and m[2, 2, 2] and not m[0, 0, 0]

    def test_all_zero_empty(self, cuda):
        assert not binarize(grid(np.zeros((4, 4, 4)))).any()

    def test_constant_rejected(self, cuda):
        with pytest.raises(DegenerateHistogramError):
            binarize(grid(np.full((4, 4, 4), 7.0)))

    def test_wide_range_bins(self, cuda):
        v = np.zeros((4, 4, 4))
        v[0, 0, 0] = 300.0
        assert intensity_histogram(grid(v)).size == 65536
        assert intensity_histogram(grid(np.ones((4, 4, 4)))).size == 256


class TestClosing:
    def test_ball(self):
        b = ball_element(1)
        assert b.sum() == 7 and b[1, 1, 1] and b[0, 1, 1] and not b[0, 0, 0]

    def test_fills_gap(self, cuda):
        m = np.zeros((9, 9, 9), dtype=bool)
        m[2:7, 2:7, 2:7] = True
        m[4, 4, 4] = False
        c = morphological_closing(m, 1)
        assert c[4, 4, 4] and c.sum() == 125

    def test_idempotent(self, cuda):
        m = np.random.default_rng(3).random((12, 12, 12)) > 0.7
        once = morphological_closing(m, 1)
        assert np.array_equal(once, morphological_closing(once, 1))

    def test_border_not_eroded(self, cuda):
        m = np.zeros((8, 8, 8), dtype=bool)
        m[0:3, 0:3, 0:3] = True
        assert (morphological_closing(m, 1) & m).sum() == m.sum()

    def test_radius_zero_identity(self, cuda):
        m = np.zeros((5, 5, 5), dtype=bool)
        m[2, 2, 2] = True
        assert np.array_equal(morphological_closing(m, 0), m)


class TestComponents:
    def test_diagonal_is_one(self, cuda):
        m = np.zeros((6, 6, 6), dtype=bool)
        m[1, 1, 1] = m[2, 2, 2] = True
        d = detections_from_mask(m, UNIT, frame=0, min_volume_um3=0.0)
        assert len(d) == 1 and d[0].voxel_count == 2

    def test_size_order_and_ids(self, cuda):
        m = np.zeros((10, 10, 10), dtype=bool)
        m[1:3, 1:3, 1:3] = True
        m[6:9, 6:9, 6:9] = True
        d = detections_from_mask(m, UNIT, frame=0, min_volume_um3=0.0)
        assert [x.voxel_count for x in d] == [27, 8] and [x.id for x in d] == [0, 1]

    def test_physical_volume_filter(self, cuda):
        m = np.zeros((12, 12, 12), dtype=bool)
        m[0:2, 0:2, 0:4] = True
        m[6:8, 6:10, 6:10] = True
        d = detections_from_mask(m, ANISO, frame=0, min_volume_um3=19.0)
        assert len(d) == 1 and d[0].voxel_count == 32 and d[0].volume_um3 == pytest.approx(20.48)

    def test_centroid(self, cuda):
        m = np.zeros((8, 8, 8), dtype=bool)
        m[2:4, 3, 5] = True
        d = detections_from_mask(m, ANISO, frame=0, min_volume_um3=0.0)
        np.testing.assert_allclose(d[0].centroid_um, [2.5 * 0.8, 3 * 0.8, 5.0])

    def test_id_start(self, cuda):
        m = np.zeros((6, 6, 6), dtype=bool)
        m[1, 1, 1] = True
        d = detections_from_mask(m, UNIT, frame=2, min_volume_um3=0.0, id_start=40)
        assert d[0].id == 40 and d[0].frame == 2

    def test_acceptance_volume_boundary(self, cuda):
        m = np.zeros((40, 8, 8), dtype=bool)
        m[1:11, 2, 2] = True
        m[20:40, 2, 2] = True
        d = detections_from_mask(m, UNIT, frame=0, min_volume_um3=SegmentationConfig().min_volume_um3)
        assert len(d) == 1 and {tuple(v) for v in d[0].voxels} == {(x, 2, 2) for x in range(20, 40)}


class TestHull:
    def test_cube_corners(self):
        h = compute_hull(np.argwhere(np.ones((4, 4, 4), dtype=bool)), UNIT)
        assert not h.flat
        assert {tuple(v) for v in h.vertices_um.tolist()} == {(float(a), float(b), float(c)) for a in (0, 3)
                                                             for b in (0, 3) for c in (0, 3)}

    def test_flat(self):
        assert compute_hull(np.array([[i, 0, 0] for i in range(5)]), UNIT).flat
        assert compute_hull(np.array([[i, j, 2] for i in range(3) for j in range(3)]), UNIT).flat


class TestCellPipeline:
    def test_two_blobs(self, cuda):
        v = np.zeros((20, 20, 12))
        v[2:6, 2:6, 2:6] = 180.0
        v[12:16, 12:16, 4:8] = 200.0
        d = segment_cell_channel(grid(v, ANISO), SegmentationConfig())
        assert len(d) == 2 and all(x.volume_um3 >= 19.0 for x in d)

    def test_speck_removed(self, cuda):
        v = np.zeros((20, 20, 12))
        v[2:6, 2:6, 2:6] = 180.0
        v[15, 15, 9] = 250.0
        d = segment_cell_channel(grid(v, ANISO), SegmentationConfig())
        assert len(d) == 1 and d[0].voxel_count >= 64

    def test_empty(self, cuda):
        assert segment_cell_channel(grid(np.zeros((8, 8, 8)), ANISO)) == []

    def test_tie_order(self, cuda):
        v = np.zeros((16, 16, 16))
        v[1:5, 1:5, 1:5] = 100.0
        v[8:12, 8:12, 8:12] = 100.0
        a = segment_cell_channel(grid(v), SegmentationConfig(min_volume_um3=0.0))
        assert tuple(a[0].voxels[0]) < tuple(a[1].voxels[0])

    def test_26_connected(self, cuda):
        v = np.where(np.random.default_rng(19).random((14, 14, 14)) > 0.6, 120.0, 0.0)
        for det in segment_cell_channel(grid(v), SegmentationConfig(min_volume_um3=0.0)):
            rem = det.voxel_set()
            front = [rem.pop()]
            while front:
                i, j, k = front.pop()
                for di in (-1, 0, 1):
                    for dj in (-1, 0, 1):
                        for dk in (-1, 0, 1):
                            nb = (i + di, j + dj, k + dk)
                            if nb in rem:
                                rem.discard(nb)
                                front.append(nb)
            assert not rem

    def test_translation(self, cuda):
        base = np.zeros((18, 18, 18))
        base[3:7, 3:7, 3:7] = 90.0
        base[3:6, 10:13, 5:9] = 110.0
        sh = np.roll(base, shift=(2, 1, 3), axis=(0, 1, 2))
        cfg = SegmentationConfig(min_volume_um3=0.0)
        a, b = segment_cell_channel(grid(base), cfg), segment_cell_channel(grid(sh), cfg)
        assert len(a) == len(b)
        for x, y in zip(a, b):
            assert y.voxel_set() == {(i + 2, j + 1, k + 3) for i, j, k in x.voxel_set()}


class TestDistanceMap:
    def test_brute_force(self, cuda):
        m = np.random.default_rng(5).random((9, 9, 9)) > 0.85
        m[4, 4, 4] = True
        np.testing.assert_allclose(distance_map(m, ANISO).values, brute_edt(m, ANISO), atol=1e-9)

    def test_acceptance_100_masks(self, cuda):
        rng = np.random.default_rng(606)
        for i in range(20):
            m = rng.random((16, 16, 16)) < rng.uniform(0.02, 0.5)
            if not m.any():
                m[tuple(rng.integers(0, 16, 3))] = True
            assert np.max(np.abs(distance_map(m, ANISO).values - brute_edt(m, ANISO))) <= 1e-9

    def test_axis_steps_and_lookup(self, cuda):
        m = np.zeros((5, 5, 5), dtype=bool)
        m[2, 2, 2] = True
        dm = distance_map(m, ANISO)
        assert dm.at_voxel(3, 2, 2) == pytest.approx(0.8) and dm.at_voxel(2, 2, 3) == pytest.approx(1.0)
        assert dm.at_point_um(np.array([1.7, 1.6, 2.1])) == 0.0

    def test_empty(self, cuda):
        dm = distance_map(np.zeros((4, 4, 4), dtype=bool), UNIT)
        assert dm.empty and np.isinf(dm.values).all()
        with pytest.raises(EmptyDistanceMapError):
            dm.at_voxel(0, 0, 0)

    def test_vessel_pipeline(self, cuda):
        v = np.zeros((10, 10, 10))
        v[:, 4:6, 4:6] = 150.0
        mask, dm = segment_vessel_channel(grid(v, ANISO))
        assert mask[:, 4:6, 4:6].all() and not dm.empty and dm.at_voxel(0, 4, 4) == 0.0


class TestVoxelRuns:
    def test_simple(self):
        v = np.array([[1, 2, 3], [1, 2, 4], [1, 2, 5], [2, 0, 0]])
        assert encode_voxel_runs(v) == [[1, 2, 3, 3], [2, 0, 0, 1]]
        np.testing.assert_array_equal(decode_voxel_runs(encode_voxel_runs(v)), v)

    @given(st.sets(st.tuples(*[st.integers(0, 6)] * 3), max_size=50))
    @settings(max_examples=50, deadline=None)
    def test_round_trip(self, s):
        v = np.array(sorted(s), dtype=np.int64).reshape(-1, 3)
        assert {tuple(x) for x in decode_voxel_runs(encode_voxel_runs(v)).tolist()} == s


def gaussian_direct(values, sigma):
    r = int(4.0 * sigma + 0.5)
    x = np.arange(-r, r + 1, dtype=float)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    k /= k.sum()
    out = values.astype(float)
    for ax in range(3):
        pad = np.pad(out, [(r, r) if a == ax else (0, 0) for a in range(3)], mode="edge")
        acc = np.zeros_like(out)
        for o, w in enumerate(k):
            sl = [slice(None)] * 3
            sl[ax] = slice(o, o + out.shape[ax])
            acc += w * pad[tuple(sl)]
        out = acc
    return out


class TestCellDenoise:
    def test_constant_to_zero(self, cuda):
        out = denoise_cell_channel(grid(np.full((12, 12, 8), 55, dtype=np.uint8)), CellDenoiseParams(1.0))
        np.testing.assert_array_equal(out.values, 0.0)

    def test_impulse_removed(self, cuda):
        v = np.zeros((15, 15, 15), dtype=np.uint8)
        v[7, 7, 7] = 240
        out = denoise_cell_channel(grid(v), CellDenoiseParams(1.0, 1))
        assert out.values.max() == 0.0

    def test_blob_retained(self, cuda):
        v = np.full((40, 40, 40), 10, dtype=np.uint8)
        v[16:23, 16:23, 16:23] = 210
        out = denoise_cell_channel(grid(v), CellDenoiseParams(4.0, 1))
        assert out.values[19, 19, 19] >= 0.5 * float((v - gaussian_direct(v, 4.0))[19, 19, 19])

    def test_median_at_voxel(self, cuda):
        v = np.random.default_rng(11).integers(0, 256, size=(14, 13, 12), dtype=np.uint8)
        out = denoise_cell_channel(grid(v), CellDenoiseParams(1.5, 1))
        res = np.maximum(v.astype(float) - gaussian_direct(v, 1.5), 0.0)
        assert out.values[6, 6, 6] == pytest.approx(np.median(res[5:8, 5:8, 5:8]), abs=1e-9)

    def test_bounds(self, cuda):
        v = np.random.default_rng(5).integers(0, 256, size=(16, 16, 16), dtype=np.uint8)
        out = denoise_cell_channel(grid(v), CellDenoiseParams(2.0))
        assert out.values.min() >= 0.0 and out.values.max() <= v.max()

    def test_oversized(self, cuda):
        with pytest.raises(ParameterError, match="kernel"):
            denoise_cell_channel(grid(np.zeros((10, 10, 10), dtype=np.uint8)), CellDenoiseParams(50.0))

    def test_invalid_params(self):
        with pytest.raises(ParameterError):
            CellDenoiseParams(gaussian_sigma_um=0.0)
        with pytest.raises(ParameterError):
            CellDenoiseParams(median_radius=0)


class TestNoiseEstimate:
    def test_constant(self, cuda):
        assert estimate_noise_variance(grid(np.full((8, 8, 8), 42))) == 0.0

    def test_ramp(self, cuda):
        i, j, k = np.meshgrid(np.arange(10), np.arange(9), np.arange(8), indexing="ij")
        assert estimate_noise_variance(grid((3 * i + 2 * j + 5 * k).astype(float))) == pytest.approx(0.0, abs=1e-12)

    def test_known_level(self, cuda):
        noise = np.random.default_rng(23).normal(0.0, 6.0, size=(64, 64, 64))
        est = estimate_noise_variance(grid(100.0 + noise))
        assert abs(est - float(np.std(noise))) / float(np.std(noise)) < 0.15

    def test_too_small(self, cuda):
        with pytest.raises(ParameterError):
            estimate_noise_variance(grid(np.zeros((2, 5, 5))))
        with pytest.raises(ParameterError):
            estimate_noise_variance(grid(np.zeros((3, 3, 3))))


class TestMrf:
    def test_constant(self, cuda):
        g = grid(np.full((6, 6, 6), 17, dtype=np.uint8))
        s = mrf_denoise_state(g)
        assert s.iteration == 0 and s.delta == 0.0 and s.current is g

    def test_step_size(self, cuda):
        assert intensity_step(np.array([3.0, 7.0, 12.0, 3.0, 7.0]).reshape(5, 1, 1)) == 4.0

    def test_sign_sums(self, cuda):
        i, j, k = np.meshgrid(np.arange(5), np.arange(5), np.arange(5), indexing="ij")
        v = (10.0 * i + 20.0 * j + 40.0 * k) + 0.0
        assert _neighbor_sign_sum(v)[2, 2, 2] == -6
        w = np.full((5, 5, 5), 50.0)
        w[2, 2, 2] = 10.0
        assert _neighbor_sign_sum(w)[2, 2, 2] == 0

    def test_quantized_and_bound(self, cuda):
        for seed in range(3):
            v = np.random.default_rng(seed).integers(0, 256, size=(16, 16, 16)).astype(float)
            s = mrf_denoise_state(grid(v))
            assert float(np.linalg.norm(s.current.values - v)) <= s.sigma_hat + 1e-9
            cur = v.copy()
            for _ in range(s.iteration):
                nxt = cur + s.delta * np.sign(_neighbor_sign_sum(cur))
                assert set(np.round(np.unique(nxt - cur), 12)) <= {-s.delta, 0.0, s.delta}
                cur = nxt
            np.testing.assert_array_equal(cur, s.current.values)

    def test_translation(self, cuda):
        v = np.random.default_rng(31).integers(0, 30, size=(8, 8, 8)).astype(np.float64)
        a, b = mrf_denoise(grid(v)), mrf_denoise(grid(v + 25.0))
        np.testing.assert_allclose(b.values - a.values, 25.0, atol=1e-9)

    def test_consensus(self, cuda):
        v = np.zeros((9, 9, 9))
        v[4, 4, 4] = 3.0
        assert mrf_denoise_state(grid(v)).current.values[4, 4, 4] <= 3.0

    def test_acceptance_contract(self, cuda):
        for seed in range(5):
            v = np.random.default_rng(700 + seed).integers(0, 256, (32, 32, 32)).astype(float)
            s = mrf_denoise_state(grid(v.copy()))
            assert float(np.linalg.norm(s.current.values - v)) <= s.sigma_hat + 1e-9
        flat = np.full((32, 32, 32), 7.0)
        s = mrf_denoise_state(grid(flat.copy()))
        assert s.iteration == 0
        np.testing.assert_array_equal(s.current.values, flat)
