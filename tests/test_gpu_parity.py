"""CUDA path vs the reference (golden fixtures) and the CPU oracle.

Bit-exact: q / histograms / thresholds / masks / canonical labels / voxel
lists / ids / centroids / volumes and the denoised float64 grid.  EDT within
1e-9 um (the reference's own contract, ref test_acceptance.py:318-332)."""

import numpy as np
import pytest
import torch

from conftest import PIPELINE_CASES, golden
from paper_1407_2089_b200 import denoise as D
from paper_1407_2089_b200 import segment as S
from paper_1407_2089_b200 import synth
from paper_1407_2089_b200.imaging import VoxelGrid, VoxelSpacing
from paper_1407_2089_b200.pipeline import FramePipeline

pytestmark = pytest.mark.gpu

ANISO = VoxelSpacing(0.8, 0.8, 1.0)
UNIT = VoxelSpacing(1.0, 1.0, 1.0)


def assert_dets(dets, g, prefix):
    assert [d.id for d in dets] == list(g[prefix + "ids"])
    assert [d.voxel_count for d in dets] == list(g[prefix + "counts"])
    vox = np.concatenate([d.voxels for d in dets]) if dets else np.empty((0, 3))
    np.testing.assert_array_equal(vox, g[prefix + "voxels"])
    np.testing.assert_array_equal(np.array([d.centroid_um for d in dets]).reshape(-1, 3), g[prefix + "centroids"])
    np.testing.assert_array_equal(np.array([d.volume_um3 for d in dets]), g[prefix + "volumes"])


def assert_rows(rows, voxels_lin, dims, g, prefix):
    """Fused-pipeline table vs golden detections."""
    _, ny, nz = dims
    assert list(rows["id"]) == list(g[prefix + "ids"])
    assert list(rows["count"]) == list(g[prefix + "counts"])
    np.testing.assert_array_equal(rows["centroid_um"].reshape(-1, 3), g[prefix + "centroids"])
    np.testing.assert_array_equal(rows["volume_um3"], g[prefix + "volumes"])
    lin = voxels_lin[: int(rows["count"].sum())]
    vox = np.stack([lin // (ny * nz), (lin // nz) % ny, lin % nz], axis=1)
    np.testing.assert_array_equal(vox, g[prefix + "voxels"])


def spec_of(case, g):
    kw = {"r_min": 2.0, "r_max": 3.0} if case == "tiny_u8" else {}
    return synth.SceneSpec(*[int(x) for x in g["dims"]], dtype=str(g["dtype"]), n_cells=int(g["n_cells"]),
                           seed=int(g["seed"]), **kw)


@pytest.mark.parametrize("case", PIPELINE_CASES)
def test_api_matches_reference_golden(cuda, case):
    g = golden(f"pipeline_{case}.npz")
    sigma = float(g["sigma_um"])
    for t in range(2):
        raw_c, raw_v = g[f"t{t}_raw_cell"], g[f"t{t}_raw_vessel"]
        den = D.denoise_cell_channel(VoxelGrid(values=raw_c, spacing=ANISO), D.CellDenoiseParams(sigma))
        np.testing.assert_array_equal(den.values, g[f"t{t}_denoised"])
        dets = S.segment_cell_channel(den, S.SegmentationConfig(), frame=t, id_start=100 * t)
        assert_dets(dets, g, f"t{t}_")
        st = D.mrf_denoise_state(VoxelGrid(values=raw_v, spacing=ANISO))
        meta = g[f"t{t}_mrf"]
        assert (st.sigma_hat, st.delta, st.iteration, float(st.converged)) == tuple(meta)
        mask, dm = S.segment_vessel_channel(st.current)
        np.testing.assert_array_equal(mask, g[f"t{t}_vmask"])
        np.testing.assert_allclose(dm.values, g[f"t{t}_vdist"], rtol=0, atol=1e-9)


@pytest.mark.parametrize("case", PIPELINE_CASES)
def test_fused_pipeline_matches_reference_golden(cuda, case):
    g = golden(f"pipeline_{case}.npz")
    spec = spec_of(case, g)
    pipe = FramePipeline(spec.dims, spec.dtype, ANISO, D.CellDenoiseParams(float(g["sigma_um"])))
    for t in range(2):
        raw_c = synth.generate(spec, t, synth.CELL)
        raw_v = synth.generate(spec, t, synth.VESSEL)
        # device generator == the frames the reference saw
        np.testing.assert_array_equal(raw_c.cpu().numpy() if spec.dtype == "u8" else
                                      raw_c.cpu().view(torch.int16).numpy().view(np.uint16), g[f"t{t}_raw_cell"])
        res = pipe.cell(raw_c, frame=t, id_start=100 * t)
        cnt, rows = pipe.finish_cell(res)
        assert_rows(rows, pipe.voxels.cpu().numpy(), spec.dims, g, f"t{t}_")
        vres = pipe.vessel(raw_v)
        mask, dm = pipe.finish_vessel(vres, raw_v)
        np.testing.assert_array_equal(mask.cpu().numpy(), g[f"t{t}_vmask"])
        np.testing.assert_allclose(dm.values.cpu().numpy(), g[f"t{t}_vdist"], rtol=0, atol=1e-9)


def test_fused_pipeline_vs_oracle_c1(cuda, oracle):
    """Full BASELINE config-1 frames (256x256x32 u8, 50 cells), both channels."""
    spec = synth.C1
    pipe = FramePipeline(spec.dims, spec.dtype, ANISO)
    for t in (0, 3):
        raw_c = synth.generate(spec, t, synth.CELL)
        raw_v = synth.generate(spec, t, synth.VESSEL)
        host_c = oracle.synth_frame(spec.dims, "u8", spec.frame_seed(t, 0), spec.vmax, balls=spec.balls(t),
                                    amp_ball=spec.amp_cell)
        host_v = oracle.synth_frame(spec.dims, "u8", spec.frame_seed(t, 1), spec.vmax, tubes=spec.tubes(),
                                    amp_tube=spec.amp_tube)
        np.testing.assert_array_equal(raw_c.cpu().numpy(), host_c)
        np.testing.assert_array_equal(raw_v.cpu().numpy(), host_v)
        o = oracle.denoise_cell(host_c, ANISO.as_array(), 10.0)
        # K1 quantised residual and K2 median, bit-exact
        res = pipe.cell(raw_c, frame=t, id_start=t * 1000)
        np.testing.assert_array_equal(pipe.q.cpu().numpy(), np.rint(o["residual"]).astype(np.uint8))
        np.testing.assert_array_equal(pipe.med.cpu().numpy(), np.rint(o["denoised"]).astype(np.uint8))
        hist = oracle.histogram(o["denoised"])
        np.testing.assert_array_equal(pipe.hist.cpu().numpy()[: hist.size], hist)
        assert int(pipe.otsu[0]) == oracle.otsu(hist)
        odets = oracle.segment_cell(o["denoised"], ANISO.as_array(), frame=t, id_start=t * 1000, intensity=host_c)
        cnt, rows = pipe.finish_cell(res)
        assert len(rows) == len(odets) > 10
        for r, d in zip(rows, odets):
            assert r["id"] == d.id and r["count"] == d.voxel_count and r["root"] == d.root
            np.testing.assert_array_equal(r["centroid_um"], d.centroid_um)
            np.testing.assert_array_equal(np.concatenate([r["bbox_lo"], r["bbox_hi"]]), d.bbox)
            assert r["intensity_sum"] == d.intensity_sum
        # canonical label volume
        lab = pipe.labels.cpu().numpy()
        for r, d in zip(rows, odets):
            assert np.all(lab[tuple(d.voxels.T)] == r["id"] - t * 1000)
        assert (lab >= 0).sum() == rows["count"].sum()
        vres = pipe.vessel(raw_v)
        mask, dm = pipe.finish_vessel(vres, raw_v)
        st = oracle.mrf(host_v)
        assert st["iteration"] == 0
        om, odist, _ = oracle.segment_vessel(st["current"], ANISO.as_array())
        np.testing.assert_array_equal(mask.cpu().numpy(), om)
        np.testing.assert_array_equal(dm.values.cpu().numpy(), odist)  # same envelope arithmetic: bit-exact


def test_u16_frame_vs_oracle(cuda, oracle):
    spec = synth.SceneSpec(96, 80, 32, "u16", n_cells=20, seed=11)
    pipe = FramePipeline(spec.dims, spec.dtype, ANISO)
    raw = synth.generate(spec, 1, synth.CELL)
    host = oracle.synth_frame(spec.dims, "u16", spec.frame_seed(1, 0), spec.vmax, balls=spec.balls(1),
                              amp_ball=spec.amp_cell)
    np.testing.assert_array_equal(raw.cpu().view(torch.int16).numpy().view(np.uint16), host)
    o = oracle.denoise_cell(host, ANISO.as_array(), 10.0)
    res = pipe.cell(raw)
    cnt, rows = pipe.finish_cell(res)
    odets = oracle.segment_cell(o["denoised"], ANISO.as_array())
    assert [int(r["count"]) for r in rows] == [d.voxel_count for d in odets]
    for r, d in zip(rows, odets):
        np.testing.assert_array_equal(r["centroid_um"], d.centroid_um)


def test_otsu_golden(cuda):
    g = golden("otsu.npz")
    for h, (nb, t) in zip(g["hists"], g["meta"]):
        assert S.otsu_threshold(h[:nb]) == t
    for h, t in zip(list(g["big"]) + [g["wrap"]], g["big_t"]):
        assert S.otsu_threshold(h) == t


def test_masks_golden(cuda):
    g = golden("masks.npz")
    for i in range(6):
        m = g[f"m{i}"]
        np.testing.assert_array_equal(S.morphological_closing(m, 1), g[f"close1_{i}"])
        np.testing.assert_array_equal(S.morphological_closing(m, 2), g[f"close2_{i}"])
        assert_dets(S.detections_from_mask(m, ANISO, frame=1, min_volume_um3=1.5, id_start=7), g, f"d{i}_")
        if m.any():
            np.testing.assert_allclose(S.distance_map(m, ANISO).values, g[f"edt{i}"], rtol=0, atol=1e-9)


def test_mrf_golden(cuda):
    g = golden("mrf.npz")
    for seed in range(4):
        st = D.mrf_denoise_state(VoxelGrid(values=g[f"v{seed}"], spacing=UNIT))
        assert (st.sigma_hat, st.delta, st.iteration, float(st.converged)) == tuple(g[f"meta{seed}"])
        np.testing.assert_array_equal(st.current.values, g[f"cur{seed}"])
    v = g["noise_v"]
    assert D.estimate_noise_variance(VoxelGrid(values=v, spacing=UNIT)) == g["noise_sigma"][0]
    assert D.intensity_step(v) == g["noise_step"][0]
    np.testing.assert_array_equal(D._neighbor_sign_sum(v), g["noise_sign"])


def test_random_masks_vs_oracle(cuda, oracle):
    rng = np.random.default_rng(2024)
    for _ in range(6):
        shape = tuple(int(x) for x in rng.integers(5, 40, 3))
        m = rng.random(shape) > rng.uniform(0.5, 0.95)
        np.testing.assert_array_equal(S.morphological_closing(m, 1), oracle.closing(m, 1))
        np.testing.assert_array_equal(S.morphological_closing(m, 3), oracle.closing(m, 3))
        d_gpu = S.detections_from_mask(m, ANISO, frame=0, min_volume_um3=0.0)
        d_ora = oracle.detections(m, ANISO.as_array(), min_volume_um3=0.0)
        assert len(d_gpu) == len(d_ora)
        for a, b in zip(d_gpu, d_ora):
            assert a.id == b.id
            np.testing.assert_array_equal(a.voxels, b.voxels)
            np.testing.assert_array_equal(a.centroid_um, b.centroid_um)
        if m.any():
            np.testing.assert_array_equal(S.distance_map(m, ANISO).values, oracle.edt(m, ANISO.as_array()))


def test_median_radii_and_dtypes_vs_oracle(cuda, oracle):
    rng = np.random.default_rng(8)
    for rad in (1, 2, 3):
        for dt in (np.uint8, np.uint16, np.float64):
            shape = (13, 11, 37)
            v = (rng.integers(0, 300, size=shape)).astype(dt) if dt != np.uint8 else rng.integers(0, 256, shape).astype(dt)
            t = torch.from_numpy(v if dt != np.uint16 else v.view(np.int16)).cuda()
            if dt == np.uint16:
                t = t.view(torch.uint16)
            out = torch.empty_like(t)
            hist = torch.zeros(65536, dtype=torch.int64, device=t.device)
            from paper_1407_2089_b200._lib import call
            from paper_1407_2089_b200 import _dev
            call("ct_median", t.data_ptr(), _dev.ct_code(t), *shape, rad, out.data_ptr(), hist.data_ptr(),
                 _dev.stream_handle())
            ref = oracle.median(v.astype(np.float64), rad)
            got = out.cpu()
            got = got.view(torch.int16).numpy().view(np.uint16) if dt == np.uint16 else got.numpy()
            np.testing.assert_array_equal(got.astype(np.float64), ref)
            if dt != np.float64:
                np.testing.assert_array_equal(hist.cpu().numpy()[:65536], np.bincount(ref.astype(np.int64).ravel(),
                                                                                      minlength=65536))


def test_gaussian_sigma_sweep_vs_oracle(cuda, oracle):
    """C5-style sigma sweep incl. radius > extent and skipped clamping paths."""
    rng = np.random.default_rng(3)
    for sig, shape in [(1.0, (40, 30, 20)), (2.0, (33, 17, 9)), (3.0, (20, 64, 40)), (4.0, (70, 20, 12))]:
        v = rng.integers(0, 256, size=shape).astype(np.uint8)
        g = D.denoise_cell_channel(VoxelGrid(values=v, spacing=UNIT), D.CellDenoiseParams(sig))
        o = oracle.denoise_cell(v, (1.0, 1.0, 1.0), sig)
        np.testing.assert_array_equal(g.values, o["denoised"])


def test_large_frame_properties(cuda):
    """BASELINE config-2 size (1024x1024x64 u8): size-independent invariants."""
    spec = synth.C2
    pipe = FramePipeline(spec.dims, spec.dtype, ANISO)
    raw = synth.generate(spec, 5, synth.CELL)
    res = pipe.cell(raw, frame=5, id_start=123)
    cnt, rows = pipe.finish_cell(res)
    labels1 = pipe.labels.clone()
    nk = len(rows)
    assert nk > 1000
    assert list(rows["id"]) == list(range(123, 123 + nk))
    key = list(zip(-rows["count"], rows["root"]))
    assert key == sorted(key)
    assert np.all(rows["volume_um3"] >= 19.0)
    lab = pipe.labels
    counts = torch.bincount(lab[lab >= 0].to(torch.int64), minlength=nk).cpu().numpy()
    np.testing.assert_array_equal(counts, rows["count"])
    vox = pipe.voxels[: int(rows["count"].sum())].cpu().numpy().astype(np.int64)
    # voxel lists: ascending within each cell, first voxel == root, label == rank
    for r in rows[:: max(1, nk // 50)]:
        seg = vox[r["voxel_offset"] : r["voxel_offset"] + r["count"]]
        assert seg[0] == r["root"] and np.all(np.diff(seg) > 0)
        assert torch.all(lab.view(-1)[torch.from_numpy(seg).cuda()] == r["id"] - 123)
        ny, nz = spec.ny, spec.nz
        pts = np.stack([seg // (ny * nz), (seg // nz) % ny, seg % nz], axis=1).astype(np.float64) * ANISO.as_array()
        np.testing.assert_array_equal(pts.mean(axis=0), r["centroid_um"])  # numpy's own mean
    # determinism: rerun gives identical labels and table
    res2 = pipe.cell(raw, frame=5, id_start=123)
    cnt2, rows2 = pipe.finish_cell(res2)
    assert torch.equal(labels1, pipe.labels)
    assert rows2.tobytes() == rows.tobytes()
    # vessel channel at full size
    rawv = synth.generate(spec, 5, synth.VESSEL)
    vres = pipe_v = FramePipeline(spec.dims, spec.dtype, ANISO, cell=False).vessel(rawv)
    assert int(vres.state[5]) == 0
    assert float(vres.state[2]) == 2.0  # decision certified without the exact sigma_hat
    assert torch.all(vres.distance[vres.mask.bool()] == 0)
    assert torch.all(vres.distance[~vres.mask.bool()] > 0)
    # the drop-in API path (exact sigma_hat, float64 grid, float histogram)
    # reaches the same decision, mask and distance map at full size
    st = D.mrf_denoise_state(VoxelGrid(values=rawv, spacing=ANISO))
    assert st.iteration == 0 and st.sigma_hat > 0
    m_api, dm_api = S.segment_vessel_channel(D.mrf_denoise(VoxelGrid(values=rawv, spacing=ANISO)))
    assert torch.equal(m_api.to(torch.uint8), vres.mask)
    assert torch.equal(dm_api.values, vres.distance)


def _q_exact_and_fast(raw, spacing, sigma_um, eps=0.0, cap=1 << 20, path=0):
    from paper_1407_2089_b200 import _dev
    from paper_1407_2089_b200._lib import call

    nx, ny, nz = (int(d) for d in raw.shape)
    sig = tuple(sigma_um / s for s in (spacing.dx, spacing.dy, spacing.dz))
    w, (rx, ry, rz) = D.device_taps(sig, raw.device)
    work = torch.empty(2 * nx * ny * nz, dtype=torch.float64, device=raw.device)
    q1 = torch.empty_like(raw)
    q2 = torch.empty_like(raw)
    fix = torch.zeros(2 + cap, dtype=torch.int64, device=raw.device)
    code = _dev.ct_code(raw)
    s = _dev.stream_handle()
    call("ct_gaussian_residual", raw.data_ptr(), code, nx, ny, nz, w.data_ptr(), rx, ry, rz, work.data_ptr(), None,
         None, q1.data_ptr(), code, s)
    call("ct_gaussian_q", raw.data_ptr(), code, nx, ny, nz, w.data_ptr(), rx, ry, rz, work.data_ptr(),
         q2.data_ptr(), fix.data_ptr(), cap, eps, path, s)
    return q1, q2, fix[:2].cpu().numpy()


@pytest.mark.parametrize("mode", [1, 0])  # FP64 FMA, auto (tensor cores where the shape fits)
def test_certified_fast_k1_matches_exact(cuda, mode):
    for spec in (synth.C1, synth.SceneSpec(128, 96, 48, "u16", n_cells=20, seed=4),
                 synth.SceneSpec(160, 96, 64, "u8", n_cells=30, seed=9)):
        raw = synth.generate(spec, 2, synth.CELL)
        q1, q2, fx = _q_exact_and_fast(raw, ANISO, 10.0, path=mode)
        assert fx[1] == 0
        assert torch.equal(q1, q2), f"{int((q1 != q2).sum())} voxels differ; flagged {fx[0]}"


@pytest.mark.parametrize("sigma,shape,seed", [(10.0, (256, 192, 64), 1), (6.0, (200, 64, 32), 2),
                                              (12.0, (130, 130, 64), 3), (3.0, (64, 32, 32), 4),
                                              (10.0, (96, 64, 96), 5),
                                              # ny % 128 == 0, and partial row / line tiles
                                              (10.0, (256, 256, 64), 6), (6.0, (130, 128, 32), 7),
                                              (12.0, (64, 384, 64), 8), (4.0, (33, 128, 64), 9)])
def test_tensor_core_k1_matches_exact(cuda, sigma, shape, seed):
    # tensor-core K1 alone (path 2) on noise and on a synthetic scene, incl.
    # row counts that are not multiples of the 128-row tile
    rng = np.random.default_rng(seed)
    noise = torch.from_numpy(rng.integers(0, 256, size=shape, dtype=np.uint8)).cuda()
    scene = synth.generate(synth.SceneSpec(*shape, "u8", n_cells=40, seed=seed), 1, synth.CELL)
    for raw in (noise, scene):
        q1, q2, fx = _q_exact_and_fast(raw, ANISO, sigma, path=2)
        assert fx[1] == 0
        assert fx[0] < 0.001 * raw.numel(), fx
        assert torch.equal(q1, q2), f"{int((q1 != q2).sum())} voxels differ; flagged {fx[0]}"


@pytest.mark.parametrize("vmax,shape,sigma,seed", [(4095, (256, 128, 64), 10.0, 21), (65535, (130, 64, 64), 10.0, 22),
                                                   (200, (96, 64, 32), 6.0, 23), (4095, (64, 192, 32), 3.0, 24)])
def test_tensor_core_k1_u16_matches_exact(cuda, vmax, shape, sigma, seed):
    """u16 tensor-core K1 (byte-interleaved pass x, 40-bit intermediates in
    5 byte planes with fraction bits from the frame's maximum: 28 for 12-bit
    data, 24 at full range) on noise and on a synthetic 12-bit scene vs the
    scipy-order exact path."""
    from paper_1407_2089_b200._lib import lib

    assert lib().ct_k1_path(2, *shape, 12, 12, 10, 0) == 2
    rng = np.random.default_rng(seed)
    noise = torch.from_numpy(rng.integers(0, vmax + 1, size=shape).astype(np.uint16).view(np.int16)).cuda()
    raws = [noise.view(torch.uint16)]
    if vmax == 4095:
        raws.append(synth.generate(synth.SceneSpec(*shape, "u16", n_cells=40, seed=seed), 1, synth.CELL))
    for raw in raws:
        q1, q2, fx = _q_exact_and_fast(raw, ANISO, sigma, path=2)
        assert fx[1] == 0
        assert fx[0] < 0.001 * raw.numel(), fx
        assert torch.equal(q1, q2), f"{int((q1 != q2).sum())} voxels differ; flagged {fx[0]}"


def test_tensor_core_k1_rejects_unfit_shape(cuda):
    """path 2 (tensor cores only) on a shape the TC kernels do not cover is an
    error, not a silent fallback; path 0 falls back to the FP64 FMA kernels."""
    from paper_1407_2089_b200._lib import LibctError, lib

    raw = torch.from_numpy(np.random.default_rng(1).integers(0, 256, (40, 36, 20), dtype=np.uint8)).cuda()
    assert lib().ct_k1_path(1, 40, 36, 20, 12, 12, 10, 0) == 1
    assert lib().ct_k1_path(1, 64, 32, 32, 12, 12, 10, 0) == 2
    assert lib().ct_k1_path(1, 64, 32, 32, 12, 12, 10, 1) == 1
    with pytest.raises(LibctError):
        _q_exact_and_fast(raw, ANISO, 3.0, path=2)
    q1, q2, fx = _q_exact_and_fast(raw, ANISO, 3.0, path=0)
    assert torch.equal(q1, q2)
    with pytest.raises(Exception):
        _q_exact_and_fast(raw, ANISO, 3.0, path=3)


@pytest.mark.parametrize("shape", [(40, 36, 20), (24, 20, 33), (12, 20, 128)])
def test_certified_fixup_recomputes_exactly(cuda, shape):
    # eps 0.6 flags every voxel: the fix-up kernels alone must reproduce K1
    # (nz = 20: plain pass-x cone; nz = 33: odd z, the unstaged pass y/z; nz = 128: the widest staged cone)
    rng = np.random.default_rng(12)
    v = torch.from_numpy(rng.integers(0, 256, size=shape, dtype=np.uint8)).cuda()
    q1, q2, fx = _q_exact_and_fast(v, ANISO, 3.0, eps=0.6)
    assert fx[0] == v.numel() and fx[1] == 0
    assert torch.equal(q1, q2)


def test_certified_fixup_tensor_cores(cuda):
    # tensor-core path: everything with residual > -0.1 is flagged and fixed
    rng = np.random.default_rng(13)
    v2 = torch.from_numpy(rng.integers(0, 256, size=(40, 36, 32), dtype=np.uint8)).cuda()
    q1, q2, fx = _q_exact_and_fast(v2, ANISO, 3.0, eps=0.6, path=2)
    assert fx[0] > v2.numel() // 3 and fx[1] == 0
    assert torch.equal(q1, q2)


@pytest.mark.parametrize("path,dtype", [(2, np.uint8), (1, np.uint8), (1, np.uint16)])
def test_fix_list_overflow_recomputed_in_stream(cuda, path, dtype):
    """Fix list too small (10 entries for thousands of flagged voxels): the
    overflow flag is set and q is still exact -- the in-stream cooperative
    recompute (k1_overflow_exact) replaced every voxel in scipy's order."""
    rng = np.random.default_rng(14)
    shape = (40, 36, 32)
    v = rng.integers(0, 256 if dtype == np.uint8 else 4096, size=shape).astype(dtype)
    t = torch.from_numpy(v if dtype == np.uint8 else v.view(np.int16)).cuda()
    if dtype == np.uint16:
        t = t.view(torch.uint16)
    q1, q2, fx = _q_exact_and_fast(t, ANISO, 3.0, eps=0.6, cap=10, path=path)
    assert fx[1] == 1 and fx[0] > 10
    assert torch.equal(q1, q2)


def test_fix_list_overflow_fused_pipeline(cuda, oracle):
    """FramePipeline with a tiny fix list on a C1 frame: the fused result
    still equals the oracle (no exception, no host-side rerun)."""
    spec = synth.C1
    pipe = FramePipeline(spec.dims, spec.dtype, ANISO)
    pipe.fix_cap = 4
    pipe.k1_eps = 0.6  # flag every voxel with residual > -0.1: the list must overflow
    raw = synth.generate(spec, 1, synth.CELL)
    res = pipe.cell(raw, frame=1)
    cnt, rows = pipe.finish_cell(res)
    assert int(pipe.fix[1]) == 1
    host = raw.cpu().numpy()
    o = oracle.denoise_cell(host, ANISO.as_array(), 10.0)
    np.testing.assert_array_equal(pipe.q.cpu().numpy(), np.rint(o["residual"]).astype(np.uint8))
    odets = oracle.segment_cell(o["denoised"], ANISO.as_array(), frame=1)
    assert [int(r["count"]) for r in rows] == [d.voxel_count for d in odets]


def _ref_encode_runs(voxels):
    """The reference's per-voxel loop (ref segment.py:321-337), restated."""
    if voxels.shape[0] == 0:
        return []
    v = voxels[np.lexsort((voxels[:, 2], voxels[:, 1], voxels[:, 0]))]
    runs, start, n = [], v[0], 1
    for prev, cur in zip(v[:-1], v[1:]):
        if cur[0] == prev[0] and cur[1] == prev[1] and cur[2] == prev[2] + 1:
            n += 1
        else:
            runs.append([int(start[0]), int(start[1]), int(start[2]), n])
            start, n = cur, 1
    runs.append([int(start[0]), int(start[1]), int(start[2]), n])
    return runs


@pytest.mark.parametrize("case", PIPELINE_CASES)
def test_gpu_voxel_runs_match_encode_voxel_runs(cuda, case):
    """ct_voxel_runs == encode_voxel_runs(det.voxels) per detection."""
    g = golden(f"pipeline_{case}.npz")
    spec = spec_of(case, g)
    pipe = FramePipeline(spec.dims, spec.dtype, ANISO, D.CellDenoiseParams(float(g["sigma_um"])))
    for t in range(2):
        res = pipe.cell(synth.generate(spec, t, synth.CELL), frame=t)
        dets = pipe.finish_cell(res, materialize=True)
        runs, offs = S.cell_runs(res.cells, spec.dims)
        assert offs.shape[0] == len(dets) + 1 and offs[-1] == runs.shape[0]
        for r, d in enumerate(dets):
            assert runs[offs[r]:offs[r + 1]].tolist() == _ref_encode_runs(d.voxels)
            assert S.encode_voxel_runs(d.voxels) == runs[offs[r]:offs[r + 1]].tolist()


def test_gpu_voxel_runs_c2_properties(cuda):
    """Full C2 frame: runs decode to exactly the C-order voxel lists."""
    spec = synth.C2
    pipe = FramePipeline(spec.dims, spec.dtype, ANISO)
    res = pipe.cell(synth.generate(spec, 0, synth.CELL))
    cnt, rows = pipe.finish_cell(res)
    runs, offs = S.cell_runs(res.cells, spec.dims)
    vox = pipe.voxels[: int(rows["count"].sum())].cpu().numpy().astype(np.int64)
    nx, ny, nz = spec.dims
    for r in range(0, len(rows), 97):
        o, c = int(rows[r]["voxel_offset"]), int(rows[r]["count"])
        lin = vox[o:o + c]
        dec = S.decode_voxel_runs(runs[offs[r]:offs[r + 1]].tolist())
        np.testing.assert_array_equal(dec, np.stack([lin // (ny * nz), (lin // nz) % ny, lin % nz], axis=1))
    assert runs[:, 3].sum() == vox.shape[0]


@pytest.mark.parametrize("shape", [(24, 40, 64), (16, 24, 32), (12, 20, 128), (10, 12, 70), (14, 18, 96)])
def test_specialised_kernel_paths_vs_oracle(cuda, oracle, shape):
    """nz-specialised kernels (SIMD MRF stream for nz in {32, 64, 128}, run-based
    CCL with the vectorised row pack for nz == 64, packed EDT pass z for
    nz in {32, 64}) and their generic fallbacks (nz = 70) against the oracle."""
    rng = np.random.default_rng(sum(shape))
    # MRF statistics on u8 volumes: smooth ramp + noise (0 iterations) and pure noise
    ramp = (np.add.outer(np.add.outer(np.arange(shape[0]), np.arange(shape[1])), np.arange(shape[2])) % 50)
    for v in ((ramp + rng.integers(0, 9, shape)).astype(np.uint8), rng.integers(0, 256, shape).astype(np.uint8)):
        st = D.mrf_denoise_state(VoxelGrid(values=v, spacing=UNIT))
        o = oracle.mrf(v)
        assert (st.sigma_hat, st.delta, st.iteration, st.converged) == \
            (o["sigma_hat"], o["delta"], o["iteration"], o["converged"])
        np.testing.assert_array_equal(np.asarray(st.current.values, dtype=np.float64), o["current"])
    # labels / detections and the EDT on random masks of two densities
    for thr in (0.55, 0.9):
        m = rng.random(shape) > thr
        d_gpu = S.detections_from_mask(m, ANISO, frame=0, min_volume_um3=0.0)
        d_ora = oracle.detections(m, ANISO.as_array(), min_volume_um3=0.0)
        assert [d.id for d in d_gpu] == [d.id for d in d_ora]
        for a, b in zip(d_gpu, d_ora):
            np.testing.assert_array_equal(a.voxels, b.voxels)
            np.testing.assert_array_equal(a.centroid_um, b.centroid_um)
        np.testing.assert_array_equal(S.distance_map(m, ANISO).values, oracle.edt(m, ANISO.as_array()))


@pytest.mark.parametrize("shape", [(24, 40, 64), (16, 24, 32), (12, 20, 128), (14, 18, 96), (9, 11, 20)])
def test_packed_rows_closing_and_ccl(cuda, oracle, shape):
    """ct_threshold_close_rows (packed z-row output of K4) and ct_ccl26_rows
    (K5 on those rows, the fused pipeline's cell path) against the byte-mask
    entry points and the oracle's closing: same words, labels, counters."""
    from paper_1407_2089_b200._lib import call, workspace_bytes
    from paper_1407_2089_b200 import _dev

    nx, ny, nz = shape
    rng = np.random.default_rng(nx * ny * nz)
    for dens in (0.5, 0.85, 0.97):
        v = (rng.random(shape) * 255).astype(np.uint8)
        t = int(255 * dens)
        dv = torch.from_numpy(v).cuda()
        otsu = torch.tensor([t, 0, 0, 0], dtype=torch.int64, device="cuda")
        work = torch.empty(workspace_bytes(1, nx, ny, nz, 1), dtype=torch.uint8, device="cuda")
        W = 1 if nz <= 64 else 2
        rows = torch.zeros(nx * ny * W, dtype=torch.int64, device="cuda")
        mask_b = torch.empty(shape, dtype=torch.uint8, device="cuda")
        mask_r = torch.empty(shape, dtype=torch.uint8, device="cuda")
        s = _dev.stream_handle()
        call("ct_threshold_close", dv.data_ptr(), 1, nx, ny, nz, otsu.data_ptr(), 0, 1, mask_b.data_ptr(),
             work.data_ptr(), s)
        call("ct_threshold_close_rows", dv.data_ptr(), 1, nx, ny, nz, otsu.data_ptr(), 0, mask_r.data_ptr(),
             rows.data_ptr(), work.data_ptr(), s)
        torch.cuda.synchronize()
        mb = mask_b.cpu().numpy()
        np.testing.assert_array_equal(mb, mask_r.cpu().numpy())
        np.testing.assert_array_equal(mb.astype(bool), oracle.closing(v > t, 1))
        # unpack the words: bit k of row (i, j)
        words = rows.cpu().numpy().view(np.uint64).reshape(nx * ny, W)
        bits = np.zeros((nx * ny, nz), dtype=np.uint8)
        for k in range(nz):
            bits[:, k] = (words[:, k // 64] >> np.uint64(k % 64)) & np.uint64(1)
        np.testing.assert_array_equal(bits.reshape(shape), mb)
        outs = []
        for name, src in (("ct_ccl26", mask_b), ("ct_ccl26_rows", rows)):
            labels = torch.empty(shape, dtype=torch.int32, device="cuda")
            fg = torch.empty(nx * ny * nz, dtype=torch.int32, device="cuda")
            cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
            if name == "ct_ccl26_rows":  # labels pre-filled by the caller (flag 1)
                labels.fill_(-1)
                call(name, src.data_ptr(), nx, ny, nz, labels.data_ptr(), fg.data_ptr(), cnt.data_ptr(), 1, s)
            else:
                call(name, src.data_ptr(), nx, ny, nz, labels.data_ptr(), fg.data_ptr(), cnt.data_ptr(), s)
            torch.cuda.synchronize()
            c = cnt.cpu().numpy()
            outs.append((labels.cpu().numpy(), c, np.sort(fg[: int(c[0])].cpu().numpy()) if c[0] else None))
        np.testing.assert_array_equal(outs[0][0], outs[1][0])
        np.testing.assert_array_equal(outs[0][1], outs[1][1])
        if outs[0][2] is not None:
            np.testing.assert_array_equal(outs[0][2], outs[1][2])


@pytest.mark.parametrize("shape", [(40, 36, 64), (16, 16, 32), (20, 18, 96), (12, 14, 70)])
def test_mrf_decide_certified_vs_exact(cuda, oracle, shape):
    """ct_mrf_decide (fused pipeline) against ct_mrf and the oracle: same
    decision, delta, nnz and norm on volumes that stop before the first step
    (certified without sigma_hat: NaN, status 2), iterate (uniform noise: the
    bound cannot decide, so the exact sigma_hat is computed) or are constant."""
    from paper_1407_2089_b200._lib import call, workspace_bytes
    from paper_1407_2089_b200 import _dev

    nx, ny, nz = shape
    rng = np.random.default_rng(nx + ny + nz)
    ramp = np.add.outer(np.add.outer(np.arange(nx), np.arange(ny)), np.arange(nz)) % 50
    vols = {"ramp": (ramp + rng.integers(0, 9, shape)).astype(np.uint8),
            "noise": rng.integers(0, 256, shape).astype(np.uint8),
            "const": np.full(shape, 7, np.uint8)}
    s = _dev.stream_handle()
    for name, v in vols.items():
        dv = torch.from_numpy(v).cuda()
        states = []
        for fn in ("ct_mrf", "ct_mrf_decide"):
            work = torch.empty(workspace_bytes(4, nx, ny, nz, 1), dtype=torch.uint8, device="cuda")
            state = torch.zeros(9, dtype=torch.float64, device="cuda")
            hist = torch.zeros(65536, dtype=torch.int64, device="cuda")
            call(fn, dv.data_ptr(), 1, nx, ny, nz, work.data_ptr(), state.data_ptr(), hist.data_ptr(), s)
            torch.cuda.synchronize()
            states.append((state.cpu().numpy(), hist.cpu().numpy()))
        (a, ha), (b, hb) = states
        np.testing.assert_array_equal(ha, hb)
        o = oracle.mrf(v)
        assert a[5] == b[5], (name, a, b)                 # decision
        assert a[0] == b[0] == o["delta"]                 # delta
        assert a[3] == b[3] and a[4] == b[4]              # nnz, first-step norm
        if b[2] == 2.0:                                   # certified: sigma skipped
            assert np.isnan(b[1]) and a[5] in (0.0, 2.0)
        else:
            assert a[1] == b[1] == o["sigma_hat"] and a[2] == b[2]
        if a[5] == 1.0:
            assert b[2] != 2.0                            # iterating volume: exact path taken
        if name == "ramp" and nz in (32, 64, 96, 128):  # (other nz: the generic stream, no quick path)
            assert b[2] == 2.0                            # smooth + noise: certified without sigma_hat


@pytest.mark.parametrize("shape,density", [((200, 24, 64), 1e-3), ((130, 20, 32), 3e-4), ((1024, 4, 64), 2e-5)])
def test_edt_sparse_masks_vs_oracle(cuda, oracle, shape, density):
    """EDT on sparse masks: pass-x segments with no foreground of their own
    (nearest from neighbouring segments only), whole lines without foreground
    (NONE throughout), and lines whose only foreground is far away -- bit-exact
    against the oracle."""
    rng = np.random.default_rng(int(1 / density))
    m = rng.random(shape) < density
    m[0, 0, 0] = True  # never empty
    np.testing.assert_array_equal(S.distance_map(m, ANISO).values, oracle.edt(m, ANISO.as_array()))


@pytest.mark.parametrize("n_keep_min", [0.0, 1.5])
def test_many_components_vs_oracle(cuda, oracle, n_keep_min):
    """More kept cells than the multi-CTA rank path holds (4096): ~16k isolated
    voxels on a lattice plus random clusters, so the single-CTA radix-sort
    path orders them; with a volume filter (1.5 um^3 drops the single voxels)
    the kept set falls back under 4096.  Ids, voxel lists, centroids and
    volumes against the oracle (API path: detections_from_mask)."""
    rng = np.random.default_rng(77)
    shape = (64, 64, 32)
    m = np.zeros(shape, dtype=bool)
    m[::2, ::2, ::2] = True                                   # 16384 isolated voxels
    for _ in range(40):                                       # clusters merging lattice points
        c = rng.integers(2, 60, 3) % np.array(shape)
        m[c[0]:c[0] + 3, c[1]:c[1] + 3, c[2]:c[2] + 2] = True
    d_gpu = S.detections_from_mask(m, ANISO, frame=0, min_volume_um3=n_keep_min)
    d_ora = oracle.detections(m, ANISO.as_array(), min_volume_um3=n_keep_min)
    assert len(d_gpu) == len(d_ora) and (n_keep_min > 0 or len(d_gpu) > 4096)
    for a, b in zip(d_gpu, d_ora):
        assert a.id == b.id and a.volume_um3 == b.volume_um3
        np.testing.assert_array_equal(a.voxels, b.voxels)
        np.testing.assert_array_equal(a.centroid_um, b.centroid_um)


def test_parallel_hulls_match_serial(cuda):
    """compute_hulls over worker processes (frames with >= HULL_POOL_MIN
    cells) returns exactly the serial compute_hull results, in order."""
    import os

    rng = np.random.default_rng(5)
    vox = []
    for _ in range(S.HULL_POOL_MIN + 40):
        r = rng.uniform(1.0, 4.5)
        g = np.mgrid[-5:6, -5:6, -5:6].reshape(3, -1).T
        v = g[((g - rng.uniform(0, 1, 3)) ** 2).sum(1) <= r * r].astype(np.int64) + 10
        vox.append(v[:rng.integers(1, len(v) + 1)])  # includes < 4 points and flat sets
    par = S.compute_hulls(vox, ANISO)
    os.environ["CT_HULL_PROCS"] = "0"
    try:
        ser = S.compute_hulls(vox, ANISO)
    finally:
        del os.environ["CT_HULL_PROCS"]
    assert len(par) == len(ser)
    for a, b in zip(par, ser):
        assert a.flat == b.flat
        np.testing.assert_array_equal(a.vertices_um, b.vertices_um)
        np.testing.assert_array_equal(a.facets, b.facets)
        if not a.flat:
            np.testing.assert_array_equal(a.equations, b.equations)
