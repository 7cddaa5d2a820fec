"""Parity at the benchmark's own configurations (BASELINE.json configs) and
for every shape-specialised kernel variant.

Full frames through ``FramePipeline`` (the fused path bench.py times) against
the CPU oracle (oracle/, pinned to the reference by tests/golden), bit-exact:
the quantised residual q, the median, the fused histogram, the Otsu
threshold, the canonical label volume, every per-cell table column (ids,
counts, roots, bbox, intensity sums, mean intensities, row-sequential
centroids, volumes), the C-order voxel lists, the vessel mask, the MRF
statistics and the distance map.

  C2   1024x1024x64 u8, cell + vessel: t = 0 (the first frame of bench.py's
       ring) and t = 5
  C3   1024x1024x64 u16, cell + vessel + the second cell channel
  C4   a 1024x1024x96 crop at C4's density (nz = 96 kernels: tensor-core K1
       pass z, median WC = 3, 128-bit CCL rows, MRF nz = 96, EDT pass z 96)

ref: denoise.py:67-89 (cell denoise), segment.py:242-318 (detections,
vessel), denoise.py:147-195 (MRF)."""

import numpy as np
import pytest
import torch

from paper_1407_2089_b200 import synth
from paper_1407_2089_b200._lib import CNT_KEPT, MRF_DECISION, MRF_DELTA, MRF_NNZ, call, workspace_bytes
from paper_1407_2089_b200 import _dev
from paper_1407_2089_b200.imaging import VoxelSpacing
from paper_1407_2089_b200.pipeline import FramePipeline

pytestmark = pytest.mark.gpu

ANISO = VoxelSpacing(0.8, 0.8, 1.0)
SP = ANISO.as_array()


def to_np(t: torch.Tensor) -> np.ndarray:
    t = t.cpu()
    if t.dtype == torch.uint16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def host_frame(oracle, spec, t, ch):
    if ch == synth.VESSEL:
        return oracle.synth_frame(spec.dims, spec.dtype, spec.frame_seed(t, ch), spec.vmax, tubes=spec.tubes(),
                                  amp_tube=spec.amp_tube)
    return oracle.synth_frame(spec.dims, spec.dtype, spec.frame_seed(t, ch), spec.vmax, balls=spec.balls(t, ch),
                              amp_ball=spec.amp_cell)


def check_cell(pipe, spec, t, ch, oracle, id_start):
    """One cell-channel frame through the fused path vs the oracle."""
    raw = synth.generate(spec, t, ch)
    host = host_frame(oracle, spec, t, ch)
    np.testing.assert_array_equal(to_np(raw), host)  # device generator == the oracle's frame
    res = pipe.cell(raw, frame=t, id_start=id_start)
    cnt, rows = pipe.finish_cell(res)
    o = oracle.denoise_cell(host, SP, 10.0)
    # K1: q = rint(max(raw - gaussian_filter(raw), 0)); K2: the median of q
    np.testing.assert_array_equal(to_np(pipe.q), np.rint(o["residual"]).astype(spec.np_dtype))
    np.testing.assert_array_equal(to_np(pipe.med), np.rint(o["denoised"]).astype(spec.np_dtype))
    hist = oracle.histogram(o["denoised"])
    np.testing.assert_array_equal(pipe.hist.cpu().numpy()[: hist.size], hist)
    assert not pipe.hist.cpu().numpy()[hist.size:].any()
    assert int(pipe.otsu[0]) == oracle.otsu(hist)
    odets = oracle.segment_cell(o["denoised"], SP, frame=t, id_start=id_start, intensity=host)
    assert int(cnt[CNT_KEPT]) == len(rows) == len(odets) > 100
    assert list(rows["id"]) == [d.id for d in odets]
    assert list(rows["count"]) == [d.voxel_count for d in odets]
    assert list(rows["root"]) == [d.root for d in odets]
    np.testing.assert_array_equal(np.concatenate([rows["bbox_lo"], rows["bbox_hi"]], axis=1),
                                  np.array([d.bbox for d in odets]))
    np.testing.assert_array_equal(rows["intensity_sum"], np.array([d.intensity_sum for d in odets]))
    hostf = host.ravel()
    nx, ny, nz = spec.dims
    lin_all = np.concatenate([(d.voxels[:, 0] * ny + d.voxels[:, 1]) * nz + d.voxels[:, 2] for d in odets])
    means = np.array([hostf[(d.voxels[:, 0] * ny + d.voxels[:, 1]) * nz + d.voxels[:, 2]].mean() for d in odets])
    np.testing.assert_array_equal(rows["mean_intensity"], means)  # numpy's own mean, bit for bit
    np.testing.assert_array_equal(rows["centroid_um"], np.array([d.centroid_um for d in odets]))
    np.testing.assert_array_equal(rows["volume_um3"], np.array([d.volume_um3 for d in odets]))
    # C-order voxel lists, concatenated in id order
    np.testing.assert_array_equal(pipe.voxels[: lin_all.size].cpu().numpy().astype(np.int64), lin_all)
    np.testing.assert_array_equal(rows["voxel_offset"], np.concatenate([[0], np.cumsum(rows["count"])[:-1]]))
    # canonical label volume: rank of the kept cell, -1 elsewhere
    lab = np.full(nx * ny * nz, -1, np.int32)
    lab[lin_all] = np.repeat(np.arange(len(odets), dtype=np.int32), [d.voxel_count for d in odets])
    np.testing.assert_array_equal(pipe.labels.cpu().numpy().ravel(), lab)
    return res, odets


def check_vessel(pipe, spec, t, oracle):
    raw = synth.generate(spec, t, synth.VESSEL)
    host = host_frame(oracle, spec, t, synth.VESSEL)
    np.testing.assert_array_equal(to_np(raw), host)
    vres = pipe.vessel(raw)
    mask, dm = pipe.finish_vessel(vres, raw)
    st = oracle.mrf(host)
    assert st["iteration"] == 0
    state = vres.state.cpu().numpy()
    assert state[MRF_DECISION] == 0.0 and state[MRF_DELTA] == st["delta"]
    ss = oracle.sign_sum(host)
    assert state[MRF_NNZ] == np.count_nonzero(ss)
    om, odist, empty = oracle.segment_vessel(st["current"], SP)
    assert not empty and 0.001 < om.mean() < 0.5
    np.testing.assert_array_equal(mask.cpu().numpy(), om)
    np.testing.assert_array_equal(dm.values.cpu().numpy(), odist)  # same envelope arithmetic: bit-exact


@pytest.fixture(scope="module")
def c2_pipe(cuda):
    return FramePipeline(synth.C2.dims, "u8", ANISO)


@pytest.mark.parametrize("t", [0, 5])
def test_c2_time_point_vs_oracle(c2_pipe, oracle, t):
    """The bench workload: full C2 time points, both channels (t = 0 is the
    first frame of bench.py's input ring)."""
    assert c2_pipe.k1_path_tc  # the tensor-core K1 the bench times
    check_cell(c2_pipe, synth.C2, t, synth.CELL, oracle, id_start=1000 * t)
    check_vessel(c2_pipe, synth.C2, t, oracle)


def test_c3_time_point_vs_oracle(cuda, oracle):
    """C3: 1024x1024x64 u16 (12-bit), three channels -- cell, vessel, and the
    second cell channel (segmented through the cell path)."""
    spec = synth.C3
    pipe = FramePipeline(spec.dims, "u16", ANISO)
    _, d1 = check_cell(pipe, spec, 2, synth.CELL, oracle, id_start=0)
    check_vessel(pipe, spec, 2, oracle)
    _, d2 = check_cell(pipe, spec, 2, synth.CELL2, oracle, id_start=len(d1))
    assert d2[0].id == len(d1)


def test_c4_crop_nz96_vs_oracle(cuda, oracle):
    """nz = 96 kernels at C4's cell density (1024x1024x96 crop)."""
    spec = synth.C4_CROP
    pipe = FramePipeline(spec.dims, "u8", ANISO)
    assert pipe.k1_path_tc and pipe.rows_path
    check_cell(pipe, spec, 1, synth.CELL, oracle, id_start=7)
    check_vessel(pipe, spec, 1, oracle)


# ---------------------------------------------------------------------------
# shape-specialised kernel variants vs the oracle
# ---------------------------------------------------------------------------
def _median(v: np.ndarray, rad: int):
    t = torch.from_numpy(v if v.dtype != np.uint16 else v.view(np.int16)).cuda()
    if v.dtype == np.uint16:
        t = t.view(torch.uint16)
    out = torch.empty_like(t)
    hist = torch.zeros(65536, dtype=torch.int64, device=t.device)
    call("ct_median", t.data_ptr(), _dev.ct_code(t), *v.shape, rad, out.data_ptr(), hist.data_ptr(),
         _dev.stream_handle())
    return to_np(out), hist.cpu().numpy()


def _scene(rng, shape, vmax):
    """Smooth blobs + noise (runs of equal values, like real q volumes) or noise."""
    nx, ny, nz = shape
    g = np.add.outer(np.add.outer(np.sin(np.arange(nx) / 3.0), np.cos(np.arange(ny) / 5.0)),
                     np.sin(np.arange(nz) / 4.0))
    return np.clip((g + 3) / 6 * vmax * 0.6 + rng.integers(0, max(2, vmax // 20), shape), 0, vmax)


@pytest.mark.parametrize("nz", [32, 64, 96, 128, 40])
@pytest.mark.parametrize("nxy", [(40, 36), (17, 19)])
def test_median_u8_nz_variants_vs_oracle(cuda, oracle, nz, nxy):
    """median3_bits<u8, 8, WC> for nz = 32/64/96/128 (WC = 1..4: the bench's
    nz = 64 kernel is WC = 2) and the generic WC = 0 (nz = 40), full and
    partial tiles, with the fused histogram."""
    rng = np.random.default_rng(nz * 7 + nxy[0])
    shape = (*nxy, nz)
    for v in (rng.integers(0, 256, shape).astype(np.uint8), _scene(rng, shape, 255).astype(np.uint8),
              (rng.random(shape) < 0.1).astype(np.uint8) * 200):
        got, hist = _median(v, 1)
        ref = oracle.median(v.astype(np.float64), 1)
        np.testing.assert_array_equal(got.astype(np.float64), ref)
        np.testing.assert_array_equal(hist, np.bincount(ref.astype(np.int64).ravel(), minlength=65536))


@pytest.mark.parametrize("nz", [32, 64, 96, 128, 150])
def test_median_u16_variants_vs_oracle(cuda, oracle, nz):
    """median3_bits<u16, 16> (nz <= 128) and median3_int (nz > 128), 12-bit and
    full 16-bit values."""
    rng = np.random.default_rng(nz)
    shape = (21, 18, nz)
    for vmax in (4095, 65535):
        v = _scene(rng, shape, vmax).astype(np.uint16)
        got, hist = _median(v, 1)
        ref = oracle.median(v.astype(np.float64), 1)
        np.testing.assert_array_equal(got.astype(np.float64), ref)
        np.testing.assert_array_equal(hist, np.bincount(ref.astype(np.int64).ravel(), minlength=65536))


@pytest.mark.parametrize("rad", [4, 5])
def test_median_large_radius_vs_oracle(cuda, oracle, rad):
    """radius > 3 (median_radix, any window size) for every dtype."""
    rng = np.random.default_rng(rad)
    shape = (11, 9, 13)
    for v in (rng.integers(0, 256, shape).astype(np.uint8), rng.integers(0, 4096, shape).astype(np.uint16),
              rng.normal(3.0, 2.0, shape).clip(0)):
        got, _ = _median(v, rad)
        np.testing.assert_array_equal(got.astype(np.float64), oracle.median(v.astype(np.float64), rad))


def test_denoise_api_large_median_radius(cuda, oracle):
    """denoise_cell_channel with median_radius 4 (the reference accepts any r >= 1)."""
    from paper_1407_2089_b200 import denoise as D
    from paper_1407_2089_b200.imaging import VoxelGrid

    v = np.random.default_rng(3).integers(0, 256, (30, 26, 20)).astype(np.uint8)
    g = D.denoise_cell_channel(VoxelGrid(values=v, spacing=VoxelSpacing(1.0, 1.0, 1.0)),
                               D.CellDenoiseParams(3.0, median_radius=4))
    np.testing.assert_array_equal(g.values, oracle.denoise_cell(v, (1.0, 1.0, 1.0), 3.0, 4)["denoised"])


@pytest.mark.parametrize("shape", [(20, 18, 150), (9, 11, 257)])
def test_long_z_lines_vs_oracle(cuda, oracle, shape):
    """nz > 128: CCL tile path, EDT pass z for long lines, the integer MRF's
    global-memory statistics, closing -- all through the drop-in API."""
    from paper_1407_2089_b200 import denoise as D
    from paper_1407_2089_b200 import segment as S
    from paper_1407_2089_b200.imaging import VoxelGrid

    rng = np.random.default_rng(sum(shape))
    for thr in (0.6, 0.93):
        m = rng.random(shape) > thr
        np.testing.assert_array_equal(S.morphological_closing(m, 1), oracle.closing(m, 1))
        d_gpu = S.detections_from_mask(m, ANISO, frame=0, min_volume_um3=0.0)
        d_ora = oracle.detections(m, SP, min_volume_um3=0.0)
        assert [d.id for d in d_gpu] == [d.id for d in d_ora]
        for a, b in zip(d_gpu, d_ora):
            np.testing.assert_array_equal(a.voxels, b.voxels)
            np.testing.assert_array_equal(a.centroid_um, b.centroid_um)
        np.testing.assert_array_equal(S.distance_map(m, ANISO).values, oracle.edt(m, SP))
    ramp = np.add.outer(np.add.outer(np.arange(shape[0]), np.arange(shape[1])), np.arange(shape[2])) % 50
    for v in ((ramp + rng.integers(0, 9, shape)).astype(np.uint8), rng.integers(0, 256, shape).astype(np.uint8),
              (ramp * 40 + rng.integers(0, 300, shape)).astype(np.uint16)):
        st = D.mrf_denoise_state(VoxelGrid(values=v, spacing=ANISO))
        o = oracle.mrf(v)
        assert (st.sigma_hat, st.delta, st.iteration, st.converged) == \
            (o["sigma_hat"], o["delta"], o["iteration"], o["converged"])
        np.testing.assert_array_equal(np.asarray(st.current.values, dtype=np.float64), o["current"])


@pytest.mark.parametrize("shape", [(24, 40, 64), (14, 18, 96), (9, 11, 20)])
def test_ccl_rows_callee_fills_labels(cuda, oracle, shape):
    """ct_ccl26_rows with flags = 0 (the call fills the -1 background itself)
    equals the byte-mask CCL (only the pre-filled form was tested)."""
    nx, ny, nz = shape
    rng = np.random.default_rng(nx + ny + nz)
    v = (rng.random(shape) * 255).astype(np.uint8)
    dv = torch.from_numpy(v).cuda()
    otsu = torch.tensor([170, 0, 0, 0], dtype=torch.int64, device="cuda")
    work = torch.empty(workspace_bytes(1, nx, ny, nz, 1), dtype=torch.uint8, device="cuda")
    W = 1 if nz <= 64 else 2
    rows = torch.zeros(nx * ny * W, dtype=torch.int64, device="cuda")
    mask = torch.empty(shape, dtype=torch.uint8, device="cuda")
    s = _dev.stream_handle()
    call("ct_threshold_close_rows", dv.data_ptr(), 1, nx, ny, nz, otsu.data_ptr(), 0, mask.data_ptr(),
         rows.data_ptr(), work.data_ptr(), s)
    outs = []
    for flags in (None, 0):
        labels = torch.full(shape, 12345, dtype=torch.int32, device="cuda")  # garbage: the call must fill
        fg = torch.empty(nx * ny * nz, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
        if flags is None:
            call("ct_ccl26", mask.data_ptr(), nx, ny, nz, labels.data_ptr(), fg.data_ptr(), cnt.data_ptr(), s)
        else:
            call("ct_ccl26_rows", rows.data_ptr(), nx, ny, nz, labels.data_ptr(), fg.data_ptr(), cnt.data_ptr(),
                 flags, s)
        outs.append((labels.cpu().numpy(), cnt.cpu().numpy()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    m = mask.cpu().numpy()
    lab, n = oracle.label26(m)
    got = outs[1][0].ravel()
    assert outs[1][1][0] == m.sum()                                   # foreground voxels
    assert int((got == np.arange(got.size)).sum()) == n               # one root per component
    # same partition as the oracle's labels (label = min voxel index of the component)
    olab = lab.ravel()
    fgm = olab > 0
    order = np.flatnonzero(fgm)
    mins = np.full(n + 1, got.size, dtype=np.int64)
    np.minimum.at(mins, olab[order], order)
    np.testing.assert_array_equal(got[fgm], mins[olab[fgm]])
    assert np.all(got[~fgm] == -1)


@pytest.mark.parametrize("nz", [32, 64, 96, 128, 70])
def test_mrf_statistics_repeatable_vs_oracle(cuda, oracle, nz):
    """ct_mrf (exact sigma_hat) and ct_mrf_decide (certified decision), 6
    times each on the same volume: every run equals the oracle (delta, nnz,
    sigma_hat / decision).  Guards the plane-ring kernels against the
    ordering hazard fixed in round 2 (a fast warp's first ring store could
    replace plane i0-1 before a slow warp had read it)."""
    shape = (256, 200, nz)
    spec = synth.SceneSpec(*shape, "u8", n_cells=10, n_tubes=12, seed=3)
    v = synth.generate(spec, 0, synth.VESSEL)
    host = to_np(v)
    o = oracle.mrf(host)
    nnz = np.count_nonzero(oracle.sign_sum(host))
    nx, ny, _ = shape
    s = _dev.stream_handle()
    for fn in ("ct_mrf", "ct_mrf_decide"):
        for _ in range(6):
            work = torch.empty(workspace_bytes(4, nx, ny, nz, 1), dtype=torch.uint8, device="cuda")
            state = torch.zeros(9, dtype=torch.float64, device="cuda")
            hist = torch.zeros(65536, dtype=torch.int64, device="cuda")
            call(fn, v.data_ptr(), 1, nx, ny, nz, work.data_ptr(), state.data_ptr(), hist.data_ptr(), s)
            st = state.cpu().numpy()
            assert st[MRF_DELTA] == o["delta"] and st[MRF_NNZ] == nnz, (fn, st)
            if fn == "ct_mrf" or st[2] != 2.0:
                assert st[1] == o["sigma_hat"], (fn, st)
            assert st[MRF_DECISION] == 0.0


UNIT = VoxelSpacing(1.0, 1.0, 1.0)


@pytest.mark.parametrize("dims,dt,sigma,radius", [
    ((128, 128, 128), "u8", 1.0, 1), ((128, 128, 128), "u16", 2.0, 2), ((128, 128, 128), "u8", 4.0, 3),
    ((96, 64, 160), "u8", 3.0, 2), ((64, 48, 256), "u16", 4.0, 1), ((128, 96, 64), "u16", 3.0, 3)])
def test_c5_sweep_points_vs_oracle(cuda, oracle, dims, dt, sigma, radius):
    """BASELINE configs[4] (C5 sweep): unit spacing, sigma 1-4 voxels, median
    radius 1-3, u8 / u16, incl. nz > 128 (the generic z pass and byte-mask
    CCL) -- the fused path vs the oracle: q, median, histogram, threshold,
    detections, label volume and the vessel channel."""
    from paper_1407_2089_b200.denoise import CellDenoiseParams

    n = dims[0] * dims[1] * dims[2]
    spec = synth.SceneSpec(*dims, dt, n_cells=max(10, n * 50 // (256 * 256 * 32)),
                           n_tubes=max(3, 3 * dims[1] * dims[2] // (256 * 32)), seed=5)
    pipe = FramePipeline(dims, dt, UNIT, denoise=CellDenoiseParams(sigma, radius))
    sp = UNIT.as_array()
    raw = synth.generate(spec, 0, synth.CELL)
    host = host_frame(oracle, spec, 0, synth.CELL)
    np.testing.assert_array_equal(to_np(raw), host)
    cnt, rows = pipe.finish_cell(pipe.cell(raw, frame=0))
    o = oracle.denoise_cell(host, sp, sigma, radius)
    np.testing.assert_array_equal(to_np(pipe.q), np.rint(o["residual"]).astype(spec.np_dtype))
    np.testing.assert_array_equal(to_np(pipe.med), np.rint(o["denoised"]).astype(spec.np_dtype))
    hist = oracle.histogram(o["denoised"])
    np.testing.assert_array_equal(pipe.hist.cpu().numpy()[: hist.size], hist)
    assert int(pipe.otsu[0]) == oracle.otsu(hist)
    odets = oracle.segment_cell(o["denoised"], sp, frame=0, intensity=host)
    assert len(rows) == len(odets) > 0
    assert list(rows["count"]) == [d.voxel_count for d in odets]
    assert list(rows["root"]) == [d.root for d in odets]
    np.testing.assert_array_equal(rows["centroid_um"], np.array([d.centroid_um for d in odets]))
    nx, ny, nz = dims
    lab = np.full(n, -1, np.int32)
    for i, d in enumerate(odets):
        lab[(d.voxels[:, 0] * ny + d.voxels[:, 1]) * nz + d.voxels[:, 2]] = i
    np.testing.assert_array_equal(pipe.labels.cpu().numpy().ravel(), lab)
    vraw = synth.generate(spec, 0, synth.VESSEL)
    vhost = host_frame(oracle, spec, 0, synth.VESSEL)
    mask, dm = pipe.finish_vessel(pipe.vessel(vraw), vraw)
    st = oracle.mrf(vhost)
    om, odist, _ = oracle.segment_vessel(st["current"] if st["current"] is not None else vhost, sp)
    np.testing.assert_array_equal(mask.cpu().numpy(), om)
    np.testing.assert_array_equal(dm.values.cpu().numpy(), odist)


def test_cuda_graph_replay_matches_eager(cuda, oracle):
    """bench.py's timed loop replays per-frame CUDA graphs (FramePipeline.capture):
    replays on two streams, alternating two captured input frames, give the
    same results as the eager launches -- q, median, label volume, the cell
    table, the vessel mask and distance map -- and the cell results equal the
    oracle's."""
    spec = synth.SceneSpec(256, 192, 64, "u8", n_cells=120, n_tubes=9, seed=11)
    pipe = FramePipeline(spec.dims, "u8", ANISO)
    raws = [{ch: synth.generate(spec, t, ch) for ch in (synth.CELL, synth.VESSEL)} for t in range(2)]
    ref = []
    for r in raws:  # eager results (also the warm-up capture needs)
        cnt, rows = pipe.finish_cell(pipe.cell(r[synth.CELL]))
        vres = pipe.vessel(r[synth.VESSEL])
        torch.cuda.synchronize()
        ref.append((pipe.q.clone(), pipe.med.clone(), pipe.labels.clone(), rows.copy(), vres.mask.clone(),
                    vres.distance.clone()))
    gc = [pipe.capture(lambda r=r: pipe.cell(r[synth.CELL])) for r in raws]
    gv = [pipe.capture(lambda r=r: pipe.vessel(r[synth.VESSEL])) for r in raws]
    s_cell = torch.cuda.Stream(priority=-1)
    s_vess = torch.cuda.Stream()
    for step in range(5):
        i = step % 2
        s_cell.wait_stream(torch.cuda.current_stream())
        s_vess.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_cell):
            gc[i].replay()
        with torch.cuda.stream(s_vess):
            gv[i].replay()
        torch.cuda.current_stream().wait_stream(s_cell)
        torch.cuda.current_stream().wait_stream(s_vess)
        torch.cuda.synchronize()
        q, med, lab, rows, vm, vd = ref[i]
        assert torch.equal(pipe.q, q) and torch.equal(pipe.med, med) and torch.equal(pipe.labels, lab)
        nk = len(rows)
        got = pipe.table[: nk * rows.itemsize].cpu().numpy().view(rows.dtype)
        assert got.tobytes() == rows.tobytes()
        assert torch.equal(pipe.vmask, vm) and torch.equal(pipe.dist, vd)
    host = host_frame(oracle, spec, 1, synth.CELL)
    o = oracle.denoise_cell(host, SP, 10.0)
    odets = oracle.segment_cell(o["denoised"], SP, frame=1, intensity=host)
    assert [int(c) for c in ref[1][3]["count"]] == [d.voxel_count for d in odets]


@pytest.mark.parametrize("nz", [32, 64, 96, 128])
def test_edt_deep_z_envelopes_vs_oracle(cuda, oracle, nz):
    """Pass-z envelopes deeper than the 32 shared-memory stack entries of
    edt_pass_zr (the rest live in the dead pass-x buffer): one foreground
    line tilted through x as it runs along z, so in slice k the nearest site
    of a far column moves by half a voxel per slice and nearly every slice's
    parabola stays on the lower envelope (~55 of 64 entries); plus a second
    tilted line and random specks."""
    from paper_1407_2089_b200 import segment as S

    shape = (96, 40, nz)
    m = np.zeros(shape, dtype=bool)
    k = np.arange(nz)
    m[(4 + k // 2) % shape[0], 3, k] = True
    m[(90 - k // 3) % shape[0], 33, k] = True
    rng = np.random.default_rng(nz)
    m |= rng.random(shape) > 0.9995
    np.testing.assert_array_equal(S.distance_map(m, ANISO).values, oracle.edt(m, SP))


@pytest.mark.parametrize("nz", [32, 64, 96, 128])
def test_ccl_rows_vs_oracle_components(cuda, oracle, nz):
    """ct_ccl26_rows (the fused path's K5, which skips the links to rows
    (i, j-1), (i-1, j+-1) that a run of row (i-1, j) already implies) against
    the oracle's 26-connected components on masks rich in diagonal-only and
    corner-only contacts: sparse random masks, diagonal voxel chains and
    random balls.  GPU label = the component's minimum voxel index; each mask
    is labelled three times (run-to-run identical)."""
    from paper_1407_2089_b200._lib import call

    rng = np.random.default_rng(1000 + nz)
    shape = (40, 48, nz)
    nx, ny, _ = shape
    masks = [rng.random(shape) > t for t in (0.9, 0.8, 0.7, 0.5)]
    chains = np.zeros(shape, dtype=bool)
    for _ in range(60):  # diagonal chains: consecutive voxels touch only at edges / corners
        p = rng.integers(0, [nx, ny, nz])
        d = rng.choice([-1, 1], size=3) * rng.integers(0, 2, size=3)
        d[rng.integers(0, 3)] = rng.choice([-1, 1])
        for _s in range(rng.integers(3, 30)):
            if not (0 <= p[0] < nx and 0 <= p[1] < ny and 0 <= p[2] < nz):
                break
            chains[tuple(p)] = True
            p = p + d
    masks.append(chains)
    balls = np.zeros(shape, dtype=bool)
    ii, jj, kk = np.indices(shape)
    for _ in range(25):
        c, r = rng.integers(0, [nx, ny, nz]), rng.uniform(1.0, 4.0)
        balls |= (ii - c[0]) ** 2 + (jj - c[1]) ** 2 + (kk - c[2]) ** 2 <= r * r
    masks.append(balls | chains)
    W = 1 if nz <= 64 else 2
    s = _dev.stream_handle()
    for m in masks:
        lab, _n = oracle.label26(m)
        flat = lab.ravel()
        fg = flat >= 0 if flat.min() < 0 else m.ravel()
        # expected: every foreground voxel carries its component's minimum index
        comp = flat[fg]
        idx = np.nonzero(fg)[0]
        mins = {}
        for c, i in zip(comp.tolist(), idx.tolist()):
            if c not in mins:
                mins[c] = i  # idx ascending: the first is the minimum
        want = np.full(m.size, -1, dtype=np.int32)
        want[idx] = [mins[c] for c in comp.tolist()]
        words = np.zeros((nx * ny, W), dtype=np.uint64)
        mb = m.reshape(nx * ny, nz)
        for k in range(nz):
            words[:, k // 64] |= mb[:, k].astype(np.uint64) << np.uint64(k % 64)
        rows = torch.from_numpy(words.view(np.int64)).cuda()
        got = []
        for _rep in range(3):
            labels = torch.full(shape, -1, dtype=torch.int32, device="cuda")
            fgl = torch.empty(m.size, dtype=torch.int32, device="cuda")
            cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
            call("ct_ccl26_rows", rows.data_ptr(), nx, ny, nz, labels.data_ptr(), fgl.data_ptr(), cnt.data_ptr(), 1, s)
            torch.cuda.synchronize()
            got.append(labels.cpu().numpy().ravel())
        for g in got:
            np.testing.assert_array_equal(g, want)
