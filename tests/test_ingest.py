"""Ingest: TIFF stacks -> (x, y, z) grids.

Mirrors ref tests/test_imaging.py (TestLoadFrame: declared dims, dtype kept,
save -> load round-trip identity; missing / unreadable file -> ManifestError
naming the path).  The reference writes and reads through tifffile, which is
not installed here; Pillow (present) is the independent TIFF implementation
the reader and writer are checked against, and numpy's transpose(2, 1, 0) is
the oracle for the (z, y, x) -> (x, y, z) step (ref imaging.py:219-220).
CPU tests cover the host reader/writer; GPU tests the device transpose,
load_tiff_volume / save_grid and the pipelined FrameIngest.
"""

import numpy as np
import pytest

from paper_1407_2089_b200 import ingest
from paper_1407_2089_b200.errors import ManifestError

Image = pytest.importorskip("PIL.Image")


def pil_pages(path):
    im = Image.open(path)
    out = []
    for i in range(im.n_frames):
        im.seek(i)
        out.append(np.array(im))
    return np.stack(out)


def pil_write(path, pages, mode=None, **kw):
    imgs = [Image.fromarray(p, mode=mode) if mode else Image.fromarray(p) for p in pages]
    imgs[0].save(path, save_all=True, append_images=imgs[1:], **kw)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.int16, np.uint32, np.int32, np.float32, np.float64])
def test_write_read_round_trip(tmp_path, dtype):
    rng = np.random.default_rng(7)
    if np.dtype(dtype).kind == "f":
        a = rng.standard_normal((4, 7, 9)).astype(dtype)
    else:
        info = np.iinfo(dtype)
        a = rng.integers(info.min, info.max, size=(4, 7, 9), dtype=dtype, endpoint=True)
    p = tmp_path / "rt.tif"
    ingest.write_tiff_pages(p, a)
    b = ingest.read_tiff_pages(p)
    assert b.dtype == a.dtype and b.shape == a.shape
    np.testing.assert_array_equal(a, b)
    with ingest.TiffStack(p) as ts:
        assert ts.dims == (9, 7, 4)
        assert ts.info.segments == 1  # pages written contiguously: one pread range


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_pillow_reads_our_files(tmp_path, dtype):
    a = np.random.default_rng(1).integers(0, np.iinfo(dtype).max, size=(5, 6, 11), dtype=dtype)
    p = tmp_path / "ours.tif"
    ingest.write_tiff_pages(p, a)
    np.testing.assert_array_equal(pil_pages(p), a)


def test_reads_pillow_files(tmp_path):
    a = np.random.default_rng(2).integers(0, 256, size=(6, 13, 10), dtype=np.uint8)
    p = tmp_path / "pil8.tif"
    pil_write(p, a)
    np.testing.assert_array_equal(ingest.read_tiff_pages(p), a)
    a16 = np.random.default_rng(3).integers(0, 65536, size=(3, 5, 8), dtype=np.uint16)
    p16 = tmp_path / "pil16.tif"
    pil_write(p16, a16)
    np.testing.assert_array_equal(ingest.read_tiff_pages(p16), a16)


def test_reads_big_endian_and_multi_strip(tmp_path):
    a16 = np.random.default_rng(4).integers(0, 65536, size=(3, 40, 24), dtype=np.uint16)
    p = tmp_path / "be.tif"
    # Pillow writes I;16B as big-endian samples in an MM file
    imgs = [Image.frombuffer("I;16B", (24, 40), x.astype(">u2").tobytes(), "raw", "I;16B", 0, 1) for x in a16]
    imgs[0].save(p, save_all=True, append_images=imgs[1:])
    with ingest.TiffStack(p) as ts:
        assert ts.dims == (24, 40, 3)
    np.testing.assert_array_equal(ingest.read_tiff_pages(p), a16)
    # several strips per page
    a8 = np.random.default_rng(5).integers(0, 256, size=(4, 50, 33), dtype=np.uint8)
    p8 = tmp_path / "strips.tif"
    pil_write(p8, a8, tiffinfo={278: 7})
    np.testing.assert_array_equal(ingest.read_tiff_pages(p8), a8)


def test_single_page_is_one_slice(tmp_path):
    a = np.arange(35, dtype=np.uint8).reshape(5, 7)
    p = tmp_path / "one.tif"
    Image.fromarray(a).save(p)
    b = ingest.read_tiff_pages(p)
    assert b.shape == (1, 5, 7)
    np.testing.assert_array_equal(b[0], a)


def test_unreadable_files_raise_manifest_error(tmp_path):
    with pytest.raises(ManifestError, match="missing.tif"):
        ingest.read_tiff_pages(tmp_path / "missing.tif")
    bad = tmp_path / "bad.tif"
    bad.write_bytes(b"not a tiff at all")
    with pytest.raises(ManifestError, match="bad.tif"):
        ingest.read_tiff_pages(bad)
    a = np.zeros((2, 8, 8), dtype=np.uint8)
    lzw = tmp_path / "lzw.tif"
    pil_write(lzw, a, compression="tiff_lzw")
    with pytest.raises(ManifestError, match="compression"):
        ingest.read_tiff_pages(lzw)
    ok = tmp_path / "trunc.tif"
    ingest.write_tiff_pages(ok, np.ones((3, 16, 16), dtype=np.uint8))
    data = ok.read_bytes()
    ok.write_bytes(data[: len(data) - 100])
    with pytest.raises(ManifestError, match="past end of file"):
        ingest.read_tiff_pages(ok)


def test_mixed_page_sizes_rejected(tmp_path):
    p = tmp_path / "mixed.tif"
    imgs = [Image.fromarray(np.zeros((8, 8), np.uint8)), Image.fromarray(np.zeros((9, 8), np.uint8))]
    imgs[0].save(p, save_all=True, append_images=imgs[1:])
    with pytest.raises(ManifestError, match="differs"):
        ingest.read_tiff_pages(p)


# ---------------------------------------------------------------------------
# device
# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.float32, np.float64])
@pytest.mark.parametrize("dims", [(9, 7, 4), (130, 3, 67), (64, 64, 64), (1, 5, 1)])
def test_gpu_load_tiff_volume_matches_transpose(tmp_path, dtype, dims):
    from paper_1407_2089_b200 import load_tiff_volume

    rng = np.random.default_rng(sum(dims))
    grid = (rng.standard_normal(dims) * 1000).astype(dtype) if np.dtype(dtype).kind == "f" else \
        rng.integers(0, np.iinfo(dtype).max, size=dims, dtype=dtype)
    p = tmp_path / "g.tif"
    ingest.write_tiff_pages(p, np.ascontiguousarray(grid.transpose(2, 1, 0)))
    got = load_tiff_volume(p)
    assert isinstance(got, np.ndarray) and got.dtype == grid.dtype and got.shape == dims
    np.testing.assert_array_equal(got, grid)
    dev = load_tiff_volume(p, device="cuda")
    assert dev.is_cuda and tuple(dev.shape) == dims


@pytest.mark.gpu
def test_gpu_big_endian_swapped_on_device(tmp_path):
    from paper_1407_2089_b200 import load_tiff_volume

    pages = np.random.default_rng(9).integers(0, 65536, size=(5, 33, 70), dtype=np.uint16)
    p = tmp_path / "be.tif"
    imgs = [Image.frombuffer("I;16B", (70, 33), x.astype(">u2").tobytes(), "raw", "I;16B", 0, 1) for x in pages]
    imgs[0].save(p, save_all=True, append_images=imgs[1:])
    np.testing.assert_array_equal(load_tiff_volume(p), pages.transpose(2, 1, 0))


@pytest.mark.gpu
def test_gpu_save_grid_round_trip(tmp_path):
    """ref test_imaging.py:120-133 round-trip identity (u16, dims (9, 7, 4))."""
    import torch

    from paper_1407_2089_b200 import VoxelGrid, VoxelSpacing, load_tiff_volume, save_grid

    values = np.random.default_rng(7).integers(0, 65536, size=(9, 7, 4), dtype=np.uint16)
    g = VoxelGrid(values=values, spacing=VoxelSpacing(1.0, 1.0, 1.0))
    save_grid(g, tmp_path / "rt.tif")
    np.testing.assert_array_equal(pil_pages(tmp_path / "rt.tif"), values.transpose(2, 1, 0))
    loaded = load_tiff_volume(tmp_path / "rt.tif")
    assert loaded.dtype == values.dtype
    np.testing.assert_array_equal(loaded, values)
    # device-resident grid (bool mask written as u8)
    m = torch.from_numpy(values > 30000).cuda()
    save_grid(VoxelGrid(values=m, spacing=g.spacing), tmp_path / "m.tif")
    np.testing.assert_array_equal(load_tiff_volume(tmp_path / "m.tif"), (values > 30000).astype(np.uint8))


@pytest.mark.gpu
@pytest.mark.parametrize("depth", [2, 3])
def test_gpu_frame_ingest_sequence(tmp_path, depth):
    import torch

    rng = np.random.default_rng(depth)
    grids, paths = [], []
    for t in range(7):
        g = rng.integers(0, 256, size=(40, 24, 16), dtype=np.uint8)
        p = tmp_path / f"t{t}.tif"
        ingest.write_tiff_pages(p, np.ascontiguousarray(g.transpose(2, 1, 0)))
        grids.append(g)
        paths.append(p)
    seen = []
    for k, grid in ingest.FrameIngest(paths, depth=depth, threads=3):
        # consume on the current stream like the pipeline does (a reduction)
        seen.append(int(grid.to(torch.int64).sum().item()))
        np.testing.assert_array_equal(grid.cpu().numpy(), grids[k])
    assert seen == [int(g.astype(np.int64).sum()) for g in grids]


@pytest.mark.gpu
def test_gpu_frame_ingest_rejects_mismatched_frame(tmp_path):
    a = np.zeros((4, 8, 8), np.uint8)
    ingest.write_tiff_pages(tmp_path / "a.tif", a)
    ingest.write_tiff_pages(tmp_path / "b.tif", np.zeros((5, 8, 8), np.uint8))
    with pytest.raises(ManifestError, match="dims"):
        for _ in ingest.FrameIngest([tmp_path / "a.tif", tmp_path / "b.tif"], depth=2):
            pass
