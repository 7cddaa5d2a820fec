"""segment_sequence (the process_experiment segmentation loop, ref
session.py:293-306) on one GPU against the reference's own per-frame loop
through the drop-in API: identical ids (the running det_counter), voxel
lists, centroids, volumes and distance maps."""

import numpy as np
import pytest
import torch

from paper_1407_2089_b200 import denoise as D
from paper_1407_2089_b200 import segment as S
from paper_1407_2089_b200 import synth
from paper_1407_2089_b200.imaging import VoxelGrid, VoxelSpacing
from paper_1407_2089_b200.sequence import segment_sequence

pytestmark = pytest.mark.gpu

ANISO = VoxelSpacing(0.8, 0.8, 1.0)


@pytest.mark.parametrize("dtype,loader", [("u8", "numpy"), ("u16", "numpy"), ("u8", "pinned"), ("u16", "cuda")])
def test_segment_sequence_matches_reference_loop(cuda, dtype, loader):
    """Pipelined two frames deep (frame t+1 queued before frame t is read
    back); numpy loaders copy synchronously, pinned / CUDA ones run async."""
    spec = synth.SceneSpec(128, 96, 32, dtype, n_cells=25, n_tubes=3, seed=21)
    T = 5
    frames_c = {t: synth.generate(spec, t, synth.CELL).cpu() for t in range(T)}
    frames_v = {t: synth.generate(spec, t, synth.VESSEL).cpu() for t in range(T)}

    def np_frame(x):
        return x.view(torch.int16).numpy().view(np.uint16) if x.dtype == torch.uint16 else x.numpy()

    if loader == "numpy":
        lc, lv = (lambda t: np_frame(frames_c[t])), (lambda t: np_frame(frames_v[t]))
    elif loader == "pinned":
        pc = {t: x.pin_memory() for t, x in frames_c.items()}
        pv = {t: x.pin_memory() for t, x in frames_v.items()}
        lc, lv = pc.__getitem__, pv.__getitem__
    else:
        dc = {t: x.cuda() for t, x in frames_c.items()}
        dv = {t: x.cuda() for t, x in frames_v.items()}
        lc, lv = dc.__getitem__, dv.__getitem__
    res = segment_sequence(lc, T, load_vessel=lv, spacing=ANISO, with_hull=True)
    # the reference loop (session.py:295-306) through the drop-in API
    det_counter = 0
    params, seg = D.CellDenoiseParams(), S.SegmentationConfig()
    for t in range(T):
        den = D.denoise_cell_channel(VoxelGrid(values=np_frame(frames_c[t]), spacing=ANISO), params)
        dets = S.segment_cell_channel(den, seg, frame=t, id_start=det_counter)
        assert res.id_starts[t] == det_counter
        det_counter += len(dets)
        got = res.detections_by_frame[t]
        assert [d.id for d in got] == [d.id for d in dets]
        assert [d.frame for d in got] == [t] * len(dets)
        for a, b in zip(got, dets):
            np.testing.assert_array_equal(a.voxels, b.voxels)
            np.testing.assert_array_equal(a.centroid_um, b.centroid_um)
            assert a.volume_um3 == b.volume_um3
            np.testing.assert_array_equal(a.hull.facets, b.hull.facets)
        rows = res.rows_by_frame[t]
        assert list(rows["id"]) == [d.id for d in dets]
        vden = D.mrf_denoise(VoxelGrid(values=np_frame(frames_v[t]), spacing=ANISO))
        _, dmap = S.segment_vessel_channel(vden, seg)
        np.testing.assert_array_equal(res.distance_maps[t].values.cpu().numpy(), dmap.values)
    assert res.det_counter == det_counter > 50
