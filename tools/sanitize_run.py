"""Small workload that launches every libct kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  fused FramePipeline, u8 and u16, nz = 32 / 64 (tensor-core K1 passes x, y,
  z with TMA / mbarrier / TMEM, certified fix-up, integer median + SMEM
  histograms, Otsu, packed-row closing, run-based union-find CCL with its
  atomics, cell table incl. the radix-sort ordering, MRF decision, EDT),
  then the drop-in API paths (scipy-order K1, float median r = 1..3, byte
  closing + CCL, MRF iterations, EDT on a sparse mask, voxel runs).

  tools/sanitize.sh runs it under each tool (logs in gpurun_out/).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_2089_b200 import synth  # noqa: E402
from paper_1407_2089_b200.denoise import CellDenoiseParams, denoise_cell_channel, mrf_denoise_state  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelGrid, VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.pipeline import FramePipeline  # noqa: E402
from paper_1407_2089_b200.segment import (  # noqa: E402
    distance_map, encode_voxel_runs, segment_cell_channel, segment_vessel_channel)

sp = VoxelSpacing(0.8, 0.8, 1.0)
torch.cuda.set_device(0)
for dims, dt, nc in (((96, 80, 32), "u8", 12), ((64, 64, 64), "u8", 10), ((64, 64, 64), "u16", 10)):
    spec = synth.SceneSpec(*dims, dt, n_cells=nc, seed=3)
    pipe = FramePipeline(spec.dims, dt, sp)
    for t in range(2):
        rc = synth.generate(spec, t, synth.CELL)
        rv = synth.generate(spec, t, synth.VESSEL)
        cnt, rows = pipe.finish_cell(pipe.cell(rc, frame=t))
        mask, dm = pipe.finish_vessel(pipe.vessel(rv), rv)
        torch.cuda.synchronize()
        print(f"fused {dims} {dt} t={t}: {len(rows)} cells, k1 {'tc' if pipe.k1_path_tc else 'fp64'}, "
              f"vessel fg {int(mask.sum())}", flush=True)
    # drop-in API (numpy in / numpy out): exact K1, float median, detections with hulls
    raw = synth.generate(spec, 0, synth.CELL).cpu().numpy().astype(np.float64) if dt == "u8" else None
    if raw is not None:
        for r in (1, 2, 3):
            den = denoise_cell_channel(VoxelGrid(values=raw, spacing=sp), CellDenoiseParams(10.0, r))
        dets = segment_cell_channel(den, frame=0)
        runs = encode_voxel_runs(dets[0].voxels) if dets else None
        print(f"api {dims}: {len(dets)} detections, runs {None if runs is None else len(runs)}", flush=True)
        vraw = synth.generate(spec, 0, synth.VESSEL).cpu().numpy().astype(np.float64)
        st = mrf_denoise_state(VoxelGrid(values=vraw, spacing=sp), max_iters=3)
        m, d = segment_vessel_channel(st.current)
        print(f"api vessel: iterations {st.iteration}, fg {int(np.asarray(m).sum())}", flush=True)
# MRF that iterates (small noisy grid) and an EDT of a sparse mask
rng = np.random.default_rng(1)
g = rng.integers(0, 4, size=(16, 16, 16)).astype(np.float64)
st = mrf_denoise_state(VoxelGrid(values=g, spacing=sp), max_iters=5)
mk = np.zeros((40, 33, 20), dtype=bool)
mk[5, 7, 3] = mk[30, 2, 19] = True
dmap = distance_map(mk, sp)
print(f"mrf iterations {st.iteration}; sparse edt max {float(np.max(dmap.values)):.3f}", flush=True)
torch.cuda.synchronize()
print("sanitize workload done")
