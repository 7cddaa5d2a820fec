"""Files -> device grids -> fused pipeline, C2 (SURVEY 8f item 3 measurement).

Writes T time points of both C2 channels as TIFF stacks (z, y, x pages, the
reference's on-disk layout), then times FrameIngest (threaded pread into
pinned memory, H2D, device transpose) feeding FramePipeline.cell/vessel.
Reported: ingest-only GB/s (no pipeline) and files->results voxels/s.  The
page cache is warm after writing (say so when quoting the number).
python tools/ingest_bench.py [--frames 6] [--dir /tmp/ct_ingest] [--threads 8]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_2089_b200 import ingest, synth  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.pipeline import FramePipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=6)
ap.add_argument("--dir", default="/tmp/ct_ingest")
ap.add_argument("--threads", type=int, default=8)
ap.add_argument("--depth", type=int, default=3)
a = ap.parse_args()
spec = synth.C2
os.makedirs(a.dir, exist_ok=True)
paths = {0: [], 1: []}
t0 = time.perf_counter()
for t in range(a.frames):
    for ch, kind in ((0, synth.CELL), (1, synth.VESSEL)):
        p = os.path.join(a.dir, f"t{t}_c{ch}.tif")
        g = synth.generate(spec, t, kind)
        pages = torch.empty((spec.nz, spec.ny, spec.nx), dtype=g.dtype, device=g.device)
        ingest.transpose_xz(g, pages, spec.nx, spec.ny, spec.nz)
        ingest.write_tiff_pages(p, pages.cpu().numpy())
        paths[ch].append(p)
torch.cuda.synchronize()
print(f"wrote {2 * a.frames} stacks in {time.perf_counter() - t0:.1f} s", file=sys.stderr)
nvox = spec.nx * spec.ny * spec.nz
order = [p for t in range(a.frames) for p in (paths[0][t], paths[1][t])]

# ingest alone
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k, grid in ingest.FrameIngest(order, depth=a.depth, threads=a.threads):
        pass
    torch.cuda.synchronize()
    dt_ing = time.perf_counter() - t0
ing_gbs = len(order) * nvox / dt_ing / 1e9

# files -> pipeline results (counters + table rows read on the host per time point)
pipe = FramePipeline(spec.dims, spec.dtype, VoxelSpacing(0.8, 0.8, 1.0))
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cells = 0
    for k, grid in ingest.FrameIngest(order, depth=a.depth, threads=a.threads):
        if k % 2 == 0:
            pipe.cell(grid, frame=k // 2)
            cells += int(pipe.counters[2].item())
        else:
            pipe.vessel(grid)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(json.dumps({
    "workload": f"C2 {a.frames} time points x 2 channels from TIFF stacks ({spec.nx}x{spec.ny}x{spec.nz} u8)",
    "ingest_only_GBps": ing_gbs, "files_to_results_voxels_per_s": len(order) * nvox / dt,
    "ms_per_time_point": dt / a.frames * 1e3, "threads": a.threads, "depth": a.depth, "cells_total": cells,
    "note": "host wall clock; page cache warm (files just written); pread -> pinned -> H2D -> device transpose",
}))
