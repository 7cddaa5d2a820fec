"""The reference's own CPU throughput on the bench workload:
the live `clonetrack` package (scipy / numpy, imported read-only from
/root/reference -- so this runs only in the build container, not on the GPU
box) on synthetic C2 time points, the process_experiment loop body
(ref session.py:296-306): denoise_cell_channel + segment_cell_channel,
mrf_denoise + segment_vessel_channel.  TIFF I/O excluded (frames in memory).

  (i)  one process, time points 0..K-1 in turn (scipy is single-threaded);
  (ii) multiprocessing.Pool(cores) over (frame, channel) volumes.

Reported with hulls (the stock segment_cell_channel, Qhull per detection)
and with compute_hull replaced by a no-op (the like-for-like number for the
GPU path's e2e, which leaves hulls to the host).  Frames come from the
oracle's synthetic generator (the same volumes the GPU bench segments).

  python tools/ref_cpu_timing.py [--frames 2] [--pool-frames 8] > profiles/r02_reference_python_cpu.json
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

SP = (0.8, 0.8, 1.0)


def frame(t, ch):
    from oracle import oracle as O
    from paper_1407_2089_b200 import synth

    spec = synth.C2
    if ch == synth.VESSEL:
        return O.synth_frame(spec.dims, spec.dtype, spec.frame_seed(t, ch), spec.vmax, tubes=spec.tubes(),
                             amp_tube=spec.amp_tube)
    return O.synth_frame(spec.dims, spec.dtype, spec.frame_seed(t, ch), spec.vmax, balls=spec.balls(t, ch),
                         amp_ball=spec.amp_cell)


def run_volume(args):
    """One (frame, channel) volume through the reference; returns seconds."""
    t, ch, hulls = args
    import _refimport

    ct = _refimport.clonetrack()
    from clonetrack import denoise, imaging, segment

    if not hulls:
        segment.compute_hull = lambda vox, spacing: None
    raw = frame(t, ch)
    grid = imaging.VoxelGrid(values=raw, spacing=imaging.VoxelSpacing(*SP))
    t0 = time.perf_counter()
    if ch == 1:
        vden = denoise.mrf_denoise(grid, max_iters=1000)
        segment.segment_vessel_channel(vden)
        n = None
    else:
        den = denoise.denoise_cell_channel(grid, denoise.CellDenoiseParams())
        n = len(segment.segment_cell_channel(den, frame=t))
    del ct
    return time.perf_counter() - t0, n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=2)
    ap.add_argument("--pool-frames", type=int, default=8)
    a = ap.parse_args()
    cores = os.cpu_count() or 1
    nvox = 1024 * 1024 * 64
    out = {"workload": "C2: 1024x1024x64 uint8, 2 channels (cell + vessel), synthetic (oracle generator)",
           "reference": "clonetrack (live, /root/reference/pkg/src) with scipy "
                        f"{__import__('scipy').__version__}, numpy {np.__version__}",
           "host": f"build container, {cores} cores (NOT the GPU box; the bench's --impl reference arm is the "
                   "OpenMP oracle port timed on the GPU box)",
           "timing": "wall clock per (frame, channel) volume, frames in memory (TIFF I/O excluded)"}
    for hulls in (False, True):
        key = "with_hulls" if hulls else "hulls_excluded"
        secs, cells = [], []
        for t in range(a.frames):
            for ch in (0, 1):
                dt, n = run_volume((t, ch, hulls))
                secs.append(dt)
                if n is not None:
                    cells.append(n)
                print(f"[ref] {key} single t={t} ch={ch}: {dt:.1f} s", file=sys.stderr, flush=True)
        single = {"volumes": len(secs), "seconds": sum(secs), "voxels_per_s": len(secs) * nvox / sum(secs),
                  "per_volume_s": secs, "cells_per_frame": cells}
        jobs = [(t, ch, hulls) for t in range(a.pool_frames) for ch in (0, 1)]
        t0 = time.perf_counter()
        with mp.get_context("spawn").Pool(cores) as pool:
            res = pool.map(run_volume, jobs, chunksize=1)
        wall = time.perf_counter() - t0
        pooled = {"processes": cores, "volumes": len(jobs), "wall_s": wall, "voxels_per_s": len(jobs) * nvox / wall,
                  "note": "wall clock incl. per-process import and frame synthesis"}
        print(f"[ref] {key} pool: {wall:.1f} s for {len(jobs)} volumes", file=sys.stderr, flush=True)
        out[key] = {"single_process": single, "pool": pooled}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
