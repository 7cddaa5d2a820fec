"""BASELINE configs[4] ("C5"): kernel roofline sweep -- unit spacing
(sigma_um = sigma_vox), Gaussian sigma 1-4, median radius 1-3, volumes 128^3,
256^3, 512^2 x 128, 1024^2 x 128, u8 and u16.

Each (dtype, volume) gets synthetic cell and vessel frames at C1's cell
density.  K1 is timed per sigma (median radius 1), K2 per median radius
(sigma 2), the other stages once; CUDA events around each stage on its
stream, mean of --reps passes after one untimed pass.  GB/s are SURVEY 8d's
algorithmic bytes per voxel / stage time; `frac` is against
MEASURED_PEAKS.json hbm_gbs.  One JSON line per (dtype, volume, stage,
parameter) plus a table on stderr.

  python tools/sweep_c5.py [--reps 3] [--sizes 128,256,512x128,1024x128] [--dtypes u8,u16]

Under ncu (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum`, --reps 1) the launch list gives each kernel's DRAM
GB/s (tools/launches.py).
"""
import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1407_2089_b200 import synth  # noqa: E402
from paper_1407_2089_b200.denoise import CellDenoiseParams  # noqa: E402
from paper_1407_2089_b200.imaging import VoxelSpacing  # noqa: E402
from paper_1407_2089_b200.pipeline import FramePipeline  # noqa: E402

SIZES = {"128": (128, 128, 128), "256": (256, 256, 256), "512x128": (512, 512, 128), "1024x128": (1024, 1024, 128)}


def peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def bytes_per_voxel(stage, b, rows_path):
    """SURVEY 8d algorithmic bytes per voxel of a fused stage (b = input bytes)."""
    return {"K1 gaussian": 2 * b, "K2 median+hist": 2 * b,
            "K4 threshold+close": (b + 0.125) if rows_path else (b + 1), "K5 ccl": 0.125 if rows_path else 1,
            "K7 mrf": b, "K3+K4 vessel otsu+close": b + 1, "K8 edt": 9}.get(stage)


def timed(pipe, fn, reps):
    fn()  # untimed: first-launch costs
    torch.cuda.synchronize()
    pipe.marks = []
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    out = pipe.stage_times_ms()
    pipe.marks = None
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--sizes", default=",".join(SIZES))
    ap.add_argument("--dtypes", default="u8,u16")
    ap.add_argument("--sigmas", default="1,2,3,4")
    ap.add_argument("--radii", default="1,2,3")
    a = ap.parse_args()
    pk, pk_src = peak_gbs()
    sp = VoxelSpacing(1.0, 1.0, 1.0)
    sigmas = [float(s) for s in a.sigmas.split(",")]
    radii = [int(r) for r in a.radii.split(",")]
    lines = []

    def emit(rec):
        lines.append(rec)
        print(json.dumps(rec), flush=True)

    for dt in a.dtypes.split(","):
        b = 1 if dt == "u8" else 2
        for sz in a.sizes.split(","):
            dims = SIZES[sz]
            n = dims[0] * dims[1] * dims[2]
            # C1's densities: 50 cells per 256 x 256 x 32 voxels, 3 tubes per 256 x 32 y-z section
            spec = synth.SceneSpec(*dims, dt, n_cells=max(10, n * 50 // (256 * 256 * 32)),
                                   n_tubes=max(3, 3 * dims[1] * dims[2] // (256 * 32)), seed=5)
            rc = synth.generate(spec, 0, synth.CELL)
            rv = synth.generate(spec, 0, synth.VESSEL)
            base = {"config": "C5", "dtype": dt, "dims": list(dims), "voxels": n}

            def rec(stage, ms, pipe, **kw):
                bb = bytes_per_voxel(stage, b, pipe.rows_path if hasattr(pipe, "rows_path") else False)
                gbs = bb * n / (ms / 1e3) / 1e9 if bb else None
                emit({**base, "stage": stage, **kw, "ms": ms, "algorithmic_bytes_per_voxel": bb, "gbs": gbs,
                      "frac": gbs / pk if gbs else None})

            # K1 per sigma (median radius 1); the rest of the cell path at sigma 2
            for sig in sigmas:
                pipe = FramePipeline(dims, dt, sp, denoise=CellDenoiseParams(sig, 1), vessel=False)
                st = timed(pipe, lambda: pipe.cell(rc), a.reps)
                rec("K1 gaussian", st["K1 gaussian"], pipe, sigma_vox=sig, r_taps=list(pipe.r),
                    k1_path="tensor" if pipe.k1_path_tc else "fp64-fma")
                if sig == 2.0:
                    for k in ("K3 otsu", "K4 threshold+close", "K5 ccl", "K6 table"):
                        rec(k, st[k], pipe, sigma_vox=sig)
                    for r in radii:
                        pipe.denoise = dataclasses.replace(pipe.denoise, median_radius=r)
                        st2 = timed(pipe, lambda: pipe.cell(rc), a.reps)
                        rec("K2 median+hist", st2["K2 median+hist"], pipe, median_radius=r)
                del pipe
                torch.cuda.empty_cache()
            vp = FramePipeline(dims, dt, sp, cell=False)
            st = timed(vp, lambda: vp.vessel(rv), a.reps)
            for k in ("K7 mrf", "K3+K4 vessel otsu+close", "K8 edt"):
                rec(k, st[k], vp)
            del vp, rc, rv
            torch.cuda.empty_cache()

    print(f"# HBM peak {pk:.0f} GB/s ({pk_src})", file=sys.stderr)
    print(f"{'dtype':5s} {'dims':16s} {'stage':26s} {'param':10s} {'ms':>8s} {'GB/s':>8s} {'frac':>6s}",
          file=sys.stderr)
    for r in lines:
        par = (f"sigma={r['sigma_vox']:g}" if "sigma_vox" in r and r["stage"] == "K1 gaussian"
               else f"r={r['median_radius']}" if "median_radius" in r else "")
        g = f"{r['gbs']:8.0f}" if r["gbs"] else "       -"
        f = f"{r['frac']:6.3f}" if r["frac"] else "     -"
        print(f"{r['dtype']:5s} {'x'.join(map(str, r['dims'])):16s} {r['stage']:26s} {par:10s} {r['ms']:8.3f} {g} {f}",
              file=sys.stderr)


if __name__ == "__main__":
    main()
