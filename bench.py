#!/usr/bin/env python
"""Benchmark: segmented voxels/s of the per-frame 3-D segmentation hot path.

Workload (BASELINE.json configs[1], "C2"): synthetic 1024x1024x64 uint8 time
points with two channels (cell + vessel), spacing (0.8, 0.8, 1.0) um, the
reference's default parameters (session.py:70-74).  One step = one time point:
the cell channel (Gaussian background, median, Otsu, closing, 26-CCL, per-cell
table) and the vessel channel (MRF statistics, Otsu, closing, EDT), the two
channels on two CUDA streams.  value = voxels of all processed (frame,
channel) volumes / device time (max over ranks).  Frames are independent:
N GPUs shard time points (weak scaling); the only collective is an
all_gather of per-frame detection counts (global id offsets).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "segmented voxels/sec (frames/sec) at 1/2/4/8 B200; % HBM roofline; vs host CPU"
UNIT = "voxels/s"
SPACING = (0.8, 0.8, 1.0)
K1_FP64_OPS_PER_VOXEL = None  # filled from the radii: 3*(rx+ry+rz) + 3


def peaks():
    # fallback: /opt/skills/guides/B200_PROFILING.md (6.65 TB/s, 1.59 PFLOP/s bf16 dense)
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        # burst figures: every roofline stage is timed alone (serialized pass)
        p = {"hbm_gbs": float(m["hbm_gbs"]), "bf16_tflops": float(m.get("bf16_tflops", 1590.0)),
             "source": "MEASURED_PEAKS.json", "sm_max_mhz": m.get("sm_max_mhz")}
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_first(self, keep_busy, timeout=10.0):
        """Keep the GPU busy (untimed) until nvidia-smi has produced a sample."""
        t_end = time.monotonic() + timeout
        while self.proc and not self.lines and time.monotonic() < t_end:
            keep_busy()

    def mark(self, which):
        setattr(self, which, time.monotonic())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        # samples inside the timed window (plus one sampling period either side)
        inside = [ln for t, ln in self.lines if t0 is None or t0 - 0.025 <= t <= t1 + 0.025]
        for ln in inside:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg / --impl reference arm)
# ---------------------------------------------------------------------------
def cpu_sample_voxels_per_s(spec, t: int, crop_nx: int, threads: int):
    """Oracle (test-only checker, oracle/) on a bounded sample: both channels of
    time point t, cropped to crop_nx x-slices.  Returns (voxels/s, seconds)."""
    os.environ["OMP_NUM_THREADS"] = str(threads)
    from oracle import oracle as O

    O.lib()
    dims = (crop_nx, spec.ny, spec.nz)
    balls = spec.balls(t)
    balls = balls[balls[:, 0] < crop_nx * 16]
    raw_c = O.synth_frame(dims, spec.dtype, spec.frame_seed(t, 0), spec.vmax, balls=balls, amp_ball=spec.amp_cell)
    raw_v = O.synth_frame(dims, spec.dtype, spec.frame_seed(t, 1), spec.vmax, tubes=spec.tubes(),
                          amp_tube=spec.amp_tube)
    t0 = time.perf_counter()
    den = O.denoise_cell(raw_c, SPACING, 10.0)["denoised"]
    O.segment_cell(den, SPACING)
    st = O.mrf(raw_v)
    cur = st["current"] if st["current"] is not None else raw_v
    O.segment_vessel(cur, SPACING)
    dt = time.perf_counter() - t0
    return 2 * crop_nx * spec.ny * spec.nz / dt, dt


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_1407_2089_b200 import synth

    O.lib()
    spec = synth.C2
    threads = os.cpu_count() or 1
    crop = args.cpu_crop
    vals = []
    for s in range(args.warmup + args.steps):
        v, dt = cpu_sample_voxels_per_s(spec, s % 100, crop, threads)
        if s >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    sample = f"oracle port, both channels of C2 time points cropped to {crop}x1024x64 per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 2 * crop * spec.ny * spec.nz / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "C2 1024x1024x64 u8, 2 channels (cell+vessel), cropped sample", "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
GATHER_ROWS = 2048  # per-cell records exchanged per frame and rank (C2: ~1,550 cells)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1407_2089_b200 import _lib, synth
    from paper_1407_2089_b200.distributed import gather_tables
    from paper_1407_2089_b200.imaging import VoxelSpacing
    from paper_1407_2089_b200.pipeline import FramePipeline

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    spec = synth.C2
    sp = VoxelSpacing(*SPACING)
    T = 100
    nvox = spec.nx * spec.ny * spec.nz
    per_rank = (T + world - 1) // world
    my_frames = [rank * per_rank + i for i in range(per_rank) if rank * per_rank + i < T] or [rank % T]
    ring = min(args.ring, len(my_frames))

    # the cell stream gets the higher priority: its persistent tensor-core K1
    # CTAs then take SMs as soon as they free up and the latency-bound vessel
    # kernels fill the gaps (1.75 vs 1.84 ms per step with equal priorities).
    # A/B knob CT_PRIO: "cell" (default), "vessel", "none"
    prio = os.environ.get("CT_PRIO", "cell")
    s_cell = torch.cuda.Stream(dev, priority=-1 if prio == "cell" else 0)
    s_vess = torch.cuda.Stream(dev, priority=-1 if prio == "vessel" else 0)
    pipe = FramePipeline(spec.dims, spec.dtype, sp)
    # inputs resident in HBM (a ring of distinct time points; 134 MB/step > L2)
    inputs = []
    for i in range(ring):
        t = my_frames[i]
        inputs.append((t, synth.generate(spec, t, synth.CELL), synth.generate(spec, t, synth.VESSEL)))
    counts_dev = torch.zeros(1, dtype=torch.int64, device=dev)
    gathered = torch.zeros(world, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()

    # Time points are queued back to back: each channel's stream runs its
    # frames in order (its buffers are reused frame to frame), the two
    # channels share no buffers, so the vessel work of time point t may still
    # run while the cell work of t+1 starts.  The timed region ends with both
    # streams joined.  (CT_STEP_JOIN=1: join both streams after every step.)
    join_each = os.environ.get("CT_STEP_JOIN", "0") == "1"

    def step(i, timing=False, coll=True, first=True):
        t, rc, rv = inputs[i % ring]
        main = torch.cuda.current_stream()
        if join_each or first:
            s_cell.wait_stream(main)
            s_vess.wait_stream(main)
        with torch.cuda.stream(s_cell):
            pipe.cell(rc, frame=t, id_start=0)
            counts_dev.copy_(pipe.counters[2:3])
        with torch.cuda.stream(s_vess):
            pipe.vessel(rv)
        if join_each:
            main.wait_stream(s_vess)
        if join_each or (world > 1 and coll):
            main.wait_stream(s_cell)  # the collectives read this step's cell results
        if world > 1 and coll:
            # the frame's detection count (global ids) and its per-cell records, over NCCL
            dist.all_gather_into_tensor(gathered, counts_dev)
            gather_tables(pipe.table, pipe.counters[2], max_rows=GATHER_ROWS)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # correctness guard: the fused path's decisions must be the fast ones
    assert int(pipe.state[5].item()) == 0, "MRF needed iterations: bench workload assumption broken"

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first(lambda: (step(0, coll=False), torch.cuda.synchronize()))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    _lib.launch_counter.update(enabled=True, count=0)
    pipe.marks = []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.mark("t0")
    e0.record()
    for i in range(args.steps):
        step(args.warmup + i, first=(i == 0))
    main_s = torch.cuda.current_stream()
    main_s.wait_stream(s_cell)
    main_s.wait_stream(s_vess)
    e1.record()
    torch.cuda.synchronize()
    clocks.mark("t1")
    _lib.launch_counter["enabled"] = False
    launches = _lib.launch_counter["count"]
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    stage_ms = pipe.stage_times_ms()
    pipe.marks = None
    t_dev = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    ms_max = float(t_dev.item())
    total_vox = world * args.steps * 2 * nvox
    value = total_vox / (ms_max / 1e3)

    # --- serialized pass (one stream) for clean per-kernel times ----------
    pipe.marks = []
    for i in range(min(3, args.steps)):
        t, rc, rv = inputs[i % ring]
        pipe.cell(rc, frame=t)
        pipe.vessel(rv)
    torch.cuda.synchronize()
    serial_ms = pipe.stage_times_ms()
    pipe.marks = None

    # --- e2e through the public pipeline API with pinned host buffers -------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, pipe, spec, sp, dev, world, s_cell, s_vess)
        e2e["materialized"] = run_materialized(args, pipe, spec, dev, world)

    # --- roofline of the dominant stage -------------------------------------
    # algorithmic HBM bytes per voxel of each stage (inputs read + outputs
    # written once) and, for K1, the int8 tensor-core work per voxel
    pk = peaks()
    rx, ry, rz = pipe.r
    nzv = spec.nz
    k1_tc = pipe.k1_path_tc
    k1_macs = (4 * 256 + 13 * 256 + 13 * nzv) if k1_tc else None  # limb-pair MMAs (see k_gauss_tc.cu)
    bpv = {"K1 gaussian": 2, "K2 median+hist": 2, "K4 threshold+close": 2, "K5 ccl": 5, "K6 table": 0,
           "K7 mrf": 3, "K3+K4 vessel otsu+close": 2, "K8 edt": 9}
    kernels, kernels_serial = {}, {}
    for src, dst in ((stage_ms, kernels), (serial_ms, kernels_serial)):
        for k, v in src.items():
            b = bpv.get(k)
            dst[k] = {"ms": v, "hbm_gbs": (b * nvox / (v / 1e3) / 1e9) if b else None,
                      "hbm_frac": (b * nvox / (v / 1e3) / 1e9 / pk["hbm_gbs"]) if b else None,
                      "algorithmic_bytes_per_voxel": b}
    dom = max(serial_ms, key=serial_ms.get)
    ms_dom = serial_ms[dom]
    if dom == "K1 gaussian" and k1_tc:
        int8_peak = 2.0 * pk["bf16_tflops"]
        achieved = 2 * k1_macs * nvox / (ms_dom / 1e3) / 1e12
        roof = {"kernel": "K1 gaussian on tcgen05 int8 (limb-split taps, 3 banded GEMM passes)", "bound": "tensor",
                "achieved": achieved, "peak": int8_peak, "unit": "TFLOP/s", "frac": achieved / int8_peak,
                "unit_note": "int8 tensor ops (multiply + add = 2), dense",
                "peak_source": "2 x measured dense bf16 (" + pk["source"] + "): B200 int8 dense = 2x bf16",
                "work_per_voxel": {"int8_macs": k1_macs, "useful_taps": (2 * rx + 1) + (2 * ry + 1) + (2 * rz + 1)}}
        # SURVEY 8d's algorithmic figure for K1: the reference's float64 ops
        # (3 (rx + ry + rz) + 3 per voxel), against the measured FP64 DADD/DMUL
        # rate of this GPU -- the roofline a float64 implementation would face
        alg = 3 * (rx + ry + rz) + 3
        fp64_pk = measured_fp64_peak(dev)
        alg_tf = alg * nvox / (ms_dom / 1e3) / 1e12
        roof["algorithmic"] = {"fp64_ops_per_voxel": alg, "achieved_tflops": alg_tf,
                               "fp64_peak_measured_tflops": fp64_pk,
                               "frac_of_fp64_peak": alg_tf / fp64_pk if fp64_pk == fp64_pk else None}
    else:
        b = bpv.get(dom) or 1
        achieved = b * nvox / (ms_dom / 1e3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "peak_source": pk["source"], "algorithmic_bytes_per_voxel": b}
    roof.update({"stage": dom, "ms_serial": ms_dom, "ms_overlapped": stage_ms.get(dom),
                 "timing": "CUDA events around the stage on its stream, serialized pass (3 time points)",
                 "traffic": ncu_traffic(dom),
                 "traffic_note": "DRAM bytes of the stage's kernels per time point, ncu launch list (profiles/)",
                 "share_of_step_serial": ms_dom / sum(serial_ms.values())})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, dt = cpu_sample_voxels_per_s(spec, 0, args.cpu_baseline_crop, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"oracle/ct_oracle.c port (OpenMP), both channels of C2 t=0 "
                         f"({args.cpu_baseline_crop}x1024x64 per channel, {dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "C2: 1024x1024x64 uint8 time points, 2 channels (cell+vessel), 1600 cells",
                       "global_batch": world, "parallelism": f"frame-sharded dp{world}",
                       "frames_per_s": world * args.steps / (ms_max / 1e3),
                       "l2": f"inputs larger than L2: {2 * nvox / 1e6:.0f} MB/step from a ring of {ring} "
                             "distinct time points, plus GB-scale intermediates"},
            "e2e": e2e, "gpu_launches": launches, "clocks": clk, "roofline": roof, "kernels": kernels,
            "kernels_serial": kernels_serial,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def measured_fp64_peak(dev) -> float:
    """TFLOP/s of independent DADD/DMUL (no FMA) measured on this GPU."""
    import torch

    from paper_1407_2089_b200._lib import lib

    L = lib()
    if not hasattr(L, "ct_fp64_peak"):
        return float("nan")
    import ctypes

    out = torch.zeros(148 * 8 * 256, dtype=torch.float64, device=dev)
    fn = L.ct_fp64_peak
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    iters = 4096
    for _ in range(2):
        fn(out.data_ptr(), iters, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    fn(out.data_ptr(), iters, torch.cuda.current_stream().cuda_stream)
    b.record()
    torch.cuda.synchronize()
    ops = out.numel() * iters * 16.0
    return ops / (a.elapsed_time(b) / 1e3) / 1e12


def ncu_traffic(pattern: str):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(pattern)
    except Exception:
        return None


def run_e2e(args, pipe, spec, sp, dev, world, s_cell, s_vess):
    """Public API end to end: pinned host frames -> H2D -> fused pipeline ->
    D2H of the step's result (counters + per-cell table rows + vessel state),
    double-buffered so step i+1's H2D overlaps step i's kernels."""
    import torch

    from paper_1407_2089_b200 import synth

    nvox = spec.nx * spec.ny * spec.nz
    nring = 2
    host = []
    for i in range(nring):
        c = torch.empty(spec.dims, dtype=torch.uint8, pin_memory=True)
        v = torch.empty(spec.dims, dtype=torch.uint8, pin_memory=True)
        c.copy_(synth.generate(spec, 50 + i, synth.CELL).cpu())
        v.copy_(synth.generate(spec, 50 + i, synth.VESSEL).cpu())
        host.append((c, v))
    NS = 3  # device input slots: H2D runs up to two time points ahead of compute
    dbuf = [(torch.empty(spec.dims, dtype=torch.uint8, device=dev), torch.empty(spec.dims, dtype=torch.uint8, device=dev))
            for _ in range(NS)]
    rows = 4096
    rbytes = rows * 128 + 64 + 72 + 32
    out_host = [torch.empty(rbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    # one copy stream per channel (two DMA engines share the PCIe link)
    s_copy = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    copied = [[torch.cuda.Event(), torch.cuda.Event()] for _ in range(NS)]
    done = [torch.cuda.Event() for _ in range(NS)]
    readable = [torch.cuda.Event() for _ in range(2)]
    for d in done:
        d.record()

    def h2d(i):
        slot = i % NS
        for ch in range(2):
            with torch.cuda.stream(s_copy[ch]):
                s_copy[ch].wait_event(done[slot])
                dbuf[slot][ch].copy_(host[i % nring][ch], non_blocking=True)
                copied[slot][ch].record()

    def compute(i):
        slot = i % NS
        main = torch.cuda.current_stream()
        main.wait_event(copied[slot][0])
        main.wait_event(copied[slot][1])
        s_cell.wait_stream(main)
        s_vess.wait_stream(main)
        with torch.cuda.stream(s_cell):
            pipe.cell(dbuf[slot][0], frame=i)
        with torch.cuda.stream(s_vess):
            pipe.vessel(dbuf[slot][1])
        main.wait_stream(s_cell)
        main.wait_stream(s_vess)
        done[slot].record()
        # the step's result to the host (host slot i % 2; read one step later)
        oh = out_host[i % 2]
        oh[: rows * 128].copy_(pipe.table[: rows * 128], non_blocking=True)
        oh[rows * 128 : rows * 128 + 64].copy_(pipe.counters.view(torch.uint8), non_blocking=True)
        oh[rows * 128 + 64 : rows * 128 + 136].copy_(pipe.state.view(torch.uint8)[:72], non_blocking=True)
        oh[rows * 128 + 136 :].copy_(pipe.votsu.view(torch.uint8), non_blocking=True)
        readable[i % 2].record()

    def run(i0, i1, seen=0):
        # every step's own H2D copy is issued inside [i0, i1): nothing is prefetched across the bracket
        h2d(i0)
        if i0 + 1 < i1:
            h2d(i0 + 1)
        for i in range(i0, i1):
            if i + 2 < i1:
                h2d(i + 2)
            compute(i)
            if i > i0:  # the previous time point's result is read on the host while this one runs
                readable[(i - 1) % 2].synchronize()
                seen += int(out_host[(i - 1) % 2][rows * 128: rows * 128 + 8].view(torch.int64)[0])
        readable[(i1 - 1) % 2].synchronize()
        return seen

    n = args.warmup + args.steps
    run(0, args.warmup)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for sc in s_copy:
        sc.wait_event(a)
    run(args.warmup, n)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    val = world * args.steps * 2 * nvox / (ms / 1e3)
    return {"value": val, "unit": UNIT, "h2d_bytes_per_step": 2 * nvox,
            "d2h_bytes_per_step": int(rbytes), "ms_per_step": ms / args.steps,
            # the H2D of the raw frames over PCIe is the e2e bound once the device step is shorter
            "h2d_gbs": 2 * nvox / (ms / args.steps / 1e3) / 1e9,
            "note": "pinned host frames, H2D up to two time points ahead of compute (3 device slots, one copy "
                    f"stream per channel); per step D2H of counters, first {rows} table rows and the vessel "
                    "state, read on the host while the next time point runs"}


def run_materialized(args, pipe, spec, dev, world):
    """Drop-in-materialised variant: per time point H2D of both
    channels, the fused pipeline, then the reference's result objects on the
    host -- the Detection list (C-order voxel arrays, centroids, volumes; hulls
    excluded) and the vessel (mask, DistanceMap) with the map left on device."""
    import time

    import torch

    from paper_1407_2089_b200 import synth

    nvox = spec.nx * spec.ny * spec.nz
    steps = max(1, min(args.steps, 10))
    host = []
    for i in range(2):
        c = torch.empty(spec.dims, dtype=torch.uint8, pin_memory=True)
        v = torch.empty(spec.dims, dtype=torch.uint8, pin_memory=True)
        c.copy_(synth.generate(spec, 60 + i, synth.CELL).cpu())
        v.copy_(synth.generate(spec, 60 + i, synth.VESSEL).cpu())
        host.append((c, v))
    dc = torch.empty(spec.dims, dtype=torch.uint8, device=dev)
    dv = torch.empty(spec.dims, dtype=torch.uint8, device=dev)
    ndet = 0

    def one(i):
        nonlocal ndet
        dc.copy_(host[i % 2][0], non_blocking=True)
        dv.copy_(host[i % 2][1], non_blocking=True)
        res = pipe.cell(dc, frame=i)
        vres = pipe.vessel(dv)
        dets = pipe.finish_cell(res, materialize=True, with_hull=False)
        mask, dmap = pipe.finish_vessel(vres, dv)
        ndet = len(dets)
        return dets

    one(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        dets = one(i + 1)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    # hulls, reported separately: host Qhull of the last frame's
    # detections, over worker processes (segment.compute_hulls; pool warmed first)
    from paper_1407_2089_b200 import segment as S

    vox = [d.voxels for d in dets]
    S.compute_hulls(vox[: S.HULL_POOL_MIN], pipe.spacing)
    th = time.perf_counter()
    S.compute_hulls(vox, pipe.spacing)
    hull_ms = (time.perf_counter() - th) * 1e3
    return {"value": world * steps * 2 * nvox / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps,
            "steps": steps, "detections_per_step": ndet,
            "hulls": {"ms_per_step": hull_ms, "procs": int(os.environ.get("CT_HULL_PROCS", min(16, os.cpu_count() or 1))),
                      "note": "host Qhull (as the reference), identical calls spread over worker processes"},
            "note": "host wall clock (the result is host Python objects): H2D both channels, pipeline, "
                    "Detection list (no hulls) + vessel (mask, device-resident DistanceMap), sequential"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default 200 (ours), 20 (--impl reference)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ring", type=int, default=6)
    ap.add_argument("--cpu-crop", type=int, default=128, help="x-slices per --impl reference step")
    ap.add_argument("--cpu-baseline-crop", type=int, default=1024, help="x-slices of the cpu_baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.steps is None:
        args.steps = 20 if args.impl == "reference" else 200
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
