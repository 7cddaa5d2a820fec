#!/usr/bin/env python
"""Benchmark: segmented voxels/s of the per-frame 3-D segmentation hot path.

Workload (BASELINE.json configs[1], "C2", the default): synthetic
1024x1024x64 uint8 time points with two channels (cell + vessel), spacing
(0.8, 0.8, 1.0) um, the reference's default parameters (session.py:70-74).
``--config C3``: 1024x1024x64 uint16 (12-bit) with three channels (cell,
vessel, second cell channel).  One step = one time point: the cell
channel(s) (Gaussian background, median, Otsu, closing, 26-CCL, per-cell
table) and the vessel channel (MRF statistics, Otsu, closing, EDT), cell and
vessel work on two CUDA streams.  value = voxels of all processed (frame,
channel) volumes / device time (max over ranks).  Frames are independent:
N GPUs shard time points (weak scaling); the collectives are an all_gather of
per-frame detection counts (global id offsets) and of the per-cell records
(SURVEY 8e).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2|C3] [--dry]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run (one process per GPU, NCCL).  --dry runs the
multi-rank host logic only (gloo on CPU, synthetic per-frame records): the
launcher, the id exchange and the record assembly, no GPU.
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


def log(msg: str):
    print(f"[bench] {msg}", file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# workloads (BASELINE.json configs)
# ---------------------------------------------------------------------------
def workload(name: str):
    """(spec, time points, channels, description)."""
    from paper_1407_2089_b200 import synth

    if name == "C2":
        return (synth.C2, 100, (synth.CELL, synth.VESSEL),
                "C2: 1024x1024x64 uint8 time points, 2 channels (cell+vessel), 1600 cells")
    if name == "C3":
        return (synth.C3, 200, (synth.CELL, synth.VESSEL, synth.CELL2),
                "C3: 1024x1024x64 uint16 (12-bit) time points, 3 channels (cell+vessel+cell#2), 1600 cells each")
    raise SystemExit(f"unknown config {name}")


def host_frame(O, spec, t: int, ch: int, crop_nx: int | None = None):
    """The oracle's copy of synthetic frame (t, ch), optionally x-cropped."""
    from paper_1407_2089_b200 import synth

    nx = crop_nx or spec.nx
    dims = (nx, spec.ny, spec.nz)
    if ch == synth.VESSEL:
        return O.synth_frame(dims, spec.dtype, spec.frame_seed(t, ch), spec.vmax, tubes=spec.tubes(),
                             amp_tube=spec.amp_tube)
    balls = spec.balls(t, ch)
    balls = balls[balls[:, 0] < nx * 16]
    return O.synth_frame(dims, spec.dtype, spec.frame_seed(t, ch), spec.vmax, balls=balls, amp_ball=spec.amp_cell)


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg / --impl reference arm)
# ---------------------------------------------------------------------------
def cpu_channel(O, raw, ch: int, keep: bool = False):
    """The reference path of one (frame, channel) volume on the oracle port
    (test-only checker, oracle/): cell = denoise_cell_channel +
    segment_cell_channel (ref denoise.py:67-89, segment.py:279-289); vessel =
    mrf_denoise + segment_vessel_channel (ref denoise.py:193-195,
    segment.py:307-318).  Returns (seconds, outputs if keep)."""
    from paper_1407_2089_b200 import synth

    t0 = time.perf_counter()
    if ch == synth.VESSEL:
        st = O.mrf(raw)
        cur = st["current"] if st["current"] is not None else raw
        out = O.segment_vessel(cur, SPACING)
    else:
        den = O.denoise_cell(raw, SPACING, 10.0)["denoised"]
        out = O.segment_cell(den, SPACING, intensity=raw)
    dt = time.perf_counter() - t0
    return dt, (out if keep else None)


def cpu_time_point(spec, channels, t: int, crop_nx: int, threads: int, keep: bool = False):
    """All channels of time point t (cropped to crop_nx x-slices).  Returns
    (voxels/s, seconds, {channel: outputs} if keep)."""
    os.environ["OMP_NUM_THREADS"] = str(threads)
    from oracle import oracle as O

    O.lib()
    total, outs = 0.0, {}
    for ch in channels:
        raw = host_frame(O, spec, t, ch, crop_nx)
        dt, out = cpu_channel(O, raw, ch, keep)
        total += dt
        if keep:
            outs[ch] = out
    return len(channels) * crop_nx * spec.ny * spec.nz / total, total, outs


def run_reference(args):
    """--impl reference: the reference path on the host cores (oracle port,
    OpenMP, all host threads).  Same workload as our arm: full-size volumes
    of the bench config; one step = one full (frame, channel) volume, the
    channels of a time point on consecutive steps (cell, vessel[, cell#2]),
    so K steps cover K / channels time points.  Warm-up steps run on a
    64-slice crop (a CPU arm has no device warm-up; this loads the library and
    touches its code without minutes of untimed work)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O

    spec, T, channels, desc = workload(args.config)
    O.lib()
    threads = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(threads)
    for s in range(args.warmup):
        cpu_channel(O, host_frame(O, spec, s % T, channels[s % len(channels)], 64), channels[s % len(channels)])
    nvox = spec.nx * spec.ny * spec.nz
    secs = []
    for s in range(args.steps):
        t, ch = s // len(channels), channels[s % len(channels)]
        raw = host_frame(O, spec, t % T, ch)
        dt, _ = cpu_channel(O, raw, ch)
        secs.append(dt)
        log(f"reference step {s}: t={t} channel={ch} {dt:.2f} s")
    value = args.steps * nvox / sum(secs)
    sample = (f"oracle/ct_oracle.c port of the reference path (OpenMP, {threads} threads) on full-size "
              f"{spec.nx}x{spec.ny}x{spec.nz} {spec.dtype} volumes: {args.steps} (frame, channel) volumes = "
              f"time points 0..{(args.steps - 1) // len(channels)}, channels in turn; {sum(secs):.1f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sum(secs) / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": spec.dtype, "data": "synthetic",
        "config": {"workload": desc, "parallelism": "cpu", "same_config": True,
                   "step": "one full-size (frame, channel) volume"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# --dry: the multi-rank host logic on CPU (gloo), no GPU
# ---------------------------------------------------------------------------
def run_dry(args):
    """Launcher + collectives + id assembly with synthetic per-frame records:
    every rank owns a contiguous frame block (distributed.frame_shard), the
    per-frame counts are exchanged (global id offsets, ref session.py:295-300)
    and rank 0 assembles every frame's records (sequence.assemble)."""
    import torch.distributed as dist

    from paper_1407_2089_b200._lib import CELL_DTYPE
    from paper_1407_2089_b200.distributed import frame_shard
    from paper_1407_2089_b200.sequence import FrameOut, assemble

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        log(f"rank {rank}/{world}: gloo group of size {dist.get_world_size()}")
    T = 100
    counts = np.random.default_rng(7).integers(0, 40, T)
    local = []
    for t in frame_shard(T, world, rank):
        rows = np.zeros(int(counts[t]), dtype=CELL_DTYPE)
        rows["id"] = np.arange(counts[t])
        rows["count"] = 1000 * t + np.arange(counts[t])
        local.append(FrameOut(t=t, rows=rows))
    res = assemble(local, T, gather_rows="rank0")
    if rank == 0:
        expect = np.concatenate([[0], np.cumsum(counts)[:-1]])
        ids_ok = res.id_starts == [int(x) for x in expect] and res.det_counter == int(counts.sum())
        rows_ok = sorted(res.rows_by_frame) == list(range(T)) and all(
            res.rows_by_frame[t]["id"].tolist() == list(range(expect[t], expect[t] + counts[t])) for t in range(T))
        print(json.dumps({"dry": True, "n_ranks": world, "backend": "gloo" if world > 1 else None,
                          "frames": T, "detections": res.det_counter, "ids_ok": bool(ids_ok),
                          "rows_ok": bool(rows_ok)}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: one process per GPU under
    torch.distributed.run (rendezvous on 127.0.0.1), same arguments."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log("launching " + " ".join(cmd[1:]))
    return subprocess.run(cmd, env=dict(os.environ, CT_BENCH_LAUNCHED="1")).returncode


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
GATHER_ROWS = 2048  # per-cell records exchanged per frame and rank (C2: ~1,550 cells)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1407_2089_b200 import _lib, synth
    from paper_1407_2089_b200.distributed import frame_shard, gather_tables
    from paper_1407_2089_b200.imaging import VoxelSpacing
    from paper_1407_2089_b200.pipeline import FramePipeline

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        probe = torch.ones(1, device=dev)
        dist.all_reduce(probe)  # communicator up: every rank contributes
        log(f"rank {rank}/{world} on cuda:{local}: NCCL communicator size {dist.get_world_size()} "
            f"(all_reduce check {int(probe.item())})")
    spec, T, channels, desc = workload(args.config)
    cell_chs = [c for c in channels if c != synth.VESSEL]
    nch = len(channels)
    sp = VoxelSpacing(*SPACING)
    nvox = spec.nx * spec.ny * spec.nz
    my_frames = list(frame_shard(T, world, rank)) or [rank % T]
    ring = min(args.ring, len(my_frames))

    # the cell stream gets the higher priority: its persistent tensor-core K1
    # CTAs then take SMs as soon as they free up and the latency-bound vessel
    # kernels fill the gaps (1.75 vs 1.84 ms per step with equal priorities)
    s_cell = torch.cuda.Stream(dev, priority=-1)
    s_vess = torch.cuda.Stream(dev, priority=0)
    pipe = FramePipeline(spec.dims, spec.dtype, sp)
    # inputs resident in HBM (a ring of distinct time points; >= 134 MB/step > L2)
    inputs = []
    for i in range(ring):
        t = my_frames[i]
        inputs.append((t, {ch: synth.generate(spec, t, ch) for ch in channels}))
    counts_dev = torch.zeros(len(cell_chs), dtype=torch.int64, device=dev)
    gathered = torch.zeros(world * len(cell_chs), dtype=torch.int64, device=dev)
    coll_done = torch.cuda.Event()
    torch.cuda.synchronize()

    # Time points are queued back to back: each channel's stream runs its
    # frames in order (its buffers are reused frame to frame) and the two
    # streams share no buffers, so the vessel work of time point t may still
    # run while the cell work of t+1 starts.  At N > 1 the collectives of a
    # step read this step's table and counters on the main stream; the next
    # step's cell work waits for them (coll_done) before overwriting those
    # buffers.  The timed region ends with both streams joined.
    graphs = {}  # (ring slot, channel) -> CUDA graph of that frame's launches (after warm-up)
    graph_launches = {}

    def cell_body(raws, t, k, ch):
        pipe.cell(raws[ch], frame=t, id_start=0)
        counts_dev[k:k + 1].copy_(pipe.counters[2:3])

    def capture_graphs():
        # one CUDA graph per (input slot, channel): a step is then one replay per
        # channel on that channel's stream (no per-kernel host launches)
        for sl in range(ring):
            t, raws = inputs[sl]
            for k, ch in enumerate(cell_chs):
                c0 = _lib.launch_counter["count"]
                _lib.launch_counter["enabled"] = True
                graphs[(sl, ch)] = pipe.capture(lambda: cell_body(raws, t, k, ch))
                graph_launches[(sl, ch)] = _lib.launch_counter["count"] - c0
                _lib.launch_counter["enabled"] = False
            c0 = _lib.launch_counter["count"]
            _lib.launch_counter["enabled"] = True
            graphs[(sl, synth.VESSEL)] = pipe.capture(lambda: pipe.vessel(raws[synth.VESSEL]))
            graph_launches[(sl, synth.VESSEL)] = _lib.launch_counter["count"] - c0
            _lib.launch_counter["enabled"] = False
        for i in range(max(2, ring)):
            step(i)
        torch.cuda.synchronize()
        log(f"captured {len(graphs)} CUDA graphs ({sum(graph_launches.values()) // ring} libct launches per step)")

    def step(i, coll=True, first=True):
        t, raws = inputs[i % ring]
        main = torch.cuda.current_stream()
        if first:
            s_cell.wait_stream(main)
            s_vess.wait_stream(main)
        elif world > 1:
            s_cell.wait_event(coll_done)
        with torch.cuda.stream(s_cell):
            for k, ch in enumerate(cell_chs):
                g = graphs.get((i % ring, ch))
                if g is not None:
                    g.replay()
                    _lib.launch_counter["count"] += graph_launches[(i % ring, ch)] * _lib.launch_counter["enabled"]
                else:
                    cell_body(raws, t, k, ch)
                if world > 1 and coll and k + 1 < len(cell_chs):
                    # the records of this channel leave before the next cell channel reuses the table
                    main.wait_stream(s_cell)
                    gather_tables(pipe.table, pipe.counters[2], max_rows=GATHER_ROWS)
                    s_cell.wait_stream(main)
        with torch.cuda.stream(s_vess):
            g = graphs.get((i % ring, synth.VESSEL))
            if g is not None:
                g.replay()
                _lib.launch_counter["count"] += graph_launches[(i % ring, synth.VESSEL)] * _lib.launch_counter["enabled"]
            else:
                pipe.vessel(raws[synth.VESSEL])
        if world > 1 and coll:
            main.wait_stream(s_cell)  # the collectives read this step's cell results
            # the frame's detection counts (global ids) and its per-cell records, over NCCL
            dist.all_gather_into_tensor(gathered, counts_dev)
            gather_tables(pipe.table, pipe.counters[2], max_rows=GATHER_ROWS)
            coll_done.record(main)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # correctness guard: the fused path's decisions must be the fast ones
    assert int(pipe.state[5].item()) == 0, "MRF needed iterations: bench workload assumption broken"
    if not args.no_graphs:
        try:
            capture_graphs()
        except Exception as exc:  # eager launches still give a valid (slower-to-issue) measurement
            graphs.clear()
            torch.cuda.synchronize()
            log(f"CUDA graph capture failed ({type(exc).__name__}: {exc}); timing eager launches")

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
    total_vox = world * args.steps * nch * nvox
    value = total_vox / (ms_max / 1e3)

    # --- overlapped per-stage times: the timed loop replays graphs (no
    # per-stage events inside them), so the same two-stream schedule runs
    # eagerly for a few steps with CUDA events around each stage on its stream
    if not stage_ms:
        pipe.marks = []
        g_saved = dict(graphs)
        graphs.clear()
        for i in range(min(2 * ring, args.steps)):
            step(args.warmup + i, coll=False, first=(i == 0))
        main_s = torch.cuda.current_stream()
        main_s.wait_stream(s_cell)
        main_s.wait_stream(s_vess)
        torch.cuda.synchronize()
        stage_ms = pipe.stage_times_ms()
        pipe.marks = None
        graphs.update(g_saved)

    # --- serialized pass (one stream) for clean per-kernel times ----------
    pipe.marks = []
    for i in range(min(3, args.steps)):
        t, raws = inputs[i % ring]
        for ch in cell_chs:
            pipe.cell(raws[ch], frame=t)
        pipe.vessel(raws[synth.VESSEL])
    torch.cuda.synchronize()
    serial_ms = pipe.stage_times_ms()
    pipe.marks = None

    # --- e2e through the public pipeline API with pinned host buffers -------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, pipe, spec, channels, dev, world, s_cell, s_vess)
        e2e["materialized"] = run_materialized(args, pipe, spec, channels, dev, world)

    # --- roofline of the dominant stage -------------------------------------
    # algorithmic HBM bytes per voxel of each stage, SURVEY 8d for the fused
    # kernels as launched (b = input bytes): K1 reads raw + writes q (2b); K2
    # reads q + writes the median (2b, histogram fused); K4 on the cell path
    # reads the median + writes packed z-rows (b + 1/8); K5 reads those rows
    # (1/8; its label writes touch only foreground voxels, the -1 background
    # fill runs on a side stream outside its window); K6 touches only the
    # foreground (latency-bound, no per-voxel bytes); K7 reads the raw vessel
    # volume once (b); vessel Otsu + closing read raw + write the byte mask
    # (b + 1); K8 reads the mask + writes float64 (9).
    pk = peaks()
    rx, ry, rz = pipe.r
    b = 1 if spec.dtype == "u8" else 2
    k1_tc = pipe.k1_path_tc
    k1_macs = (4 * 256 * b + 13 * 256 + 13 * spec.nz) if k1_tc else None  # limb-pair MMAs (see k_gauss_tc.cu)
    bpv = {"K1 gaussian": 2 * b, "K2 median+hist": 2 * b,
           "K4 threshold+close": (b + 0.125) if pipe.rows_path else (b + 1), "K5 ccl": 0.125 if pipe.rows_path else 1,
           "K6 table": None, "K7 mrf": b, "K3+K4 vessel otsu+close": b + 1, "K8 edt": 9}
    kernels, kernels_serial = {}, {}
    for src, dst in ((stage_ms, kernels), (serial_ms, kernels_serial)):
        for k, v in src.items():  # v = mean ms per call; one call = one (frame, channel) volume
            bb = bpv.get(k)
            dst[k] = {"ms": v, "hbm_gbs": (bb * nvox / (v / 1e3) / 1e9) if bb else None,
                      "hbm_frac": (bb * nvox / (v / 1e3) / 1e9 / pk["hbm_gbs"]) if bb else None,
                      "algorithmic_bytes_per_voxel": bb}
    # the dominant stage: most serial time per time point
    per_tp = {k: v * (len(cell_chs) if k.startswith(("K1", "K2", "K4 ", "K5", "K6")) else 1)
              for k, v in serial_ms.items()}
    dom = max(per_tp, key=per_tp.get)
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
                               "frac_of_fp64_peak": alg_tf / fp64_pk if fp64_pk == fp64_pk else None,
                               "hbm_gbs": 2 * b * nvox / (ms_dom / 1e3) / 1e9,
                               "hbm_frac": 2 * b * nvox / (ms_dom / 1e3) / 1e9 / pk["hbm_gbs"]}
    else:
        bb = bpv.get(dom) or 1
        achieved = bb * nvox / (ms_dom / 1e3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "peak_source": pk["source"], "algorithmic_bytes_per_voxel": bb}
    roof.update({"stage": dom, "ms_serial": ms_dom, "ms_overlapped": stage_ms.get(dom),
                 "timing": "CUDA events around the stage on its stream inside bench.py: ms_serial = serialized pass "
                           "(3 time points, the roofline's duration), ms_overlapped = the two-stream schedule of the "
                           "timed loop run eagerly (2 x ring time points; the timed loop itself replays graphs)",
                 "traffic": ncu_traffic(dom, args.config),
                 "traffic_note": "DRAM bytes of the stage's kernels per volume, ncu launch list (profiles/)",
                 "share_of_step_serial": per_tp[dom] / sum(per_tp.values())})

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        crop = args.cpu_baseline_crop
        v, dt, outs = cpu_time_point(spec, channels, 0, crop, threads, keep=(crop == spec.nx))
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"oracle/ct_oracle.c port (OpenMP), all {nch} channels of {args.config} t=0 "
                         f"({crop}x{spec.ny}x{spec.nz} per channel, {dt:.1f} s)"}
        if outs:
            parity = check_parity(pipe, spec, channels, inputs[0], outs)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": spec.dtype, "data": "synthetic",
            "config": {"workload": desc, "global_batch": world, "parallelism": f"frame-sharded dp{world}",
                       "frames_per_s": world * args.steps / (ms_max / 1e3),
                       "launch": "CUDA graph per (frame slot, channel), replayed on the channel's stream"
                                 if graphs else "eager",
                       "l2": f"inputs larger than L2: {nch * nvox * b / 1e6:.0f} MB/step from a ring of {ring} "
                             "distinct time points, plus GB-scale intermediates"},
            "parity": None if parity is None else parity["ok"], "parity_detail": parity,
            "e2e": e2e, "gpu_launches": launches, "clocks": clk, "roofline": roof, "kernels": kernels,
            "kernels_serial": kernels_serial,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def check_parity(pipe, spec, channels, inp, outs) -> dict:
    """The bench's own t = 0 time point (first frame of the input ring) on the
    fused path vs the oracle outputs of the cpu_baseline leg (same frames):
    per-cell rows (ids, counts, roots, bbox, intensity sums, mean intensities,
    centroids, volumes), C-order voxel lists, vessel mask and distance map,
    bit for bit."""
    import torch

    from paper_1407_2089_b200 import synth

    t, raws = inp
    assert t == 0
    ny, nz = spec.ny, spec.nz
    checks = {}
    for ch in channels:
        if ch == synth.VESSEL:
            vres = pipe.vessel(raws[ch])
            mask, dm = pipe.finish_vessel(vres, raws[ch])
            om, odist, _ = outs[ch]
            checks[f"vessel mask (ch {ch})"] = bool(np.array_equal(mask.cpu().numpy(), om))
            checks[f"distance map (ch {ch})"] = bool(np.array_equal(dm.values.cpu().numpy(), odist))
            continue
        res = pipe.cell(raws[ch], frame=0, id_start=0)
        cnt, rows = pipe.finish_cell(res)
        odets = outs[ch]
        ok = len(rows) == len(odets)
        if ok:
            ok &= rows["id"].tolist() == [d.id for d in odets]
            ok &= rows["count"].tolist() == [d.voxel_count for d in odets]
            ok &= rows["root"].tolist() == [d.root for d in odets]
            ok &= bool(np.array_equal(np.concatenate([rows["bbox_lo"], rows["bbox_hi"]], axis=1),
                                      np.array([d.bbox for d in odets])))
            ok &= rows["intensity_sum"].tolist() == [int(d.intensity_sum) for d in odets]
            ok &= bool(np.array_equal(rows["centroid_um"], np.array([d.centroid_um for d in odets])))
            ok &= bool(np.array_equal(rows["volume_um3"], np.array([d.volume_um3 for d in odets])))
            lin = np.concatenate([(d.voxels[:, 0] * ny + d.voxels[:, 1]) * nz + d.voxels[:, 2] for d in odets])
            ok &= bool(np.array_equal(pipe.voxels[: lin.size].cpu().numpy().astype(np.int64), lin))
            raw = raws[ch].cpu()
            rawf = (raw.view(torch.int16).numpy().view(np.uint16) if raw.dtype == torch.uint16 else raw.numpy()).ravel()
            means = [rawf[(d.voxels[:, 0] * ny + d.voxels[:, 1]) * nz + d.voxels[:, 2]].mean() for d in odets]
            ok &= bool(np.array_equal(rows["mean_intensity"], np.array(means)))
        checks[f"cell table + voxel lists (ch {ch}, {len(odets)} cells)"] = bool(ok)
    torch.cuda.synchronize()
    return {"ok": all(checks.values()), "frame": "t=0 (first frame of the timed input ring), full size",
            "vs": "oracle outputs of the cpu_baseline leg", "checks": checks}


def measured_fp64_peak(dev) -> float:
    """TFLOP/s of independent DADD/DMUL (no FMA) measured on this GPU."""
    import torch

    from paper_1407_2089_b200._lib import lib

    L = lib()
    if not hasattr(L, "ct_fp64_peak"):
        return float("nan")
    out = torch.zeros(148 * 8 * 256, dtype=torch.float64, device=dev)
    iters = 4096
    for _ in range(2):
        L.ct_fp64_peak(out.data_ptr(), iters, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    L.ct_fp64_peak(out.data_ptr(), iters, torch.cuda.current_stream().cuda_stream)
    b.record()
    torch.cuda.synchronize()
    ops = out.numel() * iters * 16.0
    return ops / (a.elapsed_time(b) / 1e3) / 1e12


def ncu_traffic(pattern: str, config: str):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return (d.get(config) or {}).get(pattern) if config in d else (d.get(pattern) if config == "C2" else None)
    except Exception:
        return None


def run_e2e(args, pipe, spec, channels, dev, world, s_cell, s_vess):
    """Public API end to end: pinned host frames -> H2D -> fused pipeline ->
    D2H of the step's result (counters + per-cell table rows of every cell
    channel + vessel state), double-buffered so step i+1's H2D overlaps step
    i's kernels."""
    import torch

    from paper_1407_2089_b200 import synth

    nvox = spec.nx * spec.ny * spec.nz
    nch = len(channels)
    cell_chs = [c for c in channels if c != synth.VESSEL]
    tdt = spec.torch_dtype
    esz = 1 if spec.dtype == "u8" else 2
    nring = 2
    host = []
    for i in range(nring):
        frames = {}
        for ch in channels:
            h = torch.empty(spec.dims, dtype=tdt, pin_memory=True)
            h.copy_(synth.generate(spec, 50 + i, ch).cpu())
            frames[ch] = h
        host.append(frames)
    NS = 3  # device input slots: H2D runs up to two time points ahead of compute
    dbuf = [{ch: torch.empty(spec.dims, dtype=tdt, device=dev) for ch in channels} for _ in range(NS)]
    rows = 4096
    rbytes_cell = rows * 128 + 64
    rbytes = len(cell_chs) * rbytes_cell + 72 + 32
    out_host = [torch.empty(rbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    # one copy stream per channel (the DMA engines share the PCIe link)
    s_copy = {ch: torch.cuda.Stream(dev) for ch in channels}
    copied = [{ch: torch.cuda.Event() for ch in channels} for _ in range(NS)]
    done = [torch.cuda.Event() for _ in range(NS)]
    readable = [torch.cuda.Event() for _ in range(2)]
    for d in done:
        d.record()

    def h2d(i):
        slot = i % NS
        for ch in channels:
            with torch.cuda.stream(s_copy[ch]):
                s_copy[ch].wait_event(done[slot])
                dbuf[slot][ch].copy_(host[i % nring][ch], non_blocking=True)
                copied[slot][ch].record()

    def compute(i):
        slot = i % NS
        main = torch.cuda.current_stream()
        for ch in channels:
            main.wait_event(copied[slot][ch])
        s_cell.wait_stream(main)
        s_vess.wait_stream(main)
        oh = out_host[i % 2]
        with torch.cuda.stream(s_vess):
            pipe.vessel(dbuf[slot][synth.VESSEL])
        with torch.cuda.stream(s_cell):
            for k, ch in enumerate(cell_chs):
                pipe.cell(dbuf[slot][ch], frame=i)
                # the channel's result to the host (host slot i % 2; read one step later)
                o = k * rbytes_cell
                oh[o: o + rows * 128].copy_(pipe.table[: rows * 128], non_blocking=True)
                oh[o + rows * 128: o + rbytes_cell].copy_(pipe.counters.view(torch.uint8), non_blocking=True)
        main.wait_stream(s_cell)
        main.wait_stream(s_vess)
        done[slot].record()
        o = len(cell_chs) * rbytes_cell
        oh[o: o + 72].copy_(pipe.state.view(torch.uint8)[:72], non_blocking=True)
        oh[o + 72:].copy_(pipe.votsu.view(torch.uint8), non_blocking=True)
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
    for sc in s_copy.values():
        sc.wait_event(a)
    run(args.warmup, n)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    val = world * args.steps * nch * nvox / (ms / 1e3)
    # the link alone: the same per-step H2D copies back to back, no compute
    # (the roofline of e2e once the device step is shorter than the copy)
    torch.cuda.synchronize()
    a.record()
    for sc in s_copy.values():
        sc.wait_event(a)
    for i in range(args.steps):
        for ch in channels:
            with torch.cuda.stream(s_copy[ch]):
                dbuf[i % NS][ch].copy_(host[i % nring][ch], non_blocking=True)
    for sc in s_copy.values():
        torch.cuda.current_stream().wait_stream(sc)
    b.record()
    torch.cuda.synchronize()
    link_gbs = nch * nvox * esz * args.steps / (a.elapsed_time(b) / 1e3) / 1e9
    return {"value": val, "unit": UNIT, "h2d_bytes_per_step": nch * nvox * esz,
            "h2d_link_gbs": link_gbs, "frac_of_link": (nch * nvox * esz / (ms / args.steps / 1e3) / 1e9) / link_gbs,
            "d2h_bytes_per_step": int(rbytes), "ms_per_step": ms / args.steps,
            # the H2D of the raw frames over PCIe is the e2e bound once the device step is shorter
            "h2d_gbs": nch * nvox * esz / (ms / args.steps / 1e3) / 1e9,
            "note": "pinned host frames, H2D up to two time points ahead of compute (3 device slots, one copy "
                    f"stream per channel); per step D2H of counters, first {rows} table rows of each cell channel "
                    "and the vessel state, read on the host while the next time point runs. The raw frames cross "
                    "PCIe once per step: at ~55 GB/s host-to-device this link, not the device step, bounds e2e"}


def run_materialized(args, pipe, spec, channels, dev, world):
    """Drop-in-materialised variant through the public sequence
    API (sequence.segment_frames, the process_experiment loop body): per time
    point the H2D of all channels from pinned host frames, the fused pipeline,
    then the reference's result objects on the host -- the Detection lists
    (C-order voxel arrays, centroids, volumes; hulls excluded) and the vessel
    (mask, DistanceMap with its values kept on the device) -- pipelined two
    frames deep (the host side of frame t overlaps the device side of t+1)."""
    import torch

    from paper_1407_2089_b200 import synth
    from paper_1407_2089_b200.sequence import segment_frames

    nvox = spec.nx * spec.ny * spec.nz
    cell_chs = [c for c in channels if c != synth.VESSEL]
    steps = max(2, min(args.steps, 20))
    host = []
    for i in range(2):
        frames = {}
        for ch in channels:
            h = torch.empty(spec.dims, dtype=spec.torch_dtype, pin_memory=True)
            h.copy_(synth.generate(spec, 60 + i, ch).cpu())
            frames[ch] = h
        host.append(frames)
    ch0 = cell_chs[0]
    ndet = 0

    last = {}

    def consume(fo):  # a streaming consumer: the frame's objects, then released
        last["fo"] = fo

    slot_pipes = []  # the sequence's two slot pipelines, created by the warm-up call and reused

    def run(frames):
        segment_frames(frames, lambda t: host[t % 2][ch0], lambda t: host[t % 2][synth.VESSEL],
                       spacing=pipe.spacing, materialize=True, with_hull=False, on_frame=consume, pipes=slot_pipes)

    run(range(3))  # warm-up: pipelines, pinned staging, first launches
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(range(steps))
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    dets = last["fo"].detections
    ndet = len(dets)
    nch_run = 2  # the first cell channel + the vessel channel per time point
    # hulls, reported separately: host Qhull of the last frame's
    # detections, over worker processes (segment.compute_hulls; pool warmed first)
    from paper_1407_2089_b200 import segment as S

    vox = [d.voxels for d in dets]
    S.compute_hulls(vox[: S.HULL_POOL_MIN], pipe.spacing)
    th = time.perf_counter()
    S.compute_hulls(vox, pipe.spacing)
    hull_ms = (time.perf_counter() - th) * 1e3
    return {"value": world * steps * nch_run * nvox / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps,
            "steps": steps, "detections_per_step": ndet, "channels_per_step": nch_run,
            "hulls": {"ms_per_step_first_cell_channel": hull_ms,
                      "procs": int(os.environ.get("CT_HULL_PROCS", min(16, os.cpu_count() or 1))),
                      "note": "host Qhull (as the reference), identical calls spread over worker processes"},
            "note": "host wall clock (the result is host Python objects), sequence.segment_frames over pinned "
                    "host frames, streaming consumer (on_frame): H2D, pipeline, Detection lists (no hulls) + "
                    "vessel (mask, device-resident DistanceMap copy per frame), two frames in flight (slot "
                    "pipelines from the warm-up call)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default 200 (ours), 20 (--impl reference)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C2", "C3"])
    ap.add_argument("--dry", action="store_true", help="multi-rank host logic only (gloo, CPU, no GPU)")
    ap.add_argument("--ring", type=int, default=6)
    ap.add_argument("--cpu-baseline-crop", type=int, default=None,
                    help="x-slices of the cpu_baseline sample (default: the full frame for C2, 256 for C3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="eager launches instead of per-frame CUDA graphs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.steps is None:
        args.steps = 20 if args.impl == "reference" else 200
    if args.cpu_baseline_crop is None:
        args.cpu_baseline_crop = 1024 if args.config == "C2" else 256
    _, world, _ = dist_env()
    if args.gpus > 1 and world == 1 and "CT_BENCH_LAUNCHED" not in os.environ:
        return relaunch(args)
    if world != args.gpus and not args.dry:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using {world} ranks")
    if args.dry:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
