"""The per-frame segmentation loop of ``process_experiment`` over a sequence
of time points, on one GPU or frame-sharded over N.

ref session.py:293-306:

    det_counter = 0
    for t in range(t_count):
        den  = denoise_cell_channel(cell(t), denoise_params)
        dets = segment_cell_channel(den, seg_config, frame=t, id_start=det_counter)
        det_counter += len(dets)
        detections_by_frame.append(dets)
        if vessel: maps[t] = segment_vessel_channel(mrf_denoise(vessel(t), max_iters))[1]

Here every frame runs through the fused ``FramePipeline`` (cell channel and
vessel channel on two CUDA streams) with ``id_start = 0``; ids are a pure
offset (id = id_start + rank by (-count, root), ref segment.py:257-264), so the
running counter is applied afterwards from the per-frame counts -- on one GPU
by a prefix sum, on N ranks by one all_gather of the counts
(``distributed.global_id_starts``) -- which reproduces the reference's ids
exactly without a host round trip between frames.

Ranks own contiguous frame blocks (``distributed.frame_shard``).  Each rank
materialises the ``Detection`` objects (voxel lists, hulls) of its own frames
(voxel lists never cross GPUs); the fixed-width per-cell records (128-B
``ct_cell`` rows, global ids) of every frame are assembled on rank 0 (or on
every rank) with one all_gather per sequence.

``assemble`` is the host/collective half and runs on CPU tensors too (the
world-2 gloo tests and ``bench.py --dry``); ``segment_frames`` is the GPU half.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from ._lib import CELL_DTYPE
from .distributed import frame_shard, global_id_starts


@dataclass
class FrameOut:
    """One time point's result before global ids are known (ids from 0)."""

    t: int
    rows: np.ndarray                 # CELL_DTYPE rows, ids 0..n-1 (id order)
    detections: list | None = None   # Detection objects (ids from 0), if materialised
    distance_map: object = None      # DistanceMap of the vessel channel (device-resident values)
    vessel_mask: object = None


@dataclass
class SequenceResult:
    """What process_experiment keeps from the segmentation loop."""

    t_count: int
    id_starts: list[int]                                        # id_start of every frame (global)
    det_counter: int                                            # total detections (ref next_detection_id)
    detections_by_frame: dict[int, list] = field(default_factory=dict)  # this rank's frames
    rows_by_frame: dict[int, np.ndarray] = field(default_factory=dict)  # every frame (on the assembling ranks)
    distance_maps: dict[int, object] = field(default_factory=dict)      # this rank's frames


def _world(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def assemble(local: list[FrameOut], t_count: int, group=None, gather_rows: str = "rank0",
             device=None) -> SequenceResult:
    """Global ids for this rank's frames and the per-cell records of all frames.

    local: this rank's FrameOuts (any order).  gather_rows: "rank0" (records of
    every frame on rank 0 only), "all" (on every rank) or "none".  Collectives:
    one all_gather of the T per-frame counts, then (unless "none") one
    all_gather of the count of rows per rank and one of the padded row bytes.
    ``device``: where the collective buffers live (the rank's GPU under NCCL,
    CPU under gloo)."""
    rank, world = _world(group)
    dev = device or torch.device("cpu")
    counts = {fo.t: int(len(fo.rows)) for fo in local}
    starts, total = global_id_starts(counts, t_count, device=dev, group=group, with_total=True)
    res = SequenceResult(t_count=t_count, id_starts=starts, det_counter=total)
    mine = sorted(local, key=lambda fo: fo.t)
    for fo in mine:
        rows = fo.rows.copy()
        rows["id"] += starts[fo.t]
        fo.rows = rows
        if fo.detections is not None:
            for d in fo.detections:
                d.id += starts[fo.t]
            res.detections_by_frame[fo.t] = fo.detections
        if fo.distance_map is not None:
            res.distance_maps[fo.t] = fo.distance_map
    if gather_rows == "none":
        return res
    if world == 1:
        res.rows_by_frame = {fo.t: fo.rows for fo in mine}
        return res
    # fixed-width records: [frame t, n rows] headers + the row bytes, one
    # padded all_gather (rows are 128 B; a C2 frame has ~1.5k cells)
    hdr = np.array([[fo.t, len(fo.rows)] for fo in mine], dtype=np.int64).reshape(-1, 2)
    body = np.concatenate([fo.rows.view(np.uint8).ravel() for fo in mine]) if mine else np.zeros(0, np.uint8)
    sizes = torch.tensor([hdr.shape[0], body.size], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [tuple(int(x) for x in s.cpu()) for s in all_sizes]
    max_h = max(s[0] for s in all_sizes)
    max_b = max(s[1] for s in all_sizes)
    hbuf = torch.zeros((max_h, 2), dtype=torch.int64, device=dev)
    hbuf[: hdr.shape[0]] = torch.from_numpy(hdr).to(dev)
    bbuf = torch.zeros(max(1, max_b), dtype=torch.uint8, device=dev)
    bbuf[: body.size] = torch.from_numpy(body).to(dev)
    hs = [torch.zeros_like(hbuf) for _ in range(world)]
    bs = [torch.zeros_like(bbuf) for _ in range(world)]
    dist.all_gather(hs, hbuf, group=group)
    dist.all_gather(bs, bbuf, group=group)
    if gather_rows == "rank0" and rank != 0:
        res.rows_by_frame = {fo.t: fo.rows for fo in mine}
        return res
    for r in range(world):
        h = hs[r][: all_sizes[r][0]].cpu().numpy()
        b = bs[r][: all_sizes[r][1]].cpu().numpy()
        off = 0
        for t, n in h:
            nb = int(n) * CELL_DTYPE.itemsize
            res.rows_by_frame[int(t)] = b[off: off + nb].copy().view(CELL_DTYPE)
            off += nb
    return res


def segment_frames(frames, load_cell, load_vessel=None, spacing=None, denoise_params=None, seg_config=None,
                   mrf_max_iters: int = 1000, materialize: bool = True, with_hull: bool = True, pipe=None,
                   depth: int = 2, on_frame=None, pipes=None):
    """The GPU half: every frame t in ``frames`` through the fused pipeline.

    load_cell(t) / load_vessel(t) return the raw frame (numpy array, pinned
    host tensor or CUDA tensor, uint8/uint16, (nx, ny, nz)).  Returns
    [FrameOut] with ids from 0, in frame order.

    Pipelined ``depth`` frames deep (one FramePipeline per slot): frame t+1's
    H2D copy and kernels are queued before the host reads frame t's results
    (rows, voxel lists, Detection objects, hulls), so the host side of frame
    t overlaps the device side of frame t+1.  The cell and vessel channels of
    a frame run on two streams; a frame's completion is an event pair, and
    its results are read on a host-side stream that waits only for those
    events.  ``pipe`` (depth 1 only) reuses a caller's FramePipeline;
    ``pipes`` (a list, filled on first use) keeps the slot pipelines across
    calls (no per-call allocation of their buffers).
    ``on_frame(fo)``: a streaming consumer -- each FrameOut is handed over as
    soon as it is read back and not kept (the returned list is empty), so its
    device copies are released frame by frame."""
    from collections import deque

    from . import _dev
    from .errors import ParameterError
    from .pipeline import FramePipeline

    if spacing is None:
        raise ParameterError("segment_frames needs the experiment's voxel spacing")
    depth = 1 if pipe is not None else max(1, int(depth))
    dev = _dev.require_cuda()
    s_cell = torch.cuda.Stream(dev, priority=-1)
    s_vess = torch.cuda.Stream(dev)
    s_copy = torch.cuda.Stream(dev)
    s_host = torch.cuda.Stream(dev)
    if pipes is None:
        pipes = [pipe] if pipe is not None else []
    elif pipe is not None and not pipes:
        pipes.append(pipe)
    slots = {}  # (slot, channel) -> device input buffer, reused every depth frames

    def stage(x, key):
        """Raw frame -> CUDA tensor: device tensors as they are, host frames
        copied on s_copy into the slot's preallocated buffer (async from
        pinned memory; allocating per frame made every copy wait for the
        allocator)."""
        if x is None:
            return None
        if not isinstance(x, torch.Tensor):
            a = np.ascontiguousarray(np.asarray(x))
            if a.dtype not in (np.uint8, np.uint16):
                raise ParameterError("raw frames must be uint8 or uint16 (ref imaging.py:211-220 TIFF frames); "
                                     "run float grids through denoise/segment directly")
            x = torch.from_numpy(a.view(np.int16)).view(torch.uint16) if a.dtype == np.uint16 else torch.from_numpy(a)
        if x.dtype not in (torch.uint8, torch.uint16):
            raise ParameterError("raw frames must be uint8 or uint16 (ref imaging.py:211-220 TIFF frames); "
                                 "run float grids through denoise/segment directly")
        if x.is_cuda:
            return x.contiguous()
        buf = slots.get(key)
        if buf is None or buf.shape != x.shape or buf.dtype != x.dtype:
            buf = slots[key] = torch.empty(x.shape, dtype=x.dtype, device=dev)
        with torch.cuda.stream(s_copy):
            buf.copy_(x, non_blocking=x.is_pinned())
        return buf

    def launch(k, t):
        raw_c = stage(load_cell(t), (k % depth, 0))
        raw_v = stage(load_vessel(t), (k % depth, 1)) if load_vessel else None
        while len(pipes) <= k % depth:
            dt = "u8" if raw_c.dtype == torch.uint8 else "u16"
            pipes.append(FramePipeline(tuple(raw_c.shape), dt, spacing, denoise_params, seg_config,
                                       vessel=load_vessel is not None, device=dev))
        p = pipes[k % depth]
        copied = torch.cuda.Event()
        copied.record(s_copy)
        s_cell.wait_event(copied)
        s_vess.wait_event(copied)
        with torch.cuda.stream(s_cell):
            cres = p.cell(raw_c, frame=t, id_start=0)
            ev_c = torch.cuda.Event()
            ev_c.record(s_cell)
        vres, ev_v = None, None
        if raw_v is not None:
            with torch.cuda.stream(s_vess):
                vres = p.vessel(raw_v)
                ev_v = torch.cuda.Event()
                ev_v.record(s_vess)
        return (t, p, raw_c, raw_v, cres, vres, ev_c, ev_v)

    def finish(item):
        t, p, raw_c, raw_v, cres, vres, ev_c, ev_v = item
        with torch.cuda.stream(s_host):
            s_host.wait_event(ev_c)
            if ev_v is not None:
                s_host.wait_event(ev_v)
            cnt, rows = p.finish_cell(cres)
            dets = p.finish_cell(cres, materialize=True, with_hull=with_hull, table=(cnt, rows)) if materialize else None
            fo = FrameOut(t=t, rows=rows, detections=dets)
            if vres is not None:
                mask, dmap = p.finish_vessel(vres, raw_v, max_iters=mrf_max_iters)
                # the slot's buffers are reused by a later frame: keep this frame's own
                # copy of the map (the bool mask is already a new tensor)
                fo.vessel_mask = mask
                dmap.values = dmap.values.clone()
                fo.distance_map = dmap
            done = torch.cuda.Event()
            done.record(s_host)
        # the slot's next frame (k + depth) reads nothing of this one, but its
        # input copy and kernels overwrite these buffers: they wait for the
        # host's reads and copies
        s_copy.wait_event(done)
        s_cell.wait_event(done)
        s_vess.wait_event(done)
        return fo

    out, inflight = [], deque()
    emit = on_frame if on_frame is not None else out.append
    for k, t in enumerate(frames):
        inflight.append(launch(k, t))
        if len(inflight) == depth:  # frame k+1 goes in before frame k-depth+1 is read back
            emit(finish(inflight.popleft()))
    while inflight:
        emit(finish(inflight.popleft()))
    return out


def segment_sequence(load_cell, t_count: int, load_vessel=None, spacing=None, denoise_params=None,
                     seg_config=None, mrf_max_iters: int = 1000, materialize: bool = True, with_hull: bool = True,
                     group=None, gather_rows: str = "rank0") -> SequenceResult:
    """process_experiment's segmentation loop (ref session.py:293-306) over
    t_count frames: this rank's contiguous block of frames on its GPU, then
    the reference's global ids and the records of all frames (``assemble``).
    Works unchanged at world size 1 (no torch.distributed group)."""
    rank, world = _world(group)
    frames = list(frame_shard(t_count, world, rank))
    local = segment_frames(frames, load_cell, load_vessel, spacing, denoise_params, seg_config, mrf_max_iters,
                           materialize, with_hull)
    dev = torch.device("cuda", torch.cuda.current_device())
    backend = dist.get_backend(group) if world > 1 else None
    return assemble(local, t_count, group=group, gather_rows=gather_rows,
                    device=dev if backend == "nccl" else torch.device("cpu"))
