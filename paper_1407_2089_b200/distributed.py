"""Frame sharding across GPUs.

Time points are independent units (ref SPEC.md:103,176,353): each rank owns a
contiguous block of frames and runs the whole per-frame path locally; volumes
never cross GPUs.  The only cross-frame dependency in the reference is the
running detection-id counter (ref session.py:295-300: frame t's ids start at
the number of detections in frames < t).  Ranks therefore segment with
id_start = 0, all_gather the per-frame detection counts (NCCL over NVLink on
the GPU box, gloo in the CPU tests), and shift their ids by the exclusive
prefix sum -- exactly the reference's ids.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def frame_shard(t_count: int, world: int, rank: int) -> range:
    """Contiguous block of frames owned by `rank` (all channels of a frame together)."""
    per = (t_count + world - 1) // world
    return range(min(rank * per, t_count), min((rank + 1) * per, t_count))


def global_id_starts(local_counts: dict[int, int], t_count: int, device=None, group=None,
                     with_total: bool = False):
    """id_start for every frame from the per-rank detection counts.

    local_counts maps the frames this rank processed to their detection
    counts.  One all_gather of a t_count-long int64 vector (owned frames
    filled, others 0); the sum over ranks is the global per-frame count and its
    exclusive prefix sum the reference's id_start per frame.  with_total:
    also return the total count (ref session.py:300, next_detection_id)."""
    dev = device or torch.device("cpu")
    mine = torch.zeros(t_count, dtype=torch.int64, device=dev)
    for t, c in local_counts.items():
        mine[t] = int(c)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        parts = [torch.zeros_like(mine) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, mine, group=group)
        total = torch.stack(parts).sum(dim=0)
    else:
        total = mine
    starts = torch.cumsum(total, 0) - total
    out = [int(x) for x in starts.cpu()]
    if with_total:  # (starts, total detections = the reference's final det_counter)
        return out, int(total.sum().item())
    return out


def relabel_rows(rows, id_start: int):
    """Shift a frame's ct_cell rows (segmented with id_start 0) to global ids."""
    out = rows.copy()
    out["id"] += id_start
    return out


def gather_tables(rows: torch.Tensor, nrows: torch.Tensor, max_rows: int, group=None):
    """All-gather of fixed-width per-cell records.

    rows: uint8 tensor holding this rank's ct_cell rows (>= max_rows * 128
    bytes; 128 B per row), nrows: int64 scalar tensor (valid rows, on the same
    device).  Exchanges max_rows rows per rank in one all_gather_into_tensor
    (fixed size: no size round trip; NCCL over NVLink on the GPU box) plus the
    counts.  Returns (gathered uint8 [world, max_rows * 128], counts int64
    [world]); rank r's valid rows are gathered[r, :counts[r] * 128]."""
    row = 128
    buf = rows[: max_rows * row].contiguous()
    cnt = nrows.reshape(1).to(torch.int64)
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world == 1:
        return buf.reshape(1, -1), cnt.clamp(max=max_rows)
    out = torch.empty(world * buf.numel(), dtype=buf.dtype, device=buf.device)
    cnts = torch.empty(world, dtype=torch.int64, device=buf.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    dist.all_gather_into_tensor(cnts, cnt, group=group)
    return out.reshape(world, -1), cnts.clamp(max=max_rows)
