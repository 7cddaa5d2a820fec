"""Multi-rank host logic on CPU: world-size-2 gloo group reproduces the
reference's sequential detection ids (ref session.py:295-300)."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_1407_2089_b200.distributed import frame_shard, gather_tables, global_id_starts


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, counts, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    T = len(counts)
    mine = {t: counts[t] for t in frame_shard(T, world, rank)}
    starts = global_id_starts(mine, T)
    q.put((rank, list(frame_shard(T, world, rank)), starts))
    dist.barrier()
    dist.destroy_process_group()


def test_shards_cover_frames_once():
    for T in (1, 7, 10, 100):
        for w in (1, 2, 3, 8):
            frames = [t for r in range(w) for t in frame_shard(T, w, r)]
            assert frames == list(range(T))


def test_id_starts_world2_gloo():
    rng = np.random.default_rng(0)
    counts = [int(x) for x in rng.integers(0, 50, 11)]
    expected, c = [], 0
    for n in counts:  # the reference's running det_counter
        expected.append(c)
        c += n
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, counts, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    owned = set()
    for rank, frames, starts in res:
        assert starts == expected
        owned |= set(frames)
    assert owned == set(range(len(counts)))


def _gather_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 3 + 2 * rank
    rows = torch.zeros(8 * 128, dtype=torch.uint8)
    for i in range(n):
        rows[i * 128:(i + 1) * 128] = 10 * rank + i
    got, cnts = gather_tables(rows, torch.tensor(n), max_rows=8)
    q.put((rank, got.numpy(), cnts.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_tables_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, got, cnts in res:
        assert cnts.tolist() == [3, 5]
        for r in range(2):
            for i in range(int(cnts[r])):
                assert (got[r, i * 128:(i + 1) * 128] == 10 * r + i).all()


def _assemble_worker(rank, world, port, counts, mode, q):
    import torch.distributed as dist

    from paper_1407_2089_b200._lib import CELL_DTYPE
    from paper_1407_2089_b200.segment import Detection
    from paper_1407_2089_b200.sequence import FrameOut, assemble

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    T = len(counts)
    local = []
    for t in frame_shard(T, world, rank):
        rows = np.zeros(counts[t], dtype=CELL_DTYPE)
        rows["id"] = np.arange(counts[t])          # a frame segmented with id_start 0
        rows["count"] = 1000 * t + np.arange(counts[t])
        dets = [Detection(id=i, frame=t, voxels=np.zeros((1, 3), np.int64), centroid_um=np.zeros(3),
                          volume_um3=1.0) for i in range(counts[t])]
        local.append(FrameOut(t=t, rows=rows, detections=dets))
    res = assemble(local[::-1], T, gather_rows=mode)  # order of the local list does not matter
    q.put((rank, res.id_starts, res.det_counter,
           {t: [d.id for d in ds] for t, ds in res.detections_by_frame.items()},
           {t: (r["id"].tolist(), r["count"].tolist()) for t, r in res.rows_by_frame.items()}))
    dist.barrier()
    dist.destroy_process_group()


def _run_assemble(counts, mode, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_assemble_worker, args=(r, world, port, counts, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _sequential_ids(counts):
    """ref session.py:295-300: frame t's ids continue the running det_counter."""
    ids, c = {}, 0
    for t, n in enumerate(counts):
        ids[t] = list(range(c, c + n))
        c += n
    return ids, c


def test_assemble_world2_gloo_rank0():
    """segment_sequence's host half (sequence.assemble) at world size 2:
    each rank's Detections get the reference's sequential ids; rank 0 holds
    the per-cell records of every frame, in frame order, with global ids."""
    counts = [3, 0, 7, 2, 5, 11, 1]
    ids, total = _sequential_ids(counts)
    res = _run_assemble(counts, "rank0")
    for rank, starts, det_counter, dets, rows in res:
        assert det_counter == total
        assert starts == [ids[t][0] if counts[t] else sum(counts[:t]) for t in range(len(counts))]
        for t, d in dets.items():
            assert t in frame_shard(len(counts), 2, rank) and d == ids[t]
        if rank == 0:
            assert sorted(rows) == list(range(len(counts)))
            for t, (rid, rcount) in rows.items():
                assert rid == ids[t]
                assert rcount == [1000 * t + i for i in range(counts[t])]
        else:
            assert sorted(rows) == list(frame_shard(len(counts), 2, 1))


def test_assemble_world2_gloo_all_and_uneven():
    counts = [4, 9, 1]  # 3 frames on 2 ranks: blocks of 2 and 1
    ids, total = _sequential_ids(counts)
    for rank, starts, det_counter, dets, rows in _run_assemble(counts, "all"):
        assert det_counter == total and sorted(rows) == [0, 1, 2]
        assert all(rows[t][0] == ids[t] for t in rows)
