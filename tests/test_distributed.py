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
