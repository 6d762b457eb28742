"""Host-side logic of the z-slab decomposition, on CPU with gloo ranks
(world size 2): slab bounds, the per-rank reduced vectors (contiguous runs of
the global reduced order), the NCCL-id broadcast pattern bench.py uses and
the rank-order reduction the device finaliser performs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2310_00177_b200 as b200
from paper_2310_00177_b200 import scenes


def test_partition_bounds():
    assert b200.partition(256, 8, 4) == [(32 * r, 32) for r in range(8)]
    assert b200.partition(64, 2, 4) == [(0, 32), (32, 32)]
    # uneven: units of 2^(depth-1) spread over the first ranks
    assert b200.partition(48, 2, 4) == [(0, 24), (24, 24)]
    assert b200.partition(40, 2, 4) == [(0, 24), (24, 16)]
    for nz, n, d in [(512, 8, 4), (128, 4, 3), (96, 3, 4)]:
        p = b200.partition(nz, n, d)
        assert p[0][0] == 0 and sum(k for _, k in p) == nz
        assert all(z0 % (1 << (d - 1)) == 0 and k % (1 << (d - 1)) == 0 for z0, k in p)
        assert all(p[i][0] + p[i][1] == p[i + 1][0] for i in range(n - 1))
    assert b200.partition(64, 3, 5) == [(0, 32), (32, 16), (48, 16)]
    with pytest.raises(ValueError):
        b200.partition(64, 5, 5)  # 4 units of 16 planes cannot feed 5 ranks
    with pytest.raises(ValueError):
        b200.partition(36, 2, 4)  # not a multiple of 8


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank: int, world: int, port: int, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t, seed = scenes.config("C3", 64)
    z0, nk = b200.partition(t.shape[0], world, 4)[rank]
    own = t[z0:z0 + nk]
    # owned fluid cells in ascending global order = a contiguous run of the
    # global reduced vector, starting after the fluid cells of lower ranks
    mine = np.flatnonzero(own.reshape(-1) == 0) + z0 * t.shape[1] * t.shape[2]
    counts = [None] * world
    dist.all_gather_object(counts, int(mine.size))
    start = int(sum(counts[:rank]))
    all_idx = np.flatnonzero(t.reshape(-1) == 0)
    ok_run = bool(np.array_equal(all_idx[start:start + mine.size], mine))
    # the id broadcast of bench.py (an opaque 128-byte blob from rank 0)
    blob = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(blob, src=0)
    # rank-order sum of per-rank partials (k_finalize) is identical on every rank
    part = torch.tensor([float(np.sum(np.sin(mine[:1000])))], dtype=torch.float64)
    parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, part)
    tot = 0.0
    for p in parts:
        tot += float(p.item())
    tots = [None] * world
    dist.all_gather_object(tots, tot)
    out[rank] = (ok_run, blob[0] == bytes(range(128)), len(set(tots)) == 1, sum(counts) == all_idx.size)
    dist.destroy_process_group()


def test_slab_host_logic_gloo_two_ranks():
    world, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_rank_main, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res == {0: (True, True, True, True), 1: (True, True, True, True)}
